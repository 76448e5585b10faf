cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "score or candidate or config_slice" > gpurun_out/pytest_k5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k5.log
python tools/kbench.py score --cands 10000 > gpurun_out/k5.txt 2>&1
tail -3 gpurun_out/pytest_k5.log; cat gpurun_out/k5.txt
