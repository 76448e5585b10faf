cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "score or candidate or config_slice" > gpurun_out/pytest_k5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k5.log
tail -30 gpurun_out/pytest_k5.log | grep -E "passed|failed|Error|assert" | head
python tools/kbench.py score --cands 10000 > gpurun_out/k5.txt 2>&1
python tools/kbench.py score --cands 10000 --layers 58 --experts 256 --gpus 32 >> gpurun_out/k5.txt 2>&1
cat gpurun_out/k5.txt
