cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/k1_modes.py --layers 58 --experts 256 --modes 0,6,8,10,1 > gpurun_out/k1m.txt 2>&1
timeout 600 python tools/k1_modes.py --modes 0,6,8,1 >> gpurun_out/k1m.txt 2>&1
timeout 600 python tools/k1_modes.py --layers 16 --experts 64 --modes 0,6,1 >> gpurun_out/k1m.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "topk_hist" > gpurun_out/pytest_k1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1.log
cat gpurun_out/k1m.txt; tail -2 gpurun_out/pytest_k1.log
