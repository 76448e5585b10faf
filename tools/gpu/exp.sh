cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "topk_hist or planted or stats_and_classes or heavy" > gpurun_out/pytest_k1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1.log
tail -2 gpurun_out/pytest_k1.log
python tools/k1_modes.py --modes 0 > gpurun_out/k1m.txt 2>&1
GEM_HIST_HEAVY_PASS=1 python tools/k1_modes.py --modes 0 >> gpurun_out/k1m.txt 2>&1
python tools/k1_modes.py --modes 0 >> gpurun_out/k1m.txt 2>&1
GEM_HIST_HEAVY_PASS=1 python tools/k1_modes.py --modes 0 >> gpurun_out/k1m.txt 2>&1
cat gpurun_out/k1m.txt
