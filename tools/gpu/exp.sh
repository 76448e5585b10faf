cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "topk_hist or planted or stats_and_classes or heavy or config_slice" > gpurun_out/pytest_k1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1.log
tail -2 gpurun_out/pytest_k1.log
python tools/k1_modes.py --layers 58 --experts 256 --modes 0,6 > gpurun_out/k1m.txt 2>&1
python tools/k1_modes.py --layers 58 --experts 256 --modes 0,6 >> gpurun_out/k1m.txt 2>&1
cat gpurun_out/k1m.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk_hist_cta" > gpurun_out/race_k1.log 2>&1; grep -E "SUMMARY|passed" gpurun_out/race_k1.log
