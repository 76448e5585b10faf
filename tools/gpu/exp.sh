cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize2
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --print-limit 5 python -m pytest tests/test_coselect.py -m gpu -x -q -p no:cacheprovider > gpurun_out/sanitize2/racecheck_k2b.log 2>&1
timeout 900 $CS --tool initcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "score or search_matches" > gpurun_out/sanitize2/initcheck_k5.log 2>&1
timeout 900 $CS --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "search_matches or topk_hist_cta" > gpurun_out/sanitize2/memcheck_new.log 2>&1
tail -3 gpurun_out/pytest_full.log
for f in gpurun_out/sanitize2/*.log; do echo $f; grep -E "SUMMARY|passed|failed" $f | tail -2; done
