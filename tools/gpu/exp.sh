# scratch experiment driver for gpurun (edited per call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_coselect.py tests/test_gpu_parity.py -q -x -k "topk_hist or stats or planted or heavy" > gpurun_out/exp_test.log 2>&1; echo "rc=$?" >> gpurun_out/exp_test.log
tail -5 gpurun_out/exp_test.log
for v in "" noheavy2; do GEM_LIB_VARIANT=$v timeout 120 python tools/kbench.py hist --reps 20; done

timeout 120 python tools/kbench.py hist --reps 10 --layers 58 --experts 256
