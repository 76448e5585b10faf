cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/config_sweep.sh > gpurun_out/sweep.txt 2>&1
tail -2 gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.json; tail -2 gpurun_out/bench.err; cat gpurun_out/sweep.txt | tail -7
