cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
bash tools/config_sweep.sh > gpurun_out/sweep.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_c5.csv python bench.py --config deepseek-v3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-coselect --no-candidates > /dev/null 2>&1
python tools/launches.py gpurun_out/ncu/launches_c5.csv > gpurun_out/launches_c5.txt 2>&1
cat gpurun_out/sweep.txt; head -30 gpurun_out/launches_c5.txt
