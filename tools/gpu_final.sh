#!/usr/bin/env bash
# Round-end evidence in one gpurun call: GPU tests, smoke, bench (ours + reference arm),
# every BASELINE config, K5 ncu captures (C4 and C5 shapes) and the bench launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final gpurun_out/sweep
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
bash tools/config_sweep.sh > $O/sweep.txt 2>&1
R=/tmp/ncu_reps; mkdir -p $R
N="timeout 900 ncu --set full --clock-control none --import-source on -c 1"
$N -k regex:maxkey -o $R/k5 python bench.py --no-search --no-e2e --no-coselect --no-cpu --steps 1 --warmup 0 > /dev/null 2>&1
$N -k regex:keysum -o $R/k5s python bench.py --no-search --no-e2e --no-coselect --no-cpu --steps 1 --warmup 0 > /dev/null 2>&1
$N -k regex:maxkey -o $R/k5c5 python bench.py --config deepseek-v3 --no-search --no-e2e --no-coselect --no-cpu --steps 1 --warmup 0 > /dev/null 2>&1
$N -k regex:keysum -o $R/k5sc5 python bench.py --config deepseek-v3 --no-search --no-e2e --no-coselect --no-cpu --steps 1 --warmup 0 > /dev/null 2>&1
for k in k5 k5s k5c5 k5sc5; do
  [ -f $R/$k.ncu-rep ] && python tools/ncu_summary.py $R/$k.ncu-rep > $O/ncu_$k.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt 2>&1
rm -f $O/launches.csv
tail -2 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/sweep.txt | tail -7; ls $O
