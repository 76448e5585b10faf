#!/usr/bin/env bash
# One ncu --set full capture per hot kernel (one launch each) + the bench launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on -c 1"
$N -k regex:topk_hist -o gpurun_out/ncu/k1 python tools/kbench.py hist --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:gram_tc -o gpurun_out/ncu/k2 python tools/kbench.py gram --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:maxkey -o gpurun_out/ncu/k5 python tools/kbench.py score --cands 10000 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:approx_scan5 -o gpurun_out/ncu/k6 python tools/kbench.py swap --runs 592 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:greedy2 -o gpurun_out/ncu/k7 python bench.py --steps 1 --warmup 3 --no-candidates --no-e2e --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/ncu
