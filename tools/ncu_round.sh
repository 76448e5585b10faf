#!/usr/bin/env bash
# One ncu --set full capture per hot kernel (one launch each) + the bench launch list,
# summarised on the box (tools/ncu_summary.py) so only small files come back.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
R=/tmp/ncu_reps; mkdir -p $R
N="timeout 900 ncu --set full --clock-control none --import-source on -c 1"
$N -k regex:topk_hist_ring -o $R/k1 python tools/kbench.py hist --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:topk_hist_creg -o $R/k1c5 python tools/kbench.py hist --layers 58 --experts 256 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:hist_heavy -o $R/k1h python tools/kbench.py hist --layers 58 --experts 256 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:gram_tc -o $R/k2 python tools/kbench.py gram --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:coselect_tc -o $R/k2b python tools/kbench.py coselect --reps 1 --warm 0 --paths gem_coselect_tc > /dev/null 2>&1
$N -k regex:maxkey -o $R/k5 python tools/kbench.py score --cands 10000 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:keysum -o $R/k5s python tools/kbench.py score --cands 10000 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:approx_scan5 -o $R/k6 python tools/kbench.py swap --runs 592 --reps 1 --warm 0 > /dev/null 2>&1
$N -k regex:greedy2 -o $R/k7 python bench.py --steps 1 --warmup 3 --no-candidates --no-e2e --no-cpu --no-coselect > /dev/null 2>&1
for k in k1 k1c5 k1h k2 k2b k5 k5s k6 k7; do
  [ -f $R/$k.ncu-rep ] && python tools/ncu_summary.py $R/$k.ncu-rep > gpurun_out/ncu/$k.json
  [ -f $R/$k.ncu-rep ] && ncu -i $R/$k.ncu-rep --page source --csv > gpurun_out/ncu/${k}_source.csv 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/ncu/launches.csv > gpurun_out/ncu/launches.txt 2>&1
ls -la gpurun_out/ncu
