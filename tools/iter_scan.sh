#!/usr/bin/env bash
# K6 iteration: scan microbench (v5 vs v4), GPU tests, per-round search trace.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ python tools/kbench.py swap --runs 592 --reps 5 --warm 2
  GEM_SCAN_NOCLAMP=1 python tools/kbench.py swap --runs 592 --reps 5 --warm 2
  GEM_SCAN_V4=1 python tools/kbench.py swap --runs 592 --reps 5 --warm 2; } > gpurun_out/swap_iter.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_iter.log 2>&1
GEM_SEARCH_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-candidates --no-e2e --no-cpu > gpurun_out/trace_iter.json 2> gpurun_out/trace_iter.err
cat gpurun_out/swap_iter.json; tail -3 gpurun_out/pytest_iter.log; grep "round [0-4]:" gpurun_out/trace_iter.err | tail -5
python -c "import json;d=json.load(open('gpurun_out/trace_iter.json'));print(d['time_to_mapping'])"
