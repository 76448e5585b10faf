#!/usr/bin/env bash
# Every BASELINE config through bench.py (short), plus the sharded code path on one GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sweep
for c in mixtral olmoe qwen3-30b qwen3-235b deepseek-v3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep/$c.json 2> gpurun_out/sweep/$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --force-dist --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep/dist.json 2> gpurun_out/sweep/dist.err
echo "force-dist rc=$?"
for f in gpurun_out/sweep/*.json; do
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split("/")[-1], "tok/s %.3g" % d["value"], "K1 frac %.3f" % d["roofline"]["frac"],
          "cand/s", d.get("candidates", {}).get("value"), "ttm", d.get("time_to_mapping", {}).get("value"),
          "agg", d.get("time_to_mapping", {}).get("aggregate_score"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
