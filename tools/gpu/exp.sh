cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "search or greedy or config_slice" > gpurun_out/pytest_k7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k7.log
tail -2 gpurun_out/pytest_k7.log
for m in a; do
  if [ $m = b ]; then export GEM_GREEDY_NOPART=1; else unset GEM_GREEDY_NOPART; fi
  GEM_SEARCH_TRACE=1 timeout 900 python bench.py --config deepseek-v3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-coselect --no-candidates > gpurun_out/tr_$m.json 2> gpurun_out/tr_$m.err
  echo "$m $(grep greedy gpurun_out/tr_$m.err | sed -n 2p) $(python -c "
import json
d=json.loads(open('gpurun_out/tr_$m.json').read().strip().splitlines()[-1]); print(d['time_to_mapping']['value'], d['time_to_mapping']['aggregate_score'])")"
done
