cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "search or greedy or refine or config_slice or fullsize or reference_suite_with" > gpurun_out/pytest_k6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6.log
tail -2 gpurun_out/pytest_k6.log
for c in deepseek-v3 qwen3-235b; do
GEM_SEARCH_TRACE=1 timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e --no-coselect --no-candidates > gpurun_out/tr_$c.json 2> gpurun_out/tr_$c.err
echo "$c $(grep 'round 0:' gpurun_out/tr_$c.err | sed -n 2p) $(python -c "
import json
d=json.loads(open('gpurun_out/tr_$c.json').read().strip().splitlines()[-1]); print(d['time_to_mapping']['value'], d['time_to_mapping']['aggregate_score'], d['time_to_mapping_w16']['value'], d['time_to_mapping_w16']['aggregate_score'])")"
done
