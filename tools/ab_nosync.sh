cd $GRAFT_REPO_ROOT
O=gpurun_out/abns; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gcn.py tests/test_gpu_explain.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/c2.json 2>&1
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/c1.json 2>&1
timeout 600 python bench.py --config C5 --steps 7 --warmup 1 > $O/c5.json 2> $O/c5.err
for f in $O/*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); e=d.get('e2e') or {}
print('$f', round(d['value']), e.get('value'), (e.get('timings_ms') or {}).get('setup_ms'), (e.get('timings_ms') or {}).get('total_ms'))"; done
grep "step seconds" $O/c5.err
