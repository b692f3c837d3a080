# C2 e2e with host vs device subgraph extraction
cd $GRAFT_REPO_ROOT
O=gpurun_out/abext; mkdir -p $O
for m in host device; do
  SF_EXTRACT=$m timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/$m.json 2>&1
  python -c "
import json; l=[x for x in open('$O/$m.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); t=d['e2e']['timings_ms']; print('$m', round(d['e2e']['value']), {k:round(v,2) for k,v in t.items()})"
done
