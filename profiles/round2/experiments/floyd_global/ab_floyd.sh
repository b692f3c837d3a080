# C4 global-memory Floyd: CTAs per SM (4 warps each) vs the sampling time
cd $GRAFT_REPO_ROOT
O=gpurun_out/abfloyd; mkdir -p $O
for g in 16 8 4 2 1; do
  SF_FLOYD_GBLOCKS=$g timeout 900 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/g$g.json 2>&1
  echo "g$g $(python -c "
import json; l=[x for x in open('$O/g$g.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(round(d['value']), d['stage_ms_per_step'])")"
done
