# fp16x2 fused kernel (SF_FUSED_TC16=1) vs 3xTF32 at C2 / C3 / C4
cd $GRAFT_REPO_ROOT
O=gpurun_out/abtc16; mkdir -p $O
for v in 0 1; do
  SF_FUSED_TC16=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_$v.json 2>&1
  SF_FUSED_TC16=$v timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_$v.json 2>&1
  SF_FUSED_TC16=$v timeout 1200 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/c4_$v.json 2>&1
done
for f in $O/*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$f', round(d.get('value',0)), d.get('stage_ms_per_step'), (d.get('config') or {}).get('accuracy_mode'))"; done
