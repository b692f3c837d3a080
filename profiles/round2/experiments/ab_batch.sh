# Inference batch budget (SF_BATCH_MB) and tail A/B at C3 / C4, then the nibble-kernel variants
cd $GRAFT_REPO_ROOT
O=gpurun_out/abbatch; mkdir -p $O
for mb in 768 3072 8192; do
  for t in 0 1; do
    SF_BATCH_MB=$mb SF_TAIL_TC=$t timeout 900 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_mb${mb}_t$t.json 2>&1
  done
done
for mb in 768 2048; do
  for t in 0 1; do
    SF_BATCH_MB=$mb SF_TAIL_TC=$t timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_mb${mb}_t$t.json 2>&1
  done
done
for mb in 768 2048; do
  SF_BATCH_MB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_mb$mb.json 2>&1
done
for f in $O/*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]) if l else {}; print('$f', d.get('value'), d.get('ms_per_step'), d.get('stage_ms_per_step'), (d.get('device_memory_gb') or {}).get('used'))"; done
bash tools/ab_nib.sh
