# DEG staging lookups: shared-memory table (base) vs __ldg global table (.scratch/degldg), C2 with u16 forced and C3
cd $GRAFT_REPO_ROOT
O=gpurun_out/abdeg; mkdir -p $O
LIB=paper_2506_22668_b200/libshapflow_b200.so
cp $LIB $O/base.so
for v in base degldg; do
  if [ "$v" = base ]; then cp $O/base.so $LIB; else cp .scratch/$v/libshapflow_b200.so $LIB; fi
  SF_ISD_U16=1 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2u_$v.json 2>&1
  timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_$v.json 2>&1
done
cp $O/base.so $LIB; rm -f $O/base.so
SF_ISD_U16=0 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_f32.json 2>&1
for f in $O/*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$f', round(d.get('value',0)), d.get('stage_ms_per_step'))"; done
