# A/B of library build variants (.scratch/<name>/libshapflow_b200.so) on the C2 value path
cd $GRAFT_REPO_ROOT
O=gpurun_out/abvar; mkdir -p $O
LIB=paper_2506_22668_b200/libshapflow_b200.so
cp $LIB $O/base.so
for v in base "$@"; do
  if [ "$v" = base ]; then cp $O/base.so $LIB; else cp .scratch/$v/libshapflow_b200.so $LIB; fi
  for rep in 1 2; do
    timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/${v}_$rep.json 2>&1
    echo "$v rep$rep $(python -c "
import json; l=[x for x in open('$O/${v}_$rep.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(round(d['value']), d['stage_ms_per_step'])")"
  done
done
cp $O/base.so $LIB
