# u16 degree rows (SF_ISD_U16=1) with either tail: parity + C2/C3/C4 A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/abu16; mkdir -p $O
SF_ISD_U16=1 timeout 1500 python -m pytest tests/test_gpu_gcn.py tests/test_gpu_explain.py -q -x > $O/tests_u16.log 2>&1; tail -2 $O/tests_u16.log
for u in 0 1; do
  SF_ISD_U16=$u timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_u$u.json 2>&1
  SF_ISD_U16=$u timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_u$u.json 2>&1
  SF_ISD_U16=$u timeout 1200 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/c4_u$u.json 2>&1
done
for f in $O/*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$f', round(d.get('value',0)), d.get('stage_ms_per_step'))"; done
