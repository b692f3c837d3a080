# CUDA-graph CGLS iteration (SF_CGLS_GRAPH) A/B: C5 targets/s, C1 and C2 e2e; solver/explain tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/abgraph; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_explain.py -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
for gph in 1 0; do
  SF_CGLS_GRAPH=$gph timeout 600 python bench.py --config C5 --steps 7 --warmup 1 > $O/c5_g$gph.json 2> $O/c5_g$gph.err
  SF_CGLS_GRAPH=$gph timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/c1_g$gph.json 2>&1
  SF_CGLS_GRAPH=$gph timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/c2_g$gph.json 2>&1
  SF_CGLS_GRAPH=$gph timeout 600 python tools/c5_stages.py > $O/c5stages_g$gph.txt 2>&1
done
for f in $O/c*_g*.json; do python -c "
import json; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; e=d.get('e2e') or {}
print('$f', round(d.get('value',0)), e.get('value'), (e.get('timings_ms') or {}).get('solve_ms'))"; done
grep "step seconds" $O/*.err; head -1 $O/c5stages_g1.txt; head -1 $O/c5stages_g0.txt
