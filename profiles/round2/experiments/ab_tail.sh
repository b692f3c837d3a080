# A/B of the tcgen05 tail (SF_TAIL_TC) at C2 / C3 / C4, plus the explain-path tests (in-place rT)
cd $GRAFT_REPO_ROOT
O=gpurun_out/abtail; mkdir -p $O
for t in 1 0; do
  SF_TAIL_TC=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_t$t.json 2>$O/c2_t$t.err
  SF_TAIL_TC=$t timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_t$t.json 2>$O/c3_t$t.err
  SF_TAIL_TC=$t timeout 1200 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_t$t.json 2>$O/c4_t$t.err
done
timeout 1500 python bench.py --config C4 --samples 1250000 --steps 2 --warmup 3 --no-cpu-baseline > $O/c4_k125.json 2>$O/c4_k125.err
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_explain.py -x -q -k "not two_gpu" > $O/tests.log 2>&1
for f in $O/*.json; do echo $f; python -c "
import json,sys; l=[x for x in open('$f').read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]) if l else {}; print(d.get('value'), d.get('ms_per_step'), d.get('stage_ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('device_memory_gb'))"; done
tail -3 $O/tests.log
