cd $GRAFT_REPO_ROOT
O=gpurun_out/abnib2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_sampler.py tests/test_gpu_configs.py -q -x -k "not c4" > $O/tests.log 2>&1; tail -2 $O/tests.log
SF_AB_PORT=1 timeout 600 python tools/cgls_ab.py C2 > $O/ab.json 2>&1; tail -1 $O/ab.json
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2.json 2>&1; python -c "
import json; l=[x for x in open('$O/c2.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(d['value'], d['stage_ms_per_step'])"
