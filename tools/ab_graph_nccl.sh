# CGLS graph with NCCL all-reduces captured (SF_CGLS_GRAPH_NCCL=1) at 2 GPUs: C2 e2e and the 2-GPU parity test
cd $GRAFT_REPO_ROOT
O=gpurun_out/abgn; mkdir -p $O
for v in 0 1; do
  SF_CGLS_GRAPH_NCCL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/c2n2_g$v.json 2> $O/c2n2_g$v.err
  echo "g$v rc=$? $(python -c "
import json; l=[x for x in open('$O/c2n2_g$v.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); e=d['e2e']; print(round(d['value']), round(e['value']), e['timings_ms']['solve_ms'])")"
done
SF_CGLS_GRAPH_NCCL=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > $O/multi.log 2>&1; tail -2 $O/multi.log
