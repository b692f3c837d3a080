#!/bin/bash
# Closing lines after the CUDA-graph CGLS iteration + the full GPU suite (4-GPU lease)
O=gpurun_out/closing3; mkdir -p $O
run() {
  local name=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then timeout 1500 python bench.py --gpus 1 "$@" > $O/$name.json 2> $O/$name.err
  else timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err; fi
}
timeout 2700 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
run c2_n1 1 --steps 10 --warmup 3
run c2_ref 1 --impl reference --steps 3 --warmup 3
run c2_n2 2 --steps 10 --warmup 3 --no-cpu-baseline
run c2_n4 4 --steps 10 --warmup 3 --no-cpu-baseline
run c1_n1 1 --config C1 --steps 10 --warmup 3
run c1_ref 1 --config C1 --impl reference --steps 3 --warmup 3
run c3_n1 1 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c3_n2 2 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c3_n4 4 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c4_n1 1 --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline
echo done > $O/done
