#!/bin/bash
# Final multi-GPU measurements after the tail/nibble changes (gpurun --gpus 4); lines in gpurun_out/final4/
O=gpurun_out/final4; mkdir -p $O
run() {  # run <name> <ngpus> <args...>
  local name=$1 n=$2; shift 2
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
}
run c2_n2 2 --steps 10 --warmup 3 --no-cpu-baseline
run c2_n4 4 --steps 10 --warmup 3 --no-cpu-baseline
run c3_n2 2 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c3_n4 4 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c5_n2 2 --config C5 --steps 5 --warmup 1
run c5_n4 4 --config C5 --steps 5 --warmup 1
run c4_n4 4 --config C4 --samples 5000000 --steps 2 --warmup 3 --no-cpu-baseline
echo done > $O/done
