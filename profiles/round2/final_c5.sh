#!/bin/bash
# C5 at 1/2/4 GPUs, 6 workers per GPU (bench default), 9 steps; also 4 workers spinning for comparison
O=gpurun_out/final6; mkdir -p $O
nproc > $O/nproc.txt
run() {
  local name=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then timeout 900 python bench.py --gpus 1 "$@" > $O/$name.json 2> $O/$name.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err; fi
}
for n in 1 2 4; do
  run c5_n$n $n --config C5 --steps 9 --warmup 1
  SF_SCHED=spin run c5_n${n}_w4spin $n --config C5 --steps 9 --warmup 1 --workers 4
done
echo done > $O/done
