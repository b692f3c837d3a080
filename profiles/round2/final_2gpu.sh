#!/bin/bash
# Final 2-GPU lease: the whole GPU suite, then the configs whose tail
# dispatch changed (C3, C4) and C5 at 1 and 2 GPUs. Lines in gpurun_out/final2/.
O=gpurun_out/final2; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
run() {  # run <name> <ngpus> <args...>
  local name=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 1500 python bench.py --gpus 1 "$@" > $O/$name.json 2> $O/$name.err
  else
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  fi
}
run c3_n1 1 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c3_n2 2 --config C3 --steps 3 --warmup 3 --no-cpu-baseline
run c4_n1 1 --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline
run c4_n1_k125 1 --config C4 --samples 1250000 --steps 2 --warmup 3 --no-cpu-baseline
run c5_n1 1 --config C5 --steps 2 --warmup 1
run c5_n2 2 --config C5 --steps 2 --warmup 1
echo done > $O/done
