#!/bin/bash
# Final 1-GPU measurements and evidence (gpurun). Lines land in gpurun_out/final/.
O=gpurun_out/final; mkdir -p $O
timeout 900 python bench.py --steps 10 --warmup 3 > $O/c2_n1.json 2> $O/c2_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/c2_ref.json 2> $O/c2_ref.err
timeout 900 python bench.py --config C1 --steps 10 --warmup 3 > $O/c1_n1.json 2> $O/c1_n1.err
timeout 900 python bench.py --config C1 --impl reference --steps 3 --warmup 3 > $O/c1_ref.json 2> $O/c1_ref.err
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 > $O/c5_n1.json 2> $O/c5_n1.err
timeout 1500 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline > $O/c4_n1.json 2> $O/c4_n1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_value.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_value.log 2>&1
SF_EXPLAIN_REPEAT=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_explain.csv \
  python bench.py --explain-only --no-cpu-baseline > $O/ncu_explain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fused_tc_kernel|isd_kernel|tail_tc_kernel|tail_finish|floyd_kernel|transpose_pairs" \
  --launch-skip 3 --launch-count 12 -o $O/kernels_value python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_value.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"floyd_kernel" --launch-skip 1 --launch-count 1 \
  -o $O/kernels_floyd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_floyd.log 2>&1
echo done > $O/single_done
