#!/bin/bash
# Closing ncu evidence on one GPU (after the same commands exited 0 without ncu)
O=gpurun_out/closing_ncu; mkdir -p $O
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_value.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_value.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_value.log 2>&1
SF_EXPLAIN_REPEAT=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_explain.csv \
  python bench.py --explain-only --no-cpu-baseline > $O/ncu_explain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fused_tc_kernel|isd_kernel|tail_tc_kernel|tail_finish|floyd_kernel|transpose_pairs" \
  --launch-skip 3 --launch-count 12 -o $O/kernels_value python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_value.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"nib_forward_kernel|nib_transpose_kernel|list_forward|list_transpose|tiles_word_major|transpose_tiles" \
  --launch-skip 20 --launch-count 8 -o $O/kernels_cgls python bench.py --explain-only --no-cpu-baseline > $O/ncu_full_cgls.log 2>&1
echo done > $O/done
