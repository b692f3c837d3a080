#!/bin/bash
# Round-2 evidence collection on one B200 (gpurun). Each ncu command runs only
# after the same program exited 0 without ncu. Outputs land in gpurun_out/.
set -x
O=gpurun_out
python -m pytest tests/test_gpu_conformance.py -q -rs -s > $O/conf_accept.log 2>&1; echo EXIT $? >> $O/conf_accept.log
python bench.py --steps 10 --warmup 3 > $O/bench_final.json 2> $O/bench_final.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_value.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_value.log 2>&1
SF_EXPLAIN_REPEAT=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_explain.csv \
  python bench.py --explain-only --no-cpu-baseline > $O/ncu_explain.log 2>&1
ncu --set full --clock-control none --import-source on \
  -k regex:"fused_tc_kernel|isd_kernel|tail_kernel|floyd_kernel|transpose_pairs" --launch-skip 40 --launch-count 10 \
  -o $O/kernels_value python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_value.log 2>&1
ncu --set full --clock-control none --import-source on \
  -k regex:"nib_forward_kernel|nib_transpose_kernel|list_forward|list_transpose|assemble_pairs|coef_kernel|transpose_tiles" \
  --launch-skip 30 --launch-count 14 -o $O/kernels_cgls python bench.py --explain-only --no-cpu-baseline > $O/ncu_full_cgls.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gram_tc_kernel|chol_update|gram_rhs" --launch-count 6 \
  -o $O/kernels_gram python profiles/solver_crossover.py 120,250 > $O/ncu_full_gram.log 2>&1
echo done
