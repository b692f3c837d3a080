#!/bin/bash
# Re-measure after the tail dispatch / nibble occupancy changes; lines in gpurun_out/final3/
O=gpurun_out/final3; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_gcn.py tests/test_gpu_parity_scale.py tests/test_gpu_explain.py -q -x -k "not two_gpu" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/c2_n1.json 2> $O/c2_n1.err
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > $O/c3_n1.json 2> $O/c3_n1.err
timeout 1500 python bench.py --config C4 --samples 1000000 --steps 2 --warmup 3 --no-cpu-baseline > $O/c4_n1.json 2> $O/c4_n1.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 1 > $O/c5_n1.json 2> $O/c5_n1.err
timeout 900 python bench.py --config C1 --steps 10 --warmup 3 > $O/c1_n1.json 2> $O/c1_n1.err
echo done > $O/done
