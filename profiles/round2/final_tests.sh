#!/bin/bash
# Closing GPU test suite on a 2-GPU lease
O=gpurun_out/closing_tests; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
