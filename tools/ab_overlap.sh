cd $GRAFT_REPO_ROOT
for ov in 1 0; do
  SF_CGLS_OVERLAP=$ov timeout 600 python tools/cgls_ab.py C2 > gpurun_out/ov$ov.json 2> gpurun_out/ov$ov.err
  cat gpurun_out/ov$ov.json; tail -n 3 gpurun_out/ov$ov.err
done
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_explain.py -x -q > gpurun_out/ov_tests.log 2>&1; tail -3 gpurun_out/ov_tests.log
