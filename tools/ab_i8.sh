# A/B of the CGLS dense-pair passes: SF_CGLS_I8 = 0 (nibble tables), 1 (i8, A in TMEM), 2 (i8, A in smem)
cd $GRAFT_REPO_ROOT
for mode in 2 1 0; do
  SF_CGLS_I8=$mode SF_AB_PORT=1 timeout 600 python tools/cgls_ab.py C2 > gpurun_out/ab_mode$mode.json 2> gpurun_out/ab_mode$mode.err
  cat gpurun_out/ab_mode$mode.json; tail -n 3 gpurun_out/ab_mode$mode.err
done
SF_CGLS_I8=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bitmat|digits_kernel|nib_" -c 40 --csv --log-file gpurun_out/i8ss_launches.csv python tools/cgls_ab.py C2 > /dev/null 2>&1
