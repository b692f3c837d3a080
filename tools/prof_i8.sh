cd $GRAFT_REPO_ROOT
export SF_AB_REPS=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bitmat|digits_kernel|absmax_partial|list_forward|list_transpose|nib_forward|nib_transpose|transpose_finish" -c 120 --csv --log-file gpurun_out/i8_launches.csv python tools/cgls_ab.py C2 > gpurun_out/i8_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bitmat_i8_kernel" --launch-skip 4 -c 2 -o gpurun_out/i8_full python tools/cgls_ab.py C2 > gpurun_out/i8_full.log 2>&1
ls -la gpurun_out/
