# overlap test: i8 forward beside the nibble forward (SF_CGLS_BOTH=1) vs each alone
cd $GRAFT_REPO_ROOT
O=gpurun_out/abboth; mkdir -p $O
for v in "base" "SF_CGLS_BOTH=1" "SF_CGLS_I8=1"; do
  if [ "$v" = base ]; then e=""; else e="$v"; fi
  env $e SF_CGLS_GRAPH=0 timeout 600 python tools/cgls_ab.py C2 > "$O/$(echo $v | tr ' =' '__').json" 2>&1
  echo "$v: $(tail -n 1 "$O/$(echo $v | tr ' =' '__').json")"
done
SF_CGLS_BOTH=1 SF_CGLS_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bitmat|nib_forward_kernel" -c 12 --csv python tools/cgls_ab.py C2 2>/dev/null | grep -E "bitmat|nib_forward" | awk -F'","' '{print $5, $NF}' | cut -c1-60,200- | tail -12
