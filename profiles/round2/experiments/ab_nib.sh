# A/B of nibble-kernel occupancy variants on the C2 solve (SF_NIB_CHUNK=1024: 32 KB forward tables; SF_NIB_T4=1: transpose at 4 CTAs/SM)
cd $GRAFT_REPO_ROOT
O=gpurun_out/abnib; mkdir -p $O
for v in "base" "SF_NIB_CHUNK=1024" "SF_NIB_T4=1" "SF_NIB_CHUNK=1024 SF_NIB_T4=1"; do
  if [ "$v" = base ]; then e=""; else e="$v"; fi
  env $e timeout 600 python tools/cgls_ab.py C2 > "$O/$(echo $v | tr ' =' '__').json" 2>&1
  echo "$v: $(tail -n 1 "$O/$(echo $v | tr ' =' '__').json")"
done
