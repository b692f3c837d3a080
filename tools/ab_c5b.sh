cd $GRAFT_REPO_ROOT
O=gpurun_out/abc5b; mkdir -p $O
nproc > $O/nproc.txt
for sch in spin yield; do
for w in 4 6 8; do
  SF_SCHED=$sch timeout 900 python bench.py --config C5 --steps 7 --warmup 1 --workers $w > $O/${sch}_w$w.json 2> $O/${sch}_w$w.err
  echo "$sch w$w $(python -c "
import json; l=[x for x in open('$O/${sch}_w$w.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(round(d['value']))") $(grep 'step seconds' $O/${sch}_w$w.err)"
done; done
cat $O/nproc.txt
