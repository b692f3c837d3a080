cd $GRAFT_REPO_ROOT
O=gpurun_out/abc5; mkdir -p $O
for w in 4 6 8 12; do
  timeout 900 python bench.py --config C5 --steps 5 --warmup 1 --workers $w > $O/w$w.json 2> $O/w$w.err
  echo "w$w $(python -c "
import json; l=[x for x in open('$O/w$w.json').read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(d['value'])") $(grep 'step seconds' $O/w$w.err)"
done
