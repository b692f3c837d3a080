"""Direct (tcgen05 Gram + device Cholesky) vs CGLS inside explain_node:
solve-stage time and phi agreement across player counts, to set the
SF_SOLVER_AUTO threshold. Targets are taken from the C5 graph (2-layer) and
C1-like densities by ball size. Prints one JSON line per target."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

d = W.build("C5")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
ctx = sf.Context(0)
rp, _ = g.csr()
deg = np.diff(rp)
want = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "30,60,120,250,500,1000,2000,3000".split(","))]
cands = np.nonzero(deg > 0)[0][:6000]
sizes = {}
for c in cands:
    sizes[int(c)] = g.extract(int(c), 2).n
picked = []
for w in want:
    best = min(sizes, key=lambda c: abs(sizes[c] - w))
    picked.append(best)
k = int(os.environ.get("SF_XOVER_K", "100000"))
for node in picked:
    out = {"node": node, "n": sizes[node], "k": k}
    res = {}
    for mode, name in ((0, "cgls"), (2, "direct")):
        opts = ExplainOptions(samples=k, seed=1, fidelity=False, solver_mode=mode)
        ctx.explain_node(g, m, node, opts)  # warm
        ts = []
        for _ in range(3):
            ex = ctx.explain_node(g, m, node, opts)
            ts.append(ex.timings["solve_ms"])
        res[name] = ex
        out[name + "_solve_ms"] = float(np.median(ts))
        out[name + "_total_ms"] = ex.timings["total_ms"]
    a, b = res["cgls"].phi, res["direct"].phi
    out["rel_l2"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))
    out["top10_same"] = [p for p, _ in res["cgls"].top] == [p for p, _ in res["direct"].top]
    out["cgls_iterations"] = res["cgls"].iterations
    print(json.dumps(out), flush=True)
