"""Diagnostic: GPU CGLS (fast loop, two-sync loop via trace, fixed order) vs
the bit-row restatement on the C2 explain system, after K steps each."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from oracle.pyoracle import Port  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

port = Port()
ctx = sf.Context(0)
d = W.build("C2")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
t = d["target"]
ctx.keep_stages(True)
ex = ctx.explain_node(g, m, t, ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False))
preds = ctx.stage_predictions()
sg = g.extract(t, cfg.hops)
n = sg.n
plan = sf.plan_sizes(n, cfg.samples, True)
bits, ros = ctx.generate_masks(plan, sf.node_sampling_seed(cfg.explain_seed, t))
w = sf.assemble_weights(n, bits, ros)
tg = preds.astype(np.float64) - ex.base_score
ct = ex.full_score - ex.base_score
print("explain iterations", ex.iterations, "residual", ex.residual, flush=True)
for K in (1, 2, 5, 10, 15, 20, 23, 24, 30):
    a = ctx.solve_cgls(n, bits, w, tg, ct, 1e6, tol=0.0, max_iter=K)
    b = ctx.solve_cgls(n, bits, w, tg, ct, 1e6, tol=0.0, max_iter=K, trace=True)
    p = port.cgls_sparse(n, bits, ros, preds.astype(np.float64), ex.base_score, ex.full_score, tol=0.0, max_iter=K)
    e = lambda x, y: float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))
    print(f"K={K:3d} fast-vs-port {e(a['phi'], p[0]):.3g}  trace-vs-port {e(b['phi'], p[0]):.3g}  "
          f"fast-vs-trace {e(a['phi'], b['phi']):.3g}  res gpu {a['relative_residual']:.4g} port {p[2]:.4g}", flush=True)
