"""A/B of the CGLS dense-pair passes (SF_CGLS_I8=1 tensor-core i8 vs 0
nibble tables) on the C2 explain system: device-resident masks, the
explain's own predictions; phi vs the bit-row restatement after the same
number of steps, and solve wall time (host round trip per iteration
included)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
ctx = sf.Context(0)
d = W.build(name)
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
t = d["target"]
ctx.keep_stages(True)
ex = ctx.explain_node(g, m, t, ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False))
preds = ctx.stage_predictions()
ctx.keep_stages(False)
n = len(ex.phi)
plan = sf.plan_sizes(n, cfg.samples, True)
nseed = sf.node_sampling_seed(cfg.explain_seed, t)
dm = ctx.masks_device(plan, nseed)
out = dict(mode=os.environ.get("SF_CGLS_I8", "1"), n=n, explain_iterations=ex.iterations,
           explain_residual=ex.residual)
times = []
for rep in range(4):
    t0 = time.perf_counter()
    r = dm.solve(preds, ex.base_score, ex.full_score)
    times.append(time.perf_counter() - t0)
out.update(solve_ms=[round(1e3 * x, 2) for x in times], iterations=r["iterations"], residual=r["relative_residual"])
fixed = dm.solve(preds, ex.base_score, ex.full_score, tol=0.0, max_iter=20)
np.save(f"gpurun_out/ab_phi_{out['mode']}.npy", r["phi"])
np.save(f"gpurun_out/ab_phi20_{out['mode']}.npy", fixed["phi"])
if os.environ.get("SF_AB_PORT"):
    from oracle.pyoracle import Port
    port = Port()
    bits, ros = ctx.generate_masks(plan, nseed)
    p = port.cgls_sparse(n, bits, ros, preds.astype(np.float64), ex.base_score, ex.full_score, tol=0.0, max_iter=20)
    out["phi20_vs_port"] = float(np.linalg.norm(fixed["phi"] - p[0]) / np.linalg.norm(p[0]))
    p = port.cgls_sparse(n, bits, ros, preds.astype(np.float64), ex.base_score, ex.full_score, tol=1e-6)
    out["phi_vs_port"] = float(np.linalg.norm(r["phi"] - p[0]) / np.linalg.norm(p[0]))
    out["port_iterations"] = p[1]
print(json.dumps(out))
