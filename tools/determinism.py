"""Run C2 explain_node twice in one process and save phi: bitwise run-to-run
determinism of the default (non fixed-order) path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

ctx = sf.Context(0)
d = W.build("C2")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
phis, preds = [], []
for rep in range(3):
    ctx.keep_stages(True)
    ex = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False))
    preds.append(ctx.stage_predictions().copy())
    ctx.keep_stages(False)
    phis.append(ex.phi.copy())
    print(rep, ex.iterations, ex.residual, flush=True)
for rep in (1, 2):
    print("phi equal", np.array_equal(phis[0], phis[rep]), "max", float(np.max(np.abs(phis[0] - phis[rep]))),
          "preds equal", np.array_equal(preds[0], preds[rep]), float(np.max(np.abs(preds[0] - preds[rep]))))
np.save(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/det_phi.npy", phis[0])
