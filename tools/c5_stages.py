"""Per-stage times of C5 targets (one worker, 64 targets): where a batch
target's ~1 ms goes."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

ctx = sf.Context(0)
d = W.build("C5")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
targets = g.select_nodes("degree-range:[4,12]:1024")[:64]
opts = ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed)
for t in targets[:4]:
    ctx.explain_node(g, m, t, opts)
rows = []
t0 = time.perf_counter()
for t in targets:
    ex = ctx.explain_node(g, m, t, opts)
    rows.append([ex.timings[k] for k in ("extract_ms", "setup_ms", "sampling_ms", "prediction_ms", "solve_ms",
                                         "fidelity_ms", "total_ms")] + [len(ex.phi), ex.iterations])
wall = (time.perf_counter() - t0) / len(targets) * 1e3
a = np.array(rows)
print("mean ms: extract %.3f setup %.3f sampling %.3f prediction %.3f solve %.3f fidelity %.3f total %.3f; "
      "wall %.3f; mean n %.0f, iterations %.1f" % tuple(list(a.mean(0)[:7]) + [wall] + list(a.mean(0)[7:])))
order = np.argsort(-a[:, 1])
print("largest setup_ms (setup, solve, n, iterations):")
for i in order[:8]:
    print("  %.3f %.3f n=%d it=%d" % (a[i, 1], a[i, 4], a[i, 7], a[i, 8]))
print("median setup %.3f solve %.3f" % (np.median(a[:, 1]), np.median(a[:, 4])))
