"""SF_TIMING laps for two C5 targets (after warm-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

ctx = sf.Context(0)
d = W.build("C5")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
targets = g.select_nodes("degree-range:[4,12]:1024")[:8]
opts = ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed)
for t in targets[:6]:
    ctx.explain_node(g, m, t, opts)
print("=== timed", flush=True)
sys.stderr.flush()
for t in targets[6:8]:
    ex = ctx.explain_node(g, m, t, opts)
    print(ex.timings, len(ex.phi), ex.iterations, flush=True)
