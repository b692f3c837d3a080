"""SF_TIMING laps of one C2 explain_node (after a warm-up call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22668_b200 as sf  # noqa: E402
from paper_2506_22668_b200 import workloads as W  # noqa: E402
from paper_2506_22668_b200.api import ExplainOptions  # noqa: E402

ctx = sf.Context(0)
d = W.build(sys.argv[1] if len(sys.argv) > 1 else "C2")
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
opts = ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed)
ctx.explain_node(g, m, d["target"], opts)
print("=== timed", flush=True)
ex = ctx.explain_node(g, m, d["target"], opts)
print(ex.timings, flush=True)
