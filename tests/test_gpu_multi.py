"""GPU, N > 1: explain_node collective over NCCL (one process per GPU,
torchrun). Every rank must return the same phi, and it must match the
single-GPU result and the reference within the BASELINE bar. Skipped when the
box has fewer than two GPUs (run with `gpurun --gpus 2`)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["SF_ROOT"])
import numpy as np
import torch.distributed as dist
import paper_2506_22668_b200 as sf
from paper_2506_22668_b200 import workloads as W
from paper_2506_22668_b200.api import ExplainOptions
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = sf.Context(local)
obj = [sf.Context.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx.join(obj[0], rank, world)
d = W.build("C1"); cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
ex = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed))
st = ctx.stats()
fx = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, solver_mode=1,
                                                        fidelity=False))
st2 = ctx.stats()
out = {"rank": rank, "phi": ex.phi.tolist(), "iterations": ex.iterations, "top": [p for p, _ in ex.top],
       "converged": ex.converged, "stats": st, "fid": ex.fidelity["plus"].tolist(),
       "fused_phi": fx.phi.tolist(), "fused_iterations": fx.iterations,
       "fused_vec": st2["vector_allreduce"] - st["vector_allreduce"],
       "fused_scalar": st2["scalar_allreduce"] - st["scalar_allreduce"]}
with open(os.path.join(os.environ["SF_OUT"], f"rank{rank}.json"), "w") as f:
    json.dump(out, f)
ctx.close()
dist.barrier()
dist.destroy_process_group()
"""


def _gpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
def test_two_gpu_explain_matches_single(tmp_path, ctx, ref):
    world = 2
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, SF_ROOT=ROOT, SF_OUT=str(tmp_path))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                   check=True, env=env, timeout=600)
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    assert res[0]["phi"] == res[1]["phi"]  # replicated, bitwise
    # single GPU and the reference
    import paper_2506_22668_b200 as sf
    from paper_2506_22668_b200 import workloads as W
    from paper_2506_22668_b200.api import ExplainOptions

    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    one = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed))
    phi2 = np.array(res[0]["phi"])
    assert np.linalg.norm(phi2 - one.phi) <= 1e-9 * np.linalg.norm(one.phi)
    assert res[0]["top"] == [p for p, _ in one.top]
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    rx = ref.explain_node(rg, rm, d["target"], samples=cfg.samples, seed=cfg.explain_seed, world=2)
    assert np.linalg.norm(phi2 - rx["phi"]) <= 1e-3 * np.linalg.norm(rx["phi"])
    # reference protocol on every rank: one scalar + one vector all-reduce per iteration (+1 vector)
    for r in res:
        it = r["iterations"]
        assert r["stats"]["scalar_allreduce"] >= it and r["stats"]["vector_allreduce"] >= it + 1
    # fused protocol: one (n+1)-double all-reduce per iteration (+1 at init), replicated phi
    assert res[0]["fused_phi"] == res[1]["fused_phi"]
    fphi = np.array(res[0]["fused_phi"])
    assert np.linalg.norm(fphi - rx["phi"]) <= 1e-3 * np.linalg.norm(rx["phi"])
    for r in res:
        assert r["fused_vec"] == r["fused_iterations"] + 1 and r["fused_scalar"] == 0
