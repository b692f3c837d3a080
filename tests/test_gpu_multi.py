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
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    rx = ref.explain_node(rg, rm, d["target"], samples=cfg.samples, seed=cfg.explain_seed, world=2)
    e_ref = np.linalg.norm(phi2 - rx["phi"]) / np.linalg.norm(rx["phi"])
    e_one = np.linalg.norm(phi2 - one.phi) / np.linalg.norm(one.phi)
    e_one_ref = np.linalg.norm(one.phi - rx["phi"]) / np.linalg.norm(rx["phi"])
    diag = (f"2-GPU vs ref {e_ref:.3g}, vs 1-GPU {e_one:.3g}, 1-GPU vs ref {e_one_ref:.3g}; iterations "
            f"2-GPU {res[0]['iterations']} 1-GPU {one.iterations} ref {rx['iterations']}")
    print(diag)
    assert e_ref <= 1e-3, diag
    assert e_one <= 1e-3, diag
    assert res[0]["top"] == [p for p, _ in one.top], diag
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


SOLVE_WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["SF_ROOT"])
import numpy as np
import torch.distributed as dist
import paper_2506_22668_b200 as sf
from oracle.pyoracle import Port
sys.path.insert(0, os.path.join(os.environ["SF_ROOT"], "tests"))
from test_gpu_solver import toy_game_values
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = sf.Context(local)
obj = [sf.Context.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx.join(obj[0], rank, world)
port = Port()
out = {}
for mode in (0, 1):
    n = 999
    p = sf.plan_sizes(n, 10000, False)
    bits, ros = ctx.generate_masks(p, 5, rank, world)
    vals = toy_game_values(bits, port)
    w = sf.assemble_weights(n, bits, ros)
    r = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6, mode=mode)
    out[mode] = {"phi": r["phi"].tolist(), "iterations": int(r["iterations"])}
with open(os.path.join(os.environ["SF_OUT"], f"solve{rank}.json"), "w") as f:
    json.dump(out, f)
ctx.close()
dist.barrier()
dist.destroy_process_group()
"""


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
def test_two_gpu_sharded_solve_matches_single(tmp_path, ctx, port):
    """The rank-sharded CGLS (rows g mod 2, NCCL all-reduces, both
    protocols) against the single-GPU solve of the whole problem."""
    import paper_2506_22668_b200 as sf
    from test_gpu_solver import toy_game_values

    world = 2
    script = tmp_path / "solve_worker.py"
    script.write_text(SOLVE_WORKER)
    env = dict(os.environ, SF_ROOT=ROOT, SF_OUT=str(tmp_path))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", "29534", str(script)],
                   check=True, env=env, timeout=600)
    res = [json.load(open(tmp_path / f"solve{r}.json")) for r in range(world)]
    n = 999
    p = sf.plan_sizes(n, 10000, False)
    bits, ros = ctx.generate_masks(p, 5)
    vals = toy_game_values(bits, port)
    w = sf.assemble_weights(n, bits, ros)
    for mode in ("0", "1"):
        assert res[0][mode]["phi"] == res[1][mode]["phi"]
        one = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6, mode=int(mode))
        two = np.array(res[0][mode]["phi"])
        err = np.linalg.norm(two - one["phi"]) / np.linalg.norm(one["phi"])
        diag = f"mode {mode}: rel {err:.3g}, iterations 2-GPU {res[0][mode]['iterations']} 1-GPU {one['iterations']}"
        print(diag)
        assert err <= 1e-6, diag


PRED_WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["SF_ROOT"])
import numpy as np
import torch.distributed as dist
import paper_2506_22668_b200 as sf
from paper_2506_22668_b200 import workloads as W
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = sf.Context(local)
d = W.build("C1"); cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
sg = g.extract(d["target"], cfg.hops)
p = sf.plan_sizes(sg.n, cfg.samples, True)
seed = sf.node_sampling_seed(cfg.explain_seed, d["target"])
bits, _ = ctx.generate_masks(p, seed, rank, world)
pred = ctx.predict_batched(m, sg, bits, 2)
np.save(os.path.join(os.environ["SF_OUT"], f"pred{rank}.npy"), pred)
np.save(os.path.join(os.environ["SF_OUT"], f"bits{rank}.npy"), bits)
ctx.close()
dist.barrier()
dist.destroy_process_group()
"""


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
def test_two_gpu_shard_predictions_match_single(tmp_path, ctx):
    """Each rank's masks and predictions equal the single-GPU rows of the
    same global pairs (pair g -> rank g mod world, sampler.cpp:177-178)."""
    import paper_2506_22668_b200 as sf
    from paper_2506_22668_b200 import workloads as W

    world = 2
    script = tmp_path / "pred_worker.py"
    script.write_text(PRED_WORKER)
    env = dict(os.environ, SF_ROOT=ROOT, SF_OUT=str(tmp_path))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", "29535", str(script)],
                   check=True, env=env, timeout=600)
    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    sg = g.extract(d["target"], cfg.hops)
    p = sf.plan_sizes(sg.n, cfg.samples, True)
    seed = sf.node_sampling_seed(cfg.explain_seed, d["target"])
    bits, _ = ctx.generate_masks(p, seed)
    pred = ctx.predict_batched(m, sg, bits, 2)
    for r in range(world):
        rb = np.load(tmp_path / f"bits{r}.npy")
        rp = np.load(tmp_path / f"pred{r}.npy")
        rows = np.concatenate([[2 * g_, 2 * g_ + 1] for g_ in range(r, bits.shape[0] // 2, world)])
        assert np.array_equal(rb, bits[rows])
        bad = np.nonzero(rp != pred[rows])[0]
        assert bad.size == 0, f"rank {r}: {bad.size} predictions differ, first rows {bad[:8]}, " \
                              f"max rel {np.max(np.abs(rp - pred[rows]) / np.abs(pred[rows])):.3g}"


TIMEOUT_WORKER = r"""
import json, os, sys, time
sys.path.insert(0, os.environ["SF_ROOT"])
import torch.distributed as dist
import paper_2506_22668_b200 as sf
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = sf.Context(local)
obj = [sf.Context.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx.join(obj[0], rank, world)
ctx.barrier()  # both ranks: a normal collective first
dist.barrier()
out = {"rank": rank}
if rank == 0:
    ctx.set_comm_timeout(3000)
    t0 = time.time()
    try:
        ctx.barrier()  # rank 1 never joins this one
        out["error"] = None
    except sf.ProtocolError as e:
        out["error"] = str(e)
    out["waited_s"] = time.time() - t0
else:
    time.sleep(6)
with open(os.path.join(os.environ["SF_OUT"], f"timeout{rank}.json"), "w") as f:
    json.dump(out, f)
dist.barrier()
os._exit(0)  # the aborted communicator is not torn down again
"""


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
def test_collective_timeout_raises_protocol_error(tmp_path):
    """A rank that never enters a collective: the waiting rank aborts its
    NCCL communicator after the configured timeout and raises ProtocolError
    (the reference Communicator's kDefaultCommTimeout behaviour,
    comm.hpp:54) instead of hanging."""
    world = 2
    script = tmp_path / "timeout_worker.py"
    script.write_text(TIMEOUT_WORKER)
    env = dict(os.environ, SF_ROOT=ROOT, SF_OUT=str(tmp_path))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", "29537", str(script)],
                   check=True, env=env, timeout=300)
    r0 = json.load(open(tmp_path / "timeout0.json"))
    assert r0["error"] and "timed out" in r0["error"]
    assert 2.5 <= r0["waited_s"] <= 30
