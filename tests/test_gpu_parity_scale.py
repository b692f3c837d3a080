"""GPU: explain_node parity at the shapes the bench numbers are quoted on.

The reference cannot run C2/C3/C5 end to end (its dense WlsProblem alone is
100 GB at C2, and its CPU inference takes ~0.3 s per C2 coalition), so parity
is pinned stage-wise, as SURVEY.md §8(c) prescribes:

1. masks: the GPU sampler's rows for the node's seed are compared with the
   compiled reference's `generate_masks` (sampler.cpp:153-210) — every row at
   C2 and C5, rank blocks at C3;
2. predictions: the predictions explain_node actually fed to its solver
   (retained with `keep_stages`) are compared with the reference's
   `predict_batched` (gcn.cpp:259-270) on >= 256 rows spread over the whole
   batch schedule (the engine's batches hold ~8K coalitions at C2; the rows are
   k/256 apart, so every batch is sampled) — bar 1e-5 relative;
3. phi: the bit-row CGLS restatement (oracle/shapflow_port.c
   `port_cgls_sparse`, pinned to the reference's solve_cgls in
   tests/test_oracle_port.py) solves the same system from those masks and
   predictions; phi must agree within 1e-3 relative L2 (solver.cpp:158-362)
   and the top-10 must be identical (rank_edges, solver.cpp:430-440);
4. Fidelity: the reference's evaluate_fidelity (fidelity.cpp:126-162) on the
   GPU's phi must equal the GPU's Fidelity+ / Fidelity- (to float rounding of
   the predictions they come from).
"""
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2506_22668_b200 as sf
from paper_2506_22668_b200 import workloads as W
from paper_2506_22668_b200.api import ExplainOptions

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRED_RTOL = 1e-5  # BASELINE north_star
PHI_RTOL = 1e-3
TRIALS = 2  # Fidelity baseline trials (keeps the reference's CPU fidelity to ~25 masks)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


def spread_rows(rows, count=256):
    """>= count rows over [0, rows): both rows of evenly spaced pairs plus the ends."""
    pairs = np.linspace(0, rows // 2 - 1, count // 2).astype(np.int64)
    pick = np.unique(np.concatenate([2 * pairs, 2 * pairs + 1, [0, 1, rows - 2, rows - 1]]))
    return pick


def ref_predict_rows(ref, rm, rg, target, bits, cls, sgr, threads=None):
    """Reference predict_batched over the rows, split across host threads
    (ctypes releases the GIL; the reference call is reentrant)."""
    threads = threads or min(32, os.cpu_count() or 1)
    chunks = np.array_split(np.arange(bits.shape[0]), threads)
    chunks = [c for c in chunks if len(c)]
    with ThreadPoolExecutor(len(chunks)) as ex:
        outs = list(ex.map(lambda c: ref.predict_batched(rm, rg, target, bits[c], cls, sg=sgr), chunks))
    return np.concatenate(outs)


def check_stagewise(ctx, ref, port, g, rg, m, rm, target, cfg, k, seed, label, full_mask_check=True):
    opts = ExplainOptions(samples=k, seed=seed, baseline_trials=TRIALS)
    ctx.keep_stages(True)
    try:
        ex = ctx.explain_node(g, m, target, opts)
        preds = ctx.stage_predictions()
    finally:
        ctx.keep_stages(False)
    sg = g.extract(target, cfg.hops)
    sgr = ref.extract(rg, target, cfg.hops, keep_handle=True)
    try:
        n = sg.n
        assert n == sgr.n and n == len(ex.phi)
        nseed = sf.node_sampling_seed(seed, target)
        plan = sf.plan_sizes(n, k, True)
        bits, ros = ctx.generate_masks(plan, nseed)
        assert preds.shape[0] == bits.shape[0] == ex.rows
        # 1. masks
        if full_mask_check:
            want, want_ros = ref.generate_masks(n, k, nseed)
            assert np.array_equal(bits, want), f"{label}: masks differ from the reference"
            assert np.array_equal(np.asarray(ros, np.uint64), np.asarray(want_ros, np.uint64))
            del want
        # 2. predictions on a spread of rows
        pick = spread_rows(bits.shape[0])
        want_p = ref_predict_rows(ref, rm, rg, target, bits[pick], ex.predicted_class, sgr)
        perr = rel_err(preds[pick], want_p)
        assert perr <= PRED_RTOL, f"{label}: predictions off by {perr:.3g}"
        # 3. phi from the bit-row restatement fed the same masks and predictions
        phi, it, res, conv = port.cgls_sparse(n, bits, ros, preds.astype(np.float64), ex.base_score,
                                              ex.full_score, tol=1e-6)
        err = float(np.linalg.norm(ex.phi - phi) / np.linalg.norm(phi))
        diag = (f"{label}: n={n} k={k} phi rel L2 {err:.3g}; iterations gpu {ex.iterations} port {it}; "
                f"pred max rel {perr:.3g} on {len(pick)} rows")
        print(diag)
        if err > PHI_RTOL and it != ex.iterations:
            # Both solvers apply the reference stop rule (solver.cpp:348-353);
            # when the residual ratio sits at the tolerance, rounding in the
            # inputs (predictions within 1e-7) moves the stop by a step, and
            # on an ill-conditioned system one step past the tolerance moves
            # phi by ~5e-3 in a rounding-dependent direction (see
            # tools/cgls_trajectory.py). Then the two solvers' trajectories
            # are compared after the common number of steps.
            assert abs(it - ex.iterations) <= 2, diag
            kc = min(it, ex.iterations)
            w = sf.assemble_weights(n, bits, ros)
            a = ctx.solve_cgls(n, bits, w, preds.astype(np.float64) - ex.base_score,
                               ex.full_score - ex.base_score, 1e6, tol=0.0, max_iter=kc)
            phi_k = port.cgls_sparse(n, bits, ros, preds.astype(np.float64), ex.base_score, ex.full_score,
                                     tol=0.0, max_iter=kc)[0]
            err = float(np.linalg.norm(a["phi"] - phi_k) / np.linalg.norm(phi_k))
            print(f"{label}: stop differs; phi after {kc} steps rel {err:.3g}")
            assert err <= PHI_RTOL, f"{label}: CGLS trajectories differ after {kc} steps: {err:.3g}"
        else:
            assert err <= PHI_RTOL, diag
            assert conv == ex.converged, diag
            top_port = port.rank_edges(phi)[:10].tolist()
            top_gpu = [p for p, _ in ex.top]
            assert top_gpu == top_port, diag
        # 4. fidelity: the reference's evaluate_fidelity on the GPU's phi
        rf = ref.evaluate_fidelity(rm, sgr, ex.predicted_class, ex.phi, seed=nseed, trials=TRIALS)
        np.testing.assert_allclose(ex.fidelity["plus"], rf["plus"], rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(ex.fidelity["plus_random"], rf["plus_random"], rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(ex.fidelity["minus"], rf["minus"], rtol=1e-4, atol=1e-6)
        return dict(n=n, err=err, perr=perr, iterations=ex.iterations)
    finally:
        ref.cg_free(sgr)


def _setup(ref, name):
    d = W.build(name)
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    return d, cfg, g, rg, m, rm


def test_c2_explain_k500k_stagewise(ctx, ref, port):
    """C2 exactly as benched: 3-layer Reddit-shaped, n ~ 50K, k = 500K."""
    d, cfg, g, rg, m, rm = _setup(ref, "C2")
    r = check_stagewise(ctx, ref, port, g, rg, m, rm, d["target"], cfg, cfg.samples, cfg.explain_seed, "C2")
    assert r["n"] > 40_000


def test_c5_eight_targets_stagewise(ctx, ref, port):
    """C5: 8 of the bench's 1,024 select_nodes targets (2-layer, d0 = 256,
    hidden 128, 40 classes), k = 100K each."""
    d, cfg, g, rg, m, rm = _setup(ref, "C5")
    targets = g.select_nodes("degree-range:[4,12]:1024")
    pick = targets[np.linspace(0, len(targets) - 1, 8).astype(int)]
    for t in pick:
        check_stagewise(ctx, ref, port, g, rg, m, rm, int(t), cfg, cfg.samples, cfg.explain_seed, f"C5 node {t}")


C3_WORKER = r"""
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
d = W.build("C3"); cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
ctx.keep_stages(True)
k = int(os.environ["SF_K"])
ex = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=k, seed=cfg.explain_seed, baseline_trials=2))
np.save(os.path.join(os.environ["SF_OUT"], f"preds{rank}.npy"), ctx.stage_predictions())
np.save(os.path.join(os.environ["SF_OUT"], f"phi{rank}.npy"), ex.phi)
out = {"rank": rank, "iterations": ex.iterations, "top": [p for p, _ in ex.top], "converged": ex.converged,
       "base": ex.base_score, "full": ex.full_score, "cls": ex.predicted_class, "rows": ex.rows,
       "stats": ctx.stats(), "plus": ex.fidelity["plus"].tolist()}
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
def test_c3_two_gpu_sharded_stagewise(tmp_path, ctx, ref, port):
    """C3 (products-shaped, n ~ 200K) sharded over 2 GPUs (pairs g mod 2,
    sampler.cpp:177-178; one NCCL all-reduce per CGLS step). k is scaled to
    256K so the host-side restatement holds all 4 GB of masks; the shard's
    rows, predictions and phi are checked like the 1-GPU cases."""
    k, world = 256_000, 2
    script = tmp_path / "worker.py"
    script.write_text(C3_WORKER)
    env = dict(os.environ, SF_ROOT=ROOT, SF_OUT=str(tmp_path), SF_K=str(k))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", "29541", str(script)],
                   check=True, env=env, timeout=1200)
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    phis = [np.load(tmp_path / f"phi{r}.npy") for r in range(world)]
    assert np.array_equal(phis[0], phis[1])  # replicated phi, bitwise
    assert res[0]["top"] == res[1]["top"]
    d, cfg, g, rg, m, rm = _setup(ref, "C3")
    target = d["target"]
    sg = g.extract(target, cfg.hops)
    n = sg.n
    nseed = sf.node_sampling_seed(cfg.explain_seed, target)
    plan = sf.plan_sizes(n, k, True)
    blocks, preds = [], []
    for r in range(world):
        b, ros = ctx.generate_masks(plan, nseed, r, world)
        p = np.load(tmp_path / f"preds{r}.npy")
        assert p.shape[0] == b.shape[0]
        blocks.append(b)
        preds.append(p)
    # whole rank blocks vs the reference sampler
    sgr = ref.extract(rg, target, cfg.hops, keep_handle=True)
    try:
        for r in range(world):
            want, _ = ref.generate_masks(n, k, nseed, r, world)
            assert np.array_equal(blocks[r], want), f"rank {r} block differs"
            del want
        cls = res[0]["cls"]
        for r in range(world):
            pick = spread_rows(blocks[r].shape[0], 128)
            want_p = ref_predict_rows(ref, rm, rg, target, blocks[r][pick], cls, sgr)
            assert rel_err(preds[r][pick], want_p) <= PRED_RTOL
        bits = np.concatenate(blocks)
        vals = np.concatenate(preds).astype(np.float64)
        phi, it, _, conv = port.cgls_sparse(n, bits, ros, vals, res[0]["base"], res[0]["full"], tol=1e-6)
        err = float(np.linalg.norm(phis[0] - phi) / np.linalg.norm(phi))
        print(f"C3 2-GPU: n={n} k={k} phi rel L2 {err:.3g}; iterations gpu {res[0]['iterations']} port {it}")
        assert err <= PHI_RTOL
        assert res[0]["top"] == port.rank_edges(phi)[:10].tolist()
        # reference protocol on both ranks: 1 vector + 1 scalar all-reduce per iteration (+1 vector at init)
        for r in res:
            assert r["stats"]["vector_allreduce"] >= r["iterations"] + 1
            assert r["stats"]["scalar_allreduce"] >= r["iterations"]
        rf = ref.evaluate_fidelity(rm, sgr, cls, phis[0], seed=nseed, trials=2)
        np.testing.assert_allclose(res[0]["plus"], rf["plus"], rtol=1e-4, atol=1e-6)
    finally:
        ref.cg_free(sgr)


def test_c2_explain_predictions_equal_predict_batched(ctx, ref):
    """The predictions explain_node feeds its solver (kept-set rows, device
    engine) equal predict_batched on the same full mask rows, for every one
    of the 500K rows (same engine, same arithmetic: bitwise)."""
    d, cfg, g, rg, m, rm = _setup(ref, "C2")
    target = d["target"]
    ctx.keep_stages(True)
    try:
        ex = ctx.explain_node(g, m, target, ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False))
        kept = ctx.stage_predictions()
    finally:
        ctx.keep_stages(False)
    sg = g.extract(target, cfg.hops)
    bits, _ = ctx.generate_masks(sf.plan_sizes(sg.n, cfg.samples, True), sf.node_sampling_seed(cfg.explain_seed, target))
    full = ctx.predict_batched(m, sg, bits, ex.predicted_class)
    bad = np.nonzero(kept != full)[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:10]}, kept {kept[bad[:5]]} full {full[bad[:5]]}"


def test_c2_explain_phi_equals_stage_solve(ctx, ref, port):
    """explain_node's phi equals the stage-level solve (solve_cgls on the
    same masks, predictions and weights): nothing between inference and the
    solver alters the solver's inputs (rows, weights, targets)."""
    d, cfg, g, rg, m, rm = _setup(ref, "C2")
    target = d["target"]
    ctx.keep_stages(True)
    try:
        ex = ctx.explain_node(g, m, target, ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False,
                                                           solver_mode=0))
        preds = ctx.stage_predictions()
    finally:
        ctx.keep_stages(False)
    sg = g.extract(target, cfg.hops)
    plan = sf.plan_sizes(sg.n, cfg.samples, True)
    nseed = sf.node_sampling_seed(cfg.explain_seed, target)
    bits, ros = ctx.generate_masks(plan, nseed)
    w = sf.assemble_weights(sg.n, bits, ros)
    t = preds.astype(np.float64) - ex.base_score
    a = ctx.solve_cgls(sg.n, bits, w, t, ex.full_score - ex.base_score, 1e6)
    dm = ctx.masks_device(plan, nseed)
    b = dm.solve(preds, ex.base_score, ex.full_score)
    e_host = float(np.linalg.norm(ex.phi - a["phi"]) / np.linalg.norm(a["phi"]))
    e_dev = float(np.linalg.norm(ex.phi - b["phi"]) / np.linalg.norm(b["phi"]))
    print(f"explain vs host-row solve {e_host:.3g} ({ex.iterations} vs {a['iterations']} it), "
          f"vs device-row solve {e_dev:.3g} ({b['iterations']} it)")
    assert e_host <= 1e-8 and e_dev <= 1e-8
