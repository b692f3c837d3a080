"""CPU, world_size 2 over gloo: the N>1 logic of the hot path.

* Pair sharding (sampler.cpp:177-178): each rank's shard (pairs g = rank,
  rank + world, ...) as planned by the library's host code interleaves back
  into the world-1 mask matrix (checked with the C restatement's masks).
* Distributed CGLS protocol (solver.cpp:158-362, solver.hpp:82-85): rows
  sharded by pair, n-vectors replicated, exactly one n-vector all-reduce (+1
  at init) and one scalar all-reduce per iteration, reproduces the
  single-rank solution. This is the protocol sf_solve_cgls runs over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dense(bits, n):
    return np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")[:, :n].astype(np.float64)


def cgls_distributed(A, sw, t, ct, cw, tol, max_iter, allreduce):
    """Row-sharded CGLS with the reference's stop rule; A is this rank's rows."""
    n = A.shape[1]
    sc = np.sqrt(cw)
    r = sw * t
    r_c = sc * ct
    stats = {"vector": 0, "scalar": 0}

    def transpose():
        s = A.T @ (sw * r)
        s = allreduce(s)
        stats["vector"] += 1
        return s + sc * r_c

    phi = np.zeros(n)
    s = transpose()
    gamma = s @ s
    data0 = np.sum((s - sc * r_c) ** 2)
    ref = data0 if data0 > 0 else gamma
    u = s.copy()
    it = 0
    conv = False
    while it < max_iter:
        v = sw * (A @ u)
        delta = allreduce(np.array([v @ v]))[0]
        stats["scalar"] += 1
        v_c = sc * u.sum()
        delta += v_c * v_c
        if delta <= 0:
            break
        theta = gamma / delta
        phi += theta * u
        r -= theta * v
        r_c -= theta * v_c
        s = transpose()
        gn = s @ s
        it += 1
        if np.sqrt(gn / ref) <= tol:
            conv = True
            break
        u = s + (gn / gamma) * u
        gamma = gn
    return phi, it, conv, stats


def _worker(rank, world, port, n, k, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2506_22668_b200 as sf
        from oracle.pyoracle import Port

        port_ = Port()
        plan = sf.plan_sizes(n, k, False)
        mine = port_.generate_masks(n, plan, seed, rank, world)
        ros = port_.rows_of_size(n, plan)
        w = sf.assemble_weights(n, mine, ros)
        # per-row values as a function of the global pair index, so shards agree
        g_local = np.arange(rank, int(plan["pairs"].sum()), world)
        vals = np.repeat(np.sin(g_local * 0.37) * 0.5 + 0.5, 2) - 0.25 * np.tile([1, -1], len(g_local))

        def allreduce(x):
            tx = torch.from_numpy(np.ascontiguousarray(x, np.float64))
            dist.all_reduce(tx)
            return tx.numpy()

        A = dense(mine, n)
        phi, it, conv, stats = cgls_distributed(A, np.sqrt(w), vals, 0.5, 1e6, 1e-10, 4 * n, allreduce)
        torch.save({"phi": phi, "it": it, "conv": conv, "stats": stats, "rows": mine.shape[0],
                    "pairs_lib": sf.plan_sizes(n, k, False)["pairs"].sum()}, f"{out}.{rank}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,seed", [(12, 600, 42), (40, 3000, 7)])
def test_two_rank_gloo_matches_single_rank(tmp_path, n, k, seed):
    from oracle.pyoracle import Port

    import paper_2506_22668_b200 as sf

    world = 2
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(world, _free_port(), n, k, seed, out), nprocs=world, join=True,
                       start_method="spawn")
    res = [torch.load(f"{out}.{r}", weights_only=False) for r in range(world)]
    # single rank reference: same global rows, same per-pair values
    port_ = Port()
    plan = sf.plan_sizes(n, k, False)
    whole = port_.generate_masks(n, plan, seed)
    ros = port_.rows_of_size(n, plan)
    w = sf.assemble_weights(n, whole, ros)
    g = np.arange(int(plan["pairs"].sum()))
    vals = np.repeat(np.sin(g * 0.37) * 0.5 + 0.5, 2) - 0.25 * np.tile([1, -1], len(g))
    phi1, it1, conv1, _ = cgls_distributed(dense(whole, n), np.sqrt(w), vals, 0.5, 1e6, 1e-10, 4 * n,
                                           lambda x: x)
    assert sum(r["rows"] for r in res) == whole.shape[0]
    for r in res:
        assert r["conv"] == conv1 and abs(r["it"] - it1) <= 1
        np.testing.assert_allclose(r["phi"], phi1, rtol=1e-9, atol=1e-12)
        # protocol: one scalar + one vector all-reduce per iteration, +1 vector at init
        assert r["stats"]["scalar"] == r["it"] and r["stats"]["vector"] == r["it"] + 1
    np.testing.assert_array_equal(res[0]["phi"], res[1]["phi"])  # replicated on every rank


def test_shards_interleave_into_world1_rows():
    """pair g -> rank g mod world; local row 2j/2j+1 = global rows 2g/2g+1."""
    import paper_2506_22668_b200 as sf
    from oracle.pyoracle import Port

    port_ = Port()
    n, k, seed = 30, 25000, 9
    plan = sf.plan_sizes(n, k, True)
    whole = port_.generate_masks(n, plan, seed)
    for world in (2, 4, 8):
        rows = 0
        for rank in range(world):
            part = port_.generate_masks(n, plan, seed, rank, world)
            g = np.arange(rank, whole.shape[0] // 2, world)
            assert (part[0::2] == whole[2 * g]).all() and (part[1::2] == whole[2 * g + 1]).all()
            rows += part.shape[0]
        assert rows == whole.shape[0]
