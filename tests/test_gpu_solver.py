"""GPU: weighted least squares on bit rows (replaces assemble_problem +
solve_cgls + solve_direct, solver.cpp:95-428). The reference's own solver tests
(test_solver.cpp) re-expressed through the C-ABI, plus parity with the
reference / bit-row restatement at larger sizes."""
import os
import pathlib

import numpy as np
import pytest

import paper_2506_22668_b200 as sf

pytestmark = pytest.mark.gpu


def toy_game_values(bits, port):
    # test_solver.cpp:23-37 hashed "toy game", any deterministic function works
    key = np.full(bits.shape[0], 0x6B43A9B5, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for w in range(bits.shape[1]):
            key = key * np.uint64(0x9E3779B97F4A7C15) + bits[:, w]
    return np.array([(int(port.philox(int(k), 3, 1)[0]) >> 11) * 2.0**-53 for k in key])


def sampled_problem(ctx, port, n, k, seed, base, full):
    p = sf.plan_sizes(n, k, False)
    bits, ros = ctx.generate_masks(p, seed)
    vals = toy_game_values(bits, port)
    w = sf.assemble_weights(n, bits, ros)
    return bits, w, vals - base, full - base


def test_identity_system_one_iteration(ctx):
    # test_solver.cpp:55-77: non-complement rows e0..e3, no pin
    bits = np.array([[1], [2], [4], [8]], np.uint64)
    r = ctx.solve_cgls(4, bits, np.ones(4), np.array([1.0, 2, 3, 4]), 0.0, 0.0)
    assert r["converged"] and r["iterations"] == 1
    assert np.allclose(r["phi"], [1, 2, 3, 4], rtol=1e-12)


def test_two_players_hand_value(ctx):
    # test_solver.cpp:79-102: f({0})=1, f({1})=2, f(both)=4 -> (1.5, 2.5)
    p = sf.plan_sizes(2, 2, True)
    bits, ros = ctx.generate_masks(p, 0)
    vals = np.where(bits[:, 0] == 1, 1.0, 2.0)
    w = sf.assemble_weights(2, bits, ros)
    r = ctx.solve_cgls(2, bits, w, vals, 4.0, 1e6, max_iter=10)
    assert r["converged"]
    assert r["phi"] == pytest.approx([1.5, 2.5], rel=1e-6)
    d = ctx.solve_direct(2, bits, w, vals, 4.0, 1e6)
    assert d == pytest.approx([1.5, 2.5], rel=1e-6)


@pytest.mark.parametrize("n", [5, 8, 13])
def test_cgls_matches_direct(ctx, port, n):
    # test_solver.cpp:104-124
    bits, w, t, ct = sampled_problem(ctx, port, n, 60 * n, 1000 + n, 0.3, 0.7)
    r = ctx.solve_cgls(n, bits, w, t, ct, 1e6, tol=1e-10, max_iter=4 * n)
    assert r["converged"]
    d = ctx.solve_direct(n, bits, w, t, ct, 1e6)
    scale = max(np.abs(d).max(), 1.0)
    assert np.abs(r["phi"] - d).max() <= 1e-8 * scale


def test_additive_game_exact(ctx):
    # test_solver.cpp:126-148
    n = 6
    p = sf.plan_sizes(n, 62, True)
    bits, ros = ctx.generate_masks(p, 0)
    vals = np.array([sum(i + 1 for i in range(n) if (int(b) >> i) & 1) for b in bits[:, 0]], float)
    w = sf.assemble_weights(n, bits, ros)
    r = ctx.solve_cgls(n, bits, w, vals, 21.0, 1e6)
    assert r["phi"] == pytest.approx(np.arange(1, n + 1), rel=1e-6)


def test_symmetric_game(ctx):
    # test_solver.cpp:150-168
    n = 6
    p = sf.plan_sizes(n, 62, True)
    bits, ros = ctx.generate_masks(p, 0)
    vals = np.array([bin(int(b)).count("1") ** 2 for b in bits[:, 0]], float)
    w = sf.assemble_weights(n, bits, ros)
    r = ctx.solve_cgls(n, bits, w, vals, 36.0, 1e6)
    assert r["phi"].max() - r["phi"].min() <= 1e-6
    assert r["phi"][0] == pytest.approx(6.0, rel=1e-4)


def test_duplicate_rows_half_weight(ctx, port):
    # test_solver.cpp:170-197
    bits, w, t, ct = sampled_problem(ctx, port, 7, 200, 5, 0.1, 0.9)
    a = ctx.solve_cgls(7, bits, w, t, ct, 1e6, tol=1e-10, max_iter=28)
    bits2 = np.repeat(bits, 2, axis=0)
    b = ctx.solve_cgls(7, bits2, np.repeat(w, 2) / 2, np.repeat(t, 2), ct, 1e6, tol=1e-10, max_iter=28)
    assert np.allclose(a["phi"], b["phi"], rtol=1e-8, atol=1e-12)


def test_monotone_row_residual(ctx, port):
    # test_solver.cpp:199-210
    bits, w, t, ct = sampled_problem(ctx, port, 10, 400, 77, 0.2, 0.8)
    r = ctx.solve_cgls(10, bits, w, t, ct, 1e6, trace=True)
    tr = r["row_residual_trace"]
    assert len(tr) >= 2
    assert all(tr[i] <= tr[i - 1] * (1 + 1e-10) + 1e-12 for i in range(1, len(tr)))


@pytest.mark.parametrize("n", [6, 12, 20])
def test_efficiency_pin(ctx, port, n):
    # test_solver.cpp:212-220
    bits, w, t, ct = sampled_problem(ctx, port, n, 50 * n, n, 0.25, 0.75)
    r = ctx.solve_cgls(n, bits, w, t, ct, 1e6)
    assert abs(r["phi"].sum() - ct) <= 1e-4


def test_validation_errors(ctx, port):
    # test_solver.cpp:258-324
    bits = np.array([[3], [4]], np.uint64)
    with pytest.raises(sf.NumericalError, match="pivot"):
        ctx.solve_direct(3, bits, np.zeros(2), np.array([1.0, 2.0]), 0.0, 0.0)
    b, w, t, ct = sampled_problem(ctx, port, 5, 100, 2, 0.0, 1.0)
    with pytest.raises(sf.DataError):
        ctx.solve_cgls(5, b[:-1], w[:-1], t[:-1], ct, 1e6)
    t2 = t.copy()
    t2[0] = np.nan
    with pytest.raises(sf.NumericalError):
        ctx.solve_cgls(5, b, w, t2, ct, 1e6)
    with pytest.raises(sf.DataError):
        sf.assemble_weights(4, np.array([[0], [15]], np.uint64))


@pytest.mark.parametrize("n,k,seed", [(11, 500, 31), (40, 3000, 3), (200, 4000, 9), (999, 10000, 1)])
def test_cgls_vs_reference(ctx, ref, port, n, k, seed):
    p = sf.plan_sizes(n, k, False)
    bits, ros = ctx.generate_masks(p, seed)
    vals = np.sin(np.arange(bits.shape[0]) * 0.37) * 0.5 + 0.5
    phi_ref, it_ref, _, conv_ref = ref.solve_cgls(n, bits, vals, 0.25, 0.75, max_iter=4 * n)
    w = sf.assemble_weights(n, bits, ros)
    r = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6, max_iter=4 * n)
    assert r["converged"] == conv_ref
    assert abs(int(r["iterations"]) - int(it_ref)) <= 1
    err = np.linalg.norm(r["phi"] - phi_ref) / np.linalg.norm(phi_ref)
    assert err <= 1e-3  # BASELINE bar; observed ~1e-12 (FP64, reordered sums)
    assert (sf.rank_edges(r["phi"])[:10] == port.rank_edges(phi_ref)[:10]).all()


def test_collective_counts_reference_protocol(ctx, port):
    # acceptance.cpp:653-677: 1 scalar + 1 vector all-reduce per iteration,
    # one more vector at init, n doubles per vector, 1 per scalar
    n = 16
    p = sf.plan_sizes(n, 2048, False)
    bits, ros = ctx.generate_masks(p, 3)
    vals = np.array([(int(port.philox(77, i, 1)[0]) >> 11) * 2.0**-53 for i in range(bits.shape[0])])
    w = sf.assemble_weights(n, bits, ros)
    before = ctx.stats()
    r = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6)
    after = ctx.stats()
    it = r["iterations"]
    assert after["scalar_allreduce"] - before["scalar_allreduce"] == it
    assert after["vector_allreduce"] - before["vector_allreduce"] == it + 1
    assert after["doubles_reduced"] - before["doubles_reduced"] == (it + 1) * n + it


@pytest.mark.parametrize("n,k,seed", [(999, 20000, 5), (3001, 40000, 6)])
def test_cgls_pass_variants_agree(ctx, ref, port, n, k, seed, monkeypatch):
    # The products run as kept-set lists on the sparse pair tiles and as
    # nibble-table lookups on the dense ones (SF_CGLS_NIB_DENSITY picks the
    # split; SF_CGLS_LISTS=0 puts the sparse tiles on set-bit loops): every
    # variant solves the same system.
    p = sf.plan_sizes(n, k, False)
    bits, ros = ctx.generate_masks(p, seed)
    vals = np.cos(np.arange(bits.shape[0]) * 0.11) * 0.5 + 0.5
    w = sf.assemble_weights(n, bits, ros)
    phi_ref, _, _, _ = ref.solve_cgls(n, bits, vals, 0.25, 0.75, max_iter=4 * n)
    out = {}
    variants = [("bits", "1e9", "0"), ("lists", "1e9", None), ("nibble", "0", None),
                ("split_bits", None, "0"), ("split", None, None)]
    for name, density, lists in variants:
        for key, val in (("SF_CGLS_NIB_DENSITY", density), ("SF_CGLS_LISTS", lists)):
            if val is None:
                monkeypatch.delenv(key, raising=False)
            else:
                monkeypatch.setenv(key, val)
        r = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6, max_iter=4 * n)
        assert r["converged"]
        out[name] = r["phi"]
        err = np.linalg.norm(r["phi"] - phi_ref) / np.linalg.norm(phi_ref)
        assert err <= 1e-3, (name, err)
        assert (sf.rank_edges(r["phi"])[:10] == port.rank_edges(phi_ref)[:10]).all()
    for name in out:
        d = np.linalg.norm(out[name] - out["bits"]) / np.linalg.norm(out["bits"])
        assert d <= 1e-8, (name, d)


I8_WORKER = r"""
import os, sys
import numpy as np
sys.path.insert(0, os.environ["SF_ROOT"])
import paper_2506_22668_b200 as sf
n, k, seed = (int(x) for x in sys.argv[1:4])
ctx = sf.Context(0)
p = sf.plan_sizes(n, k, False)
bits, ros = ctx.generate_masks(p, seed)
vals = np.cos(np.arange(bits.shape[0]) * 0.11) * 0.5 + 0.5
w = sf.assemble_weights(n, bits, ros)
r = ctx.solve_cgls(n, bits, w, vals - 0.25, 0.5, 1e6, max_iter=4 * n)
np.save(sys.argv[4], r["phi"])
"""


@pytest.mark.parametrize("n,k,seed", [(999, 20000, 5), (3001, 40000, 6)])
def test_cgls_i8_passes_agree(ctx, ref, tmp_path, n, k, seed, monkeypatch):
    """The tensor-core dense-pair passes (SF_CGLS_I8=1: A operand in TMEM,
    2: in shared memory; exact integer sums over 16 digits of the vector)
    solve the same system as the nibble tables, and the two operand paths
    give bitwise the same phi (the sums do not depend on how the work is
    staged). SF_CGLS_NIB_DENSITY=0 puts every pair tile on the dense path."""
    import subprocess
    import sys as _sys

    script = tmp_path / "i8.py"
    script.write_text(I8_WORKER)
    root = str(pathlib.Path(__file__).resolve().parents[1])
    phis = {}
    for mode in ("0", "1", "2"):
        env = dict(os.environ, SF_ROOT=root, SF_CGLS_I8=mode, SF_CGLS_NIB_DENSITY="0")
        out = tmp_path / f"phi{mode}.npy"
        subprocess.run([_sys.executable, str(script), str(n), str(k), str(seed), str(out)], check=True, env=env,
                       timeout=600)
        phis[mode] = np.load(out)
    p = sf.plan_sizes(n, k, False)
    bits, ros = ctx.generate_masks(p, seed)
    vals = np.cos(np.arange(bits.shape[0]) * 0.11) * 0.5 + 0.5
    phi_ref, _, _, _ = ref.solve_cgls(n, bits, vals, 0.25, 0.75, max_iter=4 * n)
    assert np.array_equal(phis["1"], phis["2"])
    for mode in ("1", "2"):
        d = np.linalg.norm(phis[mode] - phis["0"]) / np.linalg.norm(phis["0"])
        assert d <= 1e-8, (mode, d)
        err = np.linalg.norm(phis[mode] - phi_ref) / np.linalg.norm(phi_ref)
        assert err <= 1e-3, (mode, err)


@pytest.mark.parametrize("n", [40, 300, 1000, 2100])
def test_direct_gram_path_vs_reference(ctx, ref, port, n):
    """solve_direct (solver.cpp:364-428) on the device: tcgen05 Gram over the
    bit rows (per-size weight runs), blocked FP64 Cholesky, triangular
    solves. Bar: 1e-8 of the reference's host solve_direct. Sizes cover
    one and several 128-player tiles and the split row axis."""
    k = max(20 * n, 4000)
    p = sf.plan_sizes(n, k, False)
    bits, ros = ctx.generate_masks(p, 77 + n)
    vals = toy_game_values(bits, port)
    base, full = 0.2, 0.8
    want = ref.solve_direct(n, bits, vals, base, full)
    w = sf.assemble_weights(n, bits, ros)
    got = ctx.solve_direct(n, bits, w, vals - base, full - base, 1e6)
    scale = max(np.abs(want).max(), 1e-12)
    assert np.abs(got - want).max() <= 1e-8 * scale


def test_direct_arbitrary_rows_and_weights(ctx):
    """Caller rows (odd count, not pairs) with a distinct weight per row:
    the rows are regrouped by weight; checked against an FP64 normal-equation
    solve in numpy."""
    rng = np.random.default_rng(5)
    n, rows = 150, 901
    dense = (rng.random((rows, n)) < 0.3)
    dense[:, 0] |= ~dense.any(1)
    W = (n + 63) // 64
    bits = np.zeros((rows, W), np.uint64)
    for e in range(n):
        bits[:, e // 64] |= dense[:, e].astype(np.uint64) << np.uint64(e % 64)
    w = rng.random(rows) + 0.1
    t = rng.standard_normal(rows)
    ct, cw = 0.5, 1e3
    got = ctx.solve_direct(n, bits, w, t, ct, cw)
    A = dense.astype(np.float64)
    G = A.T @ (w[:, None] * A) + cw
    b = A.T @ (w * t) + cw * ct
    want = np.linalg.solve(G, b)
    assert np.abs(got - want).max() <= 1e-8 * max(np.abs(want).max(), 1.0)


def test_explain_direct_solver_and_dispatch(ctx, ref, port):
    """explain_node with the direct solver (tcgen05 Gram + device Cholesky):
    at C1 (n ~ 1K) phi is within the 1e-3 bar of the reference's CGLS
    explanation with the same top-10; SF_SOLVER_AUTO keeps CGLS there and
    takes the direct path for a small ball (n <= 256, the measured
    crossover)."""
    from paper_2506_22668_b200 import workloads as Wl
    from paper_2506_22668_b200.api import ExplainOptions

    d = Wl.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    base = dict(samples=cfg.samples, seed=cfg.explain_seed, fidelity=False)
    auto = ctx.explain_node(g, m, d["target"], ExplainOptions(**base))
    direct = ctx.explain_node(g, m, d["target"], ExplainOptions(solver_mode=2, **base))
    cgls = ctx.explain_node(g, m, d["target"], ExplainOptions(solver_mode=0, **base))
    assert direct.iterations == 0 and cgls.iterations > 0 and auto.iterations == cgls.iterations
    # CGLS stops at tol 1e-6 on the gradient ratio; the direct solve is exact
    assert np.linalg.norm(direct.phi - cgls.phi) <= 1e-3 * np.linalg.norm(cgls.phi)
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    rx = ref.explain_node(rg, rm, d["target"], samples=cfg.samples, seed=cfg.explain_seed, world=8)
    assert np.linalg.norm(direct.phi - rx["phi"]) <= 1e-3 * np.linalg.norm(rx["phi"])
    # a small ball: AUTO takes the direct path; same answer as forcing it
    small = next(v for v in g.select_nodes("degree-range:[2,3]:200") if 20 <= g.extract(int(v), 2).n <= 256)
    a = ctx.explain_node(g, m, int(small), ExplainOptions(**base))
    b = ctx.explain_node(g, m, int(small), ExplainOptions(solver_mode=2, **base))
    c = ctx.explain_node(g, m, int(small), ExplainOptions(solver_mode=0, **base))
    assert a.iterations == 0 and np.array_equal(a.phi, b.phi)
    assert np.linalg.norm(a.phi - c.phi) <= 1e-3 * np.linalg.norm(c.phi)


def test_fixed_order_modes(ctx, port):
    """CglsOptions::fixed_order (solver.hpp:62-65), both device schemes.
    Small systems follow the reference's folder tree (leaves in bit-reversed
    pair order, one scalar + one vector all-reduce per iteration); large ones
    use exact level sums, which make phi independent of the pair layout
    altogether: permuting the pairs (different tiles, splits, list/nibble
    split points) gives bitwise the same phi. Both agree with the default
    mode to rounding."""
    for n, k in ((40, 2400), (2100, 150_000)):
        p = sf.plan_sizes(n, k, False)
        bits, ros = ctx.generate_masks(p, 300 + n)
        vals = toy_game_values(bits, port)
        w = sf.assemble_weights(n, bits, ros)
        t, ct = vals - 0.25, 0.5
        s0 = ctx.stats()
        a = ctx.solve_cgls(n, bits, w, t, ct, 1e6, mode=2, max_iter=4 * n)
        s1 = ctx.stats()
        again = ctx.solve_cgls(n, bits, w, t, ct, 1e6, mode=2, max_iter=4 * n)
        assert np.array_equal(a["phi"], again["phi"])
        ref0 = ctx.solve_cgls(n, bits, w, t, ct, 1e6, mode=0, max_iter=4 * n)
        assert np.linalg.norm(a["phi"] - ref0["phi"]) <= 1e-8 * np.linalg.norm(ref0["phi"])
        if n == 40:  # the reference protocol: 1 scalar + 1 vector per iteration, +1 vector at init
            assert s1["scalar_allreduce"] - s0["scalar_allreduce"] == a["iterations"]
            assert s1["vector_allreduce"] - s0["vector_allreduce"] == a["iterations"] + 1
        else:
            perm = np.random.default_rng(n).permutation(bits.shape[0] // 2)
            rows = np.stack([2 * perm, 2 * perm + 1], 1).reshape(-1)
            b = ctx.solve_cgls(n, bits[rows], w[rows], t[rows], ct, 1e6, mode=2, max_iter=4 * n)
            assert a["iterations"] == b["iterations"]
            assert np.array_equal(a["phi"], b["phi"])


def test_device_resident_stages_match_host_stages(ctx, ref, port):
    """sf_masks_device -> sf_predict_dmasks -> sf_solve_dmasks (explain.cpp:
    91-114 without moving the mask block over PCIe): the downloaded block is
    the reference's MaskBlock bit for bit, the predictions equal the host-row
    path, and phi equals solve_cgls on the host-assembled system."""
    from paper_2506_22668_b200 import workloads as Wl

    d = Wl.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    sg = g.extract(d["target"], cfg.hops)
    n = sg.n
    p = sf.plan_sizes(n, 4000, True)
    seed = sf.node_sampling_seed(1, d["target"])
    dm = ctx.masks_device(p, seed)
    rows, nn, ros = dm.info()
    bits = dm.download()
    want, want_ros = ref.generate_masks(n, 4000, seed)
    assert nn == n and rows == bits.shape[0] and np.array_equal(bits, want)
    assert np.array_equal(ros, np.asarray(want_ros, np.uint64))
    pd = dm.predict(m, sg, 2)
    ph = ctx.predict_batched(m, sg, bits, 2)
    assert np.array_equal(pd, ph)
    base, full = 0.25, 0.75
    a = dm.solve(pd, base, full)
    w = sf.assemble_weights(n, bits, ros)
    b = ctx.solve_cgls(n, bits, w, pd.astype(np.float64) - base, full - base, 1e6)
    assert a["iterations"] == b["iterations"]
    assert np.linalg.norm(a["phi"] - b["phi"]) <= 1e-10 * np.linalg.norm(b["phi"])
