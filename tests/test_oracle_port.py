"""CPU: pin the C restatement (oracle/shapflow_port.c) against the reference's
golden vectors (tests/golden/golden.json) and, when it is
built, against the compiled reference itself (oracle/_ref)."""
import numpy as np
import pytest

from conftest import hex_to_u64, toy_graph_arrays


def test_philox_golden(port, golden):
    # SURVEY.md Appendix A
    assert [f"{x:016x}" for x in port.philox(0, 0, 4)] == [
        "9b00dbd8bc57ac4c", "e169c58d6627e8d5", "097eff67b1a574eb", "5cb200dbf8e4cca4"]
    for case in golden["philox"]:
        got = port.philox(case["seed"], case["stream"], len(case["out"]))
        assert (got == hex_to_u64(case["out"])).all()


def test_seed_and_binomial(port, golden):
    assert port.node_sampling_seed(1, 61) == 0x516F7AECD40A0D17
    for c in golden["node_sampling_seed"]:
        assert port.node_sampling_seed(c["seed"], c["node"]) == int(c["out"], 16)
    for c in golden["binomial"]:
        assert port.binomial_or_max(c["n"], c["s"]) == int(c["out"])


def test_plans_golden(port, golden):
    for c in golden["plans"]:
        p = port.plan_sizes(c["n"], c["k"], c["allow"])
        assert p["exhaustive"] == c["exhaustive"]
        assert p["requested"] == c["requested"]
        assert p["sizes"].tolist() == c["sizes"]
        assert p["pairs"].tolist() == c["pairs"]
        assert p["first"].tolist() == c["first"]


def test_plan_reference_cases(port):
    # test_sampler.cpp:68-80: n=4, k=110 -> rows 40/30/40 by size
    p = port.plan_sizes(4, 110, False)
    bits = port.generate_masks(4, p, 1)
    sizes = [bin(int(x)).count("1") for x in bits[:, 0]]
    assert (sizes.count(1), sizes.count(2), sizes.count(3)) == (40, 30, 40)
    # odd budgets round up (test_sampler.cpp:113-117)
    assert port.plan_sizes(6, 11, False)["requested"] == 12
    with pytest.raises(Exception):
        port.plan_sizes(1, 100)


def test_masks_golden(port, golden):
    for c in golden["masks"]:
        p = port.plan_sizes(c["n"], c["k"], c["allow"])
        bits = port.generate_masks(c["n"], p, int(c["seed"], 16), c["rank"], c["world"])
        assert list(bits.shape) == c["shape"]
        assert (bits.ravel() == hex_to_u64(c["bits"])).all()
        assert port.rows_of_size(c["n"], p).tolist() == c["rows_of_size"]


def test_acceptance_c5_balance(port, golden):
    # acceptance.cpp:387-406: n=30, k=25000, 4 workers -> 6250 rows, popcount 93750 each
    p = port.plan_sizes(30, 25000, True)
    for c in golden["acceptance_c5"]:
        bits = port.generate_masks(30, p, 9, c["rank"], 4)
        assert bits.shape[0] == c["rows"] == 6250
        assert int(sum(bin(int(x)).count("1") for x in bits.ravel())) == c["popcount"] == 93750


def test_gcn_port_hand_values(port, golden):
    # test_gcn.cpp:65-76: p0 = 1/(1+e^-4) kept, 1/(1+e^-2) dropped
    from oracle.pyoracle import Model, Subgraph
    sg = Subgraph(V=2, n=1, dim=1, row_ptr=np.array([0, 1, 2], np.uint64), col=np.array([1, 0], np.uint32),
                  edge_player=np.array([0, 0], np.uint32), players=np.array([[0, 1]], np.uint32),
                  local_to_global=np.array([0, 1], np.uint32), features=np.array([[1.0], [3.0]], np.float32))
    m = Model([1, 2], [np.array([[1.0, -1.0]], np.float32)], [np.zeros(2, np.float32)])
    kept = port.gcn_probs(sg, m, np.array([1], np.uint64))[0]
    dropped = port.gcn_probs(sg, m, np.array([0], np.uint64))[0]
    assert kept == pytest.approx(0.9820137900379085, rel=1e-6)
    assert dropped == pytest.approx(0.8807970779778823, rel=1e-6)
    assert kept == np.float32(golden["gcn_hand"]["kept"])
    assert dropped == np.float32(golden["gcn_hand"]["dropped"])


def test_gcn_port_vs_reference_toy(port, ref, golden):
    edges, feats = toy_graph_arrays()
    g = ref.graph_build(6, edges, feats)
    sg = ref.extract(g, 1, 2)
    m = ref.model_random(2, [4], 2, 17)
    allm = np.arange(1 << sg.n, dtype=np.uint64).reshape(-1, 1)
    got = port.gcn_predict(sg, m, allm, 0)
    assert (got == np.array(golden["toy"]["predictions"], np.float32)).all()  # bitwise


def test_gcn_port_vs_reference_random(port, ref):
    g = ref.graph_random(120, 420, 9, 3, 5)
    for hidden, hops in [([6], 2), ([5, 7], 3), ([], 1)]:
        m = ref.model_random(9, hidden, 3, 11)
        sg = ref.extract(g, 7, hops, keep_handle=True)
        p = port.plan_sizes(sg.n, 300, False)
        bits = port.generate_masks(sg.n, p, 4)
        a = ref.predict_batched(m, g, 7, bits, 1, sg=sg)
        b = port.gcn_predict(sg, m, bits, 1)
        assert (a == b).all()
        ref.cg_free(sg)


def test_cgls_port_golden(port, golden):
    c = golden["cgls_toy"]
    p = port.plan_sizes(c["n"], c["k"], False)
    bits = port.generate_masks(c["n"], p, c["seed"])
    ros = port.rows_of_size(c["n"], p)
    phi, it, res, conv = port.cgls(c["n"], bits, ros, np.array(c["values"]), c["base"], c["full"],
                                   max_iter=c["max_iter"])
    assert it == c["iterations"] and conv == c["converged"]
    assert (phi == np.array(c["phi"])).all()  # bitwise: same fold order as the reference


def test_cgls_port_vs_reference(port, ref):
    for n, k, seed in [(13, 780, 1013), (40, 3000, 3), (200, 4000, 9)]:
        p = port.plan_sizes(n, k, False)
        bits = port.generate_masks(n, p, seed)
        vals = np.sin(np.arange(bits.shape[0]) * 0.37) * 0.5 + 0.5
        a = ref.solve_cgls(n, bits, vals, 0.25, 0.75, max_iter=4 * n)
        b = port.cgls(n, bits, port.rows_of_size(n, p), vals, 0.25, 0.75, max_iter=4 * n)
        assert a[1] == b[1] and a[3] == b[3]
        assert (a[0] == b[0]).all()


def test_cgls_sparse_vs_reference(port, ref):
    """port_cgls_sparse (the large-shape checker used by the C2/C3/C5 parity
    tests) agrees with the compiled reference solve_cgls to rounding, for any
    thread count, on complement pairs and on non-complement (user) rows."""
    for n, k, seed in [(40, 3000, 3), (200, 4000, 9), (1000, 6000, 21)]:
        p = port.plan_sizes(n, k, False)
        bits = port.generate_masks(n, p, seed)
        ros = port.rows_of_size(n, p)
        vals = np.sin(np.arange(bits.shape[0]) * 0.37) * 0.5 + 0.5
        a = ref.solve_cgls(n, bits, vals, 0.25, 0.75, max_iter=4 * n)
        for threads in (1, 3, 8):
            b = port.cgls_sparse(n, bits, ros, vals, 0.25, 0.75, max_iter=4 * n, threads=threads)
            # same stop rule; near tol the rounding can move the stop by a few iterations
            assert b[3] == a[3] and abs(b[1] - a[1]) <= max(3, a[1] // 10)
            assert np.linalg.norm(b[0] - a[0]) <= 1e-8 * np.linalg.norm(a[0])
    # non-complement rows: swap the odd rows of two pairs
    n, k = 64, 2000
    p = port.plan_sizes(n, k, False)
    bits = port.generate_masks(n, p, 5).copy()
    bits[[1, 3]] = bits[[3, 1]]
    vals = np.cos(np.arange(bits.shape[0]) * 0.11) * 0.5 + 0.5
    ros = port.rows_of_size(n, p)
    a = ref.solve_cgls(n, bits, vals, 0.1, 0.9, max_iter=4 * n)
    b = port.cgls_sparse(n, bits, ros, vals, 0.1, 0.9, max_iter=4 * n, threads=4)
    assert np.linalg.norm(b[0] - a[0]) <= 1e-8 * np.linalg.norm(a[0])


def test_rank_edges_ties(port):
    # test_solver.cpp:278-286
    assert port.rank_edges(np.array([0.5, 0.7, 0.5, -1.0])).tolist() == [1, 0, 2, 3]
