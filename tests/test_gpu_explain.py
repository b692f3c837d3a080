"""GPU: explain_node end to end (explain.cpp:42-143) against the reference.
BASELINE bar: phi within 1e-3 relative L2, identical top-k, identical
Fidelity+ (to float rounding of the predictions it is computed from)."""
import numpy as np
import pytest

import paper_2506_22668_b200 as sf
from conftest import toy_graph_arrays
from paper_2506_22668_b200 import workloads as W
from paper_2506_22668_b200.api import ExplainOptions

pytestmark = pytest.mark.gpu


def test_exhaustive_toy_matches_exact_oracle(ctx, golden):
    # test_pipeline.cpp:61-85: exhaustive explain == exact Shapley within 1e-6
    edges, feats = toy_graph_arrays()
    g = sf.Graph.build(6, edges, feats)
    m = sf.Model.random(2, [4], 2, 17)
    ex = ctx.explain_node(g, m, 1, ExplainOptions(fidelity=False))
    assert ex.exhaustive and not ex.skipped
    assert len(ex.players) == 7
    exact = np.array(golden["toy"]["exact_shapley"])
    assert np.abs(ex.phi - exact).max() <= 1e-6
    assert ex.phi.sum() == pytest.approx(ex.full_score - ex.base_score, rel=1e-6)
    assert (ex.players[:, 0] < ex.players[:, 1]).all()
    assert ex.predicted_class == golden["toy"]["explain_class"]


def test_player_cap_and_degenerate_nodes(ctx):
    edges, feats = toy_graph_arrays()
    g = sf.Graph.build(6, edges, feats)
    m = sf.Model.random(2, [4], 2, 29)
    ex = ctx.explain_node(g, m, 1, ExplainOptions(fidelity=False, player_cap=5))
    assert ex.skipped and ex.warning and len(ex.phi) == 0
    ok = ctx.explain_node(g, m, 5, ExplainOptions(fidelity=False, player_cap=5))
    assert not ok.skipped
    # isolated node: no players
    g2 = sf.Graph.build(3, np.array([[0, 1]], np.uint64), np.ones((3, 2), np.float32))
    iso = ctx.explain_node(g2, m, 2, ExplainOptions(fidelity=False))
    assert len(iso.phi) == 0 and iso.converged
    one = ctx.explain_node(g2, m, 0, ExplainOptions(fidelity=False))
    assert len(one.phi) == 1
    assert one.phi[0] == pytest.approx(one.full_score - one.base_score)


def test_input_mismatch_rejected(ctx):
    edges, feats = toy_graph_arrays(3)
    g = sf.Graph.build(6, edges, feats)
    m = sf.Model.random(2, [4], 2, 43)
    with pytest.raises(sf.DataError):
        ctx.explain_node(g, m, 0)
    ok = sf.Graph.build(6, *toy_graph_arrays())
    with pytest.raises(sf.DataError):
        ctx.explain_node(ok, m, 6)


def test_sampled_toy_vs_reference(ctx, ref):
    edges, feats = toy_graph_arrays()
    g = sf.Graph.build(6, edges, feats)
    rg = ref.graph_build(6, edges, feats)
    m = sf.Model.random(2, [4], 2, 23)
    rm = ref.model_random(2, [4], 2, 23)
    for node in (0, 1, 5):
        ex = ctx.explain_node(g, m, node, ExplainOptions(samples=512, allow_exhaustive=False, baseline_trials=2))
        rx = ref.explain_node(rg, rm, node, samples=512, allow_exhaustive=False, trials=2, fidelity=True)
        assert ex.predicted_class == rx["predicted_class"]
        assert np.linalg.norm(ex.phi - rx["phi"]) <= 1e-3 * max(np.linalg.norm(rx["phi"]), 1e-12)
        np.testing.assert_allclose(ex.fidelity["plus"], rx["fidelity_plus"], rtol=1e-5, atol=1e-6)


def test_c1_end_to_end_vs_reference(ctx, ref, port):
    """Config C1 (2-layer Cora-shaped, n ~ 1K, k = 10K): phi within 1e-3
    relative L2, identical top-10, Fidelity+ equal (computed from predictions
    within 1e-5)."""
    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    opts = ExplainOptions(samples=cfg.samples, seed=cfg.explain_seed)
    ex = ctx.explain_node(g, m, d["target"], opts)
    rx = ref.explain_node(rg, rm, d["target"], samples=cfg.samples, seed=cfg.explain_seed, fidelity=True, world=8)
    assert ex.predicted_class == rx["predicted_class"]
    assert ex.base_score == pytest.approx(rx["base_score"], rel=1e-5)
    assert ex.full_score == pytest.approx(rx["full_score"], rel=1e-5)
    assert ex.rows == rx["rows"]
    err = np.linalg.norm(ex.phi - rx["phi"]) / np.linalg.norm(rx["phi"])
    assert err <= 1e-3, err
    top_ref = port.rank_edges(rx["phi"])[:10]
    assert [p for p, _ in ex.top] == top_ref.tolist()
    np.testing.assert_allclose(ex.fidelity["plus"], rx["fidelity_plus"], rtol=1e-4, atol=1e-6)
    assert ex.converged == bool(rx["converged"])


def test_explain_nodes_matches_explain_node(ctx):
    """explain.cpp:145-181 explain_nodes: per-node results identical to
    explain_node; an error names the node ("node N: ")."""
    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    nodes = g.select_nodes("degree-range:[4,6]:3")
    assert len(nodes) == 3
    opts = ExplainOptions(samples=2000, seed=3, baseline_trials=2)
    batch = ctx.explain_nodes(g, m, nodes, opts)
    assert [e.node for e in batch] == nodes.tolist()
    for e in batch:
        one = ctx.explain_node(g, m, e.node, opts)
        assert np.array_equal(one.phi, e.phi)
        assert one.top == e.top
    bad = sf.Model.random(cfg.feature_dim + 1, cfg.hidden, cfg.classes, 1)
    with pytest.raises(sf.DataError, match="input features"):
        ctx.explain_nodes(g, bad, nodes, opts)
    small = sf.Graph.build(3, np.array([[0, 1]], np.uint64), np.ones((3, cfg.feature_dim), np.float32))
    with pytest.raises(sf.DataError, match="^node 7: "):
        ctx.explain_nodes(small, m, [0, 7], opts)
    assert ctx.explain_nodes(g, m, [], opts) == []


@pytest.mark.parametrize("n", [40, 300])
def test_fused_solver_mode_matches_reference_protocol(ctx, port, n):
    """solver_mode 1 (one (n+1)-double all-reduce per iteration, s by
    recurrence) reaches the same phi as the reference protocol (mode 0)
    within the 1e-3 bar and uses exactly one vector all-reduce per
    iteration (+1 at init)."""
    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    res = {}
    for mode in (0, 1):
        s0 = ctx.stats()
        ex = ctx.explain_node(g, m, d["target"], ExplainOptions(samples=cfg.samples, seed=n, solver_mode=mode,
                                                                fidelity=False))
        s1 = ctx.stats()
        res[mode] = (ex, {k: s1[k] - s0[k] for k in s1})
    e0, e1 = res[0][0], res[1][0]
    assert np.linalg.norm(e1.phi - e0.phi) <= 1e-3 * np.linalg.norm(e0.phi)
    assert [p for p, _ in e1.top] == [p for p, _ in e0.top]
    assert abs(e1.iterations - e0.iterations) <= 2
    st = res[1][1]
    assert st["vector_allreduce"] == e1.iterations + 1
    assert st["scalar_allreduce"] == 0


def test_explain_nodes_workers_match_sequential(ctx):
    """sf_ctx_set_workers: targets spread over several contexts of the device
    give bitwise the explanations of the sequential loop (explain.cpp:145-181),
    in node order; an error names the lowest failing node."""
    d = W.build("C5")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    nodes = g.select_nodes("degree-range:[4,12]:24")
    opts = ExplainOptions(samples=20_000, seed=5, baseline_trials=2)
    seq = ctx.explain_nodes(g, m, nodes, opts)
    ctx.set_workers(3)
    try:
        par = ctx.explain_nodes(g, m, nodes, opts)
        assert [e.node for e in par] == [e.node for e in seq]
        for a, b in zip(seq, par):
            assert np.array_equal(a.phi, b.phi) and a.top == b.top
            assert np.array_equal(a.fidelity["plus"], b.fidelity["plus"])
        with pytest.raises(sf.DataError, match=f"^node {cfg.nodes + 5}: "):
            ctx.explain_nodes(g, m, list(nodes[:5]) + [cfg.nodes + 5, cfg.nodes + 9], opts)
    finally:
        ctx.set_workers(1)
