"""GPU: masked GCN inference (replaces evaluate_masks, gcn.cpp:40-156) within
1e-5 relative of the reference's CPU predict_batched on the same masks."""
import numpy as np
import pytest

import paper_2506_22668_b200 as sf
from conftest import toy_graph_arrays
from paper_2506_22668_b200 import workloads as W

pytestmark = pytest.mark.gpu

RTOL = 1e-5  # BASELINE north_star: predictions within 1e-5 relative


@pytest.fixture(params=["simt", "tc", "tc16"])
def kernel(request, ctx):
    """Run a parity case on every fused layer-0/1 kernel (FP32 SIMT, tcgen05
    3xTF32, tcgen05 fp16x2); the context goes back to "auto" afterwards."""
    ctx.set_fused_kernel(request.param)
    yield request.param
    ctx.set_fused_kernel("auto")


def _check_kernel(ctx, kernel, hidden):
    if len(hidden) >= 1 and hidden[0] in (64, 128):
        assert ctx.fused_kernel_used() == kernel
    elif len(hidden) >= 1 and hidden[0] == 32:
        assert ctx.fused_kernel_used() == ("tc" if kernel == "tc16" else kernel)
    elif len(hidden) >= 1 and hidden[0] in (16, 256):
        assert ctx.fused_kernel_used() == "simt"


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30))


def test_hand_case(ctx, golden):
    # test_gcn.cpp:65-76
    g = sf.Graph.build(2, np.array([[0, 1]], np.uint64), np.array([[1.0], [3.0]], np.float32))
    m = sf.Model.create([np.array([[1.0, -1.0]], np.float32)], [np.zeros(2, np.float32)])
    sg = g.extract(0, 1)
    kept = ctx.predict_probs(m, sg, np.array([1], np.uint64))
    dropped = ctx.predict_probs(m, sg, np.array([0], np.uint64))
    assert kept[0] == pytest.approx(0.9820137900379085, rel=1e-6)
    assert dropped[0] == pytest.approx(0.8807970779778823, rel=1e-6)
    assert kept[0] + kept[1] == pytest.approx(1.0, rel=1e-6)
    assert rel_err(kept[0], golden["gcn_hand"]["kept"]) <= RTOL


def test_toy_all_masks(ctx, golden):
    edges, feats = toy_graph_arrays()
    g = sf.Graph.build(6, edges, feats)
    m = sf.Model.random(2, [4], 2, 17)
    sg = g.extract(1, 2)
    allm = np.arange(1 << sg.n, dtype=np.uint64).reshape(-1, 1)
    got = ctx.predict_batched(m, sg, allm, 0)
    assert rel_err(got, golden["toy"]["predictions"]) <= RTOL


@pytest.mark.parametrize("hidden,hops,dim,classes", [
    ((6,), 2, 9, 3),          # generic widths
    ((5, 7), 3, 9, 3),        # 3-layer generic
    ((), 1, 9, 4),            # single layer (target row only)
    ((16,), 2, 33, 7),        # D = 16 fast path
    ((128,), 2, 12, 5),       # D = 128 fast path
    ((128, 128), 3, 20, 41),  # C2 widths
    ((64, 32, 8), 4, 10, 6),  # 4 layers
])
def test_random_graph_vs_reference(ctx, ref, port, kernel, hidden, hops, dim, classes):
    nodes, edges = 150, 520
    rg = ref.graph_random(nodes, edges, dim, 3, 5)
    rp, col = ref.graph_csr(rg)
    # undirected edge list for our build
    u = np.repeat(np.arange(nodes), np.diff(rp).astype(np.int64))
    e = np.stack([u, col], 1)
    e = e[e[:, 0] < e[:, 1]].astype(np.uint64)
    sgr = ref.extract(rg, 3, hops, keep_handle=True)
    g = sf.Graph.build(nodes, e, _features(nodes, dim))
    m = sf.Model.random(dim, hidden, classes, 11)
    rm = ref.model_random(dim, list(hidden), classes, 11)
    sg = g.extract(3, hops)
    assert sg.n == sgr.n
    p = sf.plan_sizes(sg.n, 700, True)
    bits, _ = ctx.generate_masks(p, 4)
    extra = np.zeros((2, bits.shape[1]), np.uint64)
    extra[1, :] = np.uint64(0xFFFFFFFFFFFFFFFF)  # full row (tail bits beyond n are ignored)
    bits = np.concatenate([bits, extra])
    cls = classes - 1
    got = ctx.predict_batched(m, sg, bits, cls)
    _check_kernel(ctx, kernel, hidden)
    want = ref.predict_batched(rm, rg, 3, bits, cls, sg=sgr)
    assert rel_err(got, want) <= RTOL
    ref.cg_free(sgr)


def _features(nodes, dim):
    # gen_random_graph's features, regenerated exactly: synthetic.cpp:71-73
    # draws float(2 * next_double() - 1) from Philox(seed, 1)
    from oracle.pyoracle import Port
    p = Port()
    raw = p.philox(5, 1, nodes * dim)
    d = (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * d - 1.0).astype(np.float32).reshape(nodes, dim)


def test_batch_size_independence(ctx):
    # test_gcn.cpp:133-165: identical results whatever the batch size
    edges, feats = toy_graph_arrays()
    g = sf.Graph.build(6, edges, feats)
    m = sf.Model.random(2, [6], 2, 5)
    sg = g.extract(1, 2)
    rng = np.random.default_rng(4)
    bits = rng.integers(0, 1 << sg.n, size=(300, 1)).astype(np.uint64)
    ref0 = ctx.predict_batched(m, sg, bits, 0, batch_size=1)
    for bs in (2, 3, 7, 50):
        assert (ctx.predict_batched(m, sg, bits, 0, batch_size=bs) == ref0).all()
    for r in range(5):
        assert ctx.predict(m, sg, bits[r], 0) == ref0[r]


def test_validation(ctx):
    g = sf.Graph.build(2, np.array([[0, 1]], np.uint64), np.array([[1.0], [3.0]], np.float32))
    m = sf.Model.create([np.array([[1.0, -1.0]], np.float32)], [np.zeros(2, np.float32)])
    sg = g.extract(0, 1)
    with pytest.raises(sf.DataError):
        ctx.predict_batched(m, sg, np.array([[1]], np.uint64), 7)
    with pytest.raises(sf.DataError):
        ctx.predict_batched(m, sg, np.array([[1]], np.uint64), 0, batch_size=0)
    wide = sf.Model.random(4, [], 2, 1)
    with pytest.raises(sf.DataError):
        ctx.predict_probs(wide, sg, np.array([1], np.uint64))


def test_c1_all_coalitions_vs_reference(ctx, ref, kernel):
    """Config C1 end to end through predict_batched: all 10,000 sampled masks."""
    d = W.build("C1")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    sg = g.extract(d["target"], cfg.hops)
    p = sf.plan_sizes(sg.n, cfg.samples, True)
    seed = sf.node_sampling_seed(cfg.explain_seed, d["target"])
    bits, _ = ctx.generate_masks(p, seed)
    got = ctx.predict_batched(m, sg, bits, 2)
    _check_kernel(ctx, kernel, cfg.hidden)
    want = ref.predict_batched(rm, rg, d["target"], bits, 2)
    assert rel_err(got, want) <= RTOL


@pytest.mark.slow
def test_c2_subset_vs_reference(ctx, ref, kernel):
    """Config C2 (3-layer, n ~ 50K): GPU predictions on the full rank shard are
    checked against the reference on a spread subset of rows."""
    d = W.build("C2")
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    sg = g.extract(d["target"], cfg.hops)
    p = sf.plan_sizes(sg.n, 20_000, True)
    bits, _ = ctx.generate_masks(p, 99)
    got = ctx.predict_batched(m, sg, bits, 5)
    _check_kernel(ctx, kernel, cfg.hidden)
    pick = np.r_[0:16, 5000:5016, 19_980:20_000]
    want = ref.predict_batched(rm, rg, d["target"], bits[pick], 5)
    assert rel_err(got[pick], want) <= RTOL


TAIL_WORKER = r"""
import os, sys
import numpy as np
sys.path.insert(0, os.environ["SF_ROOT"])
import paper_2506_22668_b200 as sf
from paper_2506_22668_b200 import workloads as W
name, k, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
ctx = sf.Context(0)
d = W.build(name)
cfg = d["cfg"]
g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
m = sf.Model.random(cfg.feature_dim, cfg.hidden, cfg.classes, cfg.model_seed)
sg = g.extract(d["target"], cfg.hops)
bits, _ = ctx.generate_masks(sf.plan_sizes(sg.n, k, True), 99)
np.save(out, ctx.predict_batched(m, sg, bits, 5))
"""


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_tail_variants_agree(ctx, ref, tmp_path, name):
    """The tcgen05 tail (SF_TAIL_TC=1: every batch) and the mma.sync tail
    (0) give the same predictions within 1e-6 at C2 and C3 (by default a
    batch takes the tcgen05 tail when it holds >= 64 tile pairs), and agree
    with the reference's predict_batched on a spread of rows."""
    import os
    import pathlib
    import subprocess
    import sys

    script = tmp_path / "tail.py"
    script.write_text(TAIL_WORKER)
    root = str(pathlib.Path(__file__).resolve().parents[1])
    preds = {}
    for t in ("0", "1"):
        out = tmp_path / f"p{t}.npy"
        subprocess.run([sys.executable, str(script), name, "20000", str(out)], check=True, timeout=900,
                       env=dict(os.environ, SF_ROOT=root, SF_TAIL_TC=t))
        preds[t] = np.load(out)
    assert rel_err(preds["1"], preds["0"]) <= 1e-6
    d = W.build(name)
    cfg = d["cfg"]
    g = sf.Graph.build(cfg.nodes, d["edges"], d["features"])
    sg = g.extract(d["target"], cfg.hops)
    bits, _ = ctx.generate_masks(sf.plan_sizes(sg.n, 20_000, True), 99)
    rg = ref.graph_build(cfg.nodes, d["edges"], d["features"])
    rm = ref.model_random(cfg.feature_dim, list(cfg.hidden), cfg.classes, cfg.model_seed)
    pick = np.r_[0:8, 10_000:10_008, 19_992:20_000]
    want = ref.predict_batched(rm, rg, d["target"], bits[pick], 5)
    for t in ("0", "1"):
        assert rel_err(preds[t][pick], want) <= RTOL
