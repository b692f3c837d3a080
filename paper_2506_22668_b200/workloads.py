"""Synthetic workloads for BASELINE.json's configs (C1-C5).

The reference ships only an Erdos-Renyi generator (synthetic.cpp:56-86), so the
"Cora / Reddit / products-shaped" graphs come from a Chung-Lu power-law
generator here (numpy PCG64, fixed seeds -> identical arrays on every box).
Both the B200 path and the CPU oracle build their Graph from the same edge
list + features (build_graph symmetrizes / dedupes identically), so parity
tests compare like with like. Models use the reference's gen_random_model
(Glorot from Philox stream 16+l, synthetic.cpp:88-118) via sf_model_random.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    nodes: int
    edges: int
    gamma: float
    feature_dim: int
    hidden: tuple
    classes: int
    hops: int
    target_players: int  # desired |E(G_c)|
    samples: int  # k coalitions
    graph_seed: int = 7
    model_seed: int = 7
    explain_seed: int = 1
    candidates: int = 64


CONFIGS = {
    # 2-layer, Cora-shaped (2,708 nodes, d 1433 -> 16 -> 7), ~1K-edge G_c, k = 10K
    "C1": Config("C1", 2708, 5429, 2.3, 1433, (16,), 7, 2, 1000, 10_000, candidates=2708),
    # 3-layer, Reddit-shaped power law (d 602 -> 128 -> 128 -> 41), ~50K-edge G_c, k = 500K
    "C2": Config("C2", 20_000, 80_000, 2.3, 602, (128, 128), 41, 3, 50_000, 500_000),
    # 3-layer, products-shaped (d 100 -> 128 -> 128 -> 47), ~200K-edge G_c, k = 2M
    "C3": Config("C3", 60_000, 330_000, 2.3, 100, (128, 128), 47, 3, 200_000, 2_000_000),
    # 3-layer, 1M-edge G_c, k = 10M
    "C4": Config("C4", 260_000, 1_500_000, 2.3, 100, (128, 128), 47, 3, 1_000_000, 10_000_000),
    # batch of 1,024 targets, 2-layer, 256-d features, k = 100K each
    "C5": Config("C5", 20_000, 100_000, 2.5, 256, (128,), 40, 2, 0, 100_000),
}


def chung_lu(nodes, edges, gamma, seed):
    """Undirected power-law edge list (u < v, unique, no self-loops)."""
    rng = np.random.default_rng(seed)
    alpha = 1.0 / (gamma - 1.0)
    w = (np.arange(nodes, dtype=np.float64) + 10.0) ** (-alpha)
    p = w / w.sum()
    m = int(edges * 1.25) + 16
    u = rng.choice(nodes, m, p=p)
    v = rng.choice(nodes, m, p=p)
    perm = rng.permutation(nodes)
    u, v = perm[u], perm[v]
    keep = u != v
    a = np.minimum(u[keep], v[keep]).astype(np.int64)
    b = np.maximum(u[keep], v[keep]).astype(np.int64)
    key = a * nodes + b
    _, first = np.unique(key, return_index=True)
    first.sort()  # keep generation order, drop duplicates
    key = key[first][:edges]
    return np.stack([key // nodes, key % nodes], 1).astype(np.uint64)


def features(nodes, dim, seed):
    rng = np.random.default_rng(seed + 1)
    return rng.uniform(-1.0, 1.0, size=(nodes, dim)).astype(np.float32)


def _csr(nodes, edges):
    u = edges[:, 0].astype(np.int64)
    v = edges[:, 1].astype(np.int64)
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rp = np.zeros(nodes + 1, np.int64)
    np.add.at(rp, src + 1, 1)
    return np.cumsum(rp), dst


def ball_edges(rp, col, target, hops):
    """(ball node count, induced undirected edge count) of the hops-ball."""
    nodes = len(rp) - 1
    seen = np.zeros(nodes, bool)
    seen[target] = True
    frontier = np.array([target])
    for _ in range(hops):
        if frontier.size == 0:
            break
        nb = np.concatenate([col[rp[x]:rp[x + 1]] for x in frontier]) if frontier.size else np.zeros(0, np.int64)
        nb = np.unique(nb)
        new = nb[~seen[nb]]
        seen[new] = True
        frontier = new
    ball = np.nonzero(seen)[0]
    deg_in = 0
    for x in ball:
        deg_in += int(seen[col[rp[x]:rp[x + 1]]].sum())
    return len(ball), deg_in // 2


def pick_target(cfg: Config, edges):
    """Node whose hops-ball has the induced-edge count closest to cfg.target_players."""
    rp, col = _csr(cfg.nodes, edges)
    rng = np.random.default_rng(cfg.graph_seed + 99)
    deg = np.diff(rp)
    cand = np.nonzero(deg > 0)[0]
    if len(cand) > cfg.candidates:
        cand = rng.choice(cand, cfg.candidates, replace=False)
    best, best_gap = None, None
    for c in sorted(int(x) for x in cand):
        _, ne = ball_edges(rp, col, c, cfg.hops)
        gap = abs(ne - cfg.target_players)
        if best is None or gap < best_gap:
            best, best_gap = c, gap
    return best


def select_degree_band(edges, nodes, lo, hi, count):
    """explain.cpp:185-202 degree-range rule: first `count` ids with degree in [lo, hi]."""
    rp, _ = _csr(nodes, edges)
    deg = np.diff(rp)
    ids = np.nonzero((deg >= lo) & (deg <= hi))[0]
    return [int(x) for x in ids[:count]]


def build(name):
    """-> dict(cfg, edges, features, target) for one config (arrays, no files)."""
    cfg = CONFIGS[name]
    e = chung_lu(cfg.nodes, cfg.edges, cfg.gamma, cfg.graph_seed)
    x = features(cfg.nodes, cfg.feature_dim, cfg.graph_seed)
    target = pick_target(cfg, e) if cfg.target_players else None
    return dict(cfg=cfg, edges=e, features=x, target=target)


def write_sfg(path, nodes, edges, feats, labels=None):
    """SFG1 binary (graph.cpp:35-64 / 165-193)."""
    with open(path, "wb") as f:
        f.write(b"SFG1")
        np.array([nodes, len(edges), feats.shape[1]], np.uint64).tofile(f)
        np.ascontiguousarray(edges, np.uint64).tofile(f)
        np.ascontiguousarray(feats, np.float32).tofile(f)
        lab = np.zeros(nodes, np.uint32) if labels is None else np.asarray(labels, np.uint32)
        lab.tofile(f)
