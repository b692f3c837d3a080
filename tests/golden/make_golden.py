"""Regenerate tests/golden/golden.json from the compiled reference (oracle/_ref).

Run in the builder container, where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/libshapflow_ref.so:

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/shapflow_port.c) and the B200 path
without needing /root/reference at test time. Every value comes from the
reference's own code paths (philox.hpp, sampler.cpp, gcn.cpp, solver.cpp,
explain.cpp, oracle.cpp, fidelity.cpp) through oracle/ref_driver.cpp.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Ref  # noqa: E402


def hexs(a):
    return [f"{int(x):016x}" for x in np.asarray(a, np.uint64).ravel()]


def toy_graph(r, dim=2):
    # test_helpers.hpp:73-91: 5-cycle + chord 1-3 + pendant 1-5, features 0.1*(i+1)
    edges = np.array([[0, 1], [1, 2], [2, 3], [3, 4], [4, 0], [1, 3], [1, 5]], np.uint64)
    feats = (0.1 * (np.arange(6 * dim, dtype=np.float32) + 1)).astype(np.float32).reshape(6, dim)
    return edges, feats, r.graph_build(6, edges, feats)


def main():
    r = Ref()
    g = {}
    g["philox"] = [
        dict(seed=0, stream=0, out=hexs(r.philox(0, 0, 8))),
        dict(seed=0x0123456789ABCDEF, stream=7, out=hexs(r.philox(0x0123456789ABCDEF, 7, 8))),
        dict(seed=0xFFFFFFFFFFFFFFFF, stream=0xFFFFFFFF00000001, out=hexs(r.philox(2**64 - 1, 0xFFFFFFFF00000001, 6))),
    ]
    g["node_sampling_seed"] = [dict(seed=s, node=n, out=f"{r.node_sampling_seed(s, n):016x}")
                               for s, n in [(1, 61), (0, 0), (7, 3), (2**63, 12345)]]
    g["binomial"] = [dict(n=n, s=s, out=str(r.binomial_or_max(n, s)))
                     for n, s in [(4, 2), (30, 15), (64, 32), (67, 33), (68, 34), (3, 7)]]
    plans = []
    for n, k, ex in [(12, 1000, False), (4, 110, False), (3, 10, False), (4, 20, True), (30, 25000, True),
                     (999, 10000, True), (49648, 500000, True), (70, 2000, False), (6, 11, False)]:
        p = r.plan_sizes(n, k, ex)
        plans.append(dict(n=n, k=k, allow=ex, exhaustive=p["exhaustive"], requested=p["requested"],
                          sizes=p["sizes"].tolist(), pairs=[int(x) for x in p["pairs"]],
                          first=[int(x) for x in p["first"]]))
    g["plans"] = plans
    masks = []
    for n, k, ex, seed, rank, world in [(12, 1000, False, 42, 0, 1), (12, 1000, False, 42, 3, 8),
                                        (70, 2000, False, 11, 1, 3), (9, 1022, True, 3, 0, 1),
                                        (6, 62, True, 0, 2, 4), (200, 400, False, 5, 0, 2),
                                        (999, 2000, True, 0x516f7aecd40a0d17, 0, 1)]:
        bits, ros = r.generate_masks(n, k, seed, rank, world, allow_exhaustive=ex)
        masks.append(dict(n=n, k=k, allow=ex, seed=f"{seed:016x}", rank=rank, world=world, shape=list(bits.shape),
                          bits=hexs(bits), rows_of_size=[int(x) for x in ros]))
    g["masks"] = masks
    # acceptance criterion 5 (acceptance.cpp:387-406)
    c5 = []
    for rk in range(4):
        bits, _ = r.generate_masks(30, 25000, 9, rk, 4, allow_exhaustive=True)
        c5.append(dict(rank=rk, rows=int(bits.shape[0]),
                       popcount=int(sum(bin(int(x)).count("1") for x in bits.ravel()))))
    g["acceptance_c5"] = c5

    # GCN hand case (test_gcn.cpp:24-76): 2 nodes, features 1 and 3, logits (x, -x)
    hg = r.graph_build(2, np.array([[0, 1]], np.uint64), np.array([[1.0], [3.0]], np.float32))
    from oracle.pyoracle import Model
    hm = Model([1, 2], [np.array([[1.0, -1.0]], np.float32)], [np.zeros(2, np.float32)])
    hsg = r.extract(hg, 0, 1, keep_handle=True)
    g["gcn_hand"] = dict(kept=float(r.predict_probs(hm, hsg, np.array([1], np.uint64))[0]),
                         dropped=float(r.predict_probs(hm, hsg, np.array([0], np.uint64))[0]))
    r.cg_free(hsg)

    # toy graph predictions for all 2^7 masks, 2-layer model (gen_random_model(2,{4},2,17))
    edges, feats, tg = toy_graph(r)
    m = r.model_random(2, [4], 2, 17)
    sg = r.extract(tg, 1, 2, keep_handle=True)
    allm = np.arange(1 << sg.n, dtype=np.uint64).reshape(-1, 1)
    pred = r.predict_batched(m, tg, 1, allm, 0, sg=sg)
    g["toy"] = dict(edges=edges.tolist(), features=feats.ravel().tolist(), target=1, hops=2,
                    model_seed=17, hidden=[4], classes=2, n=sg.n,
                    predictions=[float(x) for x in pred],
                    exact_shapley=[float(x) for x in r.exact_shapley_gnn(m, sg, 0)])
    ex = r.explain_node(tg, m, 1, seed=0, fidelity=False)
    g["toy"]["explain_phi"] = [float(x) for x in ex["phi"]]
    g["toy"]["explain_class"] = ex["predicted_class"]
    r.cg_free(sg)

    # sampled CGLS on a Philox toy game (test_solver.cpp:23-37 style), n = 11, k = 500
    n = 11
    bits, ros = r.generate_masks(n, 500, 31, 0, 1, allow_exhaustive=False)
    vals = np.array([r.philox(int(x), 3, 1)[0] >> 11 for x in bits[:, 0]], np.float64) * 2.0 ** -53
    phi, it, res, conv = r.solve_cgls(n, bits, vals, 0.2, 0.9, max_iter=44)
    g["cgls_toy"] = dict(n=n, k=500, seed=31, base=0.2, full=0.9, max_iter=44, values=vals.tolist(),
                         phi=phi.tolist(), iterations=it, converged=conv, residual=res)

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
