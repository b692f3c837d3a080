"""TEST INFRASTRUCTURE ONLY — ctypes views of the two CPU oracles.

* ``Ref``  — the unmodified reference core compiled by ``oracle/Makefile``
  into ``oracle/_ref/libshapflow_ref.so`` (driver: ``oracle/ref_driver.cpp``).
* ``Port`` — the plain-C restatement ``oracle/shapflow_port.c`` compiled into
  ``oracle/_port/libshapflow_port.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module. The product package never
does; it fails loudly when its CUDA library is missing instead.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libshapflow_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libshapflow_port.so")

u8p = C.c_void_p


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Subgraph:
    """ComputationalGraph arrays (graph.hpp:36-53)."""

    V: int
    n: int
    dim: int
    row_ptr: np.ndarray  # u64[V+1]
    col: np.ndarray  # u32[2n]
    edge_player: np.ndarray  # u32[2n]
    players: np.ndarray  # u32[n,2] local (u<v), lexicographic
    local_to_global: np.ndarray  # u32[V]
    features: np.ndarray  # f32[V,dim]
    handle: object = None


@dataclass
class Model:
    dims: list
    weights: list  # f32 [in,out] per layer
    biases: list

    @property
    def depth(self):
        return len(self.weights)

    def flat(self):
        return (np.concatenate([w.ravel() for w in self.weights]).astype(np.float32),
                np.concatenate([b.ravel() for b in self.biases]).astype(np.float32))


class Ref:
    """The compiled reference (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference oracle not built: {path} (run make -C oracle ref)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_graph_load", "ref_graph_random", "ref_graph_build", "ref_model_random",
                     "ref_model_from_arrays", "ref_model_load", "ref_extract"):
            getattr(L, name).restype = C.c_void_p
        L.ref_node_sampling_seed.restype = C.c_uint64
        L.ref_binomial_or_max.restype = C.c_uint64
        L.ref_model_depth.restype = C.c_int

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.ref_last_error().decode())

    # ----------------------------------------------------------- primitives
    def philox(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        self.L.ref_philox_u64(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(count), _p(out))
        return out

    def node_sampling_seed(self, seed, node):
        return int(self.L.ref_node_sampling_seed(C.c_uint64(seed), C.c_uint32(node)))

    def binomial_or_max(self, n, s):
        return int(self.L.ref_binomial_or_max(C.c_uint32(n), C.c_uint32(s)))

    def kernel_weight(self, n, s):
        out = C.c_double()
        self._chk(self.L.ref_kernel_weight(C.c_uint32(n), C.c_uint32(s), C.byref(out)))
        return out.value

    def plan_sizes(self, n, k, allow_exhaustive=True):
        nc, ex, req = C.c_uint64(), C.c_int(), C.c_uint64()
        self._chk(self.L.ref_plan_sizes(C.c_uint32(n), C.c_uint64(k), C.c_int(int(allow_exhaustive)),
                                        None, None, None, C.c_uint64(0), C.byref(nc), C.byref(ex),
                                        C.byref(req)))
        m = nc.value
        sizes = np.zeros(m, np.uint32)
        pairs = np.zeros(m, np.uint64)
        first = np.zeros(m, np.uint64)
        self._chk(self.L.ref_plan_sizes(C.c_uint32(n), C.c_uint64(k), C.c_int(int(allow_exhaustive)),
                                        _p(sizes), _p(pairs), _p(first), C.c_uint64(m), C.byref(nc),
                                        C.byref(ex), C.byref(req)))
        return dict(sizes=sizes, pairs=pairs, first=first, exhaustive=bool(ex.value),
                    requested=req.value)

    def generate_masks(self, n, k, seed, rank=0, world=1, allow_exhaustive=True):
        rows, words = C.c_uint64(), C.c_uint64()
        self._chk(self.L.ref_generate_masks(C.c_uint32(n), C.c_uint64(k), C.c_int(int(allow_exhaustive)),
                                            C.c_uint64(seed), C.c_int(rank), C.c_int(world), None,
                                            C.c_uint64(0), C.byref(rows), C.byref(words), None))
        out = np.zeros((rows.value, words.value), np.uint64)
        ros = np.zeros(n + 1, np.uint64)
        self._chk(self.L.ref_generate_masks(C.c_uint32(n), C.c_uint64(k), C.c_int(int(allow_exhaustive)),
                                            C.c_uint64(seed), C.c_int(rank), C.c_int(world), _p(out),
                                            C.c_uint64(out.size), C.byref(rows), C.byref(words),
                                            _p(ros)))
        return out, ros

    # ----------------------------------------------------------- graphs
    def graph_random(self, nodes, edges, dim, classes, seed):
        h = self.L.ref_graph_random(C.c_uint32(nodes), C.c_uint64(edges), C.c_uint64(dim),
                                    C.c_uint32(classes), C.c_uint64(seed))
        if not h:
            raise OracleError(2, self.L.ref_last_error().decode())
        return C.c_void_p(h)

    def graph_load(self, path):
        h = self.L.ref_graph_load(path.encode())
        if not h:
            raise OracleError(2, self.L.ref_last_error().decode())
        return C.c_void_p(h)

    def graph_build(self, num_nodes, edges_uv, features):
        edges_uv = np.ascontiguousarray(edges_uv, np.uint64).reshape(-1, 2)
        features = np.ascontiguousarray(features, np.float32)
        h = self.L.ref_graph_build(C.c_uint32(num_nodes), _p(edges_uv), C.c_uint64(len(edges_uv)),
                                   _p(features), C.c_uint64(features.shape[1]))
        if not h:
            raise OracleError(2, self.L.ref_last_error().decode())
        return C.c_void_p(h)

    def select_nodes(self, g, rule):
        cnt = C.c_uint64()
        self._chk(self.L.ref_select_nodes(g, rule.encode(), None, C.c_uint64(0), C.byref(cnt)))
        out = np.zeros(cnt.value, np.uint32)
        self._chk(self.L.ref_select_nodes(g, rule.encode(), _p(out), C.c_uint64(len(out)), C.byref(cnt)))
        return out

    def graph_save(self, g, path):
        self._chk(self.L.ref_graph_save(g, path.encode()))

    def graph_csr(self, g):
        nodes, nnz, dim = C.c_uint32(), C.c_uint64(), C.c_uint64()
        self.L.ref_graph_dims(g, C.byref(nodes), C.byref(nnz), C.byref(dim))
        rp = np.zeros(nodes.value + 1, np.uint64)
        col = np.zeros(nnz.value, np.uint32)
        self.L.ref_graph_copy(g, _p(rp), _p(col))
        return rp, col

    def graph_free(self, g):
        self.L.ref_graph_free(g)

    # ----------------------------------------------------------- models
    def model_random(self, input_dim, hidden, classes, seed):
        h = np.asarray(hidden, np.uint64)
        ptr = self.L.ref_model_random(C.c_uint64(input_dim), _p(h) if len(h) else None, C.c_int(len(h)),
                                      C.c_uint32(classes), C.c_uint64(seed))
        if not ptr:
            raise OracleError(2, self.L.ref_last_error().decode())
        return self._model_out(C.c_void_p(ptr))

    def model_load(self, path):
        ptr = self.L.ref_model_load(path.encode())
        if not ptr:
            raise OracleError(2, self.L.ref_last_error().decode())
        return self._model_out(C.c_void_p(ptr))

    def _model_out(self, ptr):
        L = self.L.ref_model_depth(ptr)
        dims, ws, bs = [], [], []
        for l in range(L):
            i, o = C.c_uint64(), C.c_uint64()
            self.L.ref_model_layer(ptr, C.c_int(l), C.byref(i), C.byref(o), None, None)
            w = np.zeros((i.value, o.value), np.float32)
            b = np.zeros(o.value, np.float32)
            self.L.ref_model_layer(ptr, C.c_int(l), C.byref(i), C.byref(o), _p(w), _p(b))
            if l == 0:
                dims.append(i.value)
            dims.append(o.value)
            ws.append(w)
            bs.append(b)
        self.L.ref_model_free(ptr)
        return Model(dims, ws, bs)

    def model_handle(self, m: Model):
        dims = np.asarray(m.dims, np.uint64)
        w, b = m.flat()
        return C.c_void_p(self.L.ref_model_from_arrays(C.c_int(m.depth), _p(dims), _p(w), _p(b)))

    def model_free(self, h):
        self.L.ref_model_free(h)

    def model_save(self, m: Model, path):
        h = self.model_handle(m)
        try:
            self._chk(self.L.ref_model_save(h, path.encode()))
        finally:
            self.model_free(h)

    # ----------------------------------------------------------- subgraph
    def extract(self, g, target, hops, keep_handle=False):
        h = self.L.ref_extract(g, C.c_uint32(target), C.c_int(hops))
        if not h:
            raise OracleError(2, self.L.ref_last_error().decode())
        h = C.c_void_p(h)
        V, n, nnz, dim = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.L.ref_cg_dims(h, C.byref(V), C.byref(n), C.byref(nnz), C.byref(dim))
        rp = np.zeros(V.value + 1, np.uint64)
        col = np.zeros(nnz.value, np.uint32)
        ep = np.zeros(nnz.value, np.uint32)
        pl = np.zeros((n.value, 2), np.uint32)
        l2g = np.zeros(V.value, np.uint32)
        feat = np.zeros((V.value, dim.value), np.float32)
        self.L.ref_cg_copy(h, _p(rp), _p(col), _p(ep), _p(pl), _p(l2g), _p(feat))
        sg = Subgraph(V.value, n.value, dim.value, rp, col, ep, pl, l2g, feat, h if keep_handle else None)
        if not keep_handle:
            self.L.ref_cg_free(h)
        return sg

    def cg_free(self, sg: Subgraph):
        if sg.handle is not None:
            self.L.ref_cg_free(sg.handle)
            sg.handle = None

    # ----------------------------------------------------------- predict
    def predict_batched(self, m: Model, g, target, bits, cls, batch=50, sg=None):
        """predict_batched on the extracted subgraph of `target` (gcn.cpp:259)."""
        bits = np.ascontiguousarray(bits, np.uint64)
        mh = self.model_handle(m)
        own = sg is None
        if own:
            sg = self.extract(g, target, m.depth, keep_handle=True)
        try:
            out = np.zeros(bits.shape[0], np.float32)
            self._chk(self.L.ref_predict_batched(mh, sg.handle, _p(bits), C.c_uint64(bits.shape[0]),
                                                 C.c_uint64(bits.shape[1]), C.c_uint32(cls),
                                                 C.c_uint64(batch), _p(out)))
            return out
        finally:
            self.model_free(mh)
            if own:
                self.cg_free(sg)

    def predict_probs(self, m: Model, sg: Subgraph, mask):
        mask = np.ascontiguousarray(mask, np.uint64)
        mh = self.model_handle(m)
        try:
            out = np.zeros(m.dims[-1], np.float32)
            self._chk(self.L.ref_predict_probs(mh, sg.handle, _p(mask), C.c_uint64(mask.size), _p(out)))
            return out
        finally:
            self.model_free(mh)

    # ----------------------------------------------------------- solve
    def solve_cgls(self, n, bits, values, base, full, cscale=1e6, tol=1e-6, max_iter=0, fixed_order=True):
        bits = np.ascontiguousarray(bits, np.uint64)
        values = np.ascontiguousarray(values, np.float64)
        phi = np.zeros(n, np.float64)
        it, res, conv = C.c_uint64(), C.c_double(), C.c_int()
        self._chk(self.L.ref_solve_cgls(C.c_uint32(n), _p(bits), C.c_uint64(bits.shape[0]),
                                        C.c_uint64(bits.shape[1]), _p(values), C.c_double(base),
                                        C.c_double(full), C.c_double(cscale), C.c_double(tol),
                                        C.c_uint64(max_iter), C.c_int(int(fixed_order)), _p(phi),
                                        C.byref(it), C.byref(res), C.byref(conv)))
        return phi, it.value, res.value, bool(conv.value)

    def solve_direct(self, n, bits, values, base, full, cscale=1e6):
        bits = np.ascontiguousarray(bits, np.uint64)
        values = np.ascontiguousarray(values, np.float64)
        phi = np.zeros(n, np.float64)
        self._chk(self.L.ref_solve_direct(C.c_uint32(n), _p(bits), C.c_uint64(bits.shape[0]),
                                          C.c_uint64(bits.shape[1]), _p(values), C.c_double(base),
                                          C.c_double(full), C.c_double(cscale), _p(phi)))
        return phi

    def exact_shapley_gnn(self, m: Model, sg: Subgraph, cls):
        mh = self.model_handle(m)
        try:
            phi = np.zeros(sg.n, np.float64)
            self._chk(self.L.ref_exact_shapley_gnn(mh, sg.handle, C.c_uint32(cls), _p(phi)))
            return phi
        finally:
            self.model_free(mh)

    def evaluate_fidelity(self, m: Model, sg: Subgraph, cls, phi, counts=(5, 10, 20),
                          sparsities=(0.1, 0.3, 0.5, 0.7, 0.9), seed=0, trials=8):
        mh = self.model_handle(m)
        counts = np.asarray(counts, np.uint32)
        sp = np.asarray(sparsities, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        outs = [np.zeros(len(counts)), np.zeros(len(counts)), np.zeros(len(sp)), np.zeros(len(sp))]
        try:
            self._chk(self.L.ref_evaluate_fidelity(mh, sg.handle, C.c_uint32(cls), _p(phi),
                                                   C.c_uint64(len(phi)), _p(counts), C.c_uint64(len(counts)),
                                                   _p(sp), C.c_uint64(len(sp)), C.c_uint64(seed),
                                                   C.c_uint32(trials), *[_p(o) for o in outs]))
        finally:
            self.model_free(mh)
        return dict(plus=outs[0], plus_random=outs[1], minus=outs[2], minus_random=outs[3])

    def explain_node(self, g, m: Model, node, samples=0, batch=50, seed=0, tol=1e-6, max_iter=0,
                     allow_exhaustive=True, fidelity=False, trials=8, world=1, phi_cap=1 << 22):
        mh = self.model_handle(m)
        phi = np.zeros(phi_cap, np.float64)
        meta = np.zeros(16, np.float64)
        try:
            self._chk(self.L.ref_explain_node(g, mh, C.c_uint32(node), C.c_uint64(samples), C.c_uint64(batch),
                                              C.c_uint64(seed), C.c_double(tol), C.c_uint64(max_iter),
                                              C.c_int(int(allow_exhaustive)), C.c_int(int(fidelity)),
                                              C.c_uint32(trials), C.c_int(world), _p(phi),
                                              C.c_uint64(phi_cap), _p(meta)))
        finally:
            self.model_free(mh)
        n = int(meta[12])
        keys = ["predicted_class", "base_score", "full_score", "iterations", "residual", "converged", "rows",
                "exhaustive", "sampling_ms", "prediction_ms", "solve_ms", "total_ms", "n"]
        out = {k: meta[i] for i, k in enumerate(keys)}
        out["predicted_class"] = int(out["predicted_class"])
        out["fidelity_plus"] = meta[13:16].copy()
        out["phi"] = phi[:n].copy()
        return out

    def sample_predict(self, m: Model, sg: Subgraph, cls, k, seed, world, infer_rows, batch=50,
                       allow_exhaustive=True):
        mh = self.model_handle(m)
        out = np.zeros(4)
        try:
            self._chk(self.L.ref_sample_predict(mh, sg.handle, C.c_uint32(cls), C.c_uint64(k), C.c_uint64(seed),
                                                C.c_int(world), C.c_uint64(infer_rows), C.c_uint64(batch),
                                                C.c_int(int(allow_exhaustive)), _p(out)))
        finally:
            self.model_free(mh)
        return dict(sampling_ms=out[0], prediction_ms=out[1], rows_predicted=int(out[2]),
                    rows_sampled=int(out[3]))


class Port:
    """The plain-C restatement (oracle/shapflow_port.c)."""

    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"port oracle not built: {path} (run make -C oracle port)")
        L = C.CDLL(path)
        self.L = L
        L.port_node_sampling_seed.restype = C.c_uint64
        L.port_binomial_or_max.restype = C.c_uint64
        L.port_generate_masks.restype = C.c_uint64

    def philox(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        self.L.port_philox_u64(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(count), _p(out))
        return out

    def node_sampling_seed(self, seed, node):
        return int(self.L.port_node_sampling_seed(C.c_uint64(seed), C.c_uint32(node)))

    def binomial_or_max(self, n, s):
        return int(self.L.port_binomial_or_max(C.c_uint32(n), C.c_uint32(s)))

    def plan_sizes(self, n, k, allow_exhaustive=True):
        cap = max(n // 2, 1)
        sizes = np.zeros(cap, np.uint32)
        pairs = np.zeros(cap, np.uint64)
        first = np.zeros(cap, np.uint64)
        nc, ex, req = C.c_uint64(), C.c_int(), C.c_uint64()
        rc = self.L.port_plan_sizes(C.c_uint32(n), C.c_uint64(k), C.c_int(int(allow_exhaustive)), _p(sizes),
                                    _p(pairs), _p(first), C.byref(nc), C.byref(ex), C.byref(req))
        if rc:
            raise OracleError(rc, "plan_sizes: invalid input")
        m = nc.value
        return dict(sizes=sizes[:m].copy(), pairs=pairs[:m].copy(), first=first[:m].copy(),
                    exhaustive=bool(ex.value), requested=req.value)

    def generate_masks(self, n, plan, seed, rank=0, world=1, g_begin=0, g_end=None):
        total = int(plan["first"][-1] + plan["pairs"][-1]) if len(plan["sizes"]) else 0
        if g_end is None:
            g_end = total
        local = len(range(g_begin + ((rank - g_begin) % world), g_end, world)) if g_end > g_begin else 0
        W = (n + 63) // 64
        out = np.zeros((2 * local, W), np.uint64)
        rows = self.L.port_generate_masks(C.c_uint32(n), _p(plan["sizes"]), _p(plan["pairs"]), _p(plan["first"]),
                                          C.c_uint64(len(plan["sizes"])), C.c_int(int(plan["exhaustive"])),
                                          C.c_uint64(seed), C.c_int(rank), C.c_int(world), C.c_uint64(g_begin),
                                          C.c_uint64(g_end), _p(out))
        assert rows == out.shape[0]
        return out

    def rows_of_size(self, n, plan):
        ros = np.zeros(n + 1, np.uint64)
        for s, p in zip(plan["sizes"], plan["pairs"]):
            s, p = int(s), int(p)
            if 2 * s == n:
                ros[s] += 2 * p
            else:
                ros[s] += p
                ros[n - s] += p
        return ros

    def gcn_predict(self, sg: Subgraph, m: Model, bits, cls):
        bits = np.ascontiguousarray(bits, np.uint64)
        dims = np.asarray(m.dims, np.uint64)
        w, b = m.flat()
        out = np.zeros(bits.shape[0], np.float32)
        self.L.port_gcn_predict(C.c_uint32(sg.V), _p(np.ascontiguousarray(sg.row_ptr, np.uint64)),
                                _p(np.ascontiguousarray(sg.col, np.uint32)),
                                _p(np.ascontiguousarray(sg.edge_player, np.uint32)),
                                _p(np.ascontiguousarray(sg.features, np.float32)), C.c_int(m.depth), _p(dims),
                                _p(w), _p(b), _p(bits), C.c_uint64(bits.shape[0]), C.c_uint64(bits.shape[1]),
                                C.c_uint32(cls), _p(out))
        return out

    def gcn_probs(self, sg: Subgraph, m: Model, mask):
        mask = np.ascontiguousarray(mask, np.uint64)
        dims = np.asarray(m.dims, np.uint64)
        w, b = m.flat()
        out = np.zeros(m.dims[-1], np.float32)
        self.L.port_gcn_probs(C.c_uint32(sg.V), _p(np.ascontiguousarray(sg.row_ptr, np.uint64)),
                              _p(np.ascontiguousarray(sg.col, np.uint32)),
                              _p(np.ascontiguousarray(sg.edge_player, np.uint32)),
                              _p(np.ascontiguousarray(sg.features, np.float32)), C.c_int(m.depth), _p(dims), _p(w),
                              _p(b), _p(mask), _p(out))
        return out

    def cgls(self, n, bits, rows_of_size, values, base, full, cscale=1e6, tol=1e-6, max_iter=0,
             fixed_order=True, global_pairs=None):
        bits = np.ascontiguousarray(bits, np.uint64)
        values = np.ascontiguousarray(values, np.float64)
        ros = np.ascontiguousarray(rows_of_size, np.uint64)
        gp = bits.shape[0] // 2 if global_pairs is None else global_pairs
        phi = np.zeros(n, np.float64)
        it, res, conv = C.c_uint64(), C.c_double(), C.c_int()
        rc = self.L.port_cgls(C.c_uint32(n), _p(bits), C.c_uint64(bits.shape[0]), C.c_uint64(bits.shape[1]),
                              _p(ros), C.c_uint64(gp), _p(values), C.c_double(base), C.c_double(full),
                              C.c_double(cscale), C.c_double(tol), C.c_uint64(max_iter), C.c_int(int(fixed_order)),
                              _p(phi), C.byref(it), C.byref(res), C.byref(conv))
        if rc:
            raise OracleError(rc, "cgls failed")
        return phi, it.value, res.value, bool(conv.value)

    def cgls_sparse(self, n, bits, rows_of_size, values, base, full, cscale=1e6, tol=1e-6, max_iter=0,
                    threads=None):
        """port_cgls_sparse: the bit-row CGLS for large k x n (set-bit passes,
        pthreads), agreeing with port_cgls / the reference to rounding."""
        bits = np.ascontiguousarray(bits, np.uint64)
        values = np.ascontiguousarray(values, np.float64)
        ros = np.ascontiguousarray(rows_of_size, np.uint64)
        threads = threads or min(64, os.cpu_count() or 1)
        phi = np.zeros(n, np.float64)
        it, res, conv = C.c_uint64(), C.c_double(), C.c_int()
        rc = self.L.port_cgls_sparse(C.c_uint32(n), _p(bits), C.c_uint64(bits.shape[0]), C.c_uint64(bits.shape[1]),
                                     _p(ros), _p(values), C.c_double(base), C.c_double(full), C.c_double(cscale),
                                     C.c_double(tol), C.c_uint64(max_iter), C.c_int(threads), _p(phi),
                                     C.byref(it), C.byref(res), C.byref(conv))
        if rc:
            raise OracleError(rc, "cgls_sparse failed")
        return phi, it.value, res.value, bool(conv.value)

    def rank_edges(self, phi):
        phi = np.ascontiguousarray(phi, np.float64)
        order = np.zeros(len(phi), np.uint32)
        self.L.port_rank_edges(_p(phi), C.c_uint32(len(phi)), _p(order))
        return order
