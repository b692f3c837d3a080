"""ctypes mirror of the shapflow API over ``libshapflow_b200.so``.

Names and argument meaning follow the reference C++ API
(/root/reference/proj/core/include/shapflow/*.hpp); status codes map back onto
the reference's exception types (error.hpp:10-27).
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(HERE, "libshapflow_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "shapflow_b200.h")


class ShapflowError(RuntimeError):
    code = 1


class DataError(ShapflowError):  # error.hpp:10-14
    code = 2


class NumericalError(ShapflowError):  # error.hpp:16-20
    code = 3


class ProtocolError(ShapflowError):  # error.hpp:22-27
    code = 4


_ERRORS = {1: ShapflowError, 2: DataError, 3: NumericalError, 4: ProtocolError}


def _header_symbols():
    """Every function the public header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", txt)))


EXPORTED_SYMBOLS = _header_symbols()


class _Lib:
    """Lazily loaded library; loading fails loudly (no fallback)."""

    def __init__(self):
        self._L = None

    def load(self):
        if self._L is None:
            if not os.path.exists(lib_path):
                raise ImportError(
                    f"{lib_path} is missing: build it with `make -C paper_2506_22668_b200/csrc` "
                    "(or __graft_entry__.build()); there is no CPU fallback")
            L = C.CDLL(lib_path)
            L.sf_last_error.restype = C.c_char_p
            L.sf_version.restype = C.c_char_p
            for name in ("sf_node_sampling_seed", "sf_auto_samples", "sf_binomial_or_max", "sf_ctx_launches"):
                getattr(L, name).restype = C.c_uint64
            L.sf_node_sampling_seed.argtypes = [C.c_uint64, C.c_uint32]
            L.sf_auto_samples.argtypes = [C.c_uint64]
            L.sf_binomial_or_max.argtypes = [C.c_uint32, C.c_uint32]
            L.sf_ctx_launches.argtypes = [C.c_void_p]
            L.sf_ctx_rank.argtypes = [C.c_void_p]
            L.sf_ctx_world.argtypes = [C.c_void_p]
            self._L = L
        return self._L

    def __getattr__(self, name):
        return getattr(self.load(), name)


lib = _Lib()


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _chk(rc):
    if rc != 0:
        msg = lib.sf_last_error().decode()
        raise _ERRORS.get(rc, ShapflowError)(msg)


def _u64(x):
    return C.c_uint64(int(x))


# ------------------------------------------------------------------ primitives
def node_sampling_seed(seed, node):  # explain.cpp:37-40
    return int(lib.sf_node_sampling_seed(int(seed) & (2**64 - 1), int(node)))


def auto_samples(n):  # explain.cpp:33-35
    return int(lib.sf_auto_samples(int(n)))


def binomial_or_max(n, s):  # sampler.cpp:67-77
    return int(lib.sf_binomial_or_max(int(n), int(s)))


def kernel_weight(n, s):  # sampler.cpp:79-91
    out = C.c_double()
    _chk(lib.sf_kernel_weight(C.c_uint32(n), C.c_uint32(s), C.byref(out)))
    return out.value


def plan_sizes(n, k, allow_exhaustive=True):
    """sampler.hpp:49-50 -> dict(sizes, pairs, first, exhaustive, requested)."""
    nc, ex, req = C.c_uint64(), C.c_int(), C.c_uint64()
    _chk(lib.sf_plan_sizes(C.c_uint32(n), _u64(k), C.c_int(int(allow_exhaustive)), None, None, None,
                           _u64(0), C.byref(nc), C.byref(ex), C.byref(req)))
    m = nc.value
    sizes = np.zeros(m, np.uint32)
    pairs = np.zeros(m, np.uint64)
    first = np.zeros(m, np.uint64)
    _chk(lib.sf_plan_sizes(C.c_uint32(n), _u64(k), C.c_int(int(allow_exhaustive)), _p(sizes), _p(pairs),
                           _p(first), _u64(m), C.byref(nc), C.byref(ex), C.byref(req)))
    return dict(n=int(n), sizes=sizes, pairs=pairs, first=first, exhaustive=bool(ex.value), requested=req.value)


def rank_edges(phi):  # solver.cpp:430-440
    phi = np.ascontiguousarray(phi, np.float64)
    order = np.zeros(len(phi), np.uint32)
    _chk(lib.sf_rank_edges(_p(phi), _u64(len(phi)), _p(order)))
    return order


def assemble_weights(n, bits, rows_of_size=None):
    """Per-row normalized weights (solver.cpp:116-151)."""
    bits = np.ascontiguousarray(bits, np.uint64)
    w = np.zeros(bits.shape[0], np.float64)
    ros = None if rows_of_size is None else np.ascontiguousarray(rows_of_size, np.uint64)
    _chk(lib.sf_assemble_weights(C.c_uint32(n), _p(bits), _u64(bits.shape[0]), _u64(bits.shape[1]),
                                 _p(ros), _p(w)))
    return w


# ------------------------------------------------------------------ objects
class Graph:
    """graph.hpp:16-31 Graph (host CSR)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    @classmethod
    def build(cls, num_nodes, edges_uv, features, labels=None):
        edges_uv = np.ascontiguousarray(edges_uv, np.uint64).reshape(-1, 2)
        features = np.ascontiguousarray(features, np.float32).reshape(num_nodes, -1)
        lab = None if labels is None else np.ascontiguousarray(labels, np.uint32)
        h = C.c_void_p()
        _chk(lib.sf_graph_build(C.c_uint32(num_nodes), _p(edges_uv), _u64(len(edges_uv)), _p(features),
                                _u64(features.shape[1]), _p(lab), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path):
        h = C.c_void_p()
        _chk(lib.sf_graph_load(str(path).encode(), C.byref(h)))
        return cls(h)

    def save(self, path):
        _chk(lib.sf_graph_save(self.h, str(path).encode()))

    def dims(self):
        n, nnz, d = C.c_uint32(), C.c_uint64(), C.c_uint64()
        _chk(lib.sf_graph_dims(self.h, C.byref(n), C.byref(nnz), C.byref(d)))
        return n.value, nnz.value, d.value

    def csr(self):
        n, nnz, _ = self.dims()
        rp = np.zeros(n + 1, np.uint64)
        col = np.zeros(nnz, np.uint32)
        _chk(lib.sf_graph_csr(self.h, _p(rp), _p(col)))
        return rp, col

    def select_nodes(self, rule):
        """explain.hpp:59-64 select_nodes: "degree-range:[lo,hi]:count" or
        a comma-separated id list."""
        cnt = C.c_uint64()
        rb = rule.encode()
        _chk(lib.sf_select_nodes(self.h, rb, None, C.c_uint64(0), C.byref(cnt)))
        out = np.zeros(cnt.value, np.uint32)
        _chk(lib.sf_select_nodes(self.h, rb, _p(out), C.c_uint64(len(out)), C.byref(cnt)))
        return out

    def extract(self, target, hops):
        h = C.c_void_p()
        _chk(lib.sf_extract(self.h, C.c_uint32(target), C.c_int(hops), C.byref(h)))
        return Subgraph(h)

    def extract_device(self, ctx, target, hops):
        """extract_computational_graph on the GPU of `ctx` (sf_extract_device)."""
        h = C.c_void_p()
        _chk(lib.sf_extract_device(ctx.h, self.h, C.c_uint32(target), C.c_int(hops), C.byref(h)))
        return Subgraph(h)

    def __del__(self):
        try:
            if self.h:
                lib.sf_graph_free(self.h)
                self.h = None
        except Exception:
            pass


class Model:
    """gcn.hpp:13-30 GcnModel."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def create(cls, weights, biases):
        dims = [weights[0].shape[0]] + [w.shape[1] for w in weights]
        for l, (w, b) in enumerate(zip(weights, biases)):  # gcn.cpp:14-33
            if w.shape[0] != dims[l] or np.size(b) != w.shape[1]:
                raise DataError(f"dimension chain broken at layer {l}: weight {w.shape}, bias {np.shape(b)}")
        d = np.asarray(dims, np.uint64)
        w = np.concatenate([np.ascontiguousarray(x, np.float32).ravel() for x in weights])
        b = np.concatenate([np.ascontiguousarray(x, np.float32).ravel() for x in biases])
        h = C.c_void_p()
        _chk(lib.sf_model_create(C.c_int(len(weights)), _p(d), _p(w), _p(b), C.byref(h)))
        return cls(h)

    @classmethod
    def random(cls, input_dim, hidden, classes, seed):  # synthetic.hpp:25-27
        hid = np.asarray(hidden, np.uint64)
        h = C.c_void_p()
        _chk(lib.sf_model_random(_u64(input_dim), _p(hid) if len(hid) else None, C.c_int(len(hid)),
                                 C.c_uint32(classes), _u64(seed), C.byref(h)))
        return cls(h)

    def dims(self):
        L = C.c_int()
        _chk(lib.sf_model_dims(self.h, C.byref(L), None))
        d = np.zeros(L.value + 1, np.uint64)
        _chk(lib.sf_model_dims(self.h, C.byref(L), _p(d)))
        return [int(x) for x in d]

    @property
    def depth(self):
        return len(self.dims()) - 1

    def layers(self):
        dims = self.dims()
        out = []
        for l in range(len(dims) - 1):
            w = np.zeros((dims[l], dims[l + 1]), np.float32)
            b = np.zeros(dims[l + 1], np.float32)
            _chk(lib.sf_model_layer(self.h, C.c_int(l), _p(w), _p(b)))
            out.append((w, b))
        return out

    def __del__(self):
        try:
            if self.h:
                lib.sf_model_free(self.h)
                self.h = None
        except Exception:
            pass


class Subgraph:
    """graph.hpp:36-53 ComputationalGraph."""

    def __init__(self, handle):
        self.h = handle
        V, n, nnz, d = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _chk(lib.sf_subgraph_dims(self.h, C.byref(V), C.byref(n), C.byref(nnz), C.byref(d)))
        self.V, self.n, self.nnz, self.dim = V.value, n.value, nnz.value, d.value

    def arrays(self):
        rp = np.zeros(self.V + 1, np.uint64)
        col = np.zeros(self.nnz, np.uint32)
        ep = np.zeros(self.nnz, np.uint32)
        pl = np.zeros((self.n, 2), np.uint32)
        l2g = np.zeros(self.V, np.uint32)
        feat = np.zeros((self.V, self.dim), np.float32)
        _chk(lib.sf_subgraph_copy(self.h, _p(rp), _p(col), _p(ep), _p(pl), _p(l2g), _p(feat)))
        return dict(row_ptr=rp, col=col, edge_player=ep, players=pl, local_to_global=l2g, features=feat)

    def ball_sizes(self, hops):
        out = np.zeros(hops + 1, np.uint64)
        _chk(lib.sf_subgraph_ball_sizes(self.h, C.c_int(hops), _p(out)))
        return [int(x) for x in out]

    @property
    def words(self):
        return (self.n + 63) // 64

    def __del__(self):
        try:
            if self.h:
                lib.sf_subgraph_free(self.h)
                self.h = None
        except Exception:
            pass


class _ExplanationC(C.Structure):
    _fields_ = [
        ("node", C.c_uint32), ("skipped", C.c_int), ("predicted_class", C.c_uint32),
        ("base_score", C.c_double), ("full_score", C.c_double), ("num_players", C.c_uint64),
        ("phi", C.POINTER(C.c_double)), ("players_global", C.POINTER(C.c_uint32)),
        ("exhaustive", C.c_int), ("rows", C.c_uint64), ("iterations", C.c_uint32),
        ("residual", C.c_double), ("converged", C.c_int), ("num_top", C.c_uint32),
        ("top_player", C.POINTER(C.c_uint32)), ("top_phi", C.POINTER(C.c_double)),
        ("has_fidelity", C.c_int), ("num_counts", C.c_uint32), ("fid_counts", C.POINTER(C.c_uint32)),
        ("fid_plus", C.POINTER(C.c_double)), ("fid_plus_random", C.POINTER(C.c_double)),
        ("num_sparsities", C.c_uint32), ("fid_sparsities", C.POINTER(C.c_double)),
        ("fid_minus", C.POINTER(C.c_double)), ("fid_minus_random", C.POINTER(C.c_double)),
        ("sampling_ms", C.c_double), ("prediction_ms", C.c_double), ("solve_ms", C.c_double),
        ("total_ms", C.c_double), ("extract_ms", C.c_double), ("setup_ms", C.c_double),
        ("fidelity_ms", C.c_double), ("warning", C.c_char * 512),
    ]


class _OptionsC(C.Structure):
    _fields_ = [
        ("samples", C.c_uint64), ("batch_size", C.c_uint64), ("top_k", C.c_uint32), ("seed", C.c_uint64),
        ("tol", C.c_double), ("max_iter", C.c_uint64), ("player_cap", C.c_uint64),
        ("allow_exhaustive", C.c_int), ("constraint_scale", C.c_double), ("fidelity", C.c_int),
        ("baseline_trials", C.c_uint32), ("solver_mode", C.c_int),
        ("top_counts", C.POINTER(C.c_uint32)), ("num_top_counts", C.c_uint32),
        ("sparsities", C.POINTER(C.c_double)), ("num_sparsities", C.c_uint32), ("fixed_order", C.c_int),
    ]


@dataclass
class Explanation:
    """document.hpp:22-44 NodeExplanation."""

    node: int
    skipped: bool
    predicted_class: int
    base_score: float
    full_score: float
    players: np.ndarray
    phi: np.ndarray
    exhaustive: bool
    rows: int
    iterations: int
    residual: float
    converged: bool
    top: list
    fidelity: dict | None
    timings: dict
    warning: str = ""


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _explanation(e):
    n = e.num_players
    fid = None
    if e.has_fidelity:
        fid = dict(top_counts=_arr(e.fid_counts, e.num_counts, np.uint32),
                   plus=_arr(e.fid_plus, e.num_counts, np.float64),
                   plus_random=_arr(e.fid_plus_random, e.num_counts, np.float64),
                   sparsities=_arr(e.fid_sparsities, e.num_sparsities, np.float64),
                   minus=_arr(e.fid_minus, e.num_sparsities, np.float64),
                   minus_random=_arr(e.fid_minus_random, e.num_sparsities, np.float64))
    top = list(zip(_arr(e.top_player, e.num_top, np.uint32).tolist(),
                   _arr(e.top_phi, e.num_top, np.float64).tolist()))
    return Explanation(
        node=e.node, skipped=bool(e.skipped), predicted_class=e.predicted_class, base_score=e.base_score,
        full_score=e.full_score, players=_arr(e.players_global, 2 * n, np.uint32).reshape(-1, 2),
        phi=_arr(e.phi, n, np.float64), exhaustive=bool(e.exhaustive), rows=e.rows, iterations=e.iterations,
        residual=e.residual, converged=bool(e.converged), top=top, fidelity=fid,
        timings=dict(extract_ms=e.extract_ms, setup_ms=e.setup_ms, sampling_ms=e.sampling_ms,
                     prediction_ms=e.prediction_ms, solve_ms=e.solve_ms, fidelity_ms=e.fidelity_ms,
                     total_ms=e.total_ms),
        warning=e.warning.decode())


@dataclass
class ExplainOptions:
    """explain.hpp:15-32 ExplainOptions."""

    samples: int = 0
    batch_size: int = 50
    top_k: int = 10
    top_counts: tuple = (5, 10, 20)
    sparsities: tuple = (0.1, 0.3, 0.5, 0.7, 0.9)
    seed: int = 0
    tol: float = 1e-6
    max_iter: int = 0
    player_cap: int = 0
    allow_exhaustive: bool = True
    constraint_scale: float = 1e6
    fidelity: bool = True
    baseline_trials: int = 8
    solver_mode: int = 3  # SF_SOLVER_AUTO (0 CGLS, 1 fused CGLS, 2 direct)
    fixed_order: bool = False  # explain.hpp:31 (exact, layout-independent CGLS sums)
    _keep: list = field(default_factory=list, repr=False)

    def c(self):
        tc = (C.c_uint32 * len(self.top_counts))(*self.top_counts)
        sp = (C.c_double * len(self.sparsities))(*self.sparsities)
        self._keep = [tc, sp]
        return _OptionsC(self.samples, self.batch_size, self.top_k, self.seed & (2**64 - 1), self.tol,
                         self.max_iter, self.player_cap, int(self.allow_exhaustive), self.constraint_scale,
                         int(self.fidelity), self.baseline_trials, self.solver_mode, tc, len(self.top_counts),
                         sp, len(self.sparsities), int(self.fixed_order))


class DeviceMasks:
    """A device-resident MaskBlock (sf_dmasks): kept-set rows in HBM."""

    def __init__(self, ctx, handle):
        self.ctx, self.h = ctx, handle

    def info(self):
        rows, n = C.c_uint64(), C.c_uint32()
        _chk(lib.sf_dmasks_info(self.h, C.byref(rows), C.byref(n), None))
        ros = np.zeros(n.value + 1, np.uint64)
        _chk(lib.sf_dmasks_info(self.h, C.byref(rows), C.byref(n), _p(ros)))
        return rows.value, n.value, ros

    def download(self):
        rows, n, _ = self.info()
        W = max(1, (n + 63) // 64)
        out = np.zeros((rows, W), np.uint64)
        _chk(lib.sf_dmasks_download(self.ctx.h, self.h, _p(out), _u64(out.size)))
        return out

    def predict(self, model, sg, class_index, batch_size=50):
        rows, _, _ = self.info()
        out = np.zeros(max(rows, 1), np.float32)
        _chk(lib.sf_predict_dmasks(self.ctx.h, model.h, sg.h, self.h, C.c_uint32(class_index), _u64(batch_size),
                                   _p(out)))
        return out[:rows]

    def solve(self, values, base, full, constraint_scale=1e6, tol=1e-6, max_iter=0, mode=0):
        rows, n, _ = self.info()
        v = np.ascontiguousarray(values, np.float32)
        phi = np.zeros(max(n, 1), np.float64)
        it, rel, conv = C.c_uint64(), C.c_double(), C.c_int()
        _chk(lib.sf_solve_dmasks(self.ctx.h, self.h, _p(v), C.c_double(base), C.c_double(full),
                                 C.c_double(constraint_scale), C.c_double(tol), _u64(max_iter), C.c_int(mode),
                                 _p(phi), C.byref(it), C.byref(rel), C.byref(conv)))
        return dict(phi=phi[:n], iterations=it.value, relative_residual=rel.value, converged=bool(conv.value))

    def __del__(self):
        try:
            if self.h:
                lib.sf_dmasks_free(self.h)
                self.h = None
        except Exception:
            pass


class Context:
    """One rank: a B200, its stream and (for world > 1) an NCCL communicator."""

    def __init__(self, device=0):
        h = C.c_void_p()
        _chk(lib.sf_ctx_create(C.c_int(device), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib.sf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- comm
    @staticmethod
    def nccl_unique_id():
        buf = (C.c_char * 128)()
        _chk(lib.sf_nccl_unique_id(buf))
        return bytes(buf)

    def join(self, unique_id, rank, world):
        buf = (C.c_char * 128).from_buffer_copy(unique_id) if unique_id else None
        _chk(lib.sf_ctx_join_nccl(self.h, buf, C.c_int(rank), C.c_int(world)))

    @property
    def rank(self):
        return lib.sf_ctx_rank(self.h)

    @property
    def world(self):
        return lib.sf_ctx_world(self.h)

    def stats(self):
        s, v, b, d = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _chk(lib.sf_ctx_stats(self.h, C.byref(s), C.byref(v), C.byref(b), C.byref(d)))
        return dict(scalar_allreduce=s.value, vector_allreduce=v.value, barriers=b.value, doubles_reduced=d.value)

    def barrier(self):
        _chk(lib.sf_ctx_barrier(self.h))

    def launches(self):
        return int(lib.sf_ctx_launches(self.h))

    def synchronize(self):
        _chk(lib.sf_ctx_synchronize(self.h))

    FUSED_KERNELS = {"auto": 0, "simt": 1, "tc": 2, "tc16": 3}

    def set_workers(self, workers):
        """Concurrent targets for explain_nodes on this device (sf_ctx_set_workers)."""
        _chk(lib.sf_ctx_set_workers(self.h, C.c_int(workers)))

    def set_comm_timeout(self, timeout_ms):
        _chk(lib.sf_ctx_set_comm_timeout(self.h, C.c_int(timeout_ms)))

    def keep_stages(self, enable=True):
        _chk(lib.sf_ctx_keep_stages(self.h, C.c_int(int(enable))))

    def stage_predictions(self):
        """This rank's predictions of the last explain_node (keep_stages on)."""
        rows = C.c_uint64()
        _chk(lib.sf_ctx_stage_predictions(self.h, None, C.c_uint64(0), C.byref(rows)))
        out = np.zeros(rows.value, np.float32)
        _chk(lib.sf_ctx_stage_predictions(self.h, _p(out), C.c_uint64(rows.value), C.byref(rows)))
        return out

    def set_fused_kernel(self, kind):
        """Select the fused layer-0/1 kernel: "auto" (tcgen05 3xTF32 where
        the hidden width allows), "simt" (FP32 SIMT), "tc" (3xTF32) or "tc16"
        (tcgen05 fp16x2 variant, widths 64 and 128)."""
        _chk(lib.sf_ctx_set_fused_kernel(self.h, self.FUSED_KERNELS[kind]))

    def fused_kernel_used(self):
        """Kernel of the last prediction: None, "simt" or "tc"."""
        return {0: None, 1: "simt", 2: "tc", 3: "tc16"}.get(lib.sf_ctx_fused_kernel_used(self.h))

    # ---- sampler
    def philox(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        _chk(lib.sf_philox_u64(self.h, _u64(seed), _u64(stream), _u64(count), _p(out)))
        return out

    def generate_masks(self, plan, seed, rank=0, world=1):
        """sampler.hpp:84-85 -> (rows u64[rows, W], global_rows_of_size)."""
        n = plan["n"]
        rows = C.c_uint64()
        ros = np.zeros(n + 1, np.uint64)
        args = (C.c_uint32(n), _p(plan["sizes"]), _p(plan["pairs"]), _p(plan["first"]), _u64(len(plan["sizes"])),
                C.c_int(int(plan["exhaustive"])), _u64(seed), C.c_int(rank), C.c_int(world))
        _chk(lib.sf_generate_masks(self.h, *args, None, _u64(0), C.byref(rows), _p(ros)))
        W = (n + 63) // 64
        out = np.zeros((rows.value, W), np.uint64)
        _chk(lib.sf_generate_masks(self.h, *args, _p(out), _u64(out.size), C.byref(rows), None))
        return out, ros

    # ---- inference
    def masks_device(self, plan, seed, rank=0, world=1):
        """sampler.hpp:84-85 generate_masks into HBM (sf_masks_device)."""
        h = C.c_void_p()
        _chk(lib.sf_masks_device(self.h, C.c_uint32(plan["n"]), _p(plan["sizes"]), _p(plan["pairs"]),
                                 _p(plan["first"]), _u64(len(plan["sizes"])), C.c_int(int(plan["exhaustive"])),
                                 _u64(seed), C.c_int(rank), C.c_int(world), C.byref(h)))
        return DeviceMasks(self, h)

    def predict_batched(self, model, sg, bits, class_index, batch_size=50):
        bits = np.ascontiguousarray(bits, np.uint64)
        if bits.ndim == 1:
            bits = bits.reshape(-1, max(sg.words, 1))
        out = np.zeros(bits.shape[0], np.float32)
        _chk(lib.sf_predict_batched(self.h, model.h, sg.h, _p(bits), _u64(bits.shape[0]), _u64(bits.shape[1]),
                                    C.c_uint32(class_index), _u64(batch_size), _p(out)))
        return out

    def predict_probs(self, model, sg, mask):
        mask = np.ascontiguousarray(mask, np.uint64).ravel()
        out = np.zeros(model.dims()[-1], np.float32)
        _chk(lib.sf_predict_probs(self.h, model.h, sg.h, _p(mask), _u64(mask.size), _p(out)))
        return out

    def predict(self, model, sg, mask, class_index):
        probs = self.predict_probs(model, sg, mask)
        if class_index >= len(probs):
            raise DataError("class index out of range")
        return probs[class_index]

    # ---- solver
    def solve_cgls(self, n, bits, weights, targets, constraint_target, constraint_weight, tol=1e-6, max_iter=0,
                   mode=0, trace=False):
        bits = np.ascontiguousarray(bits, np.uint64)
        w = np.ascontiguousarray(weights, np.float64)
        t = np.ascontiguousarray(targets, np.float64)
        phi = np.zeros(max(n, 1), np.float64)
        it, rel, conv = C.c_uint64(), C.c_double(), C.c_int()
        cap = 10000 if trace else 0
        tr = np.zeros(cap, np.float64) if trace else None
        rtr = np.zeros(cap, np.float64) if trace else None
        _chk(lib.sf_solve_cgls(self.h, C.c_uint32(n), _p(bits), _u64(bits.shape[0]),
                               _u64(bits.shape[1] if bits.ndim == 2 else 1), _p(w), _p(t),
                               C.c_double(constraint_target), C.c_double(constraint_weight), C.c_double(tol),
                               _u64(max_iter), C.c_int(mode), _p(phi), C.byref(it), C.byref(rel), C.byref(conv),
                               _p(tr), _p(rtr), _u64(cap)))
        res = dict(phi=phi[:n], iterations=it.value, relative_residual=rel.value, converged=bool(conv.value))
        if trace:
            res["trace"] = tr[: it.value]
            res["row_residual_trace"] = rtr[: it.value]
        return res

    def solve_direct(self, n, bits, weights, targets, constraint_target, constraint_weight):
        bits = np.ascontiguousarray(bits, np.uint64)
        w = np.ascontiguousarray(weights, np.float64)
        t = np.ascontiguousarray(targets, np.float64)
        phi = np.zeros(max(n, 1), np.float64)
        _chk(lib.sf_solve_direct(self.h, C.c_uint32(n), _p(bits), _u64(bits.shape[0]),
                                 _u64(bits.shape[1] if bits.ndim == 2 else 1), _p(w), _p(t),
                                 C.c_double(constraint_target), C.c_double(constraint_weight), _p(phi)))
        return phi[:n]

    # ---- pipeline
    def explain_node(self, graph, model, node, opts: ExplainOptions | None = None):
        """explain.hpp:47-49 explain_node (collective over the context's ranks)."""
        opts = opts or ExplainOptions()
        co = opts.c()
        e = _ExplanationC()
        _chk(lib.sf_explain_node(self.h, graph.h, model.h, C.c_uint32(node), C.byref(co), C.byref(e)))
        try:
            return _explanation(e)
        finally:
            lib.sf_explanation_free(C.byref(e))

    def explain_nodes(self, graph, model, nodes, opts: ExplainOptions | None = None):
        """explain.hpp:54-57 explain_nodes: one Explanation per node, in order;
        errors carry a "node N: " prefix (explain.cpp:168-180)."""
        opts = opts or ExplainOptions()
        co = opts.c()
        ids = np.ascontiguousarray(nodes, np.uint32)
        arr = (_ExplanationC * max(len(ids), 1))()
        _chk(lib.sf_explain_nodes(self.h, graph.h, model.h, _p(ids), C.c_uint64(len(ids)), C.byref(co), arr))
        out = []
        try:
            for i in range(len(ids)):
                out.append(_explanation(arr[i]))
        finally:
            for i in range(len(ids)):
                lib.sf_explanation_free(C.byref(arr[i]))
        return out

    def evaluate_fidelity(self, model, sg, class_index, phi, top_counts=(5, 10, 20),
                          sparsities=(0.1, 0.3, 0.5, 0.7, 0.9), seed=0, trials=8):
        phi = np.ascontiguousarray(phi, np.float64)
        tc = np.asarray(top_counts, np.uint32)
        sp = np.asarray(sparsities, np.float64)
        co = np.zeros(len(tc), np.uint32)
        outs = [np.zeros(len(tc)), np.zeros(len(tc)), np.zeros(len(sp)), np.zeros(len(sp))]
        _chk(lib.sf_evaluate_fidelity(self.h, model.h, sg.h, C.c_uint32(class_index), _p(phi), _p(tc),
                                      C.c_uint32(len(tc)), _p(sp), C.c_uint32(len(sp)), _u64(seed),
                                      C.c_uint32(trials), _p(co), *[_p(o) for o in outs]))
        return dict(top_counts=co, plus=outs[0], plus_random=outs[1], minus=outs[2], minus_random=outs[3])

    def sample_and_predict(self, model, sg, class_index, k, seed, allow_exhaustive=True):
        st = np.zeros(3, np.float64)
        rows = C.c_uint64()
        _chk(lib.sf_sample_and_predict(self.h, model.h, sg.h, C.c_uint32(class_index), _u64(k), _u64(seed),
                                       C.c_int(int(allow_exhaustive)), _p(st), C.byref(rows)))
        return dict(sampling_ms=st[0], prediction_ms=st[1], layer0_ms=st[2], rows=rows.value)
