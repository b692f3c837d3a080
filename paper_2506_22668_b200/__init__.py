"""B200-native DistShap explanation hot path (sampler -> masked GCN inference ->
weighted least squares), exposed through the C-ABI in ``include/shapflow_b200.h``.

The compute lives in ``libshapflow_b200.so`` (hand-written sm_100a kernels + C++
host). This package is a thin ctypes mirror of the reference ``shapflow`` C++ API
(same names, argument meaning and error types) used by the tests and the bench.
There is no CPU fallback: importing works without a GPU (so the ABI can be
inspected), but every compute call needs the CUDA library and a B200.
"""
from .api import (  # noqa: F401
    DataError,
    NumericalError,
    ProtocolError,
    ShapflowError,
    Context,
    Graph,
    Model,
    Subgraph,
    Explanation,
    lib,
    lib_path,
    node_sampling_seed,
    auto_samples,
    binomial_or_max,
    kernel_weight,
    plan_sizes,
    rank_edges,
    assemble_weights,
    EXPORTED_SYMBOLS,
)

__all__ = [
    "DataError",
    "NumericalError",
    "ProtocolError",
    "ShapflowError",
    "Context",
    "Graph",
    "Model",
    "Subgraph",
    "Explanation",
    "lib",
    "lib_path",
    "node_sampling_seed",
    "auto_samples",
    "binomial_or_max",
    "kernel_weight",
    "plan_sizes",
    "rank_edges",
    "assemble_weights",
]
