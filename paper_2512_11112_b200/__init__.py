"""B200-native GPU back end for the SPDZ online phase of arXiv 2512.11112.

Drop-in for the reference's back-end plugin (mpc::backend::Backend,
/root/reference/proj/core/include/mpc/backend.hpp:32-49), widened to the
online-phase ops that bypass it (public-constant ops, open, MAC check, linear
layer).  The compute path is hand-written sm_100a CUDA behind a C ABI
(include/spdz_b200.h, libspdz_b200.so); Python here is a thin host mirror.
"""
from . import errors  # noqa: F401
from .backend import (BackendCapability, BackendRegistry, Context, DeviceBMTriple, DeviceShare, DeviceTriple,  # noqa: F401
                      GpuBackend, ShareVec, TripleShares)
from .runtime import (ChunkedRun, Graph, LocalRun, NodeSpec, RunReport, StreamedRun, chain_graph, linear_graph,  # noqa
                      reduce_graph, run_local)

P = 4294967291
__all__ = ["errors", "GpuBackend", "BackendRegistry", "Context", "ShareVec", "TripleShares", "DeviceShare",
           "DeviceTriple", "Graph", "NodeSpec", "LocalRun", "run_local", "chain_graph", "linear_graph",
           "reduce_graph", "RunReport", "StreamedRun", "P"]
