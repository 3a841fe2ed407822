"""B200-native S-MNN hot path (arXiv 2410.06074): fused banded least-squares ODE solve.

The compute path is the C-ABI CUDA library ``lib/libsmnn.so`` (include/smnn.h);
this package is its thin PyTorch binding (``smnn``) plus multi-GPU sharding
helpers (``dist``).  It never imports ``oracle/``.
"""

from .smnn import (  # noqa: F401
    HostPlan, SMNNSolve, Weights, smnn_assemble, smnn_factor, smnn_factor_solve_fwd, smnn_solve,
    smnn_solve_bwd, smnn_substitute, workspace_bytes, kernel_path, ylo_used,
)

__version__ = "0.1.0"
