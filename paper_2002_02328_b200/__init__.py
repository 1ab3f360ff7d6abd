"""B200-native BD3MG hot path (arXiv 2002.02328): depth-variant blur H/H^T,
fused gradient, forward-only 2x2 memory-gradient Gram, device subspace solve
and block update as sm_100a CUDA kernels behind a C ABI
(include/bd3mg_b200.h), with the reference package's operator and solver
entry points kept as a drop-in (blur, objective, directions, scheduler,
runtime)."""

__version__ = "0.1.0"


def N_launches() -> int:
    """Kernels the native library has launched in this process (eager calls)."""
    from . import _native
    return int(_native.lib.bd3mg_launch_count())
