"""B200-native modal-DG Euler right-hand side and RK stage (arXiv:1601.07944).

The hot path (volume integral, edge flux with ghost states, gather with the
diagonal inverse mass, RK stage update, p=1 limiter, CFL reduction) runs as
hand-written sm_100a CUDA kernels behind the C ABI in
``include/dg2d_b200/dg2d_b200.h``; ``dg2d`` mirrors the reference solver's API.
"""
from . import dg2d  # noqa: F401

__all__ = ["dg2d"]
