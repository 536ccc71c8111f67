"""B200-native batched locomotion simulator (hot path of arXiv 1810.05762).

The product is the C-ABI shared library ``libstampede_b200.so`` (hand-written
sm_100a kernels, include/stampede_sim.h); this package is its host-side
mirror of the reference's env / physics interface.
"""
from . import abi  # noqa: F401

__all__ = ["abi", "VecEnv"]


def __getattr__(name):
    if name == "VecEnv":
        from .sim import VecEnv
        return VecEnv
    raise AttributeError(name)
