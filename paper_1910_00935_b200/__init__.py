"""B200-native differentiable MLS-MPM hot path (DiffTaichi diffmpm, arXiv 1910.00935).

The compute path is ``libmpm_b200.so`` (hand-written CUDA for sm_100a behind the
C-ABI in ``include/mpm.h``); ``mpm.py`` is its thin ctypes binding.
"""
__all__ = ["mpm", "workloads"]
