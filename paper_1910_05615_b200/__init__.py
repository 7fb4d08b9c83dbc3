"""B200-native RT-DetMCD (arXiv 1910.05615) hot path.

The method runs in libpaper_1910_05615_b200.so (sm_100a kernels behind the C
ABI of include/rtdetmcd.h); this package is its thin binding.
"""
from .api import (RTDError, chi2_quantile, choose_q, consistency_factor, csteps, fit, flag, initial,  # noqa: F401
                  partition_perm, profile, refine, set_profiling, unimcd, workspace_size)

__all__ = ["fit", "flag", "unimcd", "initial", "refine", "csteps", "chi2_quantile", "consistency_factor",
           "choose_q", "partition_perm", "workspace_size", "RTDError"]
