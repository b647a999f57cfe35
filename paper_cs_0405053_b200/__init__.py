"""B200-native synchronous-relaxation parallel n-fold way (arXiv cs/0405053).

The product is ``libising_sr.so`` (C ABI in ``include/ising_sr.h``): sm_100a
CUDA kernels for the region trajectories, the fused history diff, commit and
log replay, plus the host relaxation loop.  This package is its thin Python
binding (``binding.IsingSR``) and the multi-rank driver (``dist``).
"""
from .binding import (FLAG_DIGEST, FLAG_FRESH_WINDOW, FLAG_HALO_LOOPBACK, FLAG_JACOBI_ALL, FLAG_LOG_EVENTS,  # noqa: F401
                      FLAG_MAG_MOMENTS,
                      FLAG_OBSERVABLES, IsingSR, IsingSRError, checkerboard_run, checkerboard_sweeps, from_workload,
                      load_library, nccl_unique_id)

__all__ = ["IsingSR", "IsingSRError", "from_workload", "load_library", "FLAG_DIGEST", "FLAG_LOG_EVENTS", "FLAG_FRESH_WINDOW",
           "FLAG_OBSERVABLES", "FLAG_JACOBI_ALL", "FLAG_HALO_LOOPBACK", "FLAG_MAG_MOMENTS", "checkerboard_run", "checkerboard_sweeps",
           "nccl_unique_id"]
