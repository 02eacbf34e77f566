"""B200-native (sm_100a) hot path of DMV3D's reconstruction-based denoiser.

The product is libdmv3d.so (C ABI, include/dmv3d.h); this package is its thin
Python binding (api.py, argument marshalling only), the host-side schedule
tables (schedule.py), the seeded input generators (workloads.py) and the
multi-GPU plumbing (dist.py).  Importing it does not load the CUDA library;
the first entry-point call does, and raises if it is missing.
"""
__all__ = ["api", "schedule", "workloads"]
