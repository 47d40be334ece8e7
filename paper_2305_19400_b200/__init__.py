"""B200-native explicit phonon-BTE time step (arXiv 2305.19400).

The product is ``libbte.so`` (C ABI in ``include/bte.h``; CUDA kernels for
sm_100a in ``csrc/``).  ``bte.Solver`` is its thin ctypes binding.  There is
no CPU path: without the built library or a CUDA device, ``Solver`` raises.
"""
from .bte import (BC_DIFFUSE, BC_ISOTHERMAL, BC_PARTIAL, BC_SPECULAR, I0_BOSE_EINSTEIN, I0_LINEAR, LIB_PATH,
                  BteError, Solver, load_library, loopback_unique_id, nccl_unique_id, partition_rcb, plan_band, plan_slab, plan_umesh,
                  read_mesh)

__all__ = ["Solver", "BteError", "load_library", "loopback_unique_id", "nccl_unique_id", "plan_band", "plan_slab", "plan_umesh", "LIB_PATH",
           "read_mesh", "partition_rcb",
           "BC_ISOTHERMAL", "BC_SPECULAR", "BC_DIFFUSE", "BC_PARTIAL", "I0_LINEAR", "I0_BOSE_EINSTEIN"]
