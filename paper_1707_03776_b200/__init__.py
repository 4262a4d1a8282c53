"""paper_1707_03776_b200 -- B200-native acoustic finite-difference propagator.

The data-parallel hot path of the seismic example of Lange et al., "Optimised finite
difference computation from symbolic equations" (Devito, SciPy 2017): the explicit
leapfrog update of m u_tt - Lap u + eta u_t = q at space orders 2-16 with source
injection and receiver interpolation, its adjoint, and the FWI gradient correlation
-- hand-written CUDA for sm_100a behind the C-ABI of include/sf.h (libsf.so), with
NCCL slab halos / gradient all-reduce for multiple GPUs.

This package never imports ``oracle`` (the fp64 CPU reference used by the tests).
"""
from ._lib import EXPORTS, LIB_PATH, SfError, build, lib  # noqa: F401
from ._lib import (SF_OPT_COMM_SMS, SF_OPT_FUSE_MAX, SF_OPT_GRAPH, SF_OPT_L2_PREFETCH,  # noqa: F401
                   SF_OPT_ONE_LAUNCH, SF_OPT_P2P, SF_OPT_PDL, SF_OPT_PROF_EVERY, SF_OPT_LOOP2D, SF_OPT_TBLOCK, SF_OPT_BALANCE, SF_OPT_SNAP_HALF, SF_OPT_SPLIT, SF_OPT_ZSPLIT)
from .api import (Propagator, allreduce_gradient, fd_weights, forward_host,  # noqa: F401
                  nccl_comm_destroy, nccl_comm_info, nccl_check, nccl_comm_init, nccl_unique_id, slab_halo_plan, slab_plan,
                  local_group_create, local_group_destroy, sparse_owner, convection2d, laplace2d)

__version__ = "0.1.0"
