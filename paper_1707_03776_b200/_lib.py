"""ctypes loader for the in-tree ``libsf.so`` (the C-ABI of include/sf.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  There is no fallback -- if the shared library is missing or fails to
load, importing the package's compute API raises immediately.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# SF_LIB_PATH: load another build of the same C-ABI (A/B timing of kernel variants only;
# the tests, smoke() and bench.py use the in-tree build)
_DEFAULT_LIB = os.path.join(_HERE, "libsf.so")
LIB_PATH = os.environ.get("SF_LIB_PATH") or _DEFAULT_LIB
CSRC = os.path.join(_HERE, "csrc")

STATUS = {0: "SF_OK", 1: "SF_ERR_INVALID_ARG", 2: "SF_ERR_SHAPE", 3: "SF_ERR_ORDER",
          4: "SF_ERR_CFL", 5: "SF_ERR_OUT_OF_DOMAIN", 6: "SF_ERR_WORKSPACE", 7: "SF_ERR_CUDA",
          8: "SF_ERR_NCCL"}

# every symbol include/sf.h declares
EXPORTS = ["sf_fd_weights", "sf_create", "sf_destroy", "sf_forward", "sf_adjoint", "sf_residual",
           "sf_gradient_workspace_bytes", "sf_gradient", "sf_gradient_ckpt_workspace_bytes",
           "sf_gradient_ckpt", "sf_forward_host", "sf_forward_once", "sf_set_profiling",
           "sf_get_profile", "sf_get_profile_detail", "sf_set_tuning", "sf_set_option", "sf_get_tuning", "sf_get_tuning_modes", "sf_slab_plan", "sf_slab_halo_plan", "sf_sparse_owner",
           "sf_nccl_unique_id", "sf_nccl_comm_init", "sf_nccl_comm_destroy", "sf_nccl_comm_info",
           "sf_nccl_check", "sf_create_slab",
           "sf_allreduce_gradient", "sf_local_group_create", "sf_local_group_destroy",
           "sf_convection2d", "sf_laplace2d", "sf_debug_probe", "sf_autotune", "sf_last_error", "sf_version"]


SF_OPT_L2_PREFETCH, SF_OPT_SPLIT, SF_OPT_FUSE_MAX, SF_OPT_COMM_SMS, SF_OPT_GRAPH, SF_OPT_SNAP_HALF, SF_OPT_P2P, SF_OPT_ZSPLIT = \
    1, 2, 3, 4, 5, 7, 8, 9
SF_OPT_ONE_LAUNCH, SF_OPT_PDL, SF_OPT_PROF_EVERY, SF_OPT_LOOP2D, SF_OPT_TBLOCK, SF_OPT_BALANCE = \
    11, 12, 13, 14, 15, 16


class SfError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"{self.status}: {msg}")


class SfDesc(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("shape", ctypes.c_int64 * 3), ("h", ctypes.c_double),
                ("space_order", ctypes.c_int), ("nt", ctypes.c_int), ("dt", ctypes.c_double),
                ("m", ctypes.c_void_p), ("damp", ctypes.c_void_p), ("nsrc", ctypes.c_int),
                ("src_coords", ctypes.c_void_p), ("nrec", ctypes.c_int),
                ("rec_coords", ctypes.c_void_p), ("sigma", ctypes.c_void_p * 3)]


def build(force: bool = False, jobs: int = 8) -> str:
    """Compile libsf.so in-tree with nvcc for sm_100a (make -C csrc)."""
    args = ["make", "-C", CSRC, f"-j{jobs}"]
    if force:
        subprocess.check_call(["make", "-C", CSRC, "clean"])
    subprocess.check_call(args)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built (run __graft_entry__.build() or make -C {CSRC}); "
                              "the CUDA extension is required -- there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I, D, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        I64 = ctypes.c_int64
        sig = {
            "sf_fd_weights": [I, P],
            "sf_create": [P, P],
            "sf_forward": [P, P, P, P, P, I, P],
            "sf_adjoint": [P, P, P, P, P, I, P, P],
            "sf_residual": [P, P, P, P, P, P],
            "sf_gradient": [P, P, P, P, P, P, Z, I, P],
            "sf_gradient_ckpt": [P, P, P, P, P, P, Z, I, I, P],
            "sf_forward_host": [P, P, P, P, P],
            "sf_forward_once": [P, P, P, P, P],
            "sf_set_profiling": [P, I],
            "sf_get_profile": [P, P, P, P, I],
            "sf_get_profile_detail": [P, P, P, I],
            "sf_set_tuning": [P, I, I, I],
            "sf_set_option": [P, I, I],
            "sf_get_tuning": [P, P, P, P],
            "sf_get_tuning_modes": [P, P, P, P],
            "sf_slab_plan": [I64, I, I, I, P, P],
            "sf_slab_halo_plan": [I64, I, I, I, P],
            "sf_sparse_owner": [I64, I, I, D, D, P],
            "sf_nccl_unique_id": [P],
            "sf_nccl_comm_init": [P, I, I, P],
            "sf_nccl_comm_destroy": [P],
            "sf_nccl_comm_info": [P, P, P],
            "sf_nccl_check": [P],
            "sf_debug_probe": [P, P, P],
            "sf_autotune": [P, P, I, P, P, P],
            "sf_create_slab": [P, P, I, I, P],
            "sf_allreduce_gradient": [P, P, P, Z, P, I, P],
            "sf_local_group_create": [I, P],
            "sf_convection2d": [P, P, I64, I64, D, D, D, D, I, P],
            "sf_laplace2d": [P, P, P, I64, I64, D, D, D, I, P, P, P],
            "sf_local_group_destroy": [P],
        }
        for name, at in sig.items():
            try:
                f = getattr(L, name)
            except AttributeError:
                # an A/B build of an older revision (SF_LIB_PATH) may lack newer entry points
                if LIB_PATH != _DEFAULT_LIB:
                    continue
                raise
            f.argtypes = at
            f.restype = ctypes.c_int
        L.sf_destroy.argtypes = [P]
        L.sf_destroy.restype = None
        L.sf_gradient_workspace_bytes.argtypes = [P, I]
        L.sf_gradient_ckpt_workspace_bytes.argtypes = [P, I, I]
        L.sf_gradient_ckpt_workspace_bytes.restype = ctypes.c_size_t
        L.sf_gradient_workspace_bytes.restype = Z
        L.sf_last_error.argtypes = []
        L.sf_last_error.restype = ctypes.c_char_p
        L.sf_version.argtypes = []
        L.sf_version.restype = I
        _lib = L
    return _lib


def check(code: int):
    if code != 0:
        raise SfError(code, lib().sf_last_error().decode(errors="replace"))
