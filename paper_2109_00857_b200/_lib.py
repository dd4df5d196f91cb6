"""ctypes binding of libflowmdp_b200.so (include/flowmdp_b200.h).

The shared library is built in-tree for sm_100a by ``build_native()``
(called from ``__graft_entry__.build``).  Loading fails loudly: there is no
CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

from .errors import ContractViolation, NativeUnavailable

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("FM_LIB_PATH") or os.path.join(PKG_DIR, "libflowmdp_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")
SOURCES = [os.path.join(CSRC, "flowmdp_b200.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "fm_hypot.cuh"), os.path.join(REPO_DIR, "include", "flowmdp_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # no FMA contraction: the reference rounds every op
    "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared",
]

FM_OK, FM_SUBGRID_OVERFLOW, FM_BAD_ARG, FM_CUDA_ERROR, FM_CAPACITY = range(5)


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand == "nvcc" or os.path.exists(cand):
            return cand
    return "nvcc"


def build_native(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into the in-tree shared library (idempotent)."""
    stale = not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(d) > os.path.getmtime(LIB_PATH) for d in DEPS)
    if force or stale:
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB_PATH, *SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd, cwd=CSRC)
    return LIB_PATH


# ---------------------------------------------------------------------------
# structures (must match include/flowmdp_b200.h byte for byte)
# ---------------------------------------------------------------------------

class FmGrid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nt", C.c_int32),
                ("dx", C.c_double), ("dt", C.c_double), ("ox", C.c_double), ("oy", C.c_double)]


class FmEnv(C.Structure):
    _fields_ = [("mean", C.c_void_p), ("modes", C.c_void_p), ("coeffs", C.c_void_p),
                ("g", C.c_void_p), ("mask", C.c_void_p),
                ("n_modes", C.c_int32), ("n_real", C.c_int32)]


class FmAction(C.Structure):
    _fields_ = [("ax", C.c_double), ("ay", C.c_double), ("base", C.c_double),
                ("base_hit", C.c_double), ("neg_cff", C.c_double), ("pad", C.c_double)]


class FmReward(C.Structure):
    _fields_ = [("objective", C.c_int32), ("c_f", C.c_double), ("c_r", C.c_double),
                ("r_term", C.c_double), ("r_outbound", C.c_double),
                ("target_i", C.c_int32), ("target_j", C.c_int32)]


class FmModel(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nt", C.c_int32), ("n_actions", C.c_int32),
                ("n_real", C.c_int32), ("hx", C.c_int32), ("hy", C.c_int32),
                ("cell0", C.c_int32), ("ncell", C.c_int32),
                ("n_rows", C.c_int64),
                ("row_ptr", C.c_void_p), ("row_nnz", C.c_void_p), ("reward", C.c_void_p),
                ("entries", C.c_void_p), ("capacity", C.c_uint64), ("d_nnz", C.c_void_p)]


class FmBuildArgs(C.Structure):
    _fields_ = [("grid", FmGrid), ("env", FmEnv), ("reward", FmReward),
                ("actions", C.c_void_p), ("n_actions", C.c_int32),
                ("hx", C.c_int32), ("hy", C.c_int32), ("rx", C.c_int32), ("ry", C.c_int32),
                ("mask_sat", C.c_void_p),
                ("t0", C.c_int32), ("t1", C.c_int32), ("j0", C.c_int32), ("j1", C.c_int32),
                ("viol_flags", C.c_void_p), ("task_counter", C.c_void_p), ("d_gate_r", C.c_void_p),
                ("h_actions", C.c_void_p), ("vmax_x", C.c_double), ("vmax_y", C.c_double),
                ("envelope", C.c_void_p), ("reserve_sms", C.c_int32), ("phases", C.c_int32),
                ("reward_mode", C.c_int32)]


class FmViolation(C.Structure):
    _fields_ = [("t", C.c_int32), ("a", C.c_int32), ("di", C.c_int32), ("dj", C.c_int32)]


class FmCsr(C.Structure):
    _fields_ = [("n_g", C.c_int64), ("n_actions", C.c_int32), ("nt", C.c_int32),
                ("row_ptr", C.c_void_p), ("cols", C.c_void_p), ("vals", C.c_void_p),
                ("rewards", C.c_void_p)]


class FmRolloutArgs(C.Structure):
    _fields_ = [("grid", FmGrid), ("env", FmEnv), ("reward", FmReward),
                ("actions", C.c_void_p), ("n_actions", C.c_int32),
                ("mask_sat", C.c_void_p), ("d_gate_r", C.c_void_p), ("policy", C.c_void_p),
                ("start_i", C.c_int32), ("start_j", C.c_int32),
                ("realizations", C.c_void_p), ("n_traj", C.c_int32), ("max_rows", C.c_int32),
                ("row_cell", C.c_void_p), ("row_action", C.c_void_p), ("row_cause", C.c_void_p),
                ("row_reward", C.c_void_p), ("row_cum", C.c_void_p),
                ("n_rows", C.c_void_p), ("final_cell", C.c_void_p)]


# exported symbols and their signatures; tests check every one resolves
# fm_halo_fn: int32_t (*)(void *user, int32_t t, void *stream)
HALO_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.c_void_p)

SIGNATURES = {
    "fm_abi_version": (C.c_int32, []),
    "fm_last_error": (C.c_char_p, []),
    "fm_kernel_launches": (C.c_int64, []),
    "fm_velocity_max": (C.c_int32, [FmGrid, FmEnv, C.c_void_p, C.c_void_p]),
    "fm_velocity_max_rows": (C.c_int32, [FmGrid, FmEnv, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "fm_velocity_max_slab": (C.c_int32, [FmGrid, FmEnv, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                         C.c_void_p]),
    "fm_velocity_scan": (C.c_int32, [FmGrid, FmEnv, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    "fm_velocity_bounds": (C.c_int32, [FmGrid, FmEnv, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "fm_maxabs_segments": (C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "fm_mask_sat": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "fm_build": (C.c_int32, [C.POINTER(FmBuildArgs), C.POINTER(FmModel), C.POINTER(C.c_uint64),
                             C.POINTER(FmViolation), C.c_void_p]),
    "fm_build_launch": (C.c_int32, [C.POINTER(FmBuildArgs), C.POINTER(FmModel), C.c_void_p]),
    "fm_build_check": (C.c_int32, [C.POINTER(FmBuildArgs), C.POINTER(FmModel), C.POINTER(C.c_uint64),
                                   C.POINTER(FmViolation), C.c_void_p]),
    "fm_gate_radius": (C.c_int32, [FmGrid, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_export_coo": (C.c_int32, [C.POINTER(FmModel), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_solve_backward": (C.c_int32, [C.POINTER(FmModel), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "fm_solve_backward_halo": (C.c_int32, [C.POINTER(FmModel), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_solve_layer": (C.c_int32, [C.POINTER(FmModel), C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p]),
    "fm_prob_table": (C.c_int32, [C.c_int32, C.c_void_p, C.c_void_p]),
    "fm_solve_layer_tab": (C.c_int32, [C.POINTER(FmModel), C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_csr_row_ptr": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_void_p]),
    "fm_jacobi": (C.c_int32, [C.POINTER(FmCsr), C.c_double, C.c_int32, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p]),
    "fm_greedy": (C.c_int32, [C.POINTER(FmCsr), C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_policy_value": (C.c_int32, [C.POINTER(FmCsr), C.c_void_p, C.c_double, C.c_int32, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]),
    "fm_fp64_probe": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "fm_model_image": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                   C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "fm_rollout": (C.c_int32, [C.POINTER(FmRolloutArgs), C.c_void_p]),
}

_LIB = None


def load(require_gpu: bool = True):
    """Load the native library.  Raises NativeUnavailable when it is absent
    or (with require_gpu) when no CUDA device is visible."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                "there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return _LIB


def check(status: int, what: str) -> None:
    """Map an fm_status to the reference's exception types."""
    if status == FM_OK:
        return
    msg = load(require_gpu=False).fm_last_error().decode(errors="replace")
    if status in (FM_SUBGRID_OVERFLOW, FM_BAD_ARG):
        raise ContractViolation(msg)
    raise RuntimeError(f"{what}: {msg} (status {status})")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
