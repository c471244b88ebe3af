"""ctypes binding of libglycemlp_cuda.so (declarations: include/glycemlp_cuda.h).

The product path has no CPU fallback: if the library is missing, fails to
load, or no CUDA device is visible, every compute call raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import NumericError, ShapeError, ValidationError

LIB_PATH = Path(os.environ.get("GLX_LIB", Path(__file__).resolve().parent / "libglycemlp_cuda.so"))

GLX_OK = 0
GLX_ERR_SHAPE = -1
GLX_ERR_INVALID = -2
GLX_ERR_NUMERIC = -3
GLX_ERR_CUDA = -4
GLX_ERR_NOMEM = -5
GLX_ERR_RACE = -6  # a debug run's pipeline check failed -> RuntimeError
GLX_FLAG_DEBUG = 2

GLX_FP32 = 0
GLX_REF64 = 1
GLX_FLAG_CACHE_INPUTS = 1

NUMERICS = {"fp32": GLX_FP32, "ref64": GLX_REF64}

# every exported symbol of include/glycemlp_cuda.h with (restype, argtypes)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_int = ctypes.c_int
SIGNATURES = {
    "glx_last_error": (ctypes.c_char_p, []),
    "glx_version": (_int, []),
    "glx_device_count": (_int, []),
    "glx_sm_count": (_int, [_int]),
    "glx_run_train_segment": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i64, _dbl, _i32, _i32, _i32]),
    "glx_run_train_segment_batch": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i64, _dbl, _vp, _i32, _i32]),
    "glx_run_train_segment_eval": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i64, _dbl, _i32,
                                          _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "glx_eval_counts": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i32]),
    "glx_cache_clear": (None, []),
    "glx_train_online": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i64, _dbl, _i32, _vp]),
    "glx_train_sweep": (_int, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i64, _dbl, _i32, _vp]),
    "glx_packed_ld": (_i32, [_i32]),
    "glx_pack_rows": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "glx_train_batch": (_int, [_vp, _vp, _vp, _i64, _i32, _i32, _i64, _dbl, _vp, _vp, _vp]),
    "glx_batch_grad_len": (_i64, [_i32, _i32]),
    "glx_batch_kernel_kind": (_i32, [_i64, _i32, _i32]),
    "glx_batch_grad": (_int, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "glx_batch_apply": (_int, [_vp, _vp, _vp, _i32, _i32, _dbl, _vp, _vp]),
    "glx_eval": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp]),
    "glx_eval_packed": (_int, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "glx_tc_gemm_bf16": (_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "glx_wide_make_data": (_int, [_i64, _u64, _vp, _vp, _vp, _vp]),
    "glx_wide_train": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _dbl, _vp, _vp, _vp]),
    "glx_pack_rows_minmax": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "glx_minmax_fit": (_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "glx_forward": (_int, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp]),
    "glx_layer_forward": (_int, [_vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "glx_layer_backward": (_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "glx_layer_forward_checked": (_int, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "glx_layer_backward_checked": (_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "glx_forward_pair_debug": (_int, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp]),
    "glx_backprop_error": (_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "glx_instance_gradients": (_int, [_vp, _vp, _vp, _vp, _dbl, _i32, _i32, _vp, _vp, _vp]),
    "glx_pcg64_uniform_f32": (_int, [_u64, _u64, _u64, _u64, _i64, _i64, _vp, _vp]),
    "glx_pcg64_coin": (_int, [_u64, _u64, _u64, _u64, _i64, _i64, _vp, _vp]),
    "glx_planted_score": (_int, [_vp, _i64, _i32, _vp, _vp, _i32, _vp, _vp]),
    "glx_label_ge": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "glx_minmax_apply": (_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "glx_wide_make_shard": (_int, [_i64, _i64, _u64, _vp, _vp, _vp, _vp]),
    "glx_wide_grad_len": (_i64, []),
    "glx_wide_grad": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "glx_wide_apply": (_int, [_vp, _vp, _vp, _dbl, _vp, _vp]),
    "glx_dp_unique_id": (_int, [_vp]),
    "glx_dp_init": (_int, [_i32, _i32, _i32, _vp, _vp]),
    "glx_dp_finalize": (_int, [_vp]),
    "glx_dp_allreduce_f64": (_int, [_vp, _vp, _i64, _i32, _vp]),
    "glx_dp_train_batch": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _i64, _dbl, _vp, _vp, _vp]),
    "glx_dp_run_train_segment_batch": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _i64, _dbl, _vp,
                                              _i32]),
    "glx_wide_make_shard_tf32": (_int, [_i64, _i64, _u64, _vp, _vp, _vp, _vp]),
    "glx_wide_grad_tf32": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "glx_wide_train_tf32": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _dbl, _vp, _vp, _vp]),
    "glx_launch_count": (_u64, []),
    "glx_profile_enable": (None, [_i32]),
    "glx_set_debug": (None, [_i32]),
    "glx_profile_read": (_int, [_vp, _vp]),
    "glx_fp32_peak": (_int, [_i32, _i32, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load(require_device: bool = True):
    """Load the library (once). Raises RuntimeError if it cannot run here."""
    global _lib
    with _lock:
        if _lib is None:
            # torch first: its libnccl.so.2 must be the process's copy (the library binds
            # NCCL at run time to whatever copy is loaded, glx_abi.cu)
            import torch  # noqa: F401

            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            L = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    if require_device and _lib.glx_device_count() < 1:
        raise RuntimeError("no CUDA device visible: the glycemlp B200 engine has no CPU fallback")
    return _lib


def check(rc: int) -> None:
    """Map a GLX_ERR_* return code onto the reference's exception types."""
    if rc == GLX_OK:
        return
    msg = (_lib.glx_last_error() or b"").decode(errors="replace")
    if rc == GLX_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == GLX_ERR_INVALID:
        raise ValidationError(msg)
    if rc == GLX_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == GLX_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"glycemlp CUDA error: {msg}")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def launch_count() -> int:
    return int(load(require_device=False).glx_launch_count())
