"""ctypes front-end for the C oracle (oracle/glx_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; it is the checker, never the product. Every function
mirrors a reference kernel (file:line in glx_oracle.c) and mutates numpy
arrays in place exactly like the reference's numba kernels do.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libglx_oracle.so"
_lib = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double


def build() -> Path:
    """Compile oracle/libglx_oracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    L = ctypes.CDLL(str(_LIB_PATH))
    L.orc_train_online_seq.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _int, _int, _i64, _dbl]
    L.orc_train_online_par.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _int, _int, _i64, _dbl, _int]
    L.orc_train_batch.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _int, _int, _int, _i64, _i64, _dbl]
    L.orc_train_batch_par.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _int, _int, _int, _i64, _dbl, _int]
    L.orc_batch_grad_par.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _int, _int, _int, _f64p, _int]
    L.orc_eval.argtypes = [_f32p, _f32p, _f32p, _u8p, _i64, _int, _int, _int, _i64p,
                           ctypes.POINTER(ctypes.c_double)]
    L.orc_eval.restype = None
    L.orc_forward_row.argtypes = [_f32p, _f32p, _f32p, _int, _int, _int, _f32p, _f32p]
    L.orc_forward_row.restype = None
    L.orc_sigmoid64.argtypes = [_dbl]
    L.orc_sigmoid64.restype = _dbl
    L.orc_train_sweep.argtypes = [_i64, _i32p, _i64p, _f32p, _f32p, _f32p, _i64, _int, _i64, _dbl, _int]
    L.orc_max_threads.restype = _int
    for name in ("orc_train_online_seq", "orc_train_online_par", "orc_train_batch",
                 "orc_train_batch_par", "orc_train_sweep", "orc_batch_grad_par"):
        getattr(L, name).restype = _int
    _lib = L
    return L


def _dims(w_ih2d, w_ho2d):
    H, D1 = w_ih2d.shape
    K, H1 = w_ho2d.shape
    assert H1 == H + 1
    return D1 - 1, H, K


def _check(rc):
    if rc != 0:
        raise MemoryError("oracle allocation failed")


def train_online_seq(w_ih2d, w_ho2d, feats2d, targets, epochs, lr):
    """kernels.py:264-295 train_segment_seq, in place."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    assert K == 1 and feats2d.shape[1] == D
    _check(lib().orc_train_online_seq(w_ih2d, w_ho2d, np.ascontiguousarray(feats2d),
                                      np.ascontiguousarray(targets, dtype=np.float32),
                                      feats2d.shape[0], D, H, int(epochs), float(lr)))


def train_online_par(w_ih2d, w_ho2d, feats2d, targets, epochs, lr, workers=None):
    """kernels.py:298-349 train_segment_par (OpenMP workers + spin barrier), in place."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    assert K == 1
    nw = workers or (os.cpu_count() or 1)
    _check(lib().orc_train_online_par(w_ih2d, w_ho2d, np.ascontiguousarray(feats2d),
                                      np.ascontiguousarray(targets, dtype=np.float32),
                                      feats2d.shape[0], D, H, int(epochs), float(lr), int(nw)))


def train_batch(w_ih2d, w_ho2d, feats2d, T2d, epochs, lr, batch):
    """Batch restatement; batch=1 == train_online_seq bit-for-bit."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    T = np.ascontiguousarray(np.asarray(T2d, dtype=np.float32).reshape(feats2d.shape[0], K))
    _check(lib().orc_train_batch(w_ih2d, w_ho2d, np.ascontiguousarray(feats2d), T,
                                 feats2d.shape[0], D, H, K, int(epochs), int(batch), float(lr)))


def train_batch_par(w_ih2d, w_ho2d, feats2d, T2d, epochs, lr, workers=None):
    """Full-batch restatement, rows split over OpenMP threads (CPU baseline)."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    T = np.ascontiguousarray(np.asarray(T2d, dtype=np.float32).reshape(feats2d.shape[0], K))
    nw = workers or (os.cpu_count() or 1)
    _check(lib().orc_train_batch_par(w_ih2d, w_ho2d, np.ascontiguousarray(feats2d), T,
                                     feats2d.shape[0], D, H, K, int(epochs), float(lr), int(nw)))


def batch_grad_par(w_ih2d, w_ho2d, feats2d, T2d, workers=None):
    """One epoch's f64 gradient SUM at fixed weights, laid out like glx_batch_grad:
    [dW1 | dW2 | loss, tp, tn, fp, fn] (K == 1 counts; restatement of kernels.py:102-139)."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    T = np.ascontiguousarray(np.asarray(T2d, dtype=np.float32).reshape(feats2d.shape[0], K))
    nw = workers or (os.cpu_count() or 1)
    out = np.zeros(H * (D + 1) + K * (H + 1) + 5, np.float64)
    _check(lib().orc_batch_grad_par(np.ascontiguousarray(w_ih2d), np.ascontiguousarray(w_ho2d),
                                    np.ascontiguousarray(feats2d), T, feats2d.shape[0], D, H, K, out, int(nw)))
    return out


def eval_counts(w_ih2d, w_ho2d, feats2d, labels):
    """kernels.py:352-375 eval_counts -> ((tp, tn, fp, fn), loss_sum)."""
    D, H, K = _dims(w_ih2d, w_ho2d)
    counts = np.zeros(4, dtype=np.int64)
    loss = ctypes.c_double(0.0)
    lib().orc_eval(np.ascontiguousarray(w_ih2d), np.ascontiguousarray(w_ho2d),
                   np.ascontiguousarray(feats2d), np.ascontiguousarray(labels, dtype=np.uint8),
                   feats2d.shape[0], D, H, K, counts, ctypes.byref(loss))
    return tuple(int(c) for c in counts), float(loss.value)


def forward_row(w_ih2d, w_ho2d, x):
    D, H, K = _dims(w_ih2d, w_ho2d)
    h = np.empty(H, np.float32)
    o = np.empty(K, np.float32)
    lib().orc_forward_row(np.ascontiguousarray(w_ih2d), np.ascontiguousarray(w_ho2d),
                          np.ascontiguousarray(x, dtype=np.float32), D, H, K, h, o)
    return h, o


def sigmoid64(x: float) -> float:
    return float(lib().orc_sigmoid64(float(x)))


def train_sweep(H_per_net, w_off, w_pool, feats2d, targets, epochs, lr, workers=None):
    nw = workers or (os.cpu_count() or 1)
    _check(lib().orc_train_sweep(len(H_per_net), np.ascontiguousarray(H_per_net, dtype=np.int32),
                                 np.ascontiguousarray(w_off, dtype=np.int64), w_pool,
                                 np.ascontiguousarray(feats2d), np.ascontiguousarray(targets, dtype=np.float32),
                                 feats2d.shape[0], feats2d.shape[1], int(epochs), float(lr), int(nw)))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ------------------------------------------------------------- min-max normalisation
# numpy restatement of the reference's normalize_fit / normalize_apply
# (/root/reference/pkg/src/glycemlp/dataset.py:369-398): per-column f32 min and
# max of the training rows; (x - min) / (max - min) with every op in f32,
# constant columns -> 0.0, clamp to [-0.5, 1.5]. Pinned bit-exactly against the
# reference's outputs in tests/golden/normalize_cases.npz.
NORM_CLAMP_LO, NORM_CLAMP_HI = np.float32(-0.5), np.float32(1.5)


def normalize_fit(m: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    m = np.asarray(m, dtype=np.float32)
    return m.min(axis=0).copy(), m.max(axis=0).copy()


def normalize_apply(m: np.ndarray, col_min: np.ndarray, col_max: np.ndarray) -> np.ndarray:
    m = np.asarray(m, dtype=np.float32)
    span = (col_max - col_min).astype(np.float32)
    out = np.zeros_like(m)
    nz = span != 0
    out[:, nz] = (m[:, nz] - col_min[nz]) / span[nz]
    return np.clip(out, NORM_CLAMP_LO, NORM_CLAMP_HI)
