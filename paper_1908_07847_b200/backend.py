"""Execution backend: the drop-in for the reference's engine selection and
training-segment entry point, running on the B200 through the C ABI.

Reference counterparts (/root/reference/pkg/src/glycemlp/):
  BackendKind / sequential() / parallel()      backend.py:44-70
  run_train_segment(w_ih2d, w_ho2d, feats2d, targets, epochs, lr, kind)
                                               backend.py:208-234
  kernels.eval_counts(w_ih2d, w_ho2d, feats2d, labels)
                                               kernels.py:352-375
  LayerJob / run_layer_forward / run_layer_backward / backpropagate_error
                                               backend.py:73-205
plus run_train_segment_batch (full-batch GD) and
run_train_segment_eval (one trainer checkpoint in one device call, 8(f)1).

Engine names. The reference's two names are accepted with their meaning kept:
"sequential" and "parallel" (with a worker count, validated as the reference
does) both select the device engine in the reference's float64 operation
order ("ref64"), which is the result the reference's two CPU engines both
produce bit for bit; the worker count is recorded (effective_workers) but the
device has no host thread pool to size. "cuda" is the device engine with a
choice of numerics: "fp32" (default; packed-FP32 FMA, MUFU sigmoid, within
the 1e-4 max(1,|w|)-relative tolerance of SURVEY.md 8(c)) or "ref64". Any
other name raises ValidationError (test_backend.py:24-25). There is no CPU
engine in this package.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError, ValidationError

CUDA = "cuda"
SEQUENTIAL = "sequential"
PARALLEL = "parallel"
ENGINES = (SEQUENTIAL, PARALLEL, CUDA)
ONLINE = "online"
BATCH = "batch"


def hardware_parallelism() -> int:
    """backend.py:34-35: the host's core count (the default parallel() worker count)."""
    return os.cpu_count() or 1


def max_workers() -> int:
    """backend.py:38-40: the upper bound on a worker pool. The reference sizes it by
    numba's thread pool (the core count); the device engine has no host pool, so the
    same core-count bound is kept for the reference's clamping contract."""
    return hardware_parallelism()


@dataclass(frozen=True)
class BackendKind:
    """Engine selector (backend.py:44-62).

    name      "sequential" | "parallel" (reference-exact device engine) | "cuda"
    workers   the reference's worker-pool size (>= 1); for "cuda", the GPUs used by
              the sharded entry points (sweep, data parallel)
    numerics  "fp32" or "ref64"; forced to "ref64" for the reference's two names
    device    CUDA device ordinal for the host-pointer entry points
    """

    name: str
    workers: int = 1
    numerics: str = "fp32"
    device: int = 0

    def __post_init__(self) -> None:
        if self.name not in ENGINES:
            raise ValidationError(f"backend must be {SEQUENTIAL}, {PARALLEL} or {CUDA}, got {self.name!r}")
        if not isinstance(self.workers, (int, np.integer)) or self.workers < 1:
            raise ValidationError(f"worker_count must be >= 1, got {self.workers}")
        if self.name != CUDA:
            object.__setattr__(self, "numerics", "ref64")
        if self.numerics not in _lib.NUMERICS:
            raise ValidationError(f"numerics must be one of {tuple(_lib.NUMERICS)}, got {self.numerics!r}")
        if self.device < 0:
            raise ValidationError(f"device must be >= 0, got {self.device}")

    @property
    def effective_workers(self) -> int:
        """backend.py:57-62: 1 for sequential; the requested pool clamped to max_workers()."""
        return 1 if self.name == SEQUENTIAL else min(int(self.workers), max_workers())


def cuda(device: int = 0, numerics: str = "fp32", workers: int = 1) -> BackendKind:
    return BackendKind(CUDA, workers, numerics, device)


def sequential() -> BackendKind:
    """The reference's sequential engine: reference-exact (ref64) numerics on the device."""
    return BackendKind(SEQUENTIAL, 1)


def parallel(workers: int | None = None) -> BackendKind:
    """The reference's neuron-parallel engine (bit-identical to sequential by contract,
    SPEC.md:301): the same reference-exact device engine; `workers` validated and kept."""
    return BackendKind(PARALLEL, hardware_parallelism() if workers is None else workers)


def _f32c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _check_weights(w_ih2d: np.ndarray, w_ho2d: np.ndarray) -> tuple[int, int]:
    for name, w in (("w_ih2d", w_ih2d), ("w_ho2d", w_ho2d)):
        if w.dtype != np.float32 or w.ndim != 2 or not w.flags.c_contiguous or not w.flags.writeable:
            raise ShapeError(f"{name} must be a writeable C-contiguous 2-D float32 array (updated in place)")
    H, d1 = w_ih2d.shape
    if w_ho2d.shape != (1, H + 1):
        raise ShapeError(f"w_ho2d shape {w_ho2d.shape} != (1, {H + 1})")
    return d1 - 1, H


def _check_inputs(w_ih2d, feats2d, targets):
    if feats2d.ndim != 2 or feats2d.shape[1] != w_ih2d.shape[1] - 1:
        raise ShapeError(f"feature count {feats2d.shape[-1]} != input_dim {w_ih2d.shape[1] - 1}")
    if targets.shape[0] != feats2d.shape[0]:
        raise ShapeError("targets length must match feature rows")


def _cache_flag(enabled: bool, *arrays: np.ndarray) -> int:
    # resident-input reuse keys on host pointers: only safe for read-only
    # arrays that outlive the caller's sequence of calls (trainer.train)
    return _lib.GLX_FLAG_CACHE_INPUTS if enabled and all(not a.flags.writeable for a in arrays) else 0


def clear_input_cache() -> None:
    _lib.load(require_device=False).glx_cache_clear()


def run_train_segment(w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray, targets: np.ndarray,
                      epochs: int, lr: float, kind: BackendKind, *, cache_inputs: bool = False) -> None:
    """`epochs` passes of per-instance SGD in dataset order, weights updated in place.

    Same contract as backend.py:208-234: ShapeError on a feature-count or
    target-length mismatch, synchronous, non-finite weights are left for the
    caller to detect.
    """
    _check_inputs(w_ih2d, feats2d, targets)
    D, H = _check_weights(w_ih2d, w_ho2d)
    L = _lib.load()
    X = feats2d if (feats2d.dtype == np.float32 and feats2d.flags.c_contiguous) else _f32c(feats2d)
    T = targets if (targets.dtype == np.float32 and targets.flags.c_contiguous) else _f32c(targets)
    _lib.check(L.glx_run_train_segment(
        _lib.ptr(w_ih2d), _lib.ptr(w_ho2d), _lib.ptr(X), _lib.ptr(T), X.shape[0], D, H, int(epochs), float(lr),
        _lib.NUMERICS[kind.numerics], kind.device, _cache_flag(cache_inputs, X, T)))


def run_train_segment_batch(w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray, targets: np.ndarray,
                            epochs: int, lr: float, kind: BackendKind, stats: np.ndarray | None = None, *,
                            cache_inputs: bool = False, debug: bool = False) -> None:
    """`epochs` of full-batch gradient descent (mean gradient over all rows), in place.

    SURVEY.md 8(a) a13 (no reference implementation; parity against the
    oracle restatement). `stats`, if given, is a float64 (epochs, 5) array
    receiving loss sum, tp, tn, fp, fn at each epoch's starting weights.
    `debug` checks the tcgen05 epoch kernels' pipelines every epoch (tile hand-off
    stamps, one visit per row tile; RuntimeError on a violation) -- the device
    analogue of the reference's debug instrumentation (backend.py:122-133, 237-284).
    """
    _check_inputs(w_ih2d, feats2d, targets)
    D, H = _check_weights(w_ih2d, w_ho2d)
    L = _lib.load()
    X = feats2d if (feats2d.dtype == np.float32 and feats2d.flags.c_contiguous) else _f32c(feats2d)
    T = targets if (targets.dtype == np.float32 and targets.flags.c_contiguous) else _f32c(targets)
    sp = None
    if stats is not None:
        if stats.dtype != np.float64 or stats.shape != (int(epochs), 5) or not stats.flags.c_contiguous:
            raise ShapeError(f"stats must be a C-contiguous float64 array of shape ({int(epochs)}, 5)")
        sp = _lib.ptr(stats)
    _lib.check(L.glx_run_train_segment_batch(
        _lib.ptr(w_ih2d), _lib.ptr(w_ho2d), _lib.ptr(X), _lib.ptr(T), X.shape[0], D, H, int(epochs), float(lr),
        sp, kind.device, _cache_flag(cache_inputs, X, T) | (_lib.GLX_FLAG_DEBUG if debug else 0)))


@dataclass(frozen=True)
class CheckpointEval:
    """Result of run_train_segment_eval: exact confusion counts (tp, tn, fp, fn)
    of both splits at the segment's final weights, their loss sums, whether every
    weight is finite, and the training part's wall time."""

    train_counts: tuple[int, int, int, int]
    test_counts: tuple[int, int, int, int]
    train_loss: float
    test_loss: float
    finite: bool
    train_seconds: float


def run_train_segment_eval(w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray, targets: np.ndarray,
                           labels: np.ndarray, test_feats2d: np.ndarray, test_labels: np.ndarray, epochs: int,
                           lr: float, kind: BackendKind, *, mode: str = ONLINE,
                           cache_inputs: bool = False) -> CheckpointEval:
    """One trainer checkpoint in one device call: `epochs` of
    training (online SGD or full batch), then the finiteness test and the exact
    train/test confusion counts on the device, without a host round trip of the
    weights in between. Weights are updated in place like run_train_segment."""
    _check_inputs(w_ih2d, feats2d, targets)
    D, H = _check_weights(w_ih2d, w_ho2d)
    if labels.shape[0] != feats2d.shape[0]:
        raise ShapeError("labels length must match feature rows")
    if test_feats2d.ndim != 2 or test_feats2d.shape[1] != D or test_labels.shape[0] != test_feats2d.shape[0]:
        raise ShapeError(f"test rows must be (n, {D}) with n labels")
    if mode not in (ONLINE, BATCH):
        raise ValidationError(f"mode must be {ONLINE!r} or {BATCH!r}, got {mode!r}")
    L = _lib.load()
    X = feats2d if (feats2d.dtype == np.float32 and feats2d.flags.c_contiguous) else _f32c(feats2d)
    T = targets if (targets.dtype == np.float32 and targets.flags.c_contiguous) else _f32c(targets)
    Y = labels if (labels.dtype == np.uint8 and labels.flags.c_contiguous) else np.ascontiguousarray(labels, np.uint8)
    VX = test_feats2d if (test_feats2d.dtype == np.float32 and test_feats2d.flags.c_contiguous) else _f32c(test_feats2d)
    VY = (test_labels if (test_labels.dtype == np.uint8 and test_labels.flags.c_contiguous)
          else np.ascontiguousarray(test_labels, np.uint8))
    counts = np.zeros(8, dtype=np.int64)
    loss = np.zeros(2, dtype=np.float64)
    finite = np.zeros(1, dtype=np.int32)
    secs = np.zeros(1, dtype=np.float64)
    _lib.check(L.glx_run_train_segment_eval(
        _lib.ptr(w_ih2d), _lib.ptr(w_ho2d), _lib.ptr(X), _lib.ptr(T), _lib.ptr(Y), X.shape[0], _lib.ptr(VX),
        _lib.ptr(VY), VX.shape[0], D, H, int(epochs), float(lr), _lib.NUMERICS[kind.numerics],
        0 if mode == ONLINE else 1, kind.device, _cache_flag(cache_inputs, X, T, Y, VX, VY), _lib.ptr(counts),
        _lib.ptr(loss), _lib.ptr(finite), _lib.ptr(secs)))
    c = [int(v) for v in counts]
    return CheckpointEval(tuple(c[:4]), tuple(c[4:]), float(loss[0]), float(loss[1]), bool(finite[0]),
                          float(secs[0]))


def eval_counts_loss(w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray, labels: np.ndarray,
                     kind: BackendKind | None = None) -> tuple[tuple[int, int, int, int], float]:
    """((tp, tn, fp, fn), sum of 0.5*(t-o)^2) with poor (label 1) as the positive class."""
    kind = kind or sequential()
    if feats2d.ndim != 2 or feats2d.shape[1] != w_ih2d.shape[1] - 1:
        raise ShapeError(f"feature count {feats2d.shape[-1]} != input_dim {w_ih2d.shape[1] - 1}")
    if labels.shape[0] != feats2d.shape[0]:
        raise ShapeError("labels length must match feature rows")
    H, d1 = w_ih2d.shape
    K = w_ho2d.shape[0]
    L = _lib.load()
    W1, W2 = _f32c(w_ih2d), _f32c(w_ho2d)
    X = _f32c(feats2d)
    Y = np.ascontiguousarray(labels, dtype=np.uint8)
    counts = np.zeros(4, dtype=np.int64)
    loss = np.zeros(1, dtype=np.float64)
    _lib.check(L.glx_eval_counts(_lib.ptr(W1), _lib.ptr(W2), _lib.ptr(X), _lib.ptr(Y), X.shape[0], d1 - 1, H, K,
                                 _lib.NUMERICS[kind.numerics], _lib.ptr(counts), _lib.ptr(loss), kind.device, 0))
    return (int(counts[0]), int(counts[1]), int(counts[2]), int(counts[3])), float(loss[0])


def eval_counts(w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray, labels: np.ndarray,
                kind: BackendKind | None = None) -> tuple[int, int, int, int]:
    """Drop-in for kernels.eval_counts (kernels.py:352-375)."""
    return eval_counts_loss(w_ih2d, w_ho2d, feats2d, labels, kind)[0]


# ------------------------------------------------------- layer-level API
@dataclass
class LayerJob:
    """One dense layer pass (backend.py:73-102): weights (n_neurons x (n_inputs+1)),
    inputs, outputs; the same validation as the reference."""

    weights: np.ndarray
    inputs: np.ndarray
    outputs: np.ndarray

    def __post_init__(self) -> None:
        if self.weights.ndim != 2 or self.weights.dtype != np.float32:
            raise ShapeError("weights must be a 2-D float32 array")
        if self.inputs.ndim != 1 or self.inputs.dtype != np.float32:
            raise ShapeError("inputs must be a 1-D float32 array")
        if self.weights.shape[1] != self.inputs.shape[0] + 1:
            raise ShapeError(f"weights row length {self.weights.shape[1]} != n_inputs+1 ({self.inputs.shape[0]}+1)")
        if self.outputs.shape != (self.weights.shape[0],) or self.outputs.dtype != np.float32:
            raise ShapeError("outputs must be a float32 array with one slot per neuron")

    @classmethod
    def create(cls, weights: np.ndarray, inputs: np.ndarray) -> "LayerJob":
        w = np.ascontiguousarray(weights, dtype=np.float32)
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        return cls(weights=w, inputs=x, outputs=np.empty(w.shape[0], dtype=np.float32))


def _dev(kind: BackendKind | None):
    import torch

    return torch.device("cuda", (kind or sequential()).device)


def _check_written_once(counts) -> None:
    """The reference's write-once shadow check (backend.py:122-133)."""
    c = counts.cpu().numpy()
    if not (c == 1).all():
        bad = np.flatnonzero(c != 1)
        raise RuntimeError(f"output slots written != once: indices {bad.tolist()}")


def run_layer_forward(job: LayerJob, kind: BackendKind | None = None, debug: bool = False) -> np.ndarray:
    """outputs[j] = sigmoid(dot(weights row j, inputs) + bias_j), filled in place
    (backend.py:134-144), on the device in the reference's f64 order. `debug`: every
    output slot counts its writes on the device (glx_layer_forward_checked) and
    each must be written exactly once (backend.py:122-133)."""
    import torch

    L = _lib.load()
    dev = _dev(kind)
    n, m1 = job.weights.shape
    W = torch.from_numpy(np.ascontiguousarray(job.weights)).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(job.inputs)).to(dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    if debug:
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        _lib.check(L.glx_layer_forward_checked(W.data_ptr(), x.data_ptr(), 1, m1 - 1, n, out.data_ptr(),
                                               counts.data_ptr(), st))
        _check_written_once(counts)
    else:
        _lib.check(L.glx_layer_forward(W.data_ptr(), x.data_ptr(), 1, m1 - 1, n, out.data_ptr(), st))
    job.outputs[:] = out.cpu().numpy()
    return job.outputs


def run_layer_backward(job: LayerJob, upstream_error: np.ndarray, kind: BackendKind | None = None,
                       debug: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """Per-neuron deltas and gradient rows for one layer (backend.py:147-189):
    deltas[j] = (err_j a_j)(1 - a_j), grads[j] = deltas[j] [inputs, 1], f64, with
    job.outputs holding the layer's forward activations."""
    import torch

    n, m1 = job.weights.shape
    err = np.ascontiguousarray(upstream_error, dtype=np.float64)
    if err.shape != (n,):
        raise ShapeError(f"upstream_error must have shape ({n},), got {err.shape}")
    L = _lib.load()
    dev = _dev(kind)
    x = torch.from_numpy(np.ascontiguousarray(job.inputs)).to(dev)
    a = torch.from_numpy(np.ascontiguousarray(job.outputs)).to(dev)
    e = torch.from_numpy(err).to(dev)
    deltas = torch.empty(n, dtype=torch.float64, device=dev)
    grads = torch.empty((n, m1), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    if debug:  # each neuron's delta and gradient row written exactly once
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        _lib.check(L.glx_layer_backward_checked(x.data_ptr(), a.data_ptr(), e.data_ptr(), n, m1 - 1,
                                                deltas.data_ptr(), grads.data_ptr(), counts.data_ptr(), st))
        _check_written_once(counts)
    else:
        _lib.check(L.glx_layer_backward(x.data_ptr(), a.data_ptr(), e.data_ptr(), n, m1 - 1, deltas.data_ptr(),
                                        grads.data_ptr(), st))
    return deltas.cpu().numpy(), grads.cpu().numpy()


def forward_pair_debug(w_ih2d: np.ndarray, w_ho2d: np.ndarray, instance: np.ndarray, workers: int = 2,
                       kind: BackendKind | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Instrumented two-layer forward proving the inter-layer barrier
    (backend.py:237-284) on the device: `workers` warps write and generation-stamp
    the hidden slots, and past the layer barrier the output pass requires every
    stamp to be current (RuntimeError naming the stale slots otherwise)."""
    import torch

    if w_ih2d.ndim != 2 or w_ho2d.ndim != 2 or w_ho2d.shape[1] != w_ih2d.shape[0] + 1:
        raise ShapeError(f"weight shapes {w_ih2d.shape} / {w_ho2d.shape} do not chain")
    H, D = w_ih2d.shape[0], w_ih2d.shape[1] - 1
    K = w_ho2d.shape[0]
    x = np.ascontiguousarray(instance, dtype=np.float32).ravel()
    if x.shape[0] != D:
        raise ShapeError(f"instance has {x.shape[0]} features, network expects {D}")
    L = _lib.load()
    dev = _dev(kind)
    W1 = torch.from_numpy(_f32c(w_ih2d)).to(dev)
    W2 = torch.from_numpy(_f32c(w_ho2d)).to(dev)
    xd = torch.from_numpy(x).to(dev)
    hidden = torch.empty(H, dtype=torch.float32, device=dev)
    out = torch.empty(K, dtype=torch.float32, device=dev)
    stamps = torch.zeros(H, dtype=torch.int32, device=dev)
    status = torch.full((1,), -1, dtype=torch.int32, device=dev)
    _lib.check(L.glx_forward_pair_debug(W1.data_ptr(), W2.data_ptr(), xd.data_ptr(), D, H, K, hidden.data_ptr(),
                                        out.data_ptr(), stamps.data_ptr(), status.data_ptr(), int(workers),
                                        torch.cuda.current_stream(dev).cuda_stream))
    s = int(status.item())
    if s != 0:
        stale = np.flatnonzero(stamps.cpu().numpy() != 1)
        raise RuntimeError(f"hidden slots read before write: {stale.tolist()}")
    return hidden.cpu().numpy(), out.cpu().numpy()


def backpropagate_error(weights: np.ndarray, deltas: np.ndarray, kind: BackendKind | None = None) -> np.ndarray:
    """Fold a layer's deltas back into upstream error terms, W^T @ delta without the
    bias column, 16-blocked over neurons (backend.py:192-205)."""
    import torch

    w = np.ascontiguousarray(weights, dtype=np.float32)
    d = np.ascontiguousarray(deltas, dtype=np.float64)
    if w.ndim != 2 or d.shape != (w.shape[0],):
        raise ShapeError("weights must be (n, m+1) and deltas length n")
    n, m1 = w.shape
    L = _lib.load()
    dev = _dev(kind)
    W = torch.from_numpy(w).to(dev)
    D = torch.from_numpy(d).to(dev)
    out = torch.empty(m1 - 1, dtype=torch.float64, device=dev)
    _lib.check(L.glx_backprop_error(W.data_ptr(), D.data_ptr(), n, m1 - 1, out.data_ptr(),
                                    torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy()
