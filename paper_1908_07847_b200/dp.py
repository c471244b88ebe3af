"""Data-parallel full-batch training (configs 2/4 across GPUs, config 5).

SURVEY.md 8(e): the rows are sharded contiguously over the ranks (one
process per GPU), every epoch each rank computes the gradient SUM of its
shard with the fused streaming kernel, the P-element f64 vector (P = H(D+1) +
H + 1, plus loss and confusion counts) is summed with one NCCL all-reduce
over NVLink, and every rank applies the identical update
W <- f32(f64(W) - lr/N_total * grad). Summing in float64 keeps 1/2/4/8-GPU
results equal to ~1e-15 of each other.

The NCCL communicator belongs to the C library (NcclComm: glx_dp_init /
glx_dp_allreduce_f64 / glx_dp_train_batch); torch.distributed
is only the control plane that ships the ncclUniqueId and runs barriers. The
product epoch loop is train_data_parallel_nccl (one library call, the epoch
captured in a CUDA graph with the all-reduce inside). train_data_parallel is
the same loop written against a small engine interface so the orchestration
(sharding, all-reduce, update, statistics) is exercised on CPU with gloo and a
test engine (tests/test_dp_cpu.py), and drives the wide engine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError


def shard_bounds(n_rows: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous row range [r0, r1) of `rank`."""
    return n_rows * rank // world_size, n_rows * (rank + 1) // world_size


@dataclass
class EpochStats:
    loss_sum: float
    counts: tuple[int, ...]  # K=1: tp, tn, fp, fn; wide K=16: correct, wrong


class DeviceEngine:
    """One rank's device state: packed rows, weights and the gradient buffer."""

    def __init__(self, feats2d: np.ndarray, targets: np.ndarray, w_ih: np.ndarray, w_ho: np.ndarray,
                 device: int = 0):
        import torch

        self.torch = torch
        self.L = _lib.load()
        self.dev = torch.device("cuda", device)
        self.N, self.D = feats2d.shape
        self.H = w_ih.size // (self.D + 1)
        ld = int(self.L.glx_packed_ld(self.D))
        with torch.cuda.device(self.dev):
            self.stream = torch.cuda.current_stream(self.dev).cuda_stream
            X = torch.from_numpy(np.ascontiguousarray(feats2d, dtype=np.float32)).to(self.dev)
            T = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.float32)).to(self.dev)
            self.Xp = torch.empty((max(self.N, 1), ld), dtype=torch.float32, device=self.dev)
            _lib.check(self.L.glx_pack_rows(X.data_ptr(), T.data_ptr(), None, self.N, self.D, self.Xp.data_ptr(),
                                            self.stream))
            del X, T
            self.w1 = torch.from_numpy(np.ascontiguousarray(w_ih, dtype=np.float32)).to(self.dev)
            self.w2 = torch.from_numpy(np.ascontiguousarray(w_ho, dtype=np.float32)).to(self.dev)
            self.grad = torch.zeros(int(self.L.glx_batch_grad_len(self.D, self.H)), dtype=torch.float64,
                                    device=self.dev)
            self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)

    @classmethod
    def from_device(cls, X, labels, w_ih: np.ndarray, w_ho: np.ndarray):
        """Engine over rows already on the device (torch X (N, D) f32, labels (N,) u8,
        targets = labels): packed straight from HBM, no host round trip."""
        import torch

        self = cls.__new__(cls)
        self.torch = torch
        self.L = _lib.load()
        self.dev = X.device
        self.N, self.D = X.shape
        self.H = w_ih.size // (self.D + 1)
        ld = int(self.L.glx_packed_ld(self.D))
        with torch.cuda.device(self.dev):
            self.stream = torch.cuda.current_stream(self.dev).cuda_stream
            self.Xp = torch.empty((max(self.N, 1), ld), dtype=torch.float32, device=self.dev)
            _lib.check(self.L.glx_pack_rows(X.data_ptr(), None, labels.data_ptr(), self.N, self.D, self.Xp.data_ptr(),
                                            self.stream))
            self.w1 = torch.from_numpy(np.ascontiguousarray(w_ih, dtype=np.float32)).to(self.dev)
            self.w2 = torch.from_numpy(np.ascontiguousarray(w_ho, dtype=np.float32)).to(self.dev)
            self.grad = torch.zeros(int(self.L.glx_batch_grad_len(self.D, self.H)), dtype=torch.float64,
                                    device=self.dev)
            self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        return self

    def grad_sum(self):
        _lib.check(self.L.glx_batch_grad(self.w1.data_ptr(), self.w2.data_ptr(), self.Xp.data_ptr(), self.N,
                                         self.D, self.H, self.grad.data_ptr(), self.stream))
        return self.grad

    def apply(self, grad, lr_over_n: float) -> None:
        _lib.check(self.L.glx_batch_apply(self.w1.data_ptr(), self.w2.data_ptr(), grad.data_ptr(), self.D, self.H,
                                          float(lr_over_n), self.flag.data_ptr(), self.stream))

    def weights(self) -> tuple[np.ndarray, np.ndarray]:
        return self.w1.cpu().numpy(), self.w2.cpu().numpy()

    def nonfinite(self) -> bool:
        return bool(self.flag.item())


def train_data_parallel(engine, epochs: int, lr: float, n_total: int, all_reduce=None) -> list[EpochStats]:
    """Run `epochs` full-batch epochs; all_reduce(tensor) sums in place across ranks.

    Returns per-epoch statistics (loss sum and confusion counts over ALL rows,
    at each epoch's starting weights), identical on every rank.
    """
    # gradient layout: P sums, then loss and the counts (K=1: tp, tn, fp, fn;
    # the wide K=16 engine: correct, wrong)
    P = getattr(engine, "P", None) or engine.H * (engine.D + 1) + engine.H + 1
    ns = getattr(engine, "n_stats", 5)
    kept = []  # device-side copies: no host sync inside the epoch loop
    for _ in range(epochs):
        g = engine.grad_sum()
        if all_reduce is not None:
            all_reduce(g)
        engine.apply(g, lr / n_total)
        kept.append(g[P:P + ns].clone() if hasattr(g, "clone") else g[P:P + ns].copy())
    stats = []
    for s in kept:
        s = s.tolist()
        stats.append(EpochStats(float(s[0]), tuple(int(round(v)) for v in s[1:ns])))
    return stats


class NcclComm:
    """This rank's NCCL communicator, owned by the C library (glx_dp_init ->
    ncclCommInitRank). Rank 0 makes the 128-byte ncclUniqueId
    (glx_dp_unique_id) and the control group (any torch.distributed group that can
    broadcast_object_list, e.g. gloo) ships it to the other ranks; with one rank
    no group is needed. The data plane -- the per-epoch gradient all-reduce --
    never goes through torch."""

    def __init__(self, rank: int = 0, world_size: int = 1, device: int = 0, group=None):
        import ctypes

        import torch  # noqa: F401  (loads torch's libnccl first: the library binds the loaded copy)

        self.L = _lib.load()
        self.rank, self.world_size, self.device = rank, world_size, device
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _lib.check(self.L.glx_dp_unique_id(_lib.ptr(uid)))
        if world_size > 1:
            import torch.distributed as dist

            box = [uid.tobytes()]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = np.frombuffer(box[0], np.uint8).copy()
        h = ctypes.c_void_p()
        _lib.check(self.L.glx_dp_init(device, world_size, rank, _lib.ptr(uid), ctypes.byref(h)))
        self.handle = h.value

    def all_reduce(self, t, op: str = "sum", stream=None) -> None:
        """In-place all-reduce of a float64 device tensor (sum or max)."""
        import torch

        assert t.dtype == torch.float64 and t.is_contiguous()
        st = stream if stream is not None else torch.cuda.current_stream(t.device).cuda_stream
        _lib.check(self.L.glx_dp_allreduce_f64(self.handle, t.data_ptr(), t.numel(), 1 if op == "max" else 0, st))

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.check(self.L.glx_dp_finalize(self.handle))
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def train_data_parallel_nccl(engine: DeviceEngine, comm: NcclComm, epochs: int, lr: float,
                             n_total: int) -> list[EpochStats]:
    """`epochs` data-parallel epochs in ONE library call (glx_dp_train_batch): the
    epoch kernel over this rank's rows, the f64 gradient sum, the NCCL all-reduce
    and the update, captured once into a CUDA graph by the library and replayed.
    Same arithmetic as train_data_parallel with an all-reduce; returns the
    per-epoch statistics over all ranks' rows."""
    import torch

    if epochs <= 0:
        return []
    hist = torch.zeros((epochs, 5), dtype=torch.float64, device=engine.dev)
    _lib.check(engine.L.glx_dp_train_batch(comm.handle, engine.w1.data_ptr(), engine.w2.data_ptr(),
                                           engine.Xp.data_ptr(), engine.N, int(n_total), engine.D, engine.H,
                                           int(epochs), float(lr), hist.data_ptr(), engine.flag.data_ptr(),
                                           engine.stream))
    return [EpochStats(float(s[0]), tuple(int(round(v)) for v in s[1:5])) for s in hist.tolist()]


def run_train_segment_batch_dp(comm: NcclComm, w_ih2d: np.ndarray, w_ho2d: np.ndarray, feats2d: np.ndarray,
                               targets: np.ndarray, rows_total: int, epochs: int, lr: float,
                               stats_hist: np.ndarray | None = None) -> None:
    """Public data-parallel counterpart of backend.run_train_segment_batch: this
    rank's row shard in HOST memory (copied in), `epochs` full-batch epochs over
    all ranks' rows_total rows (glx_dp_run_train_segment_batch: pack, the
    graph-captured epoch with the NCCL all-reduce inside, update), the weights
    copied back into the caller's arrays in place -- identical on every rank.
    Collective: every rank calls it with the same epochs, lr and rows_total.
    stats_hist (epochs x 5 f64, optional): loss, tp, tn, fp, fn over all rows."""
    from .backend import _check_inputs, _check_weights, _f32c

    D, H = _check_weights(w_ih2d, w_ho2d)
    _check_inputs(w_ih2d, feats2d, targets)
    x, t = _f32c(feats2d), _f32c(targets)
    st = None
    if stats_hist is not None:
        if stats_hist.dtype != np.float64 or stats_hist.shape != (epochs, 5) or not stats_hist.flags.c_contiguous:
            raise ShapeError(f"stats_hist must be a C-contiguous float64 ({epochs}, 5) array")
        st = _lib.ptr(stats_hist)
    _lib.check(comm.L.glx_dp_run_train_segment_batch(comm.handle, _lib.ptr(w_ih2d), _lib.ptr(w_ho2d), _lib.ptr(x),
                                                     _lib.ptr(t), x.shape[0], int(rows_total), D, H, int(epochs),
                                                     float(lr), st, 0))


def torch_all_reduce(group=None):
    """all_reduce(tensor) over a torch.distributed group (the CPU/gloo tests' stand-in
    for NcclComm.all_reduce)."""
    import torch.distributed as dist

    def _ar(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return _ar
