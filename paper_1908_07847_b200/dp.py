"""Data-parallel full-batch training over torch.distributed (configs 4 and 5).

SURVEY.md 8(e): the rows are sharded contiguously over the ranks (one
process per GPU), every epoch each rank computes the gradient SUM of its
shard with the fused streaming kernel (glx_batch_grad), the P-element f64
vector (P = H(D+1) + H + 1, plus loss and confusion counts) is summed with
one NCCL all-reduce over NVLink, and every rank applies the identical
update W <- f32(f64(W) - lr/N_total * grad) (glx_batch_apply). Summing in
float64 keeps 1/2/4/8-GPU results equal to ~1e-15 of each other.

The epoch loop is written against a small engine interface so the
orchestration (sharding, all-reduce, update, statistics) is exercised on CPU
with gloo and a test engine (tests/test_dp_cpu.py); DeviceEngine is the
product engine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


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


# kernels of this library launched by CUDA-graph replays (the library's own
# glx_launch_count only sees launches issued through its C entry points)
graph_kernel_launches = 0


def train_data_parallel_graph(engine, epochs: int, lr: float, n_total: int, all_reduce) -> list[EpochStats]:
    """train_data_parallel with one epoch (gradient kernels, all-reduce, update)
    captured in a CUDA graph and replayed, removing the per-epoch host launch
    overhead. The graph is cached on the engine (keyed on the step size), so only
    the first call captures. NCCL collectives are graph-capturable; if capture
    fails the eager loop runs instead. Same arithmetic and results as
    train_data_parallel."""
    import torch

    if epochs <= 0:
        return []
    P = getattr(engine, "P", None) or engine.H * (engine.D + 1) + engine.H + 1
    ns = getattr(engine, "n_stats", 5)
    key = float(lr) / n_total
    cache = getattr(engine, "_graph_cache", None)
    if cache is None or cache[0] != key:
        side = torch.cuda.Stream(device=engine.grad.device)
        saved = engine.stream
        side.wait_stream(torch.cuda.current_stream())
        try:
            with torch.cuda.stream(side):
                engine.stream = side.cuda_stream
                # one eager epoch on the capture stream: the library allocates its
                # per-stream workspace on first use, which capture does not allow.
                # Errors here are real (kernel / NCCL) and propagate.
                first = train_data_parallel(engine, 1, lr, n_total, all_reduce)
                graph = torch.cuda.CUDAGraph()
                n0 = int(engine.L.glx_launch_count())
                try:
                    with torch.cuda.graph(graph, stream=side):
                        g = engine.grad_sum()
                        all_reduce(g)
                        engine.apply(g, key)
                except RuntimeError as e:  # only a refused capture falls back to eager epochs
                    if "captur" not in str(e).lower():
                        raise
                    graph = None
                per_replay = int(engine.L.glx_launch_count()) - n0
        finally:
            engine.stream = saved
            torch.cuda.current_stream().wait_stream(side)
        if graph is None:
            return first + train_data_parallel(engine, epochs - 1, lr, n_total, all_reduce)
        engine._graph_cache = (key, graph, side, per_replay)
        done = first
        epochs -= 1
    else:
        done = []
    global graph_kernel_launches
    _, graph, side, per_replay = engine._graph_cache
    graph_kernel_launches += per_replay * epochs
    hist = torch.zeros((max(epochs, 1), ns), dtype=torch.float64, device=engine.grad.device)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for e in range(epochs):
            graph.replay()
            hist[e].copy_(engine.grad[P:P + ns])
    torch.cuda.current_stream().wait_stream(side)
    out = list(done)
    for s in hist[:epochs].tolist():
        out.append(EpochStats(float(s[0]), tuple(int(round(v)) for v in s[1:ns])))
    return out


def nccl_all_reduce(group=None):
    import torch.distributed as dist

    def _ar(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return _ar
