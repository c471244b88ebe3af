"""Wide configuration: 1024 -> 1024 -> 16, full-batch GD on tcgen05.

Every large contraction of the epoch (hidden layer, hidden deltas, dW1) runs on
the hand-written tcgen05 GEMM of csrc/glx_tc.cu with FP32 TMEM accumulation, in
one of two precisions: "bf16" (BF16 rows and operands, H and the deltas stored
in BF16; the throughput configuration) or "tf32" (f32 U[0,1) rows, kind::tf32
MMAs, H and the deltas stored in f32; within SURVEY.md 8(c)'s 1e-4 FP32
tolerance of the f64 oracle on the f32 rows). The f32 master weights keep the reference layout
(w_ih 1024 x 1025, w_ho 16 x 1025) and take the update in f64. The rows are
generated on the device (16M x 1024 does not fit host RAM as f32): U[0,1)
features from a counter-based hash and K=16 labels = argmax of 16 planted
linear scores (a build decision; parity for K>1 is against the
oracle restatement, not the reference).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ShapeError

D, H, K = 1024, 1024, 16


PRECISIONS = ("bf16", "tf32")


class WideData:
    """Device-resident rows. bf16: Xb (N x 1024 bf16), XT ([X,1]^T, 1025 x N bf16 stored
    K-blocked as [N/64][1025][64]). tf32: Xb (N x 1024 f32, U[0,1)), XT ([X,1]^T f32,
    K-blocked [N/32][1025][32]). labels (N u8) either way."""

    def __init__(self, n_rows: int, seed: int = 0, device: int = 0, row0: int = 0, precision: str = "bf16"):
        """Rows [row0, row0 + n_rows) of the data set `seed` (row0 > 0: a data-parallel shard)."""
        import torch

        if precision not in PRECISIONS:
            raise ShapeError(f"precision must be one of {PRECISIONS}, got {precision!r}")
        blk = 64 if precision == "bf16" else 32
        if n_rows < blk or n_rows % blk:
            raise ShapeError(f"wide {precision} data needs a positive multiple of {blk} rows, got {n_rows}")
        self.N = n_rows
        self.row0 = row0
        self.precision = precision
        self.dev = torch.device("cuda", device)
        L = _lib.load()
        dt = torch.bfloat16 if precision == "bf16" else torch.float32
        make = L.glx_wide_make_shard if precision == "bf16" else L.glx_wide_make_shard_tf32
        with torch.cuda.device(self.dev):
            self.Xb = torch.empty((n_rows, D), dtype=dt, device=self.dev)
            self.XT = torch.empty((n_rows // blk, D + 1, blk), dtype=dt, device=self.dev)
            self.labels = torch.empty(n_rows, dtype=torch.uint8, device=self.dev)
            _lib.check(make(row0, n_rows, seed, self.Xb.data_ptr(), self.XT.data_ptr(), self.labels.data_ptr(),
                            torch.cuda.current_stream().cuda_stream))

    def host_rows(self) -> tuple[np.ndarray, np.ndarray]:
        """(features f32 = the exact stored values, labels u8) for CPU checking."""
        return self.Xb.float().cpu().numpy(), self.labels.cpu().numpy()


def init_wide_weights(seed: int = 0, init_range: float = 0.5) -> tuple[np.ndarray, np.ndarray]:
    """Reference-style init (network.py:110-116) for the 1024-1024-16 shape."""
    gen = np.random.default_rng(seed)
    w_ih = gen.uniform(-init_range, init_range, H * (D + 1)).astype(np.float32)
    w_ho = gen.uniform(-init_range, init_range, K * (H + 1)).astype(np.float32)
    return w_ih, w_ho


def train_wide(data: WideData, w_ih: np.ndarray, w_ho: np.ndarray, epochs: int, lr: float,
               stats: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Run `epochs` full-batch epochs; returns the updated (w_ih, w_ho) copies.

    stats, if given, is a float64 (epochs, 3) array: loss sum, correct, wrong
    at each epoch's starting weights.
    """
    import torch

    if w_ih.size != H * (D + 1) or w_ho.size != K * (H + 1):
        raise ShapeError("wide weights must be 1024 x 1025 and 16 x 1025")
    L = _lib.load()
    with torch.cuda.device(data.dev):
        st = torch.cuda.current_stream()
        w1 = torch.from_numpy(np.ascontiguousarray(w_ih, dtype=np.float32)).to(data.dev)
        w2 = torch.from_numpy(np.ascontiguousarray(w_ho, dtype=np.float32)).to(data.dev)
        sd = torch.zeros((max(epochs, 1), 3), dtype=torch.float64, device=data.dev)
        flag = torch.zeros(1, dtype=torch.int32, device=data.dev)
        train = L.glx_wide_train if data.precision == "bf16" else L.glx_wide_train_tf32
        _lib.check(train(w1.data_ptr(), w2.data_ptr(), data.Xb.data_ptr(), data.XT.data_ptr(),
                         data.labels.data_ptr(), data.N, int(epochs), float(lr), sd.data_ptr(),
                         flag.data_ptr(), st.cuda_stream))
        if stats is not None:
            stats[:] = sd[:epochs].cpu().numpy()
        return w1.cpu().numpy(), w2.cpu().numpy()


def shard_rows(n_rows: int, world_size: int, rank: int, block: int = 64) -> tuple[int, int]:
    """Contiguous shard [r0, r1) of `rank` with both ends on `block`-row boundaries
    (64 for the bf16 layout, 32 for tf32)."""
    if n_rows % block:
        raise ShapeError(f"wide data needs a multiple of {block} rows, got {n_rows}")
    blocks = n_rows // block
    return block * (blocks * rank // world_size), block * (blocks * (rank + 1) // world_size)


class WideEngine:
    """One rank's wide-network state for dp.train_data_parallel:
    the shard's device rows, f32 master weights and the f64 gradient buffer
    (P = 1,066,000 sums + loss, correct, wrong)."""

    P = H * (D + 1) + K * (H + 1)
    n_stats = 3

    def __init__(self, data: WideData, w_ih: np.ndarray, w_ho: np.ndarray):
        import torch

        if w_ih.size != H * (D + 1) or w_ho.size != K * (H + 1):
            raise ShapeError("wide weights must be 1024 x 1025 and 16 x 1025")
        self.torch = torch
        self.L = _lib.load()
        self.data = data
        self.N = data.N
        with torch.cuda.device(data.dev):
            self.stream = torch.cuda.current_stream(data.dev).cuda_stream
            self.w1 = torch.from_numpy(np.ascontiguousarray(w_ih, dtype=np.float32).reshape(-1)).to(data.dev)
            self.w2 = torch.from_numpy(np.ascontiguousarray(w_ho, dtype=np.float32).reshape(-1)).to(data.dev)
            self.grad = torch.zeros(int(self.L.glx_wide_grad_len()), dtype=torch.float64, device=data.dev)
            self.flag = torch.zeros(1, dtype=torch.int32, device=data.dev)

    def grad_sum(self):
        d = self.data
        grad = self.L.glx_wide_grad if d.precision == "bf16" else self.L.glx_wide_grad_tf32
        _lib.check(grad(self.w1.data_ptr(), self.w2.data_ptr(), d.Xb.data_ptr(), d.XT.data_ptr(),
                        d.labels.data_ptr(), d.N, self.grad.data_ptr(), self.stream))
        return self.grad

    def apply(self, grad, lr_over_n: float) -> None:
        _lib.check(self.L.glx_wide_apply(self.w1.data_ptr(), self.w2.data_ptr(), grad.data_ptr(), float(lr_over_n),
                                         self.flag.data_ptr(), self.stream))

    def weights(self) -> tuple[np.ndarray, np.ndarray]:
        return self.w1.cpu().numpy(), self.w2.cpu().numpy()

    def nonfinite(self) -> bool:
        return bool(self.flag.item())
