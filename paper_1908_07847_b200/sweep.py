"""Hidden-width x seed sweeps: many independent online-SGD networks at once.

SURVEY.md config 3 / 8(e): 4096 networks 33 -> {8..512} -> 1 (64 widths x 64
seeds) trained with the reference's per-instance semantics
(kernels.py:264-295) on one shared dataset. The networks are independent,
so multi-GPU runs shard them with no communication: longest-processing-time
(LPT) assignment on a cost model proportional to H*(D+1+K) balances the
ranks (one process per GPU under torchrun), and rank 0 gathers the trained
weights. Inside a GPU, the C ABI (glx_train_sweep) packs several networks
per CTA, each on its own warp range and named barrier, sharing one
shared-memory copy of the rows.
"""

from __future__ import annotations

import os
import heapq
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError, ValidationError
from .network import Network, NetworkConfig, init_weights


@dataclass(frozen=True)
class SweepSpec:
    input_dim: int
    hidden_dims: tuple[int, ...]
    seeds: tuple[int, ...]
    epochs: int
    learning_rate: float = 0.1
    init_range: float = 0.5
    numerics: str = "fp32"

    def __post_init__(self) -> None:
        object.__setattr__(self, "hidden_dims", tuple(int(h) for h in self.hidden_dims))
        object.__setattr__(self, "seeds", tuple(int(s) for s in self.seeds))
        if len(self.hidden_dims) != len(self.seeds):
            raise ValidationError("hidden_dims and seeds must have one entry per network")
        if self.epochs < 0:
            raise ValidationError(f"epochs must be >= 0, got {self.epochs}")
        if self.numerics not in _lib.NUMERICS:
            raise ValidationError(f"numerics must be one of {tuple(_lib.NUMERICS)}")

    def configs(self) -> list[NetworkConfig]:
        return [NetworkConfig(input_dim=self.input_dim, hidden_dim=h, seed=s, learning_rate=self.learning_rate,
                              init_range=self.init_range) for h, s in zip(self.hidden_dims, self.seeds)]

    def costs(self) -> np.ndarray:
        """Relative cost per network: FLOPs per row-step, ~ H * (D + 1 + K)."""
        return np.array([h * (self.input_dim + 2) for h in self.hidden_dims], dtype=np.float64)


def sweep_grid(widths, seeds) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """Cartesian widths x seeds, width-major (config 3: range(8, 513, 8) x range(64))."""
    hs, ss = [], []
    for h in widths:
        for s in seeds:
            hs.append(int(h))
            ss.append(int(s))
    return tuple(hs), tuple(ss)


def lpt_shards(costs, n_shards: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of items to n_shards bins.

    Items are taken in decreasing cost (ties by index) and each goes to the
    currently lightest bin (ties by bin index): deterministic, and within
    4/3 of the optimal makespan.
    """
    if n_shards < 1:
        raise ValidationError("n_shards must be >= 1")
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(costs.shape[0]), key=lambda i: (-costs[i], i))
    heap = [(0.0, b) for b in range(n_shards)]
    bins: list[list[int]] = [[] for _ in range(n_shards)]
    for i in order:
        load, b = heapq.heappop(heap)
        bins[b].append(i)
        heapq.heappush(heap, (load + costs[i], b))
    return [sorted(b) for b in bins]


def pack_pool(nets: list[Network]) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Flat weight pool [w_ih | w_ho] per network, plus H and float offsets."""
    sizes = [n.w_ih.size + n.w_ho.size for n in nets]
    off = np.zeros(len(nets), dtype=np.int64)
    if nets:
        off[1:] = np.cumsum(sizes[:-1])
    pool = np.empty(int(sum(sizes)), dtype=np.float32)
    for n, o in zip(nets, off):
        pool[o:o + n.w_ih.size] = n.w_ih
        pool[o + n.w_ih.size:o + n.w_ih.size + n.w_ho.size] = n.w_ho
    H = np.array([n.config.hidden_dim for n in nets], dtype=np.int32)
    return pool, H, off


def unpack_pool(pool: np.ndarray, nets: list[Network], off: np.ndarray) -> None:
    for n, o in zip(nets, off):
        n.w_ih[:] = pool[o:o + n.w_ih.size]
        n.w_ho[:] = pool[o + n.w_ih.size:o + n.w_ih.size + n.w_ho.size]


def train_nets_on_device(nets: list[Network], feats2d: np.ndarray, targets: np.ndarray, epochs: int, lr: float,
                         numerics: str = "fp32", device: int = 0) -> None:
    """Train `nets` in place on one GPU with glx_train_sweep (torch buffers for plumbing)."""
    import torch

    if not nets:
        return
    D = nets[0].config.input_dim
    if any(n.config.input_dim != D for n in nets) or feats2d.shape[1] != D:
        raise ShapeError("every network must share the dataset's input_dim")
    if targets.shape[0] != feats2d.shape[0]:
        raise ShapeError("targets length must match feature rows")
    L = _lib.load()
    pool, H, off = pack_pool(nets)
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        wp = torch.from_numpy(pool).to(dev)
        X = torch.from_numpy(np.ascontiguousarray(feats2d, dtype=np.float32)).to(dev)
        T = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.float32)).to(dev)
        _lib.check(L.glx_train_sweep(len(nets), _lib.ptr(H), _lib.ptr(off), wp.data_ptr(), X.data_ptr(),
                                     T.data_ptr(), X.shape[0], D, int(epochs), float(lr),
                                     _lib.NUMERICS[numerics], stream.cuda_stream))
        out = wp.cpu().numpy()
    unpack_pool(out, nets, off)


def train_sweep(spec: SweepSpec, feats2d: np.ndarray, targets: np.ndarray, *, rank: int = 0, world_size: int = 1,
                device: int | None = None, group=None, trainer=None) -> list[Network] | None:
    """Train every network of the sweep; with world_size > 1 each rank trains its
    LPT shard on its own GPU and rank 0 returns the gathered list (others None).
    `trainer(nets, feats2d, targets, epochs, lr, numerics, device)` trains a list in
    place (default: the device kernel, train_nets_on_device; tests inject a CPU
    stand-in to exercise the sharding and gather with gloo)."""
    nets = [init_weights(c) for c in spec.configs()]
    shards = lpt_shards(spec.costs(), world_size)
    mine = shards[rank]
    # the local GPU of this rank (a global rank can exceed the node's GPU count)
    dev = int(os.environ.get("LOCAL_RANK", rank)) if device is None else device
    if trainer is None:
        import torch

        if torch.cuda.is_available():
            # gather_object over NCCL stages through torch.cuda.current_device()
            torch.cuda.set_device(dev)
    (trainer or train_nets_on_device)([nets[i] for i in mine], feats2d, targets, spec.epochs, spec.learning_rate,
                                      spec.numerics, dev)
    if world_size == 1:
        return nets
    import torch.distributed as dist

    payload = {i: (nets[i].w_ih, nets[i].w_ho) for i in mine}
    gathered = [None] * world_size if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0, group=group)
    if rank != 0:
        return None
    for part in gathered:
        for i, (wi, wo) in part.items():
            nets[i].w_ih[:] = wi
            nets[i].w_ho[:] = wo
    return nets
