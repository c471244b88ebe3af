"""Dataset containers and the synthetic sample generator of the benchmark configs.

Mirrors the parts of the reference's dataset module that the training path
reads (/root/reference/pkg/src/glycemlp/dataset.py): the immutable
row-major float32 + uint8 Dataset (:77-111), SplitPair (:114-120),
NormStats (:61-74), synthetic_matrix (:260-289), which defines every
benchmark configuration's input, and the min-max normalisation
normalize_fit / normalize_apply / normalize_split (:369-410), which runs on
the device (csrc/glx_data.cu) with the reference's f32
results bit for bit. CSV ingestion, record derivation and splitting are host
plumbing outside the accelerated path; a reference-built
SplitPair can be passed straight to trainer.train.

For cohorts too large for per-row string ids (configs 2/4: 1M and 64M rows),
synthetic_arrays / iter_synthetic_chunks produce the same bytes as
synthetic_matrix without the Dataset wrapper, optionally chunk by chunk.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _lib
from .errors import ShapeError, ValidationError

SUBSET_TAGS = ("male", "female", "all", "synthetic")
LABEL_GOOD = 0
LABEL_POOR = 1


@dataclass(frozen=True)
class NormStats:
    col_min: np.ndarray
    col_max: np.ndarray

    def __post_init__(self) -> None:
        if self.col_min.shape != self.col_max.shape or self.col_min.ndim != 1:
            raise ShapeError("col_min and col_max must be 1-D arrays of equal length")

    @property
    def columns(self) -> int:
        return int(self.col_min.shape[0])


@dataclass(frozen=True)
class Dataset:
    """Immutable flat row-major float32 features + uint8 labels (dataset.py:77-111)."""

    features: np.ndarray
    labels: np.ndarray
    rows: int
    columns: int
    subset_tag: str
    row_ids: tuple
    norm_stats: NormStats | None = None

    def __post_init__(self) -> None:
        if self.subset_tag not in SUBSET_TAGS:
            raise ValidationError(f"subset_tag must be one of {SUBSET_TAGS}, got {self.subset_tag!r}")
        if self.features.dtype != np.float32 or self.features.ndim != 1:
            raise ShapeError("features must be a flat float32 array")
        if self.features.shape[0] != self.rows * self.columns:
            raise ShapeError(f"features length {self.features.shape[0]} != rows*columns ({self.rows}*{self.columns})")
        if self.labels.shape[0] != self.rows:
            raise ShapeError(f"labels length {self.labels.shape[0]} != rows {self.rows}")
        if len(self.row_ids) != self.rows:
            raise ShapeError(f"row_ids length {len(self.row_ids)} != rows {self.rows}")
        self.features.setflags(write=False)
        self.labels.setflags(write=False)

    def matrix(self) -> np.ndarray:
        return self.features.reshape(self.rows, self.columns)


@dataclass(frozen=True)
class SplitPair:
    train: Dataset
    test: Dataset
    seed: int
    fraction: float
    stratified: bool = True


def _check_synth_args(rows: int, columns: int, signal: str) -> None:
    if rows < 2:
        raise ValueError(f"rows must be >= 2, got {rows}")
    if columns < 1:
        raise ValueError(f"columns must be >= 1, got {columns}")
    if signal not in ("planted-linear", "random"):
        raise ValueError(f"signal must be planted-linear or random, got {signal!r}")


def synthetic_arrays(rows: int, columns: int, seed: int, signal: str = "random") -> tuple[np.ndarray, np.ndarray]:
    """(features (rows, columns) f32, labels (rows,) u8), byte-identical to synthetic_matrix.

    The generator call order is the reference's (dataset.py:272-281): all
    U[0,1) float32 features first, then either the planted hyperplane
    (5 distinct columns, N(0,1) weights, label = score >= median score) or
    independent fair-coin labels.
    """
    _check_synth_args(rows, columns, signal)
    gen = np.random.default_rng(seed)
    feats = gen.random((rows, columns), dtype=np.float32)
    if signal == "random":
        return feats, (gen.random(rows) < 0.5).astype(np.uint8)
    pick = gen.choice(columns, size=min(5, columns), replace=False)
    coef = gen.normal(0.0, 1.0, size=pick.shape[0])
    score = feats[:, pick].astype(np.float64) @ coef
    return feats, (score >= np.median(score)).astype(np.uint8)


def synthetic_matrix(rows: int, columns: int, seed: int, signal: str = "random") -> Dataset:
    """Benchmark / shape-test Dataset (dataset.py:260-289)."""
    feats, labels = synthetic_arrays(rows, columns, seed, signal)
    return Dataset(
        features=feats.reshape(-1),
        labels=labels,
        rows=rows,
        columns=columns,
        subset_tag="synthetic",
        row_ids=tuple(f"m{i:05d}" for i in range(rows)),
    )


def iter_synthetic_chunks(rows: int, columns: int, seed: int, signal: str = "random",
                          chunk_rows: int = 1 << 20) -> Iterator[tuple[int, np.ndarray, np.ndarray]]:
    """Yield (row0, features chunk, labels chunk) equal to synthetic_arrays' rows.

    PCG64 float32 draws are sequential, so drawing the feature matrix in row
    chunks gives the same bytes as one draw. The planted labels depend on the
    median over ALL rows and the hyperplane is drawn after the features, so
    planted-linear runs two passes: one to draw the hyperplane and the scores,
    then a replay of the saved generator state for the features.
    """
    _check_synth_args(rows, columns, signal)
    gen = np.random.default_rng(seed)
    start_state = gen.bit_generator.state
    if signal == "random":
        for r0 in range(0, rows, chunk_rows):
            gen.random((min(chunk_rows, rows - r0), columns), dtype=np.float32)
        labels = (gen.random(rows) < 0.5).astype(np.uint8)
        gen.bit_generator.state = start_state
        for r0 in range(0, rows, chunk_rows):
            n = min(chunk_rows, rows - r0)
            yield r0, gen.random((n, columns), dtype=np.float32), labels[r0:r0 + n]
        return
    # pass 1: advance past the features, draw the hyperplane, then score chunk by chunk
    for r0 in range(0, rows, chunk_rows):
        gen.random((min(chunk_rows, rows - r0), columns), dtype=np.float32)
    pick = gen.choice(columns, size=min(5, columns), replace=False)
    coef = gen.normal(0.0, 1.0, size=pick.shape[0])
    gen.bit_generator.state = start_state
    score = np.empty(rows, dtype=np.float64)
    for r0 in range(0, rows, chunk_rows):
        n = min(chunk_rows, rows - r0)
        f = gen.random((n, columns), dtype=np.float32)
        score[r0:r0 + n] = f[:, pick].astype(np.float64) @ coef
    labels = (score >= np.median(score)).astype(np.uint8)
    del score
    gen.bit_generator.state = start_state
    for r0 in range(0, rows, chunk_rows):
        n = min(chunk_rows, rows - r0)
        yield r0, gen.random((n, columns), dtype=np.float32), labels[r0:r0 + n]


# ---------------------------------------------------------------- normalisation
def _device_matrix(d: Dataset, device: int):
    import torch

    return torch.from_numpy(np.array(d.matrix(), dtype=np.float32, copy=True)).to(torch.device("cuda", device))


def normalize_fit(train: Dataset, device: int = 0) -> NormStats:
    """Per-column min/max of the training partition (dataset.py:369-372), on the device."""
    import torch

    L = _lib.load()
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev):
        m = _device_matrix(train, device)
        mn = torch.empty(train.columns, dtype=torch.float32, device=dev)
        mx = torch.empty(train.columns, dtype=torch.float32, device=dev)
        _lib.check(L.glx_minmax_fit(m.data_ptr(), train.rows, train.columns, mn.data_ptr(), mx.data_ptr(),
                                    torch.cuda.current_stream(dev).cuda_stream))
        return NormStats(col_min=mn.cpu().numpy(), col_max=mx.cpu().numpy())


def normalize_apply(d: Dataset, stats: NormStats, device: int = 0) -> Dataset:
    """Min-max scale with train-fitted stats, clamp to [-0.5, 1.5], constant columns
    -> 0.0 (dataset.py:375-398), on the device; same f32 bytes as the reference."""
    import torch

    if stats.columns != d.columns:
        raise ShapeError(f"stats have {stats.columns} columns, dataset has {d.columns}")
    L = _lib.load()
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev):
        m = _device_matrix(d, device)
        mn = torch.from_numpy(np.ascontiguousarray(stats.col_min, dtype=np.float32)).to(dev)
        mx = torch.from_numpy(np.ascontiguousarray(stats.col_max, dtype=np.float32)).to(dev)
        _lib.check(L.glx_minmax_apply(m.data_ptr(), d.rows, d.columns, mn.data_ptr(), mx.data_ptr(), m.data_ptr(),
                                      torch.cuda.current_stream(dev).cuda_stream))
        out = m.cpu().numpy()
    return Dataset(features=np.ascontiguousarray(out, dtype=np.float32).reshape(-1), labels=d.labels.copy(),
                   rows=d.rows, columns=d.columns, subset_tag=d.subset_tag, row_ids=d.row_ids, norm_stats=stats)


def normalize_split(pair: SplitPair, device: int = 0) -> SplitPair:
    """Fit on the train partition, apply to both sides (dataset.py:401-410)."""
    stats = normalize_fit(pair.train, device)
    return SplitPair(train=normalize_apply(pair.train, stats, device), test=normalize_apply(pair.test, stats, device),
                     seed=pair.seed, fraction=pair.fraction, stratified=pair.stratified)


# ------------------------------------------------------------- device generation
def _split128(v: int) -> tuple[int, int]:
    return (v >> 64) & 0xFFFFFFFFFFFFFFFF, v & 0xFFFFFFFFFFFFFFFF


def _post_feature_generator(seed: int, n_floats: int) -> np.random.Generator:
    """default_rng(seed) in the state synthetic_arrays leaves after drawing n_floats
    float32 features (PCG64.advance over the 64-bit outputs, plus the buffered
    32-bit half when n_floats is odd)."""
    k0 = (n_floats + 1) // 2
    gen = np.random.default_rng(seed)
    gen.bit_generator.advance(k0)
    if n_floats % 2:
        g = np.random.default_rng(seed)
        g.bit_generator.advance(k0 - 1)
        v = int(g.bit_generator.random_raw(1)[0])
        st = gen.bit_generator.state
        st["has_uint32"] = 1
        st["uinteger"] = v >> 32
        gen.bit_generator.state = st
    return gen


def synthetic_arrays_device(rows: int, columns: int, seed: int, signal: str = "random", device: int = 0):
    """synthetic_arrays generated on the device: (features (rows, columns) f32,
    labels (rows,) u8) as torch tensors on cuda:device, byte-identical to the host
    generator (dataset.py:260-289). The PCG64 stream is evaluated by jump-ahead on
    the GPU (csrc/glx_data.cu); the planted hyperplane's 5 columns and N(0,1)
    weights are drawn on the host from the generator advanced past the features,
    scores and labels (score >= median, numpy's two-middle-values mean) on the
    device."""
    import torch

    _check_synth_args(rows, columns, signal)
    L = _lib.load()
    dev = torch.device("cuda", device)
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s_hi, s_lo = _split128(int(st["state"]))
    i_hi, i_lo = _split128(int(st["inc"]))
    n_floats = rows * columns
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        X = torch.empty((rows, columns), dtype=torch.float32, device=dev)
        labels = torch.empty(rows, dtype=torch.uint8, device=dev)
        _lib.check(L.glx_pcg64_uniform_f32(s_hi, s_lo, i_hi, i_lo, 0, n_floats, X.data_ptr(), stream))
        if signal == "random":
            _lib.check(L.glx_pcg64_coin(s_hi, s_lo, i_hi, i_lo, (n_floats + 1) // 2, rows, labels.data_ptr(), stream))
            return X, labels
        gen = _post_feature_generator(seed, n_floats)
        pick = gen.choice(columns, size=min(5, columns), replace=False)
        coef = gen.normal(0.0, 1.0, size=pick.shape[0])
        pk = torch.from_numpy(pick.astype(np.int32)).to(dev)
        cf = torch.from_numpy(np.ascontiguousarray(coef, dtype=np.float64)).to(dev)
        score = torch.empty(rows, dtype=torch.float64, device=dev)
        _lib.check(L.glx_planted_score(X.data_ptr(), rows, columns, pk.data_ptr(), cf.data_ptr(), int(pick.shape[0]),
                                       score.data_ptr(), stream))
        # numpy median: the middle value, or the mean of the two middle values
        # (a device sort: 31 ms at 64Mi rows, where torch.kthvalue took 0.75 s)
        srt = torch.sort(score).values
        lo = srt[(rows - 1) // 2]
        med = lo if rows % 2 else (lo + srt[rows // 2]) / 2.0
        del srt
        thr = med.reshape(1).contiguous()
        _lib.check(L.glx_label_ge(score.data_ptr(), rows, thr.data_ptr(), labels.data_ptr(), stream))
        return X, labels
