"""`import glycemlp`: the reference package's import surface on the B200 engine.

The reference installs the package `glycemlp` from pkg/src
(/root/reference/pkg/pyproject.toml:5-19) and exports its API from
/root/reference/pkg/src/glycemlp/__init__.py:5-106. This package keeps that
path and those names for the training / prediction / evaluation hot path,
re-exported from `paper_1908_07847_b200` (hand-written sm_100a kernels behind
the C ABI of include/glycemlp_cuda.h), so reference call sites run unchanged:

    import glycemlp as g
    report = g.train(g.TrainSpec(config=g.NetworkConfig(input_dim=33, seed=7),
                                 epochs=100_000, backend=g.parallel()), split)

`g.sequential()` / `g.parallel(n)` select the device engine in the
reference's float64 operation order (the bytes the reference's two CPU
engines produce); `g.cuda()` selects the FP32 engine. The submodules
glycemlp.backend / network / trainer / dataset / errors / kernels / bench
resolve to their device-backed counterparts.

Out of scope (host plumbing that runs once per run, not on
the path): the clinical record schema, record synthesis, CSV I/O and the
stratified split (`schema`, `synth`, `parse_csv`, `write_csv`,
`build_dataset`, `split_by_sex`, `train_test_split`, ...). Accessing those
names raises AttributeError naming the reason; build the SplitPair with the
reference's pipeline (or any other) and pass it to `train`.
"""

from __future__ import annotations

import sys as _sys
from pathlib import Path as _Path

_ROOT = _Path(__file__).resolve().parents[3]
if str(_ROOT) not in _sys.path:
    _sys.path.insert(0, str(_ROOT))

import paper_1908_07847_b200 as _impl  # noqa: E402
from paper_1908_07847_b200 import backend, bench_report, dataset, errors, network, trainer  # noqa: E402
from paper_1908_07847_b200.backend import (  # noqa: E402
    BackendKind,
    LayerJob,
    cuda,
    hardware_parallelism,
    max_workers,
    parallel,
    run_layer_backward,
    run_layer_forward,
    sequential,
)
from paper_1908_07847_b200.bench_report import BenchReport, BenchSpec, emit_speedup_table, run_bench  # noqa: E402
from paper_1908_07847_b200.dataset import (  # noqa: E402
    Dataset,
    NormStats,
    SplitPair,
    normalize_apply,
    normalize_fit,
    normalize_split,
    synthetic_matrix,
)
from paper_1908_07847_b200.errors import (  # noqa: E402
    GlycemlpError,
    NumericError,
    ParseError,
    SchemaError,
    ShapeError,
    ValidationError,
)
from paper_1908_07847_b200.network import (  # noqa: E402
    GOOD,
    POOR,
    Activations,
    Network,
    NetworkConfig,
    backprop_update,
    forward,
    init_weights,
    load_checkpoint,
    predict,
    save_checkpoint,
    sigmoid,
)
from paper_1908_07847_b200.trainer import TrainReport, TrainSpec, epoch_sweep, evaluate, format_percent, train  # noqa: E402

from . import kernels  # noqa: E402

bench = bench_report
for _name, _mod in (("backend", backend), ("network", network), ("trainer", trainer), ("dataset", dataset),
                    ("errors", errors), ("bench", bench_report)):
    _sys.modules[f"{__name__}.{_name}"] = _mod

__version__ = _impl.__version__

# names of the reference's __init__ that belong to the out-of-scope record / CSV /
# split pipeline (dataset.py:131-366, schema.py, synth.py)
OUT_OF_SCOPE = (
    "HBA1C_POOR_CUTOFF_PCT", "ParticipantRecord", "build_dataset", "derive_features", "label_from_hba1c",
    "parse_csv", "split_by_sex", "synth_dataset", "train_test_split", "write_csv", "schema", "synth", "cli",
)


def __getattr__(name: str):
    if name in OUT_OF_SCOPE:
        raise AttributeError(
            f"glycemlp.{name} is not part of the B200 hot path (SURVEY.md 2.1: record schema, synthesis, CSV "
            f"and split are host plumbing); build the SplitPair with the reference's data pipeline and pass "
            f"it to glycemlp.train")
    raise AttributeError(f"module 'glycemlp' has no attribute {name!r}")


__all__ = [
    "Activations", "BackendKind", "BenchReport", "BenchSpec", "Dataset", "GlycemlpError", "GOOD", "LayerJob",
    "Network", "NetworkConfig", "NormStats", "NumericError", "POOR", "ParseError", "SchemaError", "ShapeError",
    "SplitPair", "TrainReport", "TrainSpec", "ValidationError", "backprop_update", "cuda", "emit_speedup_table",
    "epoch_sweep", "evaluate", "format_percent", "forward", "init_weights", "load_checkpoint", "normalize_apply",
    "normalize_fit", "normalize_split", "parallel", "predict", "run_bench", "run_layer_backward",
    "run_layer_forward", "save_checkpoint", "sequential", "sigmoid", "synthetic_matrix", "train",
]
