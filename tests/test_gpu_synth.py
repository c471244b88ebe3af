"""Device generation of the benchmark rows (dataset.synthetic_arrays_device,
csrc/glx_data.cu): numpy's PCG64 stream by jump-ahead, byte-identical to the
reference's synthetic_matrix (golden digests generated from the reference)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1908_07847_b200 as g

pytestmark = pytest.mark.gpu

GEN = json.loads((Path(__file__).parent / "golden" / "generators.json").read_text())


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", GEN["synthetic_matrix"], ids=lambda c: f"{c['rows']}x{c['columns']}-{c['signal']}")
def test_device_rows_match_reference_digests(gpu, case):
    X, lab = g.synthetic_arrays_device(case["rows"], case["columns"], case["seed"], case["signal"])
    assert _sha(X.cpu().numpy().reshape(-1)) == case["features_sha256"]
    assert _sha(lab.cpu().numpy()) == case["labels_sha256"]


@pytest.mark.parametrize("rows,cols,seed,signal", [(2, 1, 0, "random"), (3, 3, 5, "planted-linear"),
                                                   (2, 7, 9, "random"), (257, 5, 3, "planted-linear"),
                                                   (1_000_003, 33, 11, "planted-linear"), (99_999, 3, 2, "random")])
def test_device_rows_equal_host_generator(gpu, rows, cols, seed, signal):
    """Odd float counts (a buffered 32-bit half), one column, tiny and large N."""
    if signal == "planted-linear" and rows < 2:
        pytest.skip("planted labels need two rows")
    X, lab = g.synthetic_arrays_device(rows, cols, seed, signal)
    hx, hl = g.synthetic_arrays(rows, cols, seed, signal)
    assert X.cpu().numpy().tobytes() == hx.tobytes()
    assert (lab.cpu().numpy() == hl).all()
