import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def built():
    """Build (or refresh) the CUDA library and the oracle once per session."""
    from paper_1908_07847_b200 import _build
    from oracle import oracle

    _build.build()
    oracle.build()
    return True


@pytest.fixture(scope="session")
def gpu(built):
    import paper_1908_07847_b200._lib as L

    L.load()  # raises if no device: GPU tests must not silently pass on CPU
    return True


def load_case(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def make_split(train_x, train_y, test_x, test_y):
    """SplitPair from already-normalised arrays (the fixtures store the reference's
    normalised matrices; the trainer only checks that norm stats are present)."""
    import paper_1908_07847_b200 as g

    D = train_x.shape[1]
    stats = g.NormStats(col_min=np.zeros(D, np.float32), col_max=np.ones(D, np.float32))
    tr = g.Dataset(features=np.ascontiguousarray(train_x, np.float32).reshape(-1).copy(),
                   labels=np.asarray(train_y, np.uint8).copy(), rows=train_x.shape[0], columns=D,
                   subset_tag="synthetic", row_ids=tuple(f"a{i}" for i in range(train_x.shape[0])),
                   norm_stats=stats)
    te = g.Dataset(features=np.ascontiguousarray(test_x, np.float32).reshape(-1).copy(),
                   labels=np.asarray(test_y, np.uint8).copy(), rows=test_x.shape[0], columns=D,
                   subset_tag="synthetic", row_ids=tuple(f"b{i}" for i in range(test_x.shape[0])),
                   norm_stats=stats)
    return g.SplitPair(train=tr, test=te, seed=0, fraction=0.75)


def rel_err(a, b):
    """max |a-b| / max(1, |b|): the weight tolerance metric (test_gradcheck.py:50)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


PKG_SRC = ROOT / "pkg" / "src"
if str(PKG_SRC) not in sys.path:
    sys.path.insert(0, str(PKG_SRC))
