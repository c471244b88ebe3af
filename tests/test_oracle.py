"""The C oracle (oracle/glx_oracle.c) pinned against the REFERENCE's own outputs.

Fixtures in tests/golden/ were produced by running the unmodified reference
(tests/golden/make_golden.py). Everything here is CPU-only.
"""

import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, load_case

from oracle import oracle as O

ONLINE_CASES = ["paper_33_33_1", "cohort_male_30_30_1", "cohort_female_30_30_1", "wide_33_256_1"]


@pytest.fixture(scope="module", autouse=True)
def _built():
    O.build()


def _net(case):
    D, H, K, _ = case["meta"]
    return case["w_ih0"].copy().reshape(H, D + 1), case["w_ho0"].copy().reshape(1, H + 1)


@pytest.mark.parametrize("name", ONLINE_CASES)
def test_online_seq_bitexact_vs_reference(name):
    c = load_case(name)
    w1, w2 = _net(c)
    t = c["train_y"].astype(np.float32)
    prev = 0
    for cp in c["checkpoints"]:
        O.train_online_seq(w1, w2, c["train_x"], t, int(cp - prev), 0.1)
        prev = cp
        assert w1.reshape(-1).tobytes() == c[f"w_ih_{cp}"].tobytes(), f"w_ih differs at epoch {cp}"
        assert w2.reshape(-1).tobytes() == c[f"w_ho_{cp}"].tobytes(), f"w_ho differs at epoch {cp}"
        tr, _ = O.eval_counts(w1, w2, c["train_x"], c["train_y"])
        te, _ = O.eval_counts(w1, w2, c["test_x"], c["test_y"])
        assert tr == tuple(c[f"train_counts_{cp}"]) and te == tuple(c[f"test_counts_{cp}"])


@pytest.mark.parametrize("name", ["paper_33_33_1", "wide_33_256_1"])
@pytest.mark.parametrize("workers", [1, 2, 3, 8])
def test_online_par_equals_seq(name, workers):
    # kernels.py:298-349 contract: the neuron-parallel engine is byte-identical
    c = load_case(name)
    w1, w2 = _net(c)
    cp = int(c["checkpoints"][-1])
    O.train_online_par(w1, w2, c["train_x"], c["train_y"].astype(np.float32), cp, 0.1, workers)
    assert w1.reshape(-1).tobytes() == c[f"w_ih_{cp}"].tobytes()
    assert w2.reshape(-1).tobytes() == c[f"w_ho_{cp}"].tobytes()


@pytest.mark.parametrize("name", ONLINE_CASES)
def test_batch_B1_anchor_equals_online(name):
    # the batch restatement with B=1 reproduces train_segment_seq bit-for-bit
    c = load_case(name)
    w1, w2 = _net(c)
    cp = int(c["checkpoints"][-1])
    O.train_batch(w1, w2, c["train_x"], c["train_y"].astype(np.float32), cp, 0.1, 1)
    assert w1.reshape(-1).tobytes() == c[f"w_ih_{cp}"].tobytes()
    assert w2.reshape(-1).tobytes() == c[f"w_ho_{cp}"].tobytes()


def test_small_backend_case():
    c = load_case("small_7_19_1")
    w1 = c["w_ih0"].copy().reshape(19, 8)
    w2 = c["w_ho0"].copy().reshape(1, 20)
    O.train_online_seq(w1, w2, c["x"], c["t"], int(c["epochs"][0]), 0.1)
    assert w1.reshape(-1).tobytes() == c["w_ih"].tobytes()
    assert w2.reshape(-1).tobytes() == c["w_ho"].tobytes()


def test_batch_full_equals_par_rows_within_f64():
    rng = np.random.default_rng(3)
    x = rng.random((333, 7), dtype=np.float32)
    t = (rng.random(333) < 0.5).astype(np.float32)
    w1 = rng.uniform(-0.5, 0.5, (5, 8)).astype(np.float32)
    w2 = rng.uniform(-0.5, 0.5, (1, 6)).astype(np.float32)
    a1, a2, b1, b2 = w1.copy(), w2.copy(), w1.copy(), w2.copy()
    O.train_batch(a1, a2, x, t, 7, 0.5, 333)
    O.train_batch_par(b1, b2, x, t, 7, 0.5, 4)
    assert np.max(np.abs(a1 - b1)) <= 1e-6 and np.max(np.abs(a2 - b2)) <= 1e-6


def test_multi_output_eval_and_batch_shapes():
    rng = np.random.default_rng(5)
    x = rng.random((50, 6), dtype=np.float32)
    y = rng.integers(0, 4, 50).astype(np.uint8)
    w1 = rng.uniform(-0.5, 0.5, (9, 7)).astype(np.float32)
    w2 = rng.uniform(-0.5, 0.5, (4, 10)).astype(np.float32)
    (corr, wrong, z0, z1), loss = O.eval_counts(w1, w2, x, y)
    assert corr + wrong == 50 and z0 == z1 == 0 and loss > 0
    T = np.eye(4, dtype=np.float32)[y]
    before = loss
    O.train_batch(w1, w2, x, T, 200, 2.0, 50)
    _, after = O.eval_counts(w1, w2, x, y)
    assert after < before


# ---- reference known-answer tests (test_network.py / test_trainer.py) ----

def test_sigmoid_known_answers():
    assert O.sigmoid64(0.0) == 0.5
    assert abs(O.sigmoid64(20.0) - 0.9999999979388463) < 1e-12
    assert abs(O.sigmoid64(20.0) - 1.0 / (1.0 + math.exp(-20.0))) < 1e-15


def test_forward_known_answers():
    # zero weights give 0.5 everywhere (test_network.py:95-100)
    h, o = O.forward_row(np.zeros((3, 5), np.float32), np.zeros((1, 4), np.float32),
                         np.array([0.3, -1.2, 0.0, 2.0], np.float32))
    assert h.tolist() == [0.5] * 3 and o.tolist() == [0.5]
    # hand-evaluated 1-1-1 network (test_network.py:102-107)
    h, o = O.forward_row(np.array([[1.0, 0.0]], np.float32), np.array([[1.0, 0.0]], np.float32),
                         np.array([0.0], np.float32))
    assert abs(float(o[0]) - 0.6224593312018546) < 1e-6


def test_zero_net_confusion_known_answers():
    w1, w2 = np.zeros((2, 4), np.float32), np.zeros((1, 3), np.float32)
    x = np.random.default_rng(0).random((10, 3), dtype=np.float32)
    # 40% poor labels: the 0.5 boundary predicts poor everywhere -> accuracy 0.4 (test_trainer.py:137-140)
    (tp, tn, fp, fn), _ = O.eval_counts(w1, w2, x, np.array([1, 1, 1, 1, 0, 0, 0, 0, 0, 0], np.uint8))
    assert (tp + tn) / 10 == pytest.approx(0.4)
    (tp, tn, fp, fn), _ = O.eval_counts(w1, w2, x[:4], np.array([1, 0, 1, 0], np.uint8))
    assert (tp, tn, fp, fn) == (2, 0, 2, 0)  # test_trainer.py:155-160


def test_lr_zero_is_identity():
    c = load_case("paper_33_33_1")
    w1, w2 = _net(c)
    b1, b2 = w1.copy(), w2.copy()
    O.train_online_seq(w1, w2, c["train_x"], c["train_y"].astype(np.float32), 3, 0.0)
    assert w1.tobytes() == b1.tobytes() and w2.tobytes() == b2.tobytes()


def test_trainer_fixture_consistency():
    # the reference trainer's checkpoint rows equal oracle evaluation of oracle-trained weights
    doc = json.loads((GOLDEN / "trainer_paper_1000.json").read_text())
    c = load_case("paper_33_33_1")
    for row in doc["rows"]:
        cp = row["epoch"]
        counts = tuple(row["train_confusion"][k] for k in ("tp", "tn", "fp", "fn"))
        assert counts == tuple(c[f"train_counts_{cp}"])
