"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run here (the only place /root/reference exists), never on the GPU box:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records, for small fixed-seed cases, the reference's own outputs:

* online SGD weights after N epochs via backend.run_train_segment
  (kernels.train_segment_seq, kernels.py:264-295) and the parallel engine;
* eval_counts (kernels.py:352-375) at each checkpoint;
* trainer.train checkpoint rows (trainer.py:123-199);
* synthetic_matrix (dataset.py:260-289) and init_weights (network.py:110-116)
  digests, so the product's own generators can be pinned byte-for-byte.

The committed .npz/.json files are what tests/ read; this script is only
re-run when a case is added.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import glycemlp as g  # noqa: E402
from glycemlp import backend as B  # noqa: E402
from glycemlp import kernels as Kr  # noqa: E402
from glycemlp.trainer import TrainSpec  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def matrix_split(rows, cols, seed, signal="planted-linear"):
    data = g.synthetic_matrix(rows, cols, seed, signal)
    return g.normalize_split(g.train_test_split(data, 0.75, seed))


def record_split(rows, seed, signal, sex=None):
    records = g.synth_dataset(rows, seed, signal)
    if sex is not None:
        male, female = g.split_by_sex(records)
        records = male if sex == "male" else female
    data = g.build_dataset(records, "synthetic")
    return g.normalize_split(g.train_test_split(data, 0.75, seed))


def online_case(name, pair, hidden, seed, checkpoints, lr=0.1):
    cfg = g.NetworkConfig(input_dim=pair.train.columns, hidden_dim=hidden, seed=seed, learning_rate=lr)
    net = g.init_weights(cfg)
    feats = pair.train.matrix()
    targets = pair.train.labels.astype(np.float32)
    out = {
        "train_x": np.ascontiguousarray(feats), "train_y": pair.train.labels.copy(),
        "test_x": np.ascontiguousarray(pair.test.matrix()), "test_y": pair.test.labels.copy(),
        "w_ih0": net.w_ih.copy(), "w_ho0": net.w_ho.copy(),
        "checkpoints": np.array(checkpoints, dtype=np.int64),
        "meta": np.array([pair.train.columns, hidden, 1, seed], dtype=np.int64),
        "lr": np.array([lr]),
    }
    prev = 0
    for cp in checkpoints:
        B.run_train_segment(net.w_ih2d, net.w_ho2d, feats, targets, cp - prev, lr, g.sequential())
        prev = cp
        out[f"w_ih_{cp}"] = net.w_ih.copy()
        out[f"w_ho_{cp}"] = net.w_ho.copy()
        out[f"train_counts_{cp}"] = np.array(Kr.eval_counts(net.w_ih2d, net.w_ho2d, feats, pair.train.labels), np.int64)
        out[f"test_counts_{cp}"] = np.array(Kr.eval_counts(net.w_ih2d, net.w_ho2d, pair.test.matrix(), pair.test.labels), np.int64)
    # the parallel engine must agree byte-for-byte; record it too
    par = g.init_weights(cfg)
    B.run_train_segment(par.w_ih2d, par.w_ho2d, feats, targets, checkpoints[-1], lr, g.parallel(2))
    assert par.w_ih.tobytes() == net.w_ih.tobytes() and par.w_ho.tobytes() == net.w_ho.tobytes()
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: D={pair.train.columns} H={hidden} rows={pair.train.rows}/{pair.test.rows} cps={checkpoints}")


def trainer_case():
    pair = matrix_split(120, 33, 7)
    cfg = g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7)
    rep = g.train(TrainSpec(config=cfg, epochs=1000, backend=g.sequential()), pair)
    rows = [{"epoch": r.epoch, "train_accuracy": r.train_accuracy, "test_accuracy": r.test_accuracy,
             "train_confusion": r.train_confusion, "test_confusion": r.test_confusion} for r in rep.rows]
    (OUT / "trainer_paper_1000.json").write_text(json.dumps({
        "rows": rows, "w_ih_sha256": digest(rep.network.w_ih), "w_ho_sha256": digest(rep.network.w_ho),
        "diverged": rep.diverged}, indent=1))
    print("trainer_paper_1000: rows", [r["epoch"] for r in rows])


def generator_digests():
    cases = []
    for rows, cols, seed, signal in ((120, 33, 7, "planted-linear"), (1000, 33, 0, "planted-linear"),
                                     (257, 5, 3, "random"), (10_000, 33, 0, "random"),
                                     (5000, 1024, 1, "planted-linear")):
        d = g.synthetic_matrix(rows, cols, seed, signal)
        cases.append({"rows": rows, "columns": cols, "seed": seed, "signal": signal,
                      "features_sha256": digest(d.features), "labels_sha256": digest(d.labels)})
    inits = []
    for D, H, seed in ((33, 33, 7), (30, 17, 13), (33, 256, 0), (33, 512, 63), (1024, 1024, 0)):
        net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=seed))
        inits.append({"input_dim": D, "hidden_dim": H, "seed": seed,
                      "w_ih_sha256": digest(net.w_ih), "w_ho_sha256": digest(net.w_ho)})
    (OUT / "generators.json").write_text(json.dumps({"synthetic_matrix": cases, "init_weights": inits}, indent=1))
    print("generators: ok")


def small_backend_case():
    # test_backend.py:143-152 shape: 7-19-1 on 25 random rows, 40 epochs
    rng = np.random.default_rng(11)
    feats = rng.random((25, 7), dtype=np.float32)
    targets = (rng.random(25) < 0.5).astype(np.float32)
    cfg = g.NetworkConfig(input_dim=7, hidden_dim=19, seed=3)
    net = g.init_weights(cfg)
    w_ih0, w_ho0 = net.w_ih.copy(), net.w_ho.copy()
    B.run_train_segment(net.w_ih2d, net.w_ho2d, feats, targets, 40, 0.1, g.sequential())
    np.savez_compressed(OUT / "small_7_19_1.npz", x=feats, t=targets, w_ih0=w_ih0, w_ho0=w_ho0,
                        w_ih=net.w_ih, w_ho=net.w_ho, epochs=np.array([40]))
    print("small_7_19_1: ok")


def normalize_cases():
    """Reference normalize_fit / normalize_apply (dataset.py:369-398) on raw splits:
    the paper matrix split, a record-built cohort (mixed column ranges), and a
    hand-built case with a constant column, negative values and test rows
    outside the fitted range (clamp to [-0.5, 1.5])."""
    out = {}

    def record(name, pair):
        stats = g.normalize_fit(pair.train)
        out[f"{name}_train_raw"] = np.ascontiguousarray(pair.train.matrix())
        out[f"{name}_test_raw"] = np.ascontiguousarray(pair.test.matrix())
        out[f"{name}_col_min"] = stats.col_min.copy()
        out[f"{name}_col_max"] = stats.col_max.copy()
        out[f"{name}_train_norm"] = np.ascontiguousarray(g.normalize_apply(pair.train, stats).matrix())
        out[f"{name}_test_norm"] = np.ascontiguousarray(g.normalize_apply(pair.test, stats).matrix())

    record("paper", g.train_test_split(g.synthetic_matrix(120, 33, 7, "planted-linear"), 0.75, 7))
    record("cohort", g.train_test_split(g.build_dataset(g.synth_dataset(240, 3, "planted-linear"), "synthetic"),
                                        0.75, 3))
    rng = np.random.default_rng(21)
    rows, cols = 300, 37
    m = (rng.normal(0.0, 1.0, (rows, cols)) * rng.uniform(0.01, 300.0, cols)).astype(np.float32)
    m[:, 5] = 2.5  # constant column -> 0.0
    m[:, 9] = -m[:, 9]
    m[250:, 11] *= 40.0  # test rows far outside the fitted range -> clamped

    def ds(a):
        return g.Dataset(features=np.ascontiguousarray(a).reshape(-1), labels=np.zeros(a.shape[0], np.uint8),
                         rows=a.shape[0], columns=cols, subset_tag="synthetic",
                         row_ids=tuple(f"r{i}" for i in range(a.shape[0])))

    record("edge", g.SplitPair(train=ds(m[:250]), test=ds(m[250:]), seed=0, fraction=0.8))
    np.savez_compressed(OUT / "normalize_cases.npz", **out)
    print("normalize_cases: ok", sorted({k.split("_")[0] for k in out}))


def protocol_cases():
    """The paper protocol's long runs (cli.py:34-36: 100k epochs, lr 0.1): the
    reference's weights and confusion counts at 10k and 100k epochs for the
    paper 33-33-1 split and the two 30-30-1 cohorts (train_segment_seq)."""
    out = {}
    for name, pair, hidden, seed in (("paper", matrix_split(120, 33, 7), 33, 7),
                                     ("male", record_split(120, 7, "planted-linear", "male"), 30, 7),
                                     ("female", record_split(120, 7, "random", "female"), 30, 7)):
        cfg = g.NetworkConfig(input_dim=pair.train.columns, hidden_dim=hidden, seed=seed)
        net = g.init_weights(cfg)
        feats = pair.train.matrix()
        targets = pair.train.labels.astype(np.float32)
        out[f"{name}_train_x"] = np.ascontiguousarray(feats)
        out[f"{name}_train_y"] = pair.train.labels.copy()
        out[f"{name}_test_x"] = np.ascontiguousarray(pair.test.matrix())
        out[f"{name}_test_y"] = pair.test.labels.copy()
        out[f"{name}_meta"] = np.array([pair.train.columns, hidden, 1, seed], dtype=np.int64)
        prev = 0
        for cp in (10_000, 100_000):
            B.run_train_segment(net.w_ih2d, net.w_ho2d, feats, targets, cp - prev, 0.1, g.sequential())
            prev = cp
            out[f"{name}_w_ih_{cp}"] = net.w_ih.copy()
            out[f"{name}_w_ho_{cp}"] = net.w_ho.copy()
            out[f"{name}_train_counts_{cp}"] = np.array(
                Kr.eval_counts(net.w_ih2d, net.w_ho2d, feats, pair.train.labels), np.int64)
            out[f"{name}_test_counts_{cp}"] = np.array(
                Kr.eval_counts(net.w_ih2d, net.w_ho2d, pair.test.matrix(), pair.test.labels), np.int64)
        print(f"protocol {name}: 100k epochs, counts {out[f'{name}_train_counts_100000']} "
              f"{out[f'{name}_test_counts_100000']}")
    np.savez_compressed(OUT / "protocol_100k.npz", **out)


def acceptance_cases():
    """Acceptance criteria 4 and 5 (test_acceptance.py:80-115): ten seeds each of a
    planted-signal 61-row and a weak-signal 59-row record cohort (conftest.py:7-11
    make_record_split), trained by the reference's trainer for 100k epochs; the
    normalised splits, final weights, counts and accuracies per seed."""
    for crit, rows, signal in ((4, 61, "planted-linear"), (5, 59, "random")):
        out = {}
        finals = []
        for seed in range(10):
            records = g.synth_dataset(rows, seed, signal)
            pair = g.normalize_split(g.train_test_split(g.build_dataset(records, "synthetic"), 0.75, seed))
            cfg = g.NetworkConfig(input_dim=pair.train.columns, seed=seed, learning_rate=0.1)
            rep = g.train(TrainSpec(config=cfg, epochs=100_000, backend=g.sequential(), checkpoints=(100_000,)),
                          pair)
            row = rep.rows[-1]
            out[f"s{seed}_train_x"] = np.ascontiguousarray(pair.train.matrix())
            out[f"s{seed}_train_y"] = pair.train.labels.copy()
            out[f"s{seed}_test_x"] = np.ascontiguousarray(pair.test.matrix())
            out[f"s{seed}_test_y"] = pair.test.labels.copy()
            out[f"s{seed}_w_ih"] = rep.network.w_ih.copy()
            out[f"s{seed}_w_ho"] = rep.network.w_ho.copy()
            out[f"s{seed}_acc"] = np.array([row.train_accuracy, row.test_accuracy])
            out[f"s{seed}_train_counts"] = np.array([row.train_confusion[k] for k in ("tp", "tn", "fp", "fn")],
                                                    np.int64)
            out[f"s{seed}_test_counts"] = np.array([row.test_confusion[k] for k in ("tp", "tn", "fp", "fn")],
                                                   np.int64)
            finals.append((round(row.train_accuracy, 3), round(row.test_accuracy, 3)))
        np.savez_compressed(OUT / f"acceptance_c{crit}.npz", **out)
        print(f"criterion {crit}: {finals}")


def dropin_cases():
    """The reference trainer tests' splits and the reference's own results on them
    (test_trainer.py:50-121, test_acceptance.py:48-67): normalised features, labels,
    row ids and norm stats of each SplitPair, plus every checkpoint row and the final
    weights of g.train(spec, pair) with the sequential engine."""
    def spec_of(columns, epochs, checkpoints, seed):
        return TrainSpec(config=g.NetworkConfig(input_dim=columns, seed=seed), epochs=epochs,
                         backend=g.sequential(), checkpoints=checkpoints)

    runs = {
        "m30_6_2": (matrix_split(30, 6, 2), [(40, (1, 10, 40), 1)]),
        "m24_5_4": (matrix_split(24, 5, 4), [(32, (1, 2, 4, 8, 16, 32), 2), (32, (32,), 2)]),
        "r40_6": (record_split(40, 6, "planted-linear"), [(100, (1, 10, 100), 0)]),
        "m20_4_0": (matrix_split(20, 4, 0), []),
        "m20_4_1": (matrix_split(20, 4, 1), []),
        "r30_1": (record_split(30, 1, "planted-linear"), [(5, (5,), 0)]),
        "m26_5_9": (matrix_split(26, 5, 9), [(60, (60,), 3)]),
        "m24_4_5": (matrix_split(24, 4, 5), [(30, (1, 10, 30), 1), (20, (1, 20), 2)]),
        "r30_3": (record_split(30, 3, "planted-linear"), [(10, (10,), 0)]),
        "m24_4_7": (matrix_split(24, 4, 7), [(15, (5, 15), 4)]),
    }
    out = {}
    for name, (pair, specs) in runs.items():
        for part in ("train", "test"):
            d = getattr(pair, part)
            out[f"{name}_{part}_x"] = np.ascontiguousarray(d.matrix())
            out[f"{name}_{part}_y"] = d.labels.copy()
            out[f"{name}_{part}_ids"] = np.array([str(r) for r in d.row_ids])
            out[f"{name}_{part}_tag"] = np.array([d.subset_tag])
        out[f"{name}_col_min"] = pair.train.norm_stats.col_min.copy()
        out[f"{name}_col_max"] = pair.train.norm_stats.col_max.copy()
        out[f"{name}_split"] = np.array([pair.seed, pair.fraction])
        for k, (epochs, cps, seed) in enumerate(specs):
            rep = g.train(spec_of(pair.train.columns, epochs, cps, seed), pair)
            out[f"{name}_run{k}_spec"] = np.array([epochs, seed, *cps], np.int64)
            out[f"{name}_run{k}_rows"] = np.array(
                [[r.epoch, r.train_accuracy, r.test_accuracy,
                  *[r.train_confusion[c] for c in ("tp", "tn", "fp", "fn")],
                  *[r.test_confusion[c] for c in ("tp", "tn", "fp", "fn")]] for r in rep.rows], np.float64)
            out[f"{name}_run{k}_w_ih"] = rep.network.w_ih.copy()
            out[f"{name}_run{k}_w_ho"] = rep.network.w_ho.copy()
    np.savez_compressed(OUT / "dropin_splits.npz", **out)
    print("dropin_splits:", ", ".join(runs))


CASES = {
    "online": lambda: (
        online_case("paper_33_33_1", matrix_split(120, 33, 7), 33, 7, [1, 10, 100, 1000]),
        online_case("cohort_male_30_30_1", record_split(120, 7, "planted-linear", "male"), 30, 7, [1, 10, 100, 1000]),
        online_case("cohort_female_30_30_1", record_split(120, 7, "random", "female"), 30, 7, [1, 10, 100, 1000]),
        online_case("wide_33_256_1", matrix_split(200, 33, 3), 256, 5, [1, 10, 50])),
    "small": small_backend_case,
    "trainer": trainer_case,
    "generators": generator_digests,
    "normalize": normalize_cases,
    "protocol": protocol_cases,
    "acceptance": acceptance_cases,
    "dropin": dropin_cases,
}

if __name__ == "__main__":
    # no arguments: every fixture; otherwise only the named groups
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
