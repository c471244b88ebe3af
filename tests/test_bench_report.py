"""Bench harness with device cells (paper_1908_07847_b200/bench_report.py), modelled
on the reference's tests/test_bench.py: spec validation, report structure,
re-initialisation from the seed, failure isolation, the speedup table and the
v1 report format. CPU engines are injected as baselines (here: the oracle's C
restatement of the reference engines)."""

import json

import numpy as np
import pytest

import paper_1908_07847_b200 as g
from oracle import oracle as O
from paper_1908_07847_b200 import bench_report as B


def seq_engine(w1, w2, x, t, epochs, lr):
    O.train_online_seq(w1, w2, x, t, epochs, lr)


def par_engine(w1, w2, x, t, epochs, lr):
    O.train_online_par(w1, w2, x, t, epochs, lr, workers=2)


def tiny_spec(**kw):
    d = dict(config=g.NetworkConfig(input_dim=6, hidden_dim=8, seed=0), epochs_grid=(2, 4), rows=30, columns=6,
             repetitions=3, backends=(), baselines=(("sequential", seq_engine), ("parallel", par_engine)))
    d.update(kw)
    return B.BenchSpec(**d)


class TestSpec:
    def test_rejects_bad_repetitions(self):
        with pytest.raises(g.ValidationError):
            tiny_spec(repetitions=0)

    def test_rejects_unordered_grid(self):
        with pytest.raises(g.ValidationError):
            tiny_spec(epochs_grid=(4, 2))

    def test_requires_some_data(self):
        with pytest.raises(g.ValidationError):
            B.BenchSpec(config=g.NetworkConfig(input_dim=4), epochs_grid=(1,))

    def test_rejects_duplicate_cell_names(self):
        with pytest.raises(g.ValidationError):
            tiny_spec(baselines=(("sequential", seq_engine), ("sequential", par_engine)))

    def test_rejects_bad_mode(self):
        with pytest.raises(g.ValidationError):
            tiny_spec(mode="minibatch")


class TestRunCPU:
    def test_structure_and_speedups(self):
        rep = B.run_bench(tiny_spec())
        assert len(rep.cells) == 4 and len(rep.speedups) == 2
        for c in rep.cells:
            assert not c.failed and 0 < c.min_seconds <= c.median_seconds <= c.max_seconds
            assert c.sample_epochs_per_s == pytest.approx(30 * c.epochs / c.median_seconds)
        s = rep.speedups[0]
        assert s.speedup * s.parallel_seconds == pytest.approx(s.sequential_seconds, rel=1e-12)
        assert rep.environment["repetitions"] == 3 and "workers" in rep.environment
        assert rep.gpu_reference["speedup"] == 50.0

    def test_cells_reinitialize_from_seed(self, monkeypatch):
        calls = {"n": 0}
        real = B.init_weights

        def counting(cfg):
            calls["n"] += 1
            return real(cfg)

        monkeypatch.setattr(B, "init_weights", counting)
        B.run_bench(tiny_spec(epochs_grid=(2,), repetitions=2))
        assert calls["n"] == 2 * (1 + 2)  # per cell source: warm-up + repetitions

    def test_failed_engine_marks_cells_and_continues(self):
        def broken(*a):
            raise RuntimeError("injected failure")

        rep = B.run_bench(tiny_spec(epochs_grid=(2,), baselines=(("sequential", seq_engine), ("parallel", broken))))
        assert all(not c.failed for c in rep.cells if c.backend == "sequential")
        assert all(c.failed and "injected" in c.error for c in rep.cells if c.backend == "parallel")
        assert rep.speedups == ()
        with pytest.warns(UserWarning):
            text = B.emit_speedup_table(rep)
        assert text.strip().splitlines() == [",".join(B.SPEEDUP_HEADER)]

    def test_table_and_v1_format(self, tmp_path):
        rep = B.run_bench(tiny_spec(epochs_grid=(1, 2, 3), repetitions=1, fp32_peak_tflops=72.5))
        lines = B.emit_speedup_table(rep).strip().splitlines()
        assert lines[0] == ",".join(B.SPEEDUP_HEADER) and len(lines) == 4
        cols = lines[1].split(",")
        assert float(cols[3]) == pytest.approx(float(cols[1]) / float(cols[2]), rel=1e-12)
        path = tmp_path / "r.json"
        B.save_bench_report(rep, path)
        doc = json.loads(path.read_text())
        assert doc["format"] == "glycemlp-bench-report-v1"
        v1_cell = {"epochs", "backend", "workers", "median_seconds", "min_seconds", "max_seconds", "repetitions",
                   "failed", "error"}
        assert v1_cell <= set(doc["cells"][0])
        assert {"environment", "gpu_reference", "cells", "speedups"} <= set(doc)
        assert doc["workload"]["flops_per_sample_epoch"] == B.f_train(6, 8)
        assert doc["cells"][0]["frac_fp32_peak"] > 0

    def test_mismatched_config_rejected(self):
        with pytest.raises(g.ValidationError):
            B.run_bench(tiny_spec(config=g.NetworkConfig(input_dim=9)))


@pytest.mark.gpu
def test_device_cells_and_device_speedups(gpu):
    rep = B.run_bench(tiny_spec(rows=90, columns=33, config=g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7),
                                epochs_grid=(10, 100), repetitions=2, backends=(g.cuda(), g.cuda(numerics="ref64")),
                                baselines=(("sequential", seq_engine),), fp32_peak_tflops=72.5))
    names = {c.backend for c in rep.cells}
    assert names == {"sequential", "cuda-fp32", "cuda-ref64"}
    assert not any(c.failed for c in rep.cells), [c.error for c in rep.cells if c.failed]
    assert len(rep.device_speedups) == 4
    assert all(r.speedup > 0 for r in rep.device_speedups)
    lines = B.emit_device_speedup_table(rep).strip().splitlines()
    assert lines[0] == ",".join(B.DEVICE_SPEEDUP_HEADER) and len(lines) == 5


@pytest.mark.gpu
def test_batch_mode_device_cells(gpu):
    rep = B.run_bench(tiny_spec(rows=4096, columns=33, config=g.NetworkConfig(input_dim=33, hidden_dim=256, seed=0),
                                epochs_grid=(5,), repetitions=2, backends=(g.cuda(),), baselines=(), mode="batch"))
    (c,) = rep.cells
    assert c.backend == "cuda-fp32" and not c.failed and c.sample_epochs_per_s > 0


@pytest.mark.gpu
def test_bench_front_end_artifacts(gpu, tmp_path):
    """The reference's `glycemlp bench` command (cli.py:147-155, 266-288) as
    `python -m paper_1908_07847_b200.bench_report`: same arguments, same artifacts."""
    import csv

    rc = B.bench_main(["--rows", "300", "--columns", "33", "--hidden-dim", "16", "--epochs-grid", "2,4",
                       "--repetitions", "1", "--workers", "2", "--device", "--out", str(tmp_path)])
    assert rc == 0
    doc = json.loads((tmp_path / "bench_report.json").read_text())
    assert doc["format"] == "glycemlp-bench-report-v1"
    assert {c["backend"] for c in doc["cells"]} == {"sequential", "parallel", "cuda-fp32"}
    assert [s["epochs"] for s in doc["speedups"]] == [2, 4]
    rows = list(csv.reader((tmp_path / "speedup.csv").open()))
    assert rows[0] == list(B.SPEEDUP_HEADER) and len(rows) == 3
    assert (tmp_path / "device_speedup.csv").exists()
