"""Device evaluation, sweeps and the trainer mirror vs the reference / oracle."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, load_case, make_split, rel_err

import paper_1908_07847_b200 as g
from paper_1908_07847_b200.trainer import TrainSpec, report_to_dict, strip_timing
from oracle import oracle as O

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ eval
@pytest.mark.parametrize("N,D,H", [(1, 3, 2), (129, 33, 33), (100_000, 33, 256), (5000, 1024, 64), (77, 30, 1),
                                   # row split over 8 lanes (H > 112): exactly 8 blocks with a partial one, uneven
                                   # blocks per lane, 63 blocks, ragged row counts
                                   (2003, 33, 120), (3001, 17, 513), (1501, 33, 1000), (17, 33, 128)])
def test_eval_ref64_exact_vs_oracle(gpu, N, D, H):
    x, l = g.synthetic_arrays(max(N, 2), D, 3, "planted-linear")
    x, l = x[:N], l[:N]
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=5))
    counts, loss = g.eval_counts_loss(net.w_ih2d, net.w_ho2d, x, l)
    want, wloss = O.eval_counts(net.w_ih2d, net.w_ho2d, x, l)
    assert counts == want
    assert abs(loss - wloss) <= 1e-12 * max(1.0, wloss)


def test_eval_fp32_fast_path_within_tolerance(gpu):
    x, l = g.synthetic_arrays(300_000, 33, 8, "planted-linear")
    net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=2))
    counts, loss = g.eval_counts_loss(net.w_ih2d, net.w_ho2d, x, l, g.cuda(numerics="fp32"))
    want, wloss = O.eval_counts(net.w_ih2d, net.w_ho2d, x, l)
    assert sum(counts) == 300_000
    assert np.abs(np.array(counts) - np.array(want)).sum() <= 4
    assert abs(loss - wloss) <= 1e-4 * wloss


def test_eval_multi_output_argmax(gpu):
    import ctypes

    import paper_1908_07847_b200._lib as L

    rng = np.random.default_rng(1)
    x = rng.random((1000, 12), dtype=np.float32)
    y = rng.integers(0, 16, 1000).astype(np.uint8)
    w1 = rng.uniform(-0.5, 0.5, (40, 13)).astype(np.float32)
    w2 = rng.uniform(-0.5, 0.5, (16, 41)).astype(np.float32)
    counts = np.zeros(4, np.int64)
    loss = np.zeros(1)
    lib = L.load()
    L.check(lib.glx_eval_counts(L.ptr(w1), L.ptr(w2), L.ptr(x), L.ptr(y), 1000, 12, 40, 16, 1, L.ptr(counts),
                                L.ptr(loss), 0, 0))
    want, wloss = O.eval_counts(w1, w2, x, y)
    assert tuple(counts) == want and abs(loss[0] - wloss) <= 1e-12 * wloss


def test_eval_empty_dataset_rejected(gpu):
    c = load_case("paper_33_33_1")
    split = make_split(c["train_x"], c["train_y"], c["test_x"][:0], c["test_y"][:0])
    net = g.init_weights(g.NetworkConfig(input_dim=33, seed=7))
    with pytest.raises(ValueError):
        g.evaluate(net, split.test)


# ----------------------------------------------------------------- sweep
def test_sweep_vs_oracle_per_network(gpu):
    c = load_case("paper_33_33_1")
    hs, ss = g.sweep_grid([8, 24, 33, 40, 96, 200, 512], [0, 1, 2])
    for numerics, tol in (("fp32", 1e-4), ("ref64", 1e-9)):
        spec = g.SweepSpec(input_dim=33, hidden_dims=hs, seeds=ss, epochs=30, numerics=numerics)
        nets = g.train_sweep(spec, c["train_x"], c["train_y"].astype(np.float32))
        for cfg, net in zip(spec.configs(), nets):
            ref = g.init_weights(cfg)
            O.train_online_seq(ref.w_ih2d, ref.w_ho2d, c["train_x"], c["train_y"].astype(np.float32), 30, 0.1)
            err = max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho))
            assert err <= tol, f"{numerics} H={cfg.hidden_dim} seed={cfg.seed}: {err:.3e}"


def test_sweep_of_one_warp_networks_vs_oracle(gpu):
    """Every network fits one warp (H <= 64 at 2 units per thread): the launch takes the
    one-warp instantiation with no shared-memory exchange."""
    c = load_case("paper_33_33_1")
    t = c["train_y"].astype(np.float32)
    hs, ss = g.sweep_grid([1, 7, 33, 64], [0, 5])
    spec = g.SweepSpec(input_dim=33, hidden_dims=hs, seeds=ss, epochs=25)
    nets = g.train_sweep(spec, c["train_x"], t)
    for cfg, net in zip(spec.configs(), nets):
        ref = g.init_weights(cfg)
        O.train_online_seq(ref.w_ih2d, ref.w_ho2d, c["train_x"], t, 25, 0.1)
        assert max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho)) <= 1e-4, cfg


def test_sweep_full_grid_runs_and_matches_sample(gpu):
    # config 3 shape: 64 widths x 64 seeds = 4096 networks; oracle-check a stratified sample
    c = load_case("paper_33_33_1")
    t = c["train_y"].astype(np.float32)
    hs, ss = g.sweep_grid(range(8, 513, 8), range(64))
    spec = g.SweepSpec(input_dim=33, hidden_dims=hs, seeds=ss, epochs=5)
    nets = g.train_sweep(spec, c["train_x"], t)
    assert len(nets) == 4096 and all(n.weights_finite() for n in nets)
    cfgs = spec.configs()
    for i in range(0, 4096, 509):
        ref = g.init_weights(cfgs[i])
        O.train_online_seq(ref.w_ih2d, ref.w_ho2d, c["train_x"], t, 5, 0.1)
        assert max(rel_err(nets[i].w_ih, ref.w_ih), rel_err(nets[i].w_ho, ref.w_ho)) <= 1e-4


# --------------------------------------------------------------- trainer
def test_trainer_matches_reference_report(gpu):
    doc = json.loads((GOLDEN / "trainer_paper_1000.json").read_text())
    c = load_case("paper_33_33_1")
    split = make_split(c["train_x"], c["train_y"], c["test_x"], c["test_y"])
    for kind in (g.sequential(), g.cuda()):
        rep = g.train(TrainSpec(config=g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7), epochs=1000,
                                backend=kind), split)
        assert [r.epoch for r in rep.rows] == [r["epoch"] for r in doc["rows"]]
        for mine, ref in zip(rep.rows, doc["rows"]):
            assert mine.train_confusion == ref["train_confusion"]
            assert mine.test_confusion == ref["test_confusion"]
            assert mine.train_accuracy == ref["train_accuracy"] and mine.test_accuracy == ref["test_accuracy"]
        assert rel_err(rep.network.w_ih, c["w_ih_1000"]) <= (1e-9 if kind.numerics == "ref64" else 1e-4)


def test_checkpoint_evaluation_is_side_effect_free(gpu):
    c = load_case("paper_33_33_1")
    split = make_split(c["train_x"], c["train_y"], c["test_x"], c["test_y"])
    cfg = g.NetworkConfig(input_dim=33, hidden_dim=33, seed=2)
    for kind in (g.sequential(), g.cuda()):
        dense = g.train(TrainSpec(config=cfg, epochs=32, backend=kind, checkpoints=(1, 2, 4, 8, 16, 32)), split)
        sparse = g.train(TrainSpec(config=cfg, epochs=32, backend=kind, checkpoints=(32,)), split)
        assert dense.network.w_ih.tobytes() == sparse.network.w_ih.tobytes()
        assert dense.network.w_ho.tobytes() == sparse.network.w_ho.tobytes()
        a = strip_timing(report_to_dict(g.train(TrainSpec(config=cfg, epochs=15, backend=kind), split)))
        b = strip_timing(report_to_dict(g.train(TrainSpec(config=cfg, epochs=15, backend=kind), split)))
        assert json.dumps(a) == json.dumps(b)


def test_divergence_reports_last_good(gpu):
    c = load_case("paper_33_33_1")
    split = make_split(c["train_x"], c["train_y"], c["test_x"], c["test_y"])
    cfg = g.NetworkConfig(input_dim=33, seed=0)
    poisoned = g.init_weights(cfg)
    poisoned.w_ih[0] = np.float32(np.inf)
    rep = g.train(TrainSpec(config=cfg, epochs=10, checkpoints=(1, 10)), split, initial_net=poisoned)
    assert rep.diverged and rep.rows == () and rep.metadata["diverged"] is True
    assert rep.network.w_ih.tobytes() == poisoned.w_ih.tobytes()


def test_batch_mode_trainer(gpu):
    c = load_case("wide_33_256_1")
    split = make_split(c["train_x"], c["train_y"], c["test_x"], c["test_y"])
    cfg = g.NetworkConfig(input_dim=33, hidden_dim=256, seed=5, learning_rate=0.5)
    rep = g.train(TrainSpec(config=cfg, epochs=20, mode="batch"), split)
    ref = g.init_weights(cfg)
    O.train_batch(ref.w_ih2d, ref.w_ho2d, c["train_x"], c["train_y"].astype(np.float32), 20, 0.5,
                  c["train_x"].shape[0])
    assert rel_err(rep.network.w_ih, ref.w_ih) <= 1e-5
    assert rep.metadata["mode"] == "batch"


@pytest.mark.parametrize("mode", ["online", "batch"])
def test_fused_checkpoint_equals_segment_plus_eval(gpu, mode):
    """backend.run_train_segment_eval == the unfused sequence:
    segment, host finiteness test, eval_counts on train and on test."""
    from paper_1908_07847_b200.backend import run_train_segment_eval

    c = load_case("paper_33_33_1")
    x, y, vx, vy = c["train_x"], c["train_y"], c["test_x"], c["test_y"]
    t = y.astype(np.float32)
    kind = g.sequential() if mode == "online" else g.cuda()
    a = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7))
    b = a.copy()
    step = g.run_train_segment if mode == "online" else g.run_train_segment_batch
    for n in (1, 9, 90):
        r = run_train_segment_eval(a.w_ih2d, a.w_ho2d, x, t, y, vx, vy, n, 0.5, kind, mode=mode)
        step(b.w_ih2d, b.w_ho2d, x, t, n, 0.5, kind)
        assert a.w_ih.tobytes() == b.w_ih.tobytes() and a.w_ho.tobytes() == b.w_ho.tobytes()
        assert r.finite and r.train_seconds >= 0
        assert r.train_counts == g.eval_counts(b.w_ih2d, b.w_ho2d, x, y)
        assert r.test_counts == g.eval_counts(b.w_ih2d, b.w_ho2d, vx, vy)
        assert sum(r.train_counts) == x.shape[0] and sum(r.test_counts) == vx.shape[0]
        (_, l_tr), (_, l_te) = O.eval_counts(b.w_ih2d, b.w_ho2d, x, y), O.eval_counts(b.w_ih2d, b.w_ho2d, vx, vy)
        assert r.train_loss == pytest.approx(l_tr, rel=1e-12) and r.test_loss == pytest.approx(l_te, rel=1e-12)


def test_fused_checkpoint_batch_on_the_tcgen05_kernel(gpu):
    """33 -> 256 -> 1 (the tcgen05 epoch kernel): fused checkpoint segments of 1, 9 and
    90 epochs give the same bytes as the unfused segment loop, and both track the
    oracle batch restatement."""
    import paper_1908_07847_b200._lib as L
    from paper_1908_07847_b200.backend import run_train_segment_eval

    c = load_case("paper_33_33_1")
    x, y, vx, vy = c["train_x"], c["train_y"], c["test_x"], c["test_y"]
    assert L.load().glx_batch_kernel_kind(x.shape[0], 33, 256) == 2
    t = y.astype(np.float32)
    cfg = g.NetworkConfig(input_dim=33, hidden_dim=256, seed=11)
    a, b, ref = g.init_weights(cfg), g.init_weights(cfg), g.init_weights(cfg)
    for n in (1, 9, 90):
        r = run_train_segment_eval(a.w_ih2d, a.w_ho2d, x, t, y, vx, vy, n, 0.5, g.cuda(), mode="batch")
        g.run_train_segment_batch(b.w_ih2d, b.w_ho2d, x, t, n, 0.5, g.cuda())
        assert a.w_ih.tobytes() == b.w_ih.tobytes() and a.w_ho.tobytes() == b.w_ho.tobytes()
        assert r.finite and r.train_counts == g.eval_counts(b.w_ih2d, b.w_ho2d, x, y)
    O.train_batch(ref.w_ih2d, ref.w_ho2d, x, t, 100, 0.5, x.shape[0])
    assert max(rel_err(a.w_ih, ref.w_ih), rel_err(a.w_ho, ref.w_ho)) <= 1e-5


def test_fused_checkpoint_flags_nonfinite(gpu):
    from paper_1908_07847_b200.backend import run_train_segment_eval

    c = load_case("paper_33_33_1")
    x, y = c["train_x"], c["train_y"]
    net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7))
    net.w_ih[5] = np.inf
    r = run_train_segment_eval(net.w_ih2d, net.w_ho2d, x, y.astype(np.float32), y, c["test_x"], c["test_y"], 1, 0.1,
                               g.cuda(), mode="batch")
    assert not r.finite and not net.weights_finite()
