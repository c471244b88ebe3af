"""Full-batch GD kernel (configs 2/4) vs the oracle batch restatement, plus
size-independent properties at the full 1M-row benchmark size."""

import numpy as np
import pytest

from conftest import rel_err

import paper_1908_07847_b200 as g
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _case(N, D, H, seed, signal="planted-linear"):
    x, l = g.synthetic_arrays(N, D, seed, signal)
    return x, l, l.astype(np.float32), g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=seed))


@pytest.mark.parametrize("N,D,H", [
    (2, 33, 33), (65, 33, 33), (1000, 33, 33), (1000, 33, 256), (777, 33, 512), (500, 33, 19),
    (300, 7, 5), (301, 15, 16), (250, 30, 30), (4099, 33, 64), (130, 1, 1), (513, 32, 36),
    # tcgen05 kernel shapes (H = 128 / 256): exact tile, one row past a tile, D < 33
    (2, 33, 256), (63, 33, 128), (64, 33, 128), (65, 33, 256), (129, 33, 128), (1000, 33, 128), (3001, 7, 256),
    (2000, 16, 128),
])
def test_batch_vs_oracle(gpu, N, D, H):
    x, l, t, net0 = _case(N, D, H, seed=N % 97)
    epochs, lr = 6, 0.5
    ref = net0.copy()
    O.train_batch(ref.w_ih2d, ref.w_ho2d, x, t, epochs, lr, N)
    net = net0.copy()
    stats = np.zeros((epochs, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, epochs, lr, g.cuda(), stats)
    err = max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho))
    assert err <= 1e-5, f"N={N} D={D} H={H}: {err:.3e}"
    # epoch-0 statistics are the evaluation of the initial weights
    (tp, tn, fp, fn), loss = O.eval_counts(net0.w_ih2d, net0.w_ho2d, x, l)
    assert stats[0, 1:].sum() == N
    assert abs(stats[0, 0] - loss) <= 1e-4 * max(1.0, loss)
    assert np.abs(stats[0, 1:] - np.array([tp, tn, fp, fn])).sum() <= 2  # |o-0.5| < 1e-6 rows may flip


@pytest.mark.parametrize("N,H,force", [
    (3001, 160, False), (2000, 96, False), (5000, 200, False), (4099, 250, False),
    (1000, 33, False), (129, 64, False), (700, 1, True), (50_000, 40, False),
])
def test_tcgen05_kernel_any_width_vs_oracle(gpu, N, H, force, monkeypatch):
    """The tcgen05 epoch kernel for widths that are not a multiple of 128 (padded
    units: zero weights, idle epilogue warps) -- the default for 24 <= H <= 256,
    forced with GLX_BATCH_KERNEL=tc below that; H <= 128 runs two epilogue groups."""
    import paper_1908_07847_b200._lib as L

    if force:
        monkeypatch.setenv("GLX_BATCH_KERNEL", "tc")
    assert L.load().glx_batch_kernel_kind(N, 33, H) == 2
    x, l, t, net0 = _case(N, 33, H, seed=N % 89)
    ref, net = net0.copy(), net0.copy()
    O.train_batch(ref.w_ih2d, ref.w_ho2d, x, t, 6, 0.5, N)
    stats = np.zeros((6, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 6, 0.5, g.cuda(), stats)
    err = max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho))
    assert err <= 1e-5, f"N={N} H={H}: {err:.3e}"
    assert (stats[:, 1:].sum(axis=1) == N).all()


@pytest.mark.parametrize("N,D,H", [(500, 40, 64), (777, 60, 30), (300, 100, 12), (129, 127, 3)])
def test_batch_wide_inputs_vs_oracle(gpu, N, D, H):
    """D > 33 (kernels.py:264-295 takes any input width): the FP32 batch kernel with
    48-, 64- and 128-float weight rows."""
    x, l, t, net0 = _case(N, D, H, seed=D)
    ref, net = net0.copy(), net0.copy()
    O.train_batch(ref.w_ih2d, ref.w_ho2d, x, t, 5, 0.5, N)
    stats = np.zeros((5, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 5, 0.5, g.cuda(), stats)
    assert max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho)) <= 1e-5
    (tp, tn, fp, fn), loss = O.eval_counts(net0.w_ih2d, net0.w_ho2d, x, l)
    assert abs(stats[0, 0] - loss) <= 1e-4 * max(1.0, loss)


@pytest.mark.parametrize("N,H", [(200_000, 33), (150_001, 64), (131_072, 12), (300_000, 48)])
def test_rows_on_lanes_kernel_vs_oracle(gpu, N, H):
    """The narrow-layer kernel (rows on the TMEM lanes, kind 3; FAST precision from 2^17
    rows) against the f64 oracle: weights within 1e-5 after 4 epochs, epoch-0
    statistics equal to the oracle evaluation."""
    import paper_1908_07847_b200._lib as L

    assert L.load().glx_batch_kernel_kind(N, 33, H) == 3
    x, l, t, net0 = _case(N, 33, H, seed=H)
    ref, net = net0.copy(), net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, 4, 0.1)
    stats = np.zeros((4, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 4, 0.1, g.cuda(), stats)
    assert max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho)) <= 1e-5
    (tp, tn, fp, fn), loss = O.eval_counts(net0.w_ih2d, net0.w_ho2d, x, l)
    assert np.abs(stats[0, 1:] - np.array([tp, tn, fp, fn])).sum() <= 4
    assert abs(stats[0, 0] - loss) <= 1e-5 * loss


def test_tcgen05_fast_precision_padded_width(gpu, monkeypatch):
    """The large-N (FAST) precision with a padded width, 150k rows x 33 -> 192 -> 1."""
    monkeypatch.setenv("GLX_BTC_PREC", "fast")
    x, l, t, net0 = _case(150_000, 33, 192, seed=6)
    ref, net = net0.copy(), net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, 4, 0.1)
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 4, 0.1, g.cuda())
    assert max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho)) <= 1e-5


def test_tcgen05_kernel_selected_for_headline_shapes(gpu):
    """configs 2 and 4 (33 -> 33 / 128 / 256 -> 1) run the tcgen05 epoch kernel, as does any
    width 24..256; narrower and wider layers run the FP32 CUDA-core kernels
    (glx_batch_kernel_kind)."""
    import paper_1908_07847_b200._lib as L

    lib = L.load()
    assert lib.glx_batch_kernel_kind(1 << 20, 33, 256) == 2
    assert lib.glx_batch_kernel_kind(1 << 26, 33, 256) == 2
    assert lib.glx_batch_kernel_kind(1000, 33, 128) == 2
    assert lib.glx_batch_kernel_kind(1000, 33, 192) == 2 and lib.glx_batch_kernel_kind(1000, 33, 97) == 2
    assert lib.glx_batch_kernel_kind(1000, 33, 33) == 2 and lib.glx_batch_kernel_kind(1000, 33, 64) == 2
    # from 2^17 rows, narrow layers run the rows-on-lanes kernel (kind 3)
    assert lib.glx_batch_kernel_kind(1 << 20, 33, 33) == 3 and lib.glx_batch_kernel_kind(1 << 20, 33, 64) == 3
    assert lib.glx_batch_kernel_kind(1 << 20, 33, 12) == 3 and lib.glx_batch_kernel_kind(1 << 20, 33, 65) == 2
    assert lib.glx_batch_kernel_kind(1000, 33, 16) in (0, 1)
    assert lib.glx_batch_kernel_kind(1000, 33, 512) in (0, 1)
    assert lib.glx_batch_kernel_kind(1000, 40, 256) in (0, 1)  # D > 33: FP32 kernels
    assert lib.glx_batch_kernel_kind(1000, 128, 8) == 4 and lib.glx_batch_kernel_kind(1000, 33, 513) == 4  # any shape
    assert lib.glx_batch_kernel_kind(0, 33, 8) == -1


def test_tcgen05_kernel_matches_fp32_kernel(gpu, tmp_path):
    """The same 100k-row, 33-256-1 problem through the tcgen05 3xTF32 kernel (this
    process) and the FP32 three-role kernel (a subprocess with GLX_BATCH_KERNEL=3):
    weights agree within the parity tolerance and the epoch statistics' counts match."""
    import os
    import subprocess
    import sys

    x, l, t, net0 = _case(100_003, 33, 256, seed=6)
    np.savez(tmp_path / "case.npz", x=x, t=t, w1=net0.w_ih2d, w2=net0.w_ho2d)
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]); import paper_1908_07847_b200 as g\n"
        "d = np.load(sys.argv[2]); w1, w2 = d['w1'].copy(), d['w2'].copy(); st = np.zeros((5, 5))\n"
        "g.run_train_segment_batch(w1, w2, d['x'], d['t'], 5, 0.5, g.cuda(), st)\n"
        "np.savez(sys.argv[3], w1=w1, w2=w2, st=st)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GLX_BATCH_KERNEL="3")
    subprocess.run([sys.executable, "-c", code, root, str(tmp_path / "case.npz"), str(tmp_path / "fp32.npz")],
                   check=True, env=env, timeout=600)
    other = np.load(tmp_path / "fp32.npz")
    net = net0.copy()
    st = np.zeros((5, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 5, 0.5, g.cuda(), st)
    assert rel_err(net.w_ih2d, other["w1"]) <= 1e-5 and rel_err(net.w_ho2d, other["w2"]) <= 1e-5
    assert (st[:, 1:].sum(axis=1) == x.shape[0]).all()
    assert np.abs(st[:, 1:] - other["st"][:, 1:]).sum(axis=1).max() <= 4  # |o - 0.5| ~ 0 rows may flip
    assert np.allclose(st[:, 0], other["st"][:, 0], rtol=1e-5)


def test_batch_is_deterministic(gpu):
    x, l, t, net0 = _case(100_003, 33, 256, seed=4)
    a, b = net0.copy(), net0.copy()
    g.run_train_segment_batch(a.w_ih2d, a.w_ho2d, x, t, 3, 0.1, g.cuda())
    g.run_train_segment_batch(b.w_ih2d, b.w_ho2d, x, t, 3, 0.1, g.cuda())
    assert a.w_ih.tobytes() == b.w_ih.tobytes() and a.w_ho.tobytes() == b.w_ho.tobytes()


@pytest.mark.parametrize("H", [33, 256])
def test_full_size_1M_properties(gpu, H):
    # config 2 at full size: 1M rows; the oracle checks a bounded 2-epoch run on the same data
    x, l, t, net0 = _case(1_000_000, 33, H, seed=0)
    net = net0.copy()
    stats = np.zeros((2, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 2, 0.1, g.cuda(), stats)
    assert net.weights_finite()
    assert (stats[:, 1:].sum(axis=1) == 1_000_000).all()
    ref = net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, 2, 0.1)
    assert max(rel_err(net.w_ih, ref.w_ih), rel_err(net.w_ho, ref.w_ho)) <= 1e-5


def test_loss_decreases_over_epochs(gpu):
    x, l, t, net0 = _case(200_000, 33, 33, seed=1)
    stats = np.zeros((40, 5))
    net = net0.copy()
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 40, 2.0, g.cuda(), stats)
    assert stats[-1, 0] < stats[0, 0]


def test_dp_split_equals_fused_single_gpu(gpu):
    """glx_batch_grad + glx_batch_apply over 2 row shards (summed on the host, as the
    all-reduce would) == the fused single-GPU epoch loop."""
    import torch

    from paper_1908_07847_b200 import dp

    x, l, t, net0 = _case(20_001, 33, 64, seed=9)
    fused = net0.copy()
    g.run_train_segment_batch(fused.w_ih2d, fused.w_ho2d, x, t, 4, 0.5, g.cuda())
    engines = []
    for r in range(2):
        r0, r1 = dp.shard_bounds(x.shape[0], 2, r)
        engines.append(dp.DeviceEngine(x[r0:r1], t[r0:r1], net0.w_ih, net0.w_ho))
    for _ in range(4):
        total = engines[0].grad_sum().clone() + engines[1].grad_sum().clone()
        for e in engines:
            e.apply(total, 0.5 / x.shape[0])
    torch.cuda.synchronize()
    w1, w2 = engines[0].weights()
    assert rel_err(w1, fused.w_ih) <= 1e-6 and rel_err(w2, fused.w_ho) <= 1e-6
    v1, v2 = engines[1].weights()
    assert w1.tobytes() == v1.tobytes() and w2.tobytes() == v2.tobytes()


def test_dp_path_over_library_nccl_one_rank(gpu):
    """The library-owned NCCL data plane (glx_dp_init, glx_dp_train_batch: epoch kernel,
    f64 gradient, ncclAllReduce, update, captured in a CUDA graph) with one rank
    matches the fused single-GPU loop; eager (GLX_DP_GRAPH=0) and graph replays are
    byte-identical, including across calls (cached graphs) and the epoch statistics."""
    import os

    from paper_1908_07847_b200 import dp

    x, l, t, net0 = _case(50_000, 33, 256, seed=2)
    fused = net0.copy()
    fstats = np.zeros((7, 5))
    g.run_train_segment_batch(fused.w_ih2d, fused.w_ho2d, x, t, 7, 0.5, g.cuda(), fstats)
    with dp.NcclComm(0, 1, 0) as comm:
        a = dp.DeviceEngine(x, t, net0.w_ih, net0.w_ho)
        sa = dp.train_data_parallel_nccl(a, comm, 3, 0.5, x.shape[0])
        sa += dp.train_data_parallel_nccl(a, comm, 4, 0.5, x.shape[0])  # cached graphs
        os.environ["GLX_DP_GRAPH"] = "0"
        try:
            b = dp.DeviceEngine(x, t, net0.w_ih, net0.w_ho)
            sb = dp.train_data_parallel_nccl(b, comm, 7, 0.5, x.shape[0])
        finally:
            del os.environ["GLX_DP_GRAPH"]
        # the generic loop with the library all-reduce as its collective
        c = dp.DeviceEngine(x, t, net0.w_ih, net0.w_ho)
        sc = dp.train_data_parallel(c, 7, 0.5, x.shape[0], comm.all_reduce)
        wa, wb, wc = a.weights(), b.weights(), c.weights()
    assert wa[0].tobytes() == wb[0].tobytes() == wc[0].tobytes()
    assert wa[1].tobytes() == wb[1].tobytes() == wc[1].tobytes()
    assert [(s.loss_sum, s.counts) for s in sa] == [(s.loss_sum, s.counts) for s in sb] == \
           [(s.loss_sum, s.counts) for s in sc]
    assert rel_err(wa[0], fused.w_ih) <= 1e-6 and rel_err(wa[1], fused.w_ho) <= 1e-6
    assert all(sum(st.counts) == x.shape[0] for st in sa)
    assert np.abs(np.array([[s.loss_sum, *s.counts] for s in sa]) - fstats).max() <= 1e-6 * fstats[:, 0].max()


def test_dp_rank_without_rows_and_host_api(gpu):
    """A rank with no rows still joins the all-reduce (zero gradient: weights
    unchanged when it is the only rank); the host-buffer DP entry point
    (glx_dp_run_train_segment_batch) equals the device one."""
    from paper_1908_07847_b200 import _lib, dp

    x, l, t, net0 = _case(30_000, 33, 128, seed=4)
    with dp.NcclComm(0, 1, 0) as comm:
        e0 = dp.DeviceEngine(x[:0], t[:0], net0.w_ih, net0.w_ho)
        s0 = dp.train_data_parallel_nccl(e0, comm, 2, 0.5, 1000)
        w1, w2 = e0.weights()
        assert w1.tobytes() == net0.w_ih.tobytes() and w2.tobytes() == net0.w_ho.tobytes()
        assert all(s.loss_sum == 0 and sum(s.counts) == 0 for s in s0)
        dev = dp.DeviceEngine(x, t, net0.w_ih, net0.w_ho)
        dp.train_data_parallel_nccl(dev, comm, 5, 0.3, x.shape[0])
        host = net0.copy()
        st = np.zeros((5, 5))
        L = _lib.load()
        _lib.check(L.glx_dp_run_train_segment_batch(comm.handle, _lib.ptr(host.w_ih), _lib.ptr(host.w_ho),
                                                     _lib.ptr(x), _lib.ptr(t), x.shape[0], x.shape[0], 33, 128, 5,
                                                     0.3, _lib.ptr(st), 0))
        v1, v2 = dev.weights()
    assert host.w_ih.tobytes() == v1.tobytes() and host.w_ho.tobytes() == v2.tobytes()
    assert (st[:, 1:].sum(axis=1) == x.shape[0]).all()


@pytest.mark.parametrize("N,H", [(1 << 20, 256), (100_000, 256), (300_000, 128), (1 << 18, 33), (200_000, 60)])
def test_pipeline_checker_debug_runs(gpu, N, H):
    """debug=True: the tcgen05 epoch kernels stamp every tile hand-off between their
    roles and count the tiles each role handled (the device analogue of the
    reference's debug instrumentation, backend.py:122-133, 237-284); a clean run
    passes every check and trains the same bytes as the unchecked run."""
    import paper_1908_07847_b200._lib as L

    kind = L.load().glx_batch_kernel_kind(N, 33, H)
    assert kind in (2, 3)
    x, l, t, net0 = _case(N, 33, H, seed=H)
    a, b = net0.copy(), net0.copy()
    g.run_train_segment_batch(a.w_ih2d, a.w_ho2d, x, t, 3, 0.5, g.cuda())
    g.run_train_segment_batch(b.w_ih2d, b.w_ho2d, x, t, 3, 0.5, g.cuda(), debug=True)
    assert a.w_ih.tobytes() == b.w_ih.tobytes() and a.w_ho.tobytes() == b.w_ho.tobytes()


@pytest.mark.parametrize("N,H", [(1 << 20, 256), (1 << 18, 33)])
def test_pipeline_checker_catches_a_stale_hand_off(gpu, N, H, monkeypatch):
    """Fault injection: the producer stamps one row tile wrongly; the debug run must
    fail with the checker's RuntimeError naming the hand-off."""
    monkeypatch.setenv("GLX_DEBUG_INJECT_TILE", "37")
    x, l, t, net0 = _case(N, 33, H, seed=1)
    net = net0.copy()
    with pytest.raises(RuntimeError, match="pipeline check"):
        g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 1, 0.5, g.cuda(), debug=True)
