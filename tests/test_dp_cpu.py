"""Data-parallel orchestration (paper_1908_07847_b200/dp.py) on CPU: gloo, world_size 2.

The product's epoch loop (shard -> per-rank gradient sum -> all-reduce(sum)
-> identical update) is run with a numpy test engine standing in for the
device kernels; the result must equal single-process full-batch GD (the
oracle restatement) to f64 rounding, and every rank must hold identical
weights and statistics.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_07847_b200 import dp


class NumpyEngine:
    """Test stand-in for dp.DeviceEngine: f64 gradient sums of one row shard."""

    def __init__(self, x, t, w_ih, w_ho):
        self.x = x.astype(np.float64)
        self.t = t.astype(np.float64)
        self.N, self.D = x.shape
        self.H = w_ih.size // (self.D + 1)
        self.w1 = w_ih.copy().reshape(self.H, self.D + 1)
        self.w2 = w_ho.copy().reshape(-1)

    def grad_sum(self):
        W1 = self.w1.astype(np.float64)
        w2 = self.w2.astype(np.float64)
        xa = np.hstack([self.x, np.ones((self.N, 1))])
        h = 1.0 / (1.0 + np.exp(-(xa @ W1.T)))
        o = 1.0 / (1.0 + np.exp(-(h @ w2[:-1] + w2[-1])))
        d_o = (o - self.t) * o * (1.0 - o)
        d_h = (d_o[:, None] * w2[None, :-1]) * h * (1.0 - h)
        g1 = d_h.T @ xa
        g2 = np.concatenate([d_o @ h, [d_o.sum()]])
        pred, pos = o >= 0.5, self.t >= 0.5
        stats = [0.5 * np.sum((self.t - o) ** 2), np.sum(pred & pos), np.sum(~pred & ~pos), np.sum(pred & ~pos),
                 np.sum(~pred & pos)]
        return torch.from_numpy(np.concatenate([g1.reshape(-1), g2, np.array(stats, np.float64)]))

    def apply(self, grad, lr_over_n):
        g = grad.numpy()
        P1 = self.H * (self.D + 1)
        self.w1 = (self.w1.astype(np.float64) - lr_over_n * g[:P1].reshape(self.w1.shape)).astype(np.float32)
        self.w2 = (self.w2.astype(np.float64) - lr_over_n * g[P1:P1 + self.H + 1]).astype(np.float32)


def _data():
    rng = np.random.default_rng(17)
    x = rng.random((203, 6), dtype=np.float32)
    t = (x[:, 0] + 0.3 * x[:, 3] > 0.65).astype(np.float32)
    w1 = rng.uniform(-0.5, 0.5, 5 * 7).astype(np.float32)
    w2 = rng.uniform(-0.5, 0.5, 6).astype(np.float32)
    return x, t, w1, w2


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, t, w1, w2 = _data()
    r0, r1 = dp.shard_bounds(x.shape[0], world, rank)
    eng = NumpyEngine(x[r0:r1], t[r0:r1], w1, w2)
    stats = dp.train_data_parallel(eng, 25, 2.0, x.shape[0], dp.torch_all_reduce())
    out_q.put((rank, eng.w1.copy(), eng.w2.copy(), [(s.loss_sum, s.counts) for s in stats]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(240)
def test_gloo_world2_equals_single_process_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=200) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, a1, a2, sa), (_, b1, b2, sb) = res
    # every rank holds identical weights and statistics
    assert a1.tobytes() == b1.tobytes() and a2.tobytes() == b2.tobytes()
    assert [c for _, c in sa] == [c for _, c in sb]
    # ... equal to single-process full-batch GD (oracle restatement, B = N)
    from oracle import oracle as O

    x, t, w1, w2 = _data()
    r1 = w1.copy().reshape(5, 7)
    r2 = w2.copy().reshape(1, 6)
    O.train_batch(r1, r2, x, t, 25, 2.0, x.shape[0])
    assert np.max(np.abs(a1.reshape(-1) - r1.reshape(-1))) <= 1e-6
    assert np.max(np.abs(a2.reshape(-1) - r2.reshape(-1))) <= 1e-6
    # statistics cover all rows: counts sum to N every epoch
    assert all(sum(c) == x.shape[0] for _, c in sa)


def test_world1_no_allreduce_matches():
    x, t, w1, w2 = _data()
    eng = NumpyEngine(x, t, w1, w2)
    dp.train_data_parallel(eng, 5, 2.0, x.shape[0], None)
    from oracle import oracle as O

    r1 = w1.copy().reshape(5, 7)
    r2 = w2.copy().reshape(1, 6)
    O.train_batch(r1, r2, x, t, 5, 2.0, x.shape[0])
    assert np.max(np.abs(eng.w1.reshape(-1) - r1.reshape(-1))) <= 1e-6


class NumpyKEngine:
    """Test stand-in for wide.WideEngine: K sigmoid outputs, one-hot targets, the
    wide gradient layout (P sums, then loss, correct, wrong)."""

    n_stats = 3

    def __init__(self, x, y, w_ih, w_ho, H, K):
        self.x = x.astype(np.float64)
        self.y = y
        self.N, self.D = x.shape
        self.H, self.K = H, K
        self.P = H * (self.D + 1) + K * (H + 1)
        self.w1 = w_ih.copy().reshape(H, self.D + 1)
        self.w2 = w_ho.copy().reshape(K, H + 1)

    def grad_sum(self):
        W1, W2 = self.w1.astype(np.float64), self.w2.astype(np.float64)
        xa = np.hstack([self.x, np.ones((self.N, 1))])
        h = 1.0 / (1.0 + np.exp(-(xa @ W1.T)))
        ha = np.hstack([h, np.ones((self.N, 1))])
        o = 1.0 / (1.0 + np.exp(-(ha @ W2.T)))
        t = np.eye(self.K)[self.y]
        d_o = (o - t) * o * (1.0 - o)
        d_h = (d_o @ W2[:, :-1]) * h * (1.0 - h)
        correct = np.sum(np.argmax(o, axis=1) == self.y)
        stats = [0.5 * np.sum((t - o) ** 2), correct, self.N - correct]
        return torch.from_numpy(np.concatenate([(d_h.T @ xa).reshape(-1), (d_o.T @ ha).reshape(-1),
                                                np.array(stats, np.float64)]))

    def apply(self, grad, lr_over_n):
        g = grad.numpy()
        P1 = self.w1.size
        self.w1 = (self.w1.astype(np.float64) - lr_over_n * g[:P1].reshape(self.w1.shape)).astype(np.float32)
        self.w2 = (self.w2.astype(np.float64) - lr_over_n * g[P1:self.P].reshape(self.w2.shape)).astype(np.float32)


def _kdata():
    rng = np.random.default_rng(5)
    x = rng.random((256, 9), dtype=np.float32)
    y = np.argmax(x[:, :4] + 0.1 * rng.random((256, 4)), axis=1).astype(np.uint8)
    w1 = rng.uniform(-0.5, 0.5, 6 * 10).astype(np.float32)
    w2 = rng.uniform(-0.5, 0.5, 4 * 7).astype(np.float32)
    return x, y, w1, w2


def _kworker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_07847_b200 import wide

    x, y, w1, w2 = _kdata()
    r0, r1 = wide.shard_rows(x.shape[0], world, rank)  # 64-row aligned shards, as the wide path uses
    eng = NumpyKEngine(x[r0:r1], y[r0:r1], w1, w2, 6, 4)
    stats = dp.train_data_parallel(eng, 10, 1.5, x.shape[0], dp.torch_all_reduce())
    out_q.put((rank, eng.w1.copy(), eng.w2.copy(), [(s.loss_sum, s.counts) for s in stats]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_gloo_world2_k_outputs_wide_layout():
    """The C5 data-parallel loop (K=16 engine layout: P sums + loss, correct, wrong)
    over gloo equals the oracle's single-process K-output full-batch restatement."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kworker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=200) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, a1, a2, sa), (_, b1, b2, sb) = res
    assert a1.tobytes() == b1.tobytes() and a2.tobytes() == b2.tobytes()
    assert [c for _, c in sa] == [c for _, c in sb]
    from oracle import oracle as O

    x, y, w1, w2 = _kdata()
    r1, r2 = w1.copy().reshape(6, 10), w2.copy().reshape(4, 7)
    O.train_batch_par(r1, r2, x, np.eye(4, dtype=np.float32)[y], 10, 1.5)
    assert np.max(np.abs(a1.reshape(-1) - r1.reshape(-1))) <= 1e-6
    assert np.max(np.abs(a2.reshape(-1) - r2.reshape(-1))) <= 1e-6
    assert all(len(c) == 2 and sum(c) == x.shape[0] for _, c in sa)


def test_wide_shard_rows_cover_and_align():
    from paper_1908_07847_b200 import wide

    for n, world in [(64 * 100, 8), (64 * 7, 4), (1 << 24, 8), (64, 1)]:
        spans = [wide.shard_rows(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all(r0 % 64 == 0 and r1 % 64 == 0 for r0, r1 in spans)
    with pytest.raises(Exception):
        wide.shard_rows(100, 2, 0)


def _oracle_trainer(nets, feats2d, targets, epochs, lr, numerics, device):
    """CPU stand-in for sweep.train_nets_on_device: the reference's sequential engine."""
    from oracle import oracle as O

    for n in nets:
        O.train_online_seq(n.w_ih2d, n.w_ho2d, feats2d, targets, epochs, lr)


def _sweep_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1908_07847_b200 as g

    x, y = g.synthetic_arrays(40, 6, 2, "planted-linear")
    hs, ss = g.sweep_grid([3, 8, 17, 30], [0, 1, 2])
    spec = g.SweepSpec(input_dim=6, hidden_dims=hs, seeds=ss, epochs=7)
    nets = g.train_sweep(spec, x, y.astype(np.float32), rank=rank, world_size=world, trainer=_oracle_trainer)
    out_q.put((rank, None if nets is None else [(n.w_ih.copy(), n.w_ho.copy()) for n in nets]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_gloo_world2_sweep_sharding_and_gather():
    """Config 3 across ranks: LPT shards trained independently (no
    data-path collective), gathered on rank 0, equal to the single-process sweep."""
    import paper_1908_07847_b200 as g

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=200) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None and res[0] is not None
    x, y = g.synthetic_arrays(40, 6, 2, "planted-linear")
    hs, ss = g.sweep_grid([3, 8, 17, 30], [0, 1, 2])
    spec = g.SweepSpec(input_dim=6, hidden_dims=hs, seeds=ss, epochs=7)
    single = g.train_sweep(spec, x, y.astype(np.float32), trainer=_oracle_trainer)
    assert len(res[0]) == len(single) == 12
    for (wi, wo), n in zip(res[0], single):
        assert wi.tobytes() == n.w_ih.tobytes() and wo.tobytes() == n.w_ho.tobytes()


def test_bench_spawns_ranks_itself():
    """`python bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run on 127.0.0.1); rank 0 prints one JSON line with n_gpus 2.
    GLX_BENCH_DRYRUN=1 stops after the rank plumbing (no GPU here)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, GLX_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["max_rank"] == 1.0
    assert rec["config"]["parallelism"] == "dp2" and rec["config"]["rows_per_gpu"] * 2 == rec["config"]["global_rows"]


def test_bench_scaling_rows():
    """`python bench.py --scaling 1,2` runs the headline once per GPU count (each its
    own ranks) and prints one line of scaling rows (GLX_BENCH_DRYRUN=1: plumbing only)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, GLX_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--scaling", "1,2", "--steps", "4", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert [r["n_gpus"] for r in rec["scaling_rows"]] == [1, 2]
    assert not any(r.get("failed") for r in rec["scaling_rows"]), rec
