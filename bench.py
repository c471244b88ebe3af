"""Benchmark: train sample-epochs/s of full-batch GD on B200 (BASELINE.json configs 4 / 2).

Default workload (config 4, the configuration BASELINE.json quotes at 1/2/4/8
B200): synthetic_matrix(67_108_864, 33, seed=0, "planted-linear") rows,
generated on the device (byte-identical to the host generator), network
33 -> 256 -> 1, full-batch gradient descent, lr 0.1. The rows are sharded
contiguously over the ranks (strong scaling: the global row count is fixed);
one step = one epoch over all rows (forward, output/hidden deltas, dW/db
reduction, SGD update, loss/accuracy of the epoch-start weights). N = 1 runs the
fused single-GPU loop (epoch kernel + update kernel); N > 1 runs the library's
data-parallel epoch (epoch kernel, f64 gradient, NCCL all-reduce owned by the C
library, update) captured in a CUDA graph. `--workload c2` is config 2 (1M rows).

`python bench.py --gpus N` spawns N ranks itself (torch.distributed.run,
127.0.0.1) when it is not already running under torchrun.

Prints ONE JSON line (rank 0). `value` is measured with the packed rows
resident in HBM; `e2e` is the public host-pointer API
(backend.run_train_segment_batch -> glx_run_train_segment_batch at N = 1,
dp.run_train_segment_batch_dp -> glx_dp_run_train_segment_batch on every rank
at N > 1) with this rank's rows in pinned host memory and the host<->device
copies inside the timed region, E_E2E epochs per step (the reference bench's
default epoch grid, bench.py:147-155 of the reference CLI). `--impl reference`
times the reference's own CPU training engine (a C port of
kernels.train_segment_par, oracle/glx_oracle.c) on the host cores for the same
shape and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "c4": {"rows": 1 << 26, "name": "config 4: synthetic_matrix(67_108_864, 33, seed=0, planted-linear), "
                                    "33->256->1 sigmoid MLP, full-batch GD lr 0.1, K=1, rows sharded over the GPUs"},
    "c2": {"rows": 1_000_000, "name": "config 2: synthetic_matrix(1_000_000, 33, seed=0, planted-linear), "
                                      "33->256->1 sigmoid MLP, full-batch GD lr 0.1, K=1, rows sharded over the GPUs"},
}
D, H, K = 33, 256, 1
LR = 0.1
E_E2E = 100
CPU_ROWS = 1_000_000  # rows the CPU legs sample from
METRIC = "train sample-epochs/sec (full-batch GD, 33->256->1)"
UNIT = "sample-epochs/s"


def f_train(d=D, h=H, k=K) -> int:
    """Algorithmic flops per sample-epoch: 4H(D+1) + 4K(H+1) + 2HK."""
    return 4 * h * (d + 1) + 4 * k * (h + 1) + 2 * h * k


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        rows = []
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) < 8:
                continue
            try:
                rows.append((float(p[0]), float(p[1]), p[3:7], float(p[7])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [r for r in rows if r[3] >= 50] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in loaded for n, v in zip(names, r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(loaded)}


# --------------------------------------------------------- CPU baselines
def cpu_baseline_batch(feats, targets, target_s=20.0):  # the 4096-row calibration overestimates ~2x
    """Oracle port of the full-batch restatement, all host cores, bounded sample."""
    from oracle import oracle as O

    nw = os.cpu_count() or 1
    w1 = np.random.default_rng(0).uniform(-0.5, 0.5, (H, D + 1)).astype(np.float32)
    w2 = np.random.default_rng(1).uniform(-0.5, 0.5, (1, H + 1)).astype(np.float32)
    n = 4096
    t0 = time.perf_counter()
    O.train_batch_par(w1, w2, feats[:n], targets[:n], 1, LR, nw)
    dt = max(time.perf_counter() - t0, 1e-6)
    want = n * target_s / dt  # sample-epochs for ~target_s of CPU work
    n = int(min(feats.shape[0], max(4096, want)))
    epochs = max(1, int(round(want / n)))  # all rows fit: repeat epochs to fill the budget
    t0 = time.perf_counter()
    O.train_batch_par(w1, w2, feats[:n], targets[:n], epochs, LR, nw)
    dt = time.perf_counter() - t0
    return {"value": n * epochs / dt, "unit": UNIT, "cores": nw, "kind": "port",
            "sample": f"oracle train_batch_par (full-batch restatement, f64 reference op order), "
                      f"{n} of the rows x {epochs} epochs, {dt:.1f} s"}


def _reference_engines(nw):
    from oracle import oracle as O

    return (("train_segment_par", nw, lambda w1, w2, x, t: O.train_online_par(w1, w2, x, t, 1, LR, nw)),
            ("train_segment_seq", 1, lambda w1, w2, x, t: O.train_online_seq(w1, w2, x, t, 1, LR)))


def _fresh_weights():
    w1 = np.random.default_rng(0).uniform(-0.5, 0.5, (H, D + 1)).astype(np.float32)
    w2 = np.random.default_rng(1).uniform(-0.5, 0.5, (1, H + 1)).astype(np.float32)
    return w1, w2


def reference_calibrate(feats, targets, nw):
    """Pick the faster of the reference's two engines (C ports of kernels.py:264-349) on
    this host and its rows/s on a small sample."""
    best = None
    for name, cores, fn in _reference_engines(nw):
        w1, w2 = _fresh_weights()
        fn(w1, w2, feats[:64], targets[:64])  # spin up the thread team
        n = 2000
        t0 = time.perf_counter()
        fn(w1, w2, feats[:n], targets[:n])
        rate = n / max(time.perf_counter() - t0, 1e-6)
        if best is None or rate > best[3]:
            best = (name, cores, fn, rate)
    return best


def run_reference(args):
    """Reference arm: the reference's own CPU training engine (online SGD, the only
    training loop the reference has; same flops per sample-epoch as the batch
    epoch), C port pinned byte-identical to it, all host cores, bounded samples."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1908_07847_b200 import synthetic_arrays
    from oracle import oracle as O

    O.build()
    feats, labels = synthetic_arrays(CPU_ROWS, D, 0, "planted-linear")
    targets = labels.astype(np.float32)
    nw = os.cpu_count() or 1
    name, cores, fn, rate = reference_calibrate(feats, targets, nw)
    per_step_s = min(2.0, max(0.05, 150.0 / (args.steps + args.warmup)))
    n = int(min(feats.shape[0], max(64, rate * per_step_s)))
    for _ in range(args.warmup):
        w1, w2 = _fresh_weights()
        fn(w1, w2, feats[:n], targets[:n])
    times = []
    for _ in range(args.steps):
        w1, w2 = _fresh_weights()
        t0 = time.perf_counter()
        fn(w1, w2, feats[:n], targets[:n])
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    v = n / dt
    base = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{name} (C port of the reference engine, online SGD, same flops per sample-epoch as "
                      f"the 33->256->1 batch epoch), {n} rows x 1 epoch per step, median of {args.steps}"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.workload, args.gpus), "cpu_baseline": base,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(workload, n):
    rows = WORKLOADS[workload]["rows"]
    return {"workload": WORKLOADS[workload]["name"], "global_rows": rows, "rows_per_gpu": rows // n,
            "input_dim": D, "hidden_dim": H, "output_dim": K, "parallelism": f"dp{n}",
            "l2": f"packed rows {rows * 144 / n / 1e6:.0f} MB per GPU > 126 MB L2 (no flush needed)"}


def tf32_peak_cublas(dev) -> float:
    """Dense TF32 throughput of cuBLAS on this GPU now (8192^3 fp32 GEMM with TF32
    tensor cores), the measured TF32 roofline denominator (TFLOP/s)."""
    import torch

    n = 8192
    a = torch.rand((n, n), device=dev)
    b = torch.rand((n, n), device=dev)
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        for _ in range(3):
            torch.matmul(a, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        return 2 * n ** 3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
        del a, b


# -------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch

    import paper_1908_07847_b200 as g
    from paper_1908_07847_b200 import _lib, dp

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    # GLX_BENCH_FORCE_DP=1: the data-parallel (NCCL) branch even with one rank
    use_dp = world > 1 or os.environ.get("GLX_BENCH_FORCE_DP") == "1"
    ctrl = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # control plane only: id exchange, barriers, max over ranks
        ctrl = dist
    L = _lib.load()
    rows = WORKLOADS[args.workload]["rows"]
    r0, r1 = dp.shard_bounds(rows, world, rank)
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0, learning_rate=LR))

    # rows on the device (byte-identical to synthetic_matrix), this rank's shard packed;
    # a pinned host copy of the shard for the end-to-end leg
    X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear", device=local)
    Xs, ls = X[r0:r1].contiguous(), lab[r0:r1].contiguous()
    del X, lab
    eng = dp.DeviceEngine.from_device(Xs, ls, net.w_ih, net.w_ho)
    host_x = torch.empty((r1 - r0, D), dtype=torch.float32, pin_memory=True)
    host_t = torch.empty((r1 - r0,), dtype=torch.float32, pin_memory=True)
    host_x.copy_(Xs)
    host_t.copy_(ls.to(torch.float32))
    del Xs, ls
    torch.cuda.empty_cache()
    comm = dp.NcclComm(rank, world, local) if use_dp else None

    stream = torch.cuda.current_stream()
    stats_dev = torch.zeros((max(args.steps, args.warmup), 5), dtype=torch.float64, device="cuda")

    def epochs(k):
        if comm is None:  # fused single-GPU loop: epoch kernel + reduce/update kernel per epoch
            _lib.check(L.glx_train_batch(eng.w1.data_ptr(), eng.w2.data_ptr(), eng.Xp.data_ptr(), eng.N, D, H, k,
                                         LR, stats_dev.data_ptr(), eng.flag.data_ptr(), stream.cuda_stream))
        else:
            _lib.check(L.glx_dp_train_batch(comm.handle, eng.w1.data_ptr(), eng.w2.data_ptr(), eng.Xp.data_ptr(),
                                            eng.N, rows, D, H, k, LR, stats_dev.data_ptr(), eng.flag.data_ptr(),
                                            stream.cuda_stream))

    def barrier():
        if ctrl is not None:
            ctrl.barrier()

    def max_over_ranks(v: float) -> float:
        if ctrl is None:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        ctrl.all_reduce(t, op=ctrl.ReduceOp.MAX)
        return float(t.item())

    # roofline denominators measured on this GPU now
    tfl = np.zeros(1)
    ms = np.zeros(1)
    _lib.check(L.glx_fp32_peak(local, 50_000, _lib.ptr(tfl), _lib.ptr(ms)))
    fp32_peak = float(tfl[0])
    tf32_meas = tf32_peak_cublas(torch.device("cuda", local))

    epochs(args.warmup)
    torch.cuda.synchronize()
    launches0 = int(L.glx_launch_count())
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        epochs(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = int(L.glx_launch_count()) - launches0
    elapsed = max_over_ranks(e0.elapsed_time(e1))
    value = rows * args.steps / (elapsed * 1e-3)
    assert not eng.nonfinite(), "non-finite weights during the benchmark"
    final_loss = float(stats_dev[args.steps - 1, 0].item())

    # the dominant kernel (the epoch kernel), per launch: CUDA events around each launch
    # on its stream, in eager epochs right after the timed region (the timed region
    # itself runs without per-launch events; N > 1 replays a CUDA graph)
    os.environ["GLX_DP_GRAPH"] = "0"
    L.glx_profile_enable(1)
    L.glx_profile_read(None, None)
    epochs(10)
    kms = np.zeros(1)
    kn = np.zeros(1, dtype=np.int64)
    _lib.check(L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn)))
    L.glx_profile_enable(0)
    del os.environ["GLX_DP_GRAPH"]
    k_ms = float(kms[0]) / max(1, int(kn[0]))
    n_local = r1 - r0
    flops_per_launch = n_local * f_train()
    achieved = flops_per_launch / (k_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    tr_file = ROOT / "profiles" / "traffic.json"
    if tr_file.exists():
        tr = json.loads(tr_file.read_text())
        per_row = tr.get("batch_epoch_kernel_bytes_per_row")
        if per_row:
            traffic = per_row * n_local
            traffic_src = tr.get("source")
    kind = int(L.glx_batch_kernel_kind(n_local, D, H))
    step_ms = elapsed / args.steps
    common = {"traffic": traffic, "traffic_source": traffic_src, "kernel_ms_per_launch": k_ms,
              "kernel_share_of_step": k_ms / step_ms if step_ms else None,
              "kernel_timing": "CUDA events around each epoch-kernel launch on its stream, 10 eager epochs right "
                               "after the timed region (which ran without per-launch events)",
              "algorithmic_flops_per_launch": flops_per_launch,
              "algorithmic_hbm_bytes_per_launch": n_local * (4 * D + 1),
              "hbm_frac": n_local * (4 * D + 1) / (k_ms * 1e-3) / 1e9 / peaks().get("hbm_gbs", 6545.9),
              "fp32_peak_tflops": fp32_peak, "fp32_frac": achieved / fp32_peak}
    if kind == 2:
        # tcgen05 kind::tf32: per 64-row tile and 128-unit half, FAST precision
        # (>= 2^17 rows) runs 10 forward MMAs (M=128 units, N=64 rows, K=8: hi(W) x + lo(W) x over
        # K=40) and 8 backward MMAs (M=128, N=48 features, K=8 rows); FULL (3xTF32) 15 + 24
        tf32_derived = peaks().get("bf16_tflops_sustained", 1355.8) / 2
        tf32_peak = max(tf32_meas, tf32_derived)
        tiles = -(-n_local // 64)
        fast = n_local >= (1 << 17)
        nf, nb = (10, 8) if fast else (15, 24)
        mma_flops = tiles * (H // 128) * (nf * 2 * 128 * 64 * 8 + nb * 2 * 128 * 48 * 8)
        mufu_peak = 148 * 16 * clk_mhz_for_peak(local) * 1e6
        roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": achieved / tf32_peak,
                    "kernel": f"batchtc_kernel<2, {'FAST' if fast else 'FULL'}> (tcgen05 kind::tf32, deltas in TMEM)",
                    "tf32_cublas_measured_tflops": tf32_meas, "tf32_half_of_bf16_tflops": tf32_derived,
                    "executed_mma_flops_per_launch": mma_flops,
                    "executed_mma_frac": mma_flops / (k_ms * 1e-3) / 1e12 / tf32_peak,
                    "mufu_ops_per_launch": 1.5 * n_local * H,
                    "mufu_frac": 1.5 * n_local * H / (k_ms * 1e-3) / mufu_peak,
                    "binding_resource": "the epilogue (sigmoid on MUFU, shuffle/FMA row and delta passes), "
                                        "not the tensor pipe: mufu_frac and the ncu capture in profiles/",
                    "peak_source": "dense TF32 = max(cuBLAS 8192^3 TF32 GEMM measured in this run, half of "
                                   "MEASURED_PEAKS.json bf16_tflops_sustained); executed_mma_frac counts the MMA "
                                   "work incl. K/N padding; mufu_frac = 1.5 MUFU ops per hidden activation (ex2 "
                                   "+ one reciprocal per pair) / (148 SMs x 16/clk x max SM clock)",
                    **common}
    else:
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak,
                    "kernel": "batch3_kernel<34,4,4> (three warp-specialised roles)" if kind == 1 else
                              "batch_epoch_kernel (two roles)",
                    "peak_source": "glx_fp32_peak FFMA2 microbenchmark on this GPU in this run (MEASURED_PEAKS.json "
                                   "has no FP32 figure)", **common}

    # end-to-end through the public API, this rank's rows in pinned host memory
    e2e = run_e2e(g, dp, comm, host_x.numpy(), host_t.numpy(), rows, barrier, max_over_ranks)
    e2e["gpu_launches"] = None
    # config 3 sharded the way it scales: every rank its LPT share of the 4096 networks
    sweep = run_sweep_sharded(L, rank, world, barrier, max_over_ranks)

    if rank == 0:
        cpu = None
        secondary = None
        if world == 1:
            n_cpu = min(CPU_ROWS, host_x.shape[0])
            cpu = cpu_baseline_batch(host_x.numpy()[:n_cpu], host_t.numpy()[:n_cpu])
            if not args.no_secondary:
                del eng, host_x, host_t
                torch.cuda.empty_cache()
                secondary = secondary_configs(L, fp32_peak)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
                "config": config_dict(args.workload, world), "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "final_loss_sum": final_loss,
                "secondary_configs": secondary, "sweep_sharded": sweep,
                "path": "glx_train_batch (fused single-GPU loop)" if comm is None else
                        "glx_dp_train_batch (epoch kernel, f64 gradient, library-owned ncclAllReduce, update; "
                        "CUDA graph replay)"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if ctrl is not None:
        ctrl.barrier()
        ctrl.destroy_process_group()


def secondary_configs(L, fp32_peak):
    """The other named configurations measured in the same run on the same GPU (BASELINE.json
    configs 1, 3, 5 and config 2 at the reference's default width H = 33), device-timed,
    bounded to a few seconds each (tools/bench_configs.py; CPU legs: bench.py --suite)."""
    import torch

    import paper_1908_07847_b200 as g
    from paper_1908_07847_b200 import _lib

    sys.path.insert(0, str(ROOT / "tools"))
    sys.path.insert(0, str(ROOT / "tests"))
    import bench_configs as bc

    out = {}
    # config 2 at the reference default width (33 -> 33 -> 1, 1M rows; the rows-on-lanes
    # tcgen05 kernel), first: after config 5's BF16 GEMMs the power cap lowers the clocks
    rows, h33 = 1_000_000, 33
    X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
    Xp = torch.empty((rows, int(L.glx_packed_ld(D))), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=h33, seed=0))
    w1, w2 = torch.from_numpy(net.w_ih).cuda(), torch.from_numpy(net.w_ho).cuda()
    run = lambda k: _lib.check(L.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, h33, k, LR,
                                                 None, None, st))
    run(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(200)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    out["config2_h33"] = {"config": "2 at H = 33: synthetic_matrix(1_000_000, 33, 0, planted-linear), 33->33->1",
                          "ms_per_epoch": ms, "sample_epochs_per_s": rows / (ms * 1e-3),
                          "kernel_kind": int(L.glx_batch_kernel_kind(rows, D, h33)),
                          "frac_fp32_peak": rows * f_train(D, h33) / (ms * 1e-3) / 1e12 / fp32_peak}
    del X, lab, Xp, w1, w2
    torch.cuda.empty_cache()
    for name, fn in (("config1", lambda: bc.config1(L, fp32_peak)), ("config3", lambda: bc.config3(L, fp32_peak)),
                     ("config5_bf16", lambda: bc.config5(L, fp32_peak))):
        try:
            out[name] = fn()
        except Exception as e:  # reported, never fatal to the headline line
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()
    return out


def run_sweep_sharded(L, rank, world, barrier, max_over_ranks, epochs=200, reps=3):
    """Config 3 at this GPU count: 4096 networks 33 -> {8..512} -> 1 (64 widths x 64 seeds)
    on the paper's 90-row split, online fp32; the networks are LPT-sharded over the ranks
    by cost (sweep.lpt_shards, no communication), every rank trains its share with
    glx_train_sweep, time = max over ranks of the median device time; value = all
    networks' sample-epochs / that time."""
    import torch

    import paper_1908_07847_b200 as g
    from paper_1908_07847_b200 import _lib
    from paper_1908_07847_b200.sweep import lpt_shards, pack_pool

    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import load_case

    c = load_case("paper_33_33_1")
    x, t = c["train_x"], c["train_y"].astype(np.float32)
    N, Dx = x.shape
    hs, ss = g.sweep_grid(range(8, 513, 8), range(64))
    spec = g.SweepSpec(input_dim=Dx, hidden_dims=hs, seeds=ss, epochs=epochs)
    mine = lpt_shards(spec.costs(), world)[rank]
    nets = [g.init_weights(g.NetworkConfig(input_dim=Dx, hidden_dim=hs[i], seed=ss[i])) for i in mine]
    pool, Hs, off = pack_pool(nets)
    wp = torch.from_numpy(pool).cuda()
    X = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    T = torch.from_numpy(t).cuda()
    st = torch.cuda.current_stream().cuda_stream
    run = lambda: _lib.check(L.glx_train_sweep(len(nets), _lib.ptr(Hs), _lib.ptr(off), wp.data_ptr(), X.data_ptr(),
                                               T.data_ptr(), N, Dx, epochs, 0.1, _lib.NUMERICS["fp32"], st))
    run()
    times = []
    for _ in range(reps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        times.append(max_over_ranks(e0.elapsed_time(e1)))
    ms = statistics.median(times)
    flops = sum(f_train(Dx, h) for h in hs) * N * epochs
    return {"config": "3: sweep 4096 nets 33->{8..512}->1, 90 rows, online fp32, LPT-sharded over the GPUs",
            "n_gpus": world, "epochs": epochs, "ms": ms, "nets_this_rank": len(nets),
            "net_sample_epochs_per_s": len(hs) * N * epochs / (ms * 1e-3),
            "tflops": flops / (ms * 1e-3) / 1e12, "scaling": "strong",
            "timing": "CUDA events per rank, max over ranks, median of 3"}


def run_e2e(g, dp, comm, x, t, rows_total, barrier, max_over_ranks, reps=3):
    """Public-API step with this rank's rows in pinned host memory: E_E2E epochs of
    run_train_segment_batch (N = 1) or dp.run_train_segment_batch_dp (data parallel,
    every rank), host->device copy of the rows and the weights, packing, training,
    device->host copy of the weights and the per-epoch statistics; step time = max
    over ranks, value over all ranks' rows."""
    net0 = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    times = []
    for it in range(reps + 1):  # the first repetition is the warm-up
        net = net0.copy()
        stats = np.zeros((E_E2E, 5))
        barrier()
        t0 = time.perf_counter()
        if comm is None:
            g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, E_E2E, LR, g.cuda(), stats)
        else:
            dp.run_train_segment_batch_dp(comm, net.w_ih2d, net.w_ho2d, x, t, rows_total, E_E2E, LR, stats)
        dt = max_over_ranks(time.perf_counter() - t0)
        if it:
            times.append(dt)
    dt = statistics.median(times)
    w_bytes = 4 * (net.w_ih.size + net.w_ho.size)
    return {"value": rows_total * E_E2E / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(x.nbytes + t.nbytes + w_bytes),
            "d2h_bytes_per_step": int(w_bytes + stats.nbytes), "epochs_per_step": E_E2E,
            "seconds_per_step": dt, "bytes_per_rank": comm is not None,
            "api": "backend.run_train_segment_batch -> glx_run_train_segment_batch" if comm is None else
                   "dp.run_train_segment_batch_dp -> glx_dp_run_train_segment_batch (every rank)"}


def clk_mhz_for_peak(dev) -> float:
    """SM clock (MHz) for the MUFU peak: the max SM clock nvidia-smi reports, else MEASURED_PEAKS."""
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(dev), "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=20).stdout.strip()
        return float(out.splitlines()[0])
    except Exception:
        return float(peaks().get("sm_max_mhz", 1965.0))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


class SuiteCpuLegs:
    """CPU reference legs of the secondary-config suite (tools/bench_configs.py):
    the C restatement of the reference engines (oracle/, pinned byte-identical to
    kernels.train_segment_seq / _par / eval_counts), timed beside the device."""

    def __init__(self):
        from oracle import oracle as O

        self.O = O

    def online_seq(self, *a):
        self.O.train_online_seq(*a)

    def online_par(self, *a):
        self.O.train_online_par(*a)

    def sweep(self, *a):
        self.O.train_sweep(*a)

    def eval_counts(self, *a):
        return self.O.eval_counts(*a)


def run_suite(which: str, out: str | None):
    sys.path.insert(0, str(ROOT / "tools"))
    sys.path.insert(0, str(ROOT / "tests"))
    import bench_configs

    bench_configs.run_suite(which, out, SuiteCpuLegs())


def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-launch this script as N ranks (one process per
    GPU) with torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args):
    """GLX_BENCH_DRYRUN=1: the launch / rank plumbing only (no GPU): every rank joins
    the gloo control group, rank 0 prints the line skeleton (tests/test_dp_cpu.py)."""
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = __import__("torch").tensor([float(rank)], dtype=__import__("torch").float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        top = float(t.item())
    else:
        top = 0.0
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_rank": top, "steps": args.steps,
                          "warmup": args.warmup, "config": config_dict(args.workload, world)}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_scaling(args) -> None:
    """`--scaling 1,2,4,8`: the headline at each GPU count, each a separate
    `bench.py --gpus N` run (its own ranks), and one JSON line of scaling rows
    (n_gpus, value, ms_per_step, speedup over the first N, efficiency) -- the
    report-side 1/2/4/8 rows of SURVEY.md 8(f)3. The driver's SCALE run computes
    its own efficiency from the per-N lines; this is the builder-side table."""
    rows = []
    for n in [int(v) for v in args.scaling.split(",") if v]:
        cmd = [sys.executable, str(Path(__file__).resolve()), "--gpus", str(n), "--steps", str(args.steps),
               "--warmup", str(args.warmup), "--workload", args.workload, "--no-secondary"]
        env = dict(os.environ)
        for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
            env.pop(k, None)
        out = subprocess.run(cmd, capture_output=True, text=True, env=env)
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if out.returncode != 0 or not lines:
            rows.append({"n_gpus": n, "failed": True, "error": (out.stderr or out.stdout)[-400:]})
            continue
        rec = json.loads(lines[-1])
        sw = rec.get("sweep_sharded") or {}
        rows.append({"n_gpus": rec.get("n_gpus", n), "value": rec.get("value"), "ms_per_step": rec.get("ms_per_step"),
                     "e2e": (rec.get("e2e") or {}).get("value"), "scaling": rec.get("scaling"),
                     "sweep_net_sample_epochs_per_s": sw.get("net_sample_epochs_per_s")})
    base = next((r for r in rows if r.get("value")), None)
    sbase = next((r for r in rows if r.get("sweep_net_sample_epochs_per_s")), None)
    for r in rows:
        if base and r.get("value"):
            r["speedup"] = r["value"] / base["value"]
            r["efficiency"] = r["speedup"] * base["n_gpus"] / r["n_gpus"]
        if sbase and r.get("sweep_net_sample_epochs_per_s"):
            r["sweep_speedup"] = r["sweep_net_sample_epochs_per_s"] / sbase["sweep_net_sample_epochs_per_s"]
    line = {"metric": METRIC, "unit": "sample-epochs/s", "workload": args.workload, "scaling_rows": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="c4")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other configurations measured after the headline (N = 1)")
    ap.add_argument("--suite", default=None,
                    help="secondary configurations instead of the headline, e.g. 1,3,4,5,eval,norm")
    ap.add_argument("--out", default=None, help="with --suite / --scaling: write the results JSON here")
    ap.add_argument("--scaling", default=None, help="GPU counts, e.g. 1,2,4,8: one headline run per count and "
                    "a table of scaling rows")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.suite:
        run_suite(args.suite, args.out)
    elif args.scaling:
        run_scaling(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    elif os.environ.get("GLX_BENCH_DRYRUN") == "1":
        run_dry(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
