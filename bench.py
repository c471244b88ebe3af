"""Benchmark: train sample-epochs/s of full-batch GD on the B200 (BASELINE.json config 2).

Workload (per GPU): synthetic_matrix(1_000_000, 33, seed=rank, "planted-linear")
rows, network 33 -> 256 -> 1, full-batch gradient descent, lr 0.1. One step =
one epoch over all of a GPU's rows (forward, output/hidden deltas, dW/db
reduction over the rows, SGD update, loss/accuracy of the epoch-start
weights). N > 1 (torchrun, one process per GPU) is weak scaling: each rank
owns 1M rows and the per-epoch gradient is summed with one NCCL all-reduce
(paper_1908_07847_b200/dp.py).

Prints ONE JSON line (rank 0). `value` is measured with the packed rows
resident in HBM; `e2e` is the public host-pointer API
(backend.run_train_segment_batch -> glx_run_train_segment_batch) with the
inputs in pinned host memory, host<->device copies inside the timed region,
one call of E_E2E epochs per step (the reference bench's default epoch grid,
bench.py:147-155 of the reference CLI). `--impl reference` times the
reference's own CPU training engine (a C port of kernels.train_segment_par,
oracle/glx_oracle.c) on the host cores for the same shape and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ROWS_PER_GPU = 1_000_000
D, H, K = 33, 256, 1
LR = 0.1
E_E2E = 100
METRIC = "train sample-epochs/sec (full-batch GD, 33->256->1, 1M rows per GPU)"
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
    feats, labels = synthetic_arrays(ROWS_PER_GPU, D, 0, "planted-linear")
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
                      f"config 2), {n} rows x 1 epoch per step, median of {args.steps}"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.gpus), "cpu_baseline": base,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(n):
    return {"workload": "config 2: synthetic_matrix(1_000_000, 33, seed=rank, planted-linear) per GPU, "
                        "33->256->1 sigmoid MLP, full-batch GD lr 0.1, K=1",
            "rows_per_gpu": ROWS_PER_GPU, "input_dim": D, "hidden_dim": H, "output_dim": K,
            "global_rows": ROWS_PER_GPU * n, "parallelism": f"dp{n}",
            "l2": "packed rows 144 MB per GPU > 126 MB L2 (no flush needed)"}


# -------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1908_07847_b200 as g
    from paper_1908_07847_b200 import _lib, dp

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    # GLX_BENCH_FORCE_DP=1: take the data-parallel branch even with one rank (a
    # one-rank NCCL group), to exercise the N > 1 code path on a single GPU
    use_dp = world > 1 or os.environ.get("GLX_BENCH_FORCE_DP") == "1"
    if use_dp:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.load()
    feats, labels = g.synthetic_arrays(ROWS_PER_GPU, D, rank, "planted-linear")
    targets = labels.astype(np.float32)
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0, learning_rate=LR))
    eng = dp.DeviceEngine(feats, targets, net.w_ih, net.w_ho, device=local)
    stream = torch.cuda.current_stream()
    n_total = ROWS_PER_GPU * world
    stats_dev = torch.zeros((max(args.steps, args.warmup), 5), dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")

    ar = dp.nccl_all_reduce() if use_dp else None

    def epochs(k, stats):
        if not use_dp:  # fused single-GPU loop: epoch kernel + reduce/update kernel per epoch
            _lib.check(L.glx_train_batch(eng.w1.data_ptr(), eng.w2.data_ptr(), eng.Xp.data_ptr(), eng.N, D, H, k,
                                         LR, stats.data_ptr() if stats is not None else None, flag.data_ptr(),
                                         stream.cuda_stream))
        else:
            dp.train_data_parallel_graph(eng, k, LR, n_total, ar)

    # FP32 roofline denominator: packed-FFMA throughput on this GPU, now
    tfl = np.zeros(1)
    ms = np.zeros(1)
    _lib.check(L.glx_fp32_peak(local, 50_000, _lib.ptr(tfl), _lib.ptr(ms)))
    fp32_peak = float(tfl[0])

    epochs(args.warmup, stats_dev)
    torch.cuda.synchronize()
    L.glx_profile_enable(1)
    L.glx_profile_read(None, None)
    launches0 = int(L.glx_launch_count()) + dp.graph_kernel_launches
    with ClockSampler(local) as clk:
        if use_dp:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        epochs(args.steps, stats_dev)
        e1.record(stream)
        torch.cuda.synchronize()
        if use_dp:
            dist.barrier()
    launches = int(L.glx_launch_count()) + dp.graph_kernel_launches - launches0
    kms = np.zeros(1)
    kn = np.zeros(1, dtype=np.int64)
    _lib.check(L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn)))
    L.glx_profile_enable(0)
    elapsed = e0.elapsed_time(e1)
    if use_dp:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    value = n_total * args.steps / (elapsed * 1e-3)
    assert not eng.nonfinite() and not bool(flag.item()), "non-finite weights during the benchmark"

    # roofline of the dominant kernel (the epoch kernel), per launch
    kernel_timing = "CUDA events around every epoch-kernel launch in the timed region"
    if int(kn[0]) == 0 and use_dp:
        # the timed region replayed a CUDA graph (no per-launch host events): time the
        # same kernel on eager data-parallel epochs right after it
        L.glx_profile_enable(1)
        L.glx_profile_read(None, None)
        dp.train_data_parallel(eng, 5, LR, n_total, ar)
        _lib.check(L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn)))
        L.glx_profile_enable(0)
        kernel_timing = "CUDA events around 5 eager epochs right after the timed region (which replays a CUDA graph)"
    k_ms = float(kms[0]) / max(1, int(kn[0]))
    flops_per_launch = ROWS_PER_GPU * f_train()
    achieved = flops_per_launch / (k_ms * 1e-3) / 1e12
    traffic = None
    tr_file = ROOT / "profiles" / "traffic.json"
    if tr_file.exists():
        traffic = json.loads(tr_file.read_text()).get("batch_epoch_kernel_bytes_per_launch")
    kind = int(L.glx_batch_kernel_kind(ROWS_PER_GPU, D, H))
    common = {"traffic": traffic, "kernel_ms_per_launch": k_ms,
              "kernel_share_of_step": k_ms / (elapsed / args.steps) if elapsed else None,
              "kernel_timing": kernel_timing, "algorithmic_flops_per_launch": flops_per_launch,
              "algorithmic_hbm_bytes_per_launch": ROWS_PER_GPU * (4 * D + 1),
              "hbm_frac": ROWS_PER_GPU * (4 * D + 1) / (k_ms * 1e-3) / 1e9 / peaks().get("hbm_gbs", 6545.9),
              "fp32_peak_tflops": fp32_peak, "fp32_frac": achieved / fp32_peak}
    if kind == 2:
        # tcgen05 kind::tf32, 3xTF32: per 64-row tile 30 forward MMAs (M=128 units, N=64 rows,
        # K=8) and 48 backward MMAs (M=128, N=48 features, K=8 rows) per 128-unit half pair
        tf32_peak = peaks().get("bf16_tflops_sustained", 1355.8) / 2
        tiles = -(-ROWS_PER_GPU // 64)
        mma_flops = tiles * (H // 128) * (15 * 2 * 128 * 64 * 8 + 24 * 2 * 128 * 48 * 8)
        mufu_peak = 148 * 16 * clk_mhz_for_peak(local) * 1e6
        roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": achieved / tf32_peak,
                    "kernel": "batchtc_kernel<2> (tcgen05 kind::tf32, 3xTF32, deltas in TMEM)",
                    "fp32_accurate_peak": tf32_peak / 3,
                    "frac_of_fp32_accurate_peak": achieved / (tf32_peak / 3),
                    "executed_mma_flops_per_launch": mma_flops,
                    "executed_mma_frac": mma_flops / (k_ms * 1e-3) / 1e12 / tf32_peak,
                    "mufu_frac": 2 * ROWS_PER_GPU * H / (k_ms * 1e-3) / mufu_peak,
                    "peak_source": "dense TF32 = half of MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, "
                                   "back to back); fp32_accurate_peak = TF32 / 3 (3xTF32 spends three TF32 MMAs "
                                   "per fp32-accurate product); executed_mma_frac counts the 3xTF32 MMA work incl. "
                                   "K/N padding; "
                                   "mufu_frac = 2 MUFU ops per hidden activation / (148 SMs x 16/clk x SM clock)",
                    **common}
    else:
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak,
                    "kernel": "batch3_kernel<34,4,4> (three warp-specialised roles)" if kind == 1 else
                              "batch_epoch_kernel (two roles)",
                    "peak_source": "glx_fp32_peak FFMA2 microbenchmark on this GPU in this run (MEASURED_PEAKS.json "
                                   "has no FP32 figure)", **common}

    # end-to-end through the public API, inputs in pinned host memory: the host
    # segment API on one GPU, the data-parallel engine (every rank) on N
    e2e = run_e2e_dp(g, torch, dp, feats, targets, n_total, world) if use_dp else run_e2e(g, torch, feats, targets)

    line = None
    if rank == 0:
        cpu = cpu_baseline_batch(feats, targets) if world == 1 else None
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": elapsed / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
                "config": config_dict(world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(),
                "final_loss_sum": float(stats_dev[args.steps - 1, 0].item()) if not use_dp else None}
        print(json.dumps(line), flush=True)
    if use_dp:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(g, torch, feats, targets, reps=3):
    """Public API step: run_train_segment_batch(host arrays, E_E2E epochs), copies included."""
    pin_x = torch.empty(feats.shape, dtype=torch.float32, pin_memory=True)
    pin_t = torch.empty(targets.shape, dtype=torch.float32, pin_memory=True)
    pin_x.numpy()[:] = feats
    pin_t.numpy()[:] = targets
    x, t = pin_x.numpy(), pin_t.numpy()
    net0 = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    kind = g.cuda()
    net = net0.copy()
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 2, LR, kind)  # warm-up
    times = []
    for _ in range(reps):
        net = net0.copy()
        stats = np.zeros((E_E2E, 5))
        t0 = time.perf_counter()
        g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, E_E2E, LR, kind, stats)
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    w_bytes = 4 * (net.w_ih.size + net.w_ho.size)
    return {"value": feats.shape[0] * E_E2E / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(feats.nbytes + targets.nbytes + w_bytes),
            "d2h_bytes_per_step": int(w_bytes + stats.nbytes), "epochs_per_step": E_E2E,
            "seconds_per_step": dt, "api": "backend.run_train_segment_batch -> glx_run_train_segment_batch"}


def run_e2e_dp(g, torch, dp, feats, targets, n_total, world, reps=3):
    """N-GPU public-API step: every rank builds a dp.DeviceEngine from its pinned host
    shard (host->device copy and row packing), runs E_E2E data-parallel epochs
    (gradient kernel, NCCL all-reduce, update) and reads the weights back; the step
    time is the max over ranks and the value covers all ranks' rows."""
    import torch.distributed as dist

    pin_x = torch.empty(feats.shape, dtype=torch.float32, pin_memory=True)
    pin_t = torch.empty(targets.shape, dtype=torch.float32, pin_memory=True)
    pin_x.numpy()[:] = feats
    pin_t.numpy()[:] = targets
    x, t = pin_x.numpy(), pin_t.numpy()
    net0 = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    times = []
    for it in range(reps + 1):  # the first repetition is the warm-up
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng = dp.DeviceEngine(x, t, net0.w_ih, net0.w_ho, device=torch.cuda.current_device())
        # eager epochs: a fresh engine per step would pay graph instantiation in-step
        dp.train_data_parallel(eng, E_E2E, LR, n_total, dp.nccl_all_reduce())
        w1, w2 = eng.weights()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if it:
            times.append(float(dt.item()))
        del eng
    dt = statistics.median(times)
    w_bytes = 4 * (w1.size + w2.size)
    return {"value": n_total * E_E2E / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(feats.nbytes + targets.nbytes + w_bytes),
            "d2h_bytes_per_step": int(w_bytes + 5 * 8 * E_E2E), "epochs_per_step": E_E2E, "seconds_per_step": dt,
            "per_rank": True, "ranks": world,
            "api": "dp.DeviceEngine + dp.train_data_parallel (glx_batch_grad, NCCL all-reduce, glx_batch_apply)"}


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--suite", default=None,
                    help="secondary configurations instead of the headline, e.g. 1,3,4,5,eval,norm")
    ap.add_argument("--out", default=None, help="with --suite: write the results JSON here")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.suite:
        run_suite(args.suite, args.out)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
