"""Per-config device measurements beyond bench.py's headline (SURVEY.md 8(d)
configs 1, 3, 4, 5, eval, normalisation).

Device timings use CUDA events on the launching stream. The CPU reference
numbers beside them come from `cpu` legs passed in by `python bench.py --suite`
(bench.py owns the reference-engine timing); run directly, this module reports
device numbers only. Prints one JSON object per config; --out writes them all.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

import paper_1908_07847_b200 as g  # noqa: E402
from paper_1908_07847_b200 import _lib, dp  # noqa: E402
from paper_1908_07847_b200.sweep import pack_pool  # noqa: E402


def f_train(d, h, k=1):
    return 4 * h * (d + 1) + 4 * k * (h + 1) + 2 * h * k


def fp32_peak(L):
    tfl = np.zeros(1)
    ms = np.zeros(1)
    _lib.check(L.glx_fp32_peak(0, 50_000, _lib.ptr(tfl), _lib.ptr(ms)))
    return float(tfl[0])


def timed(fn, reps=1):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_rate(fn, rows, budget_s=5.0):
    t0 = time.perf_counter()
    fn(1)
    dt = time.perf_counter() - t0
    ep = max(1, int(budget_s / max(dt, 1e-6)))
    t0 = time.perf_counter()
    fn(ep)
    return rows * ep / (time.perf_counter() - t0)


def config1(L, peak, cpu=None):
    """Paper shape online SGD, one network (33-33-1, 90 rows) + both 30-30-1 cohorts."""
    from conftest import load_case  # fixture data produced by the reference

    out = []
    for name in ("paper_33_33_1", "cohort_male_30_30_1", "cohort_female_30_30_1"):
        c = load_case(name)
        D, H = int(c["meta"][0]), int(c["meta"][1])
        x, t = c["train_x"], c["train_y"].astype(np.float32)
        N = x.shape[0]
        dev = torch.device("cuda")
        X = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        T = torch.from_numpy(t).to(dev)
        res = {"config": f"1: {name} online SGD, {N} rows, {D}-{H}-1"}
        for numerics in ("fp32", "ref64"):
            net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=7))
            w1 = torch.from_numpy(net.w_ih).to(dev)
            w2 = torch.from_numpy(net.w_ho).to(dev)
            E = 2000
            st = torch.cuda.current_stream().cuda_stream
            run = lambda: _lib.check(L.glx_train_online(w1.data_ptr(), w2.data_ptr(), X.data_ptr(), T.data_ptr(), N,
                                                        D, H, E, 0.1, _lib.NUMERICS[numerics], st))
            run()
            ms = timed(run)
            res[f"gpu_{numerics}_sample_epochs_per_s"] = N * E / (ms * 1e-3)
        if cpu is not None:
            w1 = net.w_ih2d.copy()
            w2 = net.w_ho2d.copy()
            res["cpu_seq_sample_epochs_per_s"] = cpu_rate(lambda e: cpu.online_seq(w1, w2, x, t, e, 0.1), N)
            res["cpu_par_sample_epochs_per_s"] = cpu_rate(lambda e: cpu.online_par(w1, w2, x, t, e, 0.1), N)
            res["cpu_cores"] = os.cpu_count()
        res["note"] = "latency-bound: rows are serial in online SGD; one network uses one CTA"
        out.append(res)
    return out


def config3(L, peak, cpu=None, epochs=200):
    """4096 networks (64 widths 8..512 x 64 seeds), paper 90-row split, online fp32."""
    from conftest import load_case

    c = load_case("paper_33_33_1")
    x, t = c["train_x"], c["train_y"].astype(np.float32)
    N, D = x.shape
    hs, ss = g.sweep_grid(range(8, 513, 8), range(64))
    nets = [g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=h, seed=s)) for h, s in zip(hs, ss)]
    pool, H, off = pack_pool(nets)
    dev = torch.device("cuda")
    wp = torch.from_numpy(pool).to(dev)
    X = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    T = torch.from_numpy(t).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    res = {"config": f"3: sweep 4096 nets 33->{{8..512}}->1, {N} rows, online", "epochs": epochs}
    for numerics in ("fp32", "ref64"):
        ep = epochs if numerics == "fp32" else max(1, epochs // 10)
        run = lambda: _lib.check(L.glx_train_sweep(len(nets), _lib.ptr(H), _lib.ptr(off), wp.data_ptr(),
                                                   X.data_ptr(), T.data_ptr(), N, D, ep, 0.1,
                                                   _lib.NUMERICS[numerics], st))
        run()
        ms = timed(run)
        flops = sum(f_train(D, h) for h in hs) * N * ep
        res[f"gpu_{numerics}_net_sample_epochs_per_s"] = len(nets) * N * ep / (ms * 1e-3)
        res[f"gpu_{numerics}_tflops"] = flops / (ms * 1e-3) / 1e12
        res[f"gpu_{numerics}_frac_fp32_peak"] = flops / (ms * 1e-3) / 1e12 / peak
        res[f"gpu_{numerics}_ms"] = ms
    if cpu is None:
        return res
    # CPU: the reference engine on a cost-stratified sample of networks, extrapolated by flops
    idx = list(range(0, 4096, 128))
    sub = [nets[i].copy() for i in idx]
    spool, sH, soff = pack_pool(sub)
    t0 = time.perf_counter()
    cpu.sweep(sH, soff, spool, x, t, 20, 0.1, os.cpu_count())
    dt = time.perf_counter() - t0
    sub_flops = sum(f_train(D, int(h)) for h in sH) * N * 20
    cpu_tflops = sub_flops / dt / 1e12
    all_flops = sum(f_train(D, h) for h in hs) * N
    res["cpu_net_sample_epochs_per_s"] = 4096 * N * (cpu_tflops * 1e12 / all_flops)
    res["cpu_cores"] = os.cpu_count()
    res["cpu_sample"] = f"{len(sub)} stratified networks x 20 epochs, train_segment_seq per network, OpenMP over nets"
    return res


def config4_1gpu(L, peak, cpu=None, rows=67_108_864, epochs=5):
    """64Mi rows, 33->256->1, full batch, on one GPU (the DP config's per-run total)."""
    dev = torch.device("cuda")
    D, H = 33, 256
    ld = int(L.glx_packed_ld(D))
    Xp = torch.empty((rows, ld), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    # the rows of synthetic_matrix(rows, 33, 0, "planted-linear"), generated on the device
    # (numpy's PCG64 stream by jump-ahead; byte-identical, tests/test_gpu_synth.py) and packed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
    _lib.check(L.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    del X, lab
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    w1 = torch.from_numpy(net.w_ih).to(dev)
    w2 = torch.from_numpy(net.w_ho).to(dev)
    run = lambda: _lib.check(L.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, H, epochs, 0.1,
                                               None, None, st))
    run()
    ms = timed(run) / epochs
    flops = rows * f_train(D, H)
    return {"config": "4 (1 GPU): 64Mi rows synthetic_matrix(...,33,0,planted-linear), 33->256->1 full batch",
            "ms_per_epoch": ms, "sample_epochs_per_s": rows / (ms * 1e-3),
            "tflops": flops / (ms * 1e-3) / 1e12, "frac_fp32_peak": flops / (ms * 1e-3) / 1e12 / peak,
            "kernel": ["two-role FP32", "batch3 FP32", "batchtc tcgen05 3xTF32"][L.glx_batch_kernel_kind(rows, D, H)],
            "frac_tf32_dense_sustained": flops / (ms * 1e-3) / 1e12 / (_peaks().get("bf16_tflops_sustained", 1355.8) / 2),
            "data_gen_and_pack_s": gen_s,
            "data_gen_note": "device generation + packing (host numpy generation + upload of the same rows: 19.4 s)"}


def _peaks():
    import json
    from pathlib import Path

    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def config5(L, peak, cpu=None, rows=16_777_216, epochs=3):
    """Wide 1024 -> 1024 -> 16 on 16Mi rows, full batch, tcgen05 BF16 (device-generated rows)."""
    from paper_1908_07847_b200 import wide

    data = wide.WideData(rows, seed=0)
    w1, w2 = wide.init_wide_weights(seed=0)
    dev = torch.device("cuda")
    W1 = torch.from_numpy(w1).to(dev)
    W2 = torch.from_numpy(w2).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    run = lambda e: _lib.check(L.glx_wide_train(W1.data_ptr(), W2.data_ptr(), data.Xb.data_ptr(),
                                                data.XT.data_ptr(), data.labels.data_ptr(), rows, e, 0.1, None,
                                                None, st))
    run(1)
    L.glx_profile_enable(1)
    L.glx_profile_read(None, None)
    ms = timed(lambda: run(epochs)) / epochs
    kms = np.zeros(1)
    kn = np.zeros(1, dtype=np.int64)
    _lib.check(L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn)))
    L.glx_profile_enable(0)
    flops = rows * f_train(1024, 1024, 16)
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    bf16 = pk.get("bf16_tflops", 1654.1)
    return {"config": "5: wide 1024->1024->16, 16Mi rows, full batch, tcgen05 BF16 operands / FP32 TMEM accumulation",
            "ms_per_epoch": ms, "sample_epochs_per_s": rows / (ms * 1e-3),
            "tflops_algorithmic": flops / (ms * 1e-3) / 1e12, "frac_bf16_peak": flops / (ms * 1e-3) / 1e12 / bf16,
            "tc_gemm_ms_per_epoch": float(kms[0]) / epochs, "bf16_peak_tflops": bf16,
            "note": "tc_gemm_ms covers the three tcgen05 launches per 1Mi-row chunk (hidden-layer GEMM, the fused tail "
                    "kernel: output layer + delta_o + dH + dW2 in one pass over H, split-K dW1 GEMM); the remainder is "
                    "the per-epoch derive/reduce/update kernels. frac_bf16_peak is against MEASURED_PEAKS.json "
                    "bf16_tflops (cuBLAS burst)"}


def config5_tf32(L, peak, cpu=None, rows=16_777_216, epochs=2):
    """Wide 1024 -> 1024 -> 16 on 16Mi f32 rows, full batch, tcgen05 kind::tf32 with f32 H and
    deltas (the precision held to the 1e-4 FP32 tolerance, tests/test_gpu_tc.py)."""
    from paper_1908_07847_b200 import wide

    data = wide.WideData(rows, seed=0, precision="tf32")
    w1, w2 = wide.init_wide_weights(seed=0)
    dev = torch.device("cuda")
    W1 = torch.from_numpy(w1).to(dev)
    W2 = torch.from_numpy(w2).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    run = lambda e: _lib.check(L.glx_wide_train_tf32(W1.data_ptr(), W2.data_ptr(), data.Xb.data_ptr(),
                                                     data.XT.data_ptr(), data.labels.data_ptr(), rows, e, 0.1, None,
                                                     None, st))
    run(1)
    ms = timed(lambda: run(epochs)) / epochs
    flops = rows * f_train(1024, 1024, 16)
    import bench as _bench

    tf32 = _bench.tf32_peak_cublas(dev)
    return {"config": "5 (tf32): wide 1024->1024->16, 16Mi f32 rows, full batch, tcgen05 kind::tf32, f32 H / deltas",
            "ms_per_epoch": ms, "sample_epochs_per_s": rows / (ms * 1e-3),
            "tflops_algorithmic": flops / (ms * 1e-3) / 1e12, "tf32_peak_tflops_cublas": tf32,
            "frac_tf32_peak": flops / (ms * 1e-3) / 1e12 / tf32}


def eval_rate(L, peak, cpu=None):
    x, l = g.synthetic_arrays(1_000_000, 33, 0, "planted-linear")
    out = {}
    dev = torch.device("cuda")
    for H in (33, 256):
        net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=H, seed=0))
        w1 = torch.from_numpy(net.w_ih).to(dev)
        w2 = torch.from_numpy(net.w_ho).to(dev)
        X = torch.from_numpy(x).to(dev)
        Y = torch.from_numpy(l).to(dev)
        cnt = torch.zeros(4, dtype=torch.int64, device=dev)
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        run = lambda: _lib.check(L.glx_eval(w1.data_ptr(), w2.data_ptr(), X.data_ptr(), Y.data_ptr(), x.shape[0], 33,
                                            H, 1, cnt.data_ptr(), loss.data_ptr(), st))
        run()
        ms = timed(run)
        Xp = torch.empty((x.shape[0], int(L.glx_packed_ld(33))), dtype=torch.float32, device=dev)
        T = torch.from_numpy(l.astype(np.float32)).to(dev)
        _lib.check(L.glx_pack_rows(X.data_ptr(), T.data_ptr(), None, x.shape[0], 33, Xp.data_ptr(), st))
        stats = torch.zeros(5, dtype=torch.float64, device=dev)
        run2 = lambda: _lib.check(L.glx_eval_packed(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), x.shape[0], 33, H,
                                                    stats.data_ptr(), st))
        run2()
        ms2 = timed(run2)
        f_eval = 2 * H * 34 + 2 * (H + 1)
        out[f"H{H}"] = {"ref64_rows_per_s": x.shape[0] / (ms * 1e-3), "fp32_rows_per_s": x.shape[0] / (ms2 * 1e-3),
                        "fp32_frac_fp32_peak": x.shape[0] * f_eval / (ms2 * 1e-3) / 1e12 / peak}
        if cpu is not None:
            w1h, w2h = net.w_ih2d.copy(), net.w_ho2d.copy()
            t0 = time.perf_counter()
            cpu.eval_counts(w1h, w2h, x[:100_000], l[:100_000])
            out[f"H{H}"]["cpu_rows_per_s_1core"] = 100_000 / (time.perf_counter() - t0)
    return {"config": "eval_counts, 1M rows x 33", **out}


def norm_rate(L, peak, cpu=None, rows=67_108_864, D=33):
    """Device min-max normalisation at config 4's size (64Mi x 33 f32, 8.9 GB): fit
    (reads X) and apply (reads X, writes Y) against the measured HBM copy peak."""
    dev = torch.device("cuda")
    X = torch.rand((rows, D), device=dev) * 100.0
    Y = torch.empty_like(X)
    mn = torch.empty(D, device=dev)
    mx = torch.empty(D, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    fit = lambda: _lib.check(L.glx_minmax_fit(X.data_ptr(), rows, D, mn.data_ptr(), mx.data_ptr(), st))
    app = lambda: _lib.check(L.glx_minmax_apply(X.data_ptr(), rows, D, mn.data_ptr(), mx.data_ptr(), Y.data_ptr(), st))
    fit()
    app()
    t_fit = timed(fit, 5)
    t_app = timed(app, 5)
    ld = int(L.glx_packed_ld(D))
    T = torch.rand(rows, device=dev)
    Xp = torch.empty((rows, ld), device=dev)
    pack = lambda: _lib.check(L.glx_pack_rows(X.data_ptr(), T.data_ptr(), None, rows, D, Xp.data_ptr(), st))
    packn = lambda: _lib.check(L.glx_pack_rows_minmax(X.data_ptr(), T.data_ptr(), None, rows, D, mn.data_ptr(),
                                                     mx.data_ptr(), Xp.data_ptr(), st))
    pack()
    packn()
    t_pack = timed(pack, 5)
    t_packn = timed(packn, 5)
    pb = rows * (D * 4 + 4 + ld * 4)
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = pk.get("hbm_gbs", 6545.9)
    b = rows * D * 4
    return {"config": f"min-max normalisation, {rows} x {D} f32 (config 4 rows)",
            "fit_ms": t_fit, "fit_gbs": b / (t_fit * 1e-3) / 1e9, "fit_frac_hbm": b / (t_fit * 1e-3) / 1e9 / hbm,
            "apply_ms": t_app, "apply_gbs": 2 * b / (t_app * 1e-3) / 1e9,
            "apply_frac_hbm": 2 * b / (t_app * 1e-3) / 1e9 / hbm, "hbm_peak_gbs": hbm,
            "pack_rows_ms": t_pack, "pack_rows_gbs": pb / (t_pack * 1e-3) / 1e9,
            "pack_rows_minmax_ms": t_packn, "pack_rows_minmax_gbs": pb / (t_packn * 1e-3) / 1e9}


SUITE = {"1": config1, "3": config3, "4": config4_1gpu, "5": config5, "5tf32": config5_tf32, "eval": eval_rate,
         "norm": norm_rate}


def run_suite(which: str, out: str | None = None, cpu=None) -> dict:
    L = _lib.load()
    peak = fp32_peak(L)
    results = {"fp32_peak_tflops": peak}
    for w in which.split(","):
        r = SUITE[w](L, peak, cpu)
        results[f"config_{w}"] = r
        print(json.dumps({w: r}), flush=True)
    if out:
        Path(out).write_text(json.dumps(results, indent=1))
    return results


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="1,3,4,eval")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    run_suite(args.which, args.out)


if __name__ == "__main__":
    main()
