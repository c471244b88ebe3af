"""Numerical design study for the tcgen05 epoch kernel's TF32 operand splits.

Emulates, in numpy, the full-batch epoch of glx_batchtc.cu with each GEMM
operand split into tf32 hi + lo parts and a chosen subset of the split
products (hi.hi always, plus hi.lo / lo.hi cross terms) -- for the forward
Z = W1s [x,1] and the backward dW1 = sum_r dh_r x_r -- and trains for E epochs
against the f64 oracle restatement (oracle.train_batch_par). The accumulation
is done in float64 so only the operand-split error is measured.

    python tools/tf32_split_error.py [rows] [epochs]

Split modes: "trunc" (hi = mantissa truncated to 10 bits, the kernel up to
round 1) and "rn" (hi = round-to-nearest tf32, cvt.rna.tf32.f32).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def tf32(v: np.ndarray, mode: str) -> np.ndarray:
    b = np.ascontiguousarray(v, np.float32).view(np.uint32)
    if mode == "rn":  # round half away from zero on the 13 dropped bits (cvt.rna)
        b = (b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    else:
        b = b & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def split(v, mode):
    hi = tf32(v, mode)
    lo = (np.asarray(v, np.float32) - hi).astype(np.float32)
    return hi.astype(np.float64), tf32(lo, "trunc").astype(np.float64)  # the MMA reads lo as tf32 too


def gemm(a, b, mode, terms):
    """a @ b with split operands; terms among 'hh', 'hl' (a hi . b lo), 'lh' (a lo . b hi)."""
    ah, al = split(a, mode)
    bh, bl = split(b, mode)
    out = ah @ bh
    if "hl" in terms:
        out += ah @ bl
    if "lh" in terms:
        out += al @ bh
    return out


def epoch_grad(w1, w2, x1, t, mode, fwd_terms, bwd_terms):
    """One epoch's gradient sums as the kernel forms them (f64 accumulation)."""
    log2e = 1.4426950408889634
    w1s = (-log2e * w1).astype(np.float32)
    z = gemm(x1, w1s.T, mode, fwd_terms)  # [N, H], prescaled by -log2 e
    h = (1.0 / (1.0 + np.exp2(z))).astype(np.float32).astype(np.float64)
    zo = h @ w2[0, :-1].astype(np.float64) + w2[0, -1]
    o = 1.0 / (1.0 + np.exp(-zo))
    do = (o - t) * o * (1.0 - o)
    dh = (do[:, None] * h * (1.0 - h)).astype(np.float32)  # w2_j folded in later (batch_update)
    g1 = gemm(dh.T, x1, mode, bwd_terms) * w2[0, :-1, None].astype(np.float64)
    g2 = np.concatenate([(do[:, None] * h).sum(0), [do.sum()]])
    return g1, g2


def run(rows=100_000, epochs=20, lr=0.1, schemes=None):
    import paper_1908_07847_b200 as g
    from oracle import oracle as O

    x, l = g.synthetic_arrays(rows, 33, 3, "planted-linear")
    t = l.astype(np.float64)
    x1 = np.concatenate([x, np.ones((rows, 1), np.float32)], axis=1)
    net0 = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=256, seed=3))
    ref = net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, l.astype(np.float32), epochs, lr)
    schemes = schemes or [("trunc", "hl lh", "hl lh"), ("rn", "hl lh", "hl lh"), ("rn", "hl lh", "hl"),
               ("rn", "hl lh", "lh"), ("rn", "hl", "hl"), ("trunc", "hl lh", "hl"), ("rn", "", "hl"),
               ("rn", "hl", "")]
    for mode, ft, bt in schemes:
        w1 = net0.w_ih2d.astype(np.float32).copy()
        w2 = net0.w_ho2d.astype(np.float32).copy()
        for _ in range(epochs):
            g1, g2 = epoch_grad(w1, w2, x1, t, mode, ft.split(), bt.split())
            w1 = (w1.astype(np.float64) - lr / rows * g1).astype(np.float32)
            w2 = (w2.astype(np.float64) - lr / rows * g2[None, :]).astype(np.float32)
        err = max(np.max(np.abs(w1 - ref.w_ih2d) / np.maximum(1, np.abs(ref.w_ih2d))),
                  np.max(np.abs(w2 - ref.w_ho2d) / np.maximum(1, np.abs(ref.w_ho2d))))
        print(f"split {mode:5s} forward hh+{ft or '-':6s} backward hh+{bt or '-':6s}: "
              f"max rel weight err after {epochs} epochs {err:.2e}", flush=True)


if __name__ == "__main__":
    run(*(int(a) for a in sys.argv[1:3]), *(float(a) for a in sys.argv[3:4]))
