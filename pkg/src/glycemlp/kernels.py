"""glycemlp.kernels on the device: the reference's hot-path kernel entry points
(/root/reference/pkg/src/glycemlp/kernels.py) with their signatures, each one
call into libglycemlp_cuda.so.

  train_segment_seq(w_ih2d, w_ho2d, feats2d, targets, epochs, lr)      kernels.py:264-295
  train_segment_par(w_ih2d, w_ho2d, feats2d, targets, epochs, lr, ...) kernels.py:298-349
  eval_counts(w_ih2d, w_ho2d, feats2d, labels) -> (tp, tn, fp, fn)     kernels.py:352-375

Both training entry points run the reference-order (ref64) device engine and
update the weights in place; the parallel one's worker/scratch arguments are
accepted and unused (one CUDA thread per hidden neuron replaces the worker pool).
"""

from __future__ import annotations

from paper_1908_07847_b200.backend import eval_counts as _eval_counts
from paper_1908_07847_b200.backend import parallel, run_train_segment, sequential

BLOCK = 16  # kernels.py:31: the blocked-f64 accumulation width the device engine reproduces


def train_segment_seq(w_ih2d, w_ho2d, feats2d, targets, epochs, lr) -> None:
    run_train_segment(w_ih2d, w_ho2d, feats2d, targets, int(epochs), float(lr), sequential())


def train_segment_par(w_ih2d, w_ho2d, feats2d, targets, epochs, lr, *unused) -> None:
    run_train_segment(w_ih2d, w_ho2d, feats2d, targets, int(epochs), float(lr), parallel(1))


def eval_counts(w_ih2d, w_ho2d, feats2d, labels) -> tuple[int, int, int, int]:
    return _eval_counts(w_ih2d, w_ho2d, feats2d, labels, sequential())
