"""Per-instance API on the device (network.forward / predict / loss_gradients /
backprop_update, reference network.py:100-197), modelled on the reference's
tests/test_network.py, checked against the oracle's row forward and one-row
online step and against an f64 restatement of the reference's gradient code."""

import numpy as np
import pytest

import paper_1908_07847_b200 as g
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_zero_weights_give_half(gpu):
    cfg = g.NetworkConfig(input_dim=4, hidden_dim=3)
    net = g.Network(cfg, np.zeros(cfg.w_ih_len, np.float32), np.zeros(cfg.w_ho_len, np.float32))
    acts = g.forward(net, [0.3, -1.2, 0.0, 2.0])
    assert acts.hidden.tolist() == [0.5, 0.5, 0.5] and acts.output.tolist() == [0.5]


def test_1_1_1_hand_evaluation(gpu):
    cfg = g.NetworkConfig(input_dim=1, hidden_dim=1)
    net = g.Network(cfg, np.array([1.0, 0.0], np.float32), np.array([1.0, 0.0], np.float32))
    assert abs(float(g.forward(net, [0.0]).output[0]) - 0.6224593312018546) < 1e-6


@pytest.mark.parametrize("D,H,seed", [(33, 33, 7), (30, 30, 1), (7, 19, 3), (33, 256, 0), (5, 40, 2)])
def test_forward_matches_oracle_bitwise(gpu, D, H, seed):
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=seed))
    x = np.random.default_rng(seed).random(D, dtype=np.float32)
    acts = g.forward(net, x)
    h, o = O.forward_row(net.w_ih2d, net.w_ho2d, x)
    assert acts.hidden.tobytes() == h.tobytes() and acts.output.tobytes() == o.tobytes()


def test_predict_boundary_and_batch(gpu):
    cfg = g.NetworkConfig(input_dim=2, hidden_dim=2)
    zero = g.Network(cfg, np.zeros(cfg.w_ih_len, np.float32), np.zeros(cfg.w_ho_len, np.float32))
    assert g.predict(zero, [0.0, 0.0]) == g.POOR  # output exactly 0.5
    hi = g.Network(cfg, np.zeros(cfg.w_ih_len, np.float32), np.array([0.0, 0.0, 3.0], np.float32))
    lo = g.Network(cfg, np.zeros(cfg.w_ih_len, np.float32), np.array([0.0, 0.0, -3.0], np.float32))
    assert g.predict(hi, [0.1, 0.9]) == g.POOR and g.predict(lo, [0.1, 0.9]) == g.GOOD
    net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=4))
    X, lab = g.synthetic_arrays(500, 33, 1, "planted-linear")
    pb = g.predict_batch(net, X)
    assert [g.POOR if p else g.GOOD for p in pb[:20]] == [g.predict(net, X[i]) for i in range(20)]
    (tp, tn, fp, fn), _ = O.eval_counts(net.w_ih2d, net.w_ho2d, X, lab)
    assert int(pb.sum()) == tp + fp


def _ref_gradients(net, x, t):
    """f64 restatement of network.loss_gradients (network.py:144-165)."""
    h, o = O.forward_row(net.w_ih2d, net.w_ho2d, x)
    od = float(o[0])
    d_o = ((od - float(t)) * od) * (1.0 - od)
    hd = h.astype(np.float64)
    g_ho = np.concatenate([d_o * hd, [d_o]])[None, :]
    err_h = net.w_ho2d[0, :-1].astype(np.float64) * d_o
    d_h = (err_h * hd) * (1.0 - hd)
    g_ih = np.hstack([d_h[:, None] * x.astype(np.float64)[None, :], d_h[:, None]])
    return g_ih, g_ho, 0.5 * (float(t) - od) ** 2


@pytest.mark.parametrize("D,H,t", [(33, 33, 1), (7, 19, 0), (4, 1, 1)])
def test_loss_gradients_match_reference_formula(gpu, D, H, t):
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=D + H))
    before = (net.w_ih.tobytes(), net.w_ho.tobytes())
    x = np.random.default_rng(H).random(D, dtype=np.float32)
    g_ih, g_ho, err = g.loss_gradients(net, x, t)
    r_ih, r_ho, r_err = _ref_gradients(net, x, t)
    assert g_ih.shape == (H, D + 1) and g_ho.shape == (1, H + 1)
    assert g_ih.tobytes() == r_ih.tobytes() and g_ho.tobytes() == r_ho.tobytes() and err == r_err
    assert (net.w_ih.tobytes(), net.w_ho.tobytes()) == before  # no side effect


def test_backprop_update_is_one_reference_row_step(gpu):
    net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7))
    ref = net.copy()
    x = np.random.default_rng(1).random(33, dtype=np.float32)
    err = g.backprop_update(net, x, 1.0, lr=0.3)
    _, o = O.forward_row(ref.w_ih2d, ref.w_ho2d, x)
    O.train_online_seq(ref.w_ih2d, ref.w_ho2d, x[None, :], np.array([1.0], np.float32), 1, 0.3)
    assert net.w_ih.tobytes() == ref.w_ih.tobytes() and net.w_ho.tobytes() == ref.w_ho.tobytes()
    assert err == 0.5 * (1.0 - float(o[0])) ** 2


def test_backprop_update_contract(gpu):
    net = g.init_weights(g.NetworkConfig(input_dim=4, seed=5))
    before = (net.w_ih.tobytes(), net.w_ho.tobytes())
    g.backprop_update(net, [0.1, 0.2, 0.3, 0.4], 1.0, lr=0.0)
    assert (net.w_ih.tobytes(), net.w_ho.tobytes()) == before
    one = g.init_weights(g.NetworkConfig(input_dim=1, hidden_dim=1, seed=2))
    errors = [g.backprop_update(one, [1.0], 1.0, lr=0.1) for _ in range(30)]
    assert all(b < a for a, b in zip(errors, errors[1:]))
    with pytest.raises(g.ValidationError):
        g.backprop_update(net, [0.1, 0.2, 0.3, 0.4], 0.5)
    with pytest.raises(g.ShapeError):
        g.forward(net, [0.1, 0.2])


# ------------------------------------------------------- layer-level API
def _np_activation(W, x):
    """f64 restatement of kernels._activation for every neuron (kernels.py:102-122)."""
    from oracle import oracle as O

    n, m1 = W.shape
    out = np.empty(n, np.float32)
    for j in range(n):
        acc = 0.0
        for b0 in range(0, m1 - 1, 16):
            part = 0.0
            for i in range(b0, min(b0 + 16, m1 - 1)):
                part += float(W[j, i]) * float(x[i])
            acc += part
        out[j] = np.float32(O.sigmoid64(acc + float(W[j, m1 - 1])))
    return out


def test_layer_forward_backward_backprop_error(gpu):
    rng = np.random.default_rng(9)
    W = rng.uniform(-0.5, 0.5, (37, 34)).astype(np.float32)
    x = rng.random(33, dtype=np.float32)
    job = g.LayerJob.create(W, x)
    out = g.run_layer_forward(job, g.sequential())
    assert out is job.outputs and out.tobytes() == _np_activation(W, x).tobytes()
    err = rng.normal(size=37)
    deltas, grads = g.run_layer_backward(job, err, g.sequential())
    a = out.astype(np.float64)
    want_d = (err * a) * (1.0 - a)
    assert deltas.tobytes() == want_d.tobytes()
    want_g = np.hstack([want_d[:, None] * x.astype(np.float64)[None, :], want_d[:, None]])
    assert grads.tobytes() == want_g.tobytes()
    ep = g.backpropagate_error(W, deltas, g.sequential())
    want_e = np.empty(33)
    for i in range(33):
        acc = 0.0
        for b0 in range(0, 37, 16):
            part = 0.0
            for j in range(b0, min(b0 + 16, 37)):
                part += float(W[j, i]) * deltas[j]
            acc += part
        want_e[i] = acc
    assert ep.tobytes() == want_e.tobytes()
    with pytest.raises(g.ShapeError):
        g.LayerJob(W, x[:5], np.empty(37, np.float32))
    with pytest.raises(g.ShapeError):
        g.run_layer_backward(job, err[:3], g.sequential())
