"""Host-side logic of the product package (no GPU needed)."""

import hashlib
import os
import json

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1908_07847_b200 as g
from paper_1908_07847_b200 import backend as B
from paper_1908_07847_b200 import dp
from paper_1908_07847_b200.errors import ShapeError, ValidationError
from paper_1908_07847_b200.trainer import TrainSpec, default_checkpoints


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


GEN = json.loads((GOLDEN / "generators.json").read_text())


@pytest.mark.parametrize("case", GEN["synthetic_matrix"], ids=lambda c: f"{c['rows']}x{c['columns']}-{c['signal']}")
def test_synthetic_matrix_matches_reference(case):
    d = g.synthetic_matrix(case["rows"], case["columns"], case["seed"], case["signal"])
    assert sha(d.features) == case["features_sha256"]
    assert sha(d.labels) == case["labels_sha256"]


@pytest.mark.parametrize("signal", ["planted-linear", "random"])
@pytest.mark.parametrize("chunk", [1, 7, 333, 10_000])
def test_chunked_generation_is_byte_identical(signal, chunk):
    f, l = g.synthetic_arrays(1000, 33, 0, signal)
    parts = list(g.iter_synthetic_chunks(1000, 33, 0, signal, chunk_rows=chunk))
    assert [p[0] for p in parts] == list(range(0, 1000, chunk))
    assert np.concatenate([p[1] for p in parts]).tobytes() == f.tobytes()
    assert np.concatenate([p[2] for p in parts]).tobytes() == l.tobytes()


@pytest.mark.parametrize("case", GEN["init_weights"], ids=lambda c: f"{c['input_dim']}-{c['hidden_dim']}-{c['seed']}")
def test_init_weights_matches_reference(case):
    net = g.init_weights(g.NetworkConfig(input_dim=case["input_dim"], hidden_dim=case["hidden_dim"],
                                         seed=case["seed"]))
    assert sha(net.w_ih) == case["w_ih_sha256"] and sha(net.w_ho) == case["w_ho_sha256"]


def test_network_config_contract():
    assert g.NetworkConfig(input_dim=7).hidden_dim == 7
    c = g.NetworkConfig(input_dim=3, hidden_dim=4)
    assert (c.w_ih_len, c.w_ho_len) == (16, 5)
    for bad in (dict(input_dim=0), dict(input_dim=3, learning_rate=0.0), dict(input_dim=3, momentum=0.5),
                dict(input_dim=3, output_dim=2), dict(input_dim=3, hidden_dim=0)):
        with pytest.raises(ValidationError):
            g.NetworkConfig(**bad)
    with pytest.raises(ShapeError):
        g.Network(c, np.zeros(15, np.float32), np.zeros(5, np.float32))
    with pytest.raises(ShapeError):
        g.Network(c, np.zeros(16, np.float64), np.zeros(5, np.float32))


def test_checkpoint_round_trip(tmp_path):
    net = g.init_weights(g.NetworkConfig(input_dim=30, hidden_dim=17, seed=13))
    p = tmp_path / "net.json"
    g.save_checkpoint(net, p)
    back = g.load_checkpoint(p)
    assert back.w_ih.tobytes() == net.w_ih.tobytes() and back.w_ho.tobytes() == net.w_ho.tobytes()
    assert json.dumps(g.checkpoint_dict(back)) == json.dumps(g.checkpoint_dict(net))
    with pytest.raises(ValidationError):
        g.network_from_dict({"version": "nope"})


def test_sigmoid_known_answers():
    assert g.sigmoid(0.0) == 0.5
    assert abs(g.sigmoid(20.0) - 0.9999999979388463) < 1e-12


def test_backend_kind_contract():
    """The reference's names and validation (backend.py:44-70, test_backend.py:18-32) plus "cuda"."""
    assert g.cuda().name == "cuda"
    assert g.sequential().numerics == "ref64" and g.parallel(4).numerics == "ref64"
    assert B.BackendKind("sequential", 1) == g.sequential()
    assert B.BackendKind("parallel", 3).effective_workers == 3 and g.sequential().effective_workers == 1
    assert g.parallel().workers == (os.cpu_count() or 1)
    assert B.BackendKind("parallel", 2, "fp32").numerics == "ref64"  # the reference engines are exact
    for bad in (("gpu", 1), ("parallel", 0), ("cuda", 0), ("sequential", -1)):
        with pytest.raises(ValidationError):
            B.BackendKind(*bad)
    with pytest.raises(ValidationError):
        B.BackendKind("cuda", 1, "fp16")


def test_train_spec_contract():
    assert default_checkpoints(100_000) == (1, 10, 100, 1_000, 10_000, 100_000)
    assert default_checkpoints(500) == (1, 10, 100, 500)
    assert default_checkpoints(1) == (1,)
    cfg = g.NetworkConfig(input_dim=4)
    with pytest.raises(ValidationError):
        TrainSpec(config=cfg, epochs=0)
    for cps in ((1, 20), (5, 5), (0, 5)):
        with pytest.raises(ValidationError):
            TrainSpec(config=cfg, epochs=10, checkpoints=cps)
    with pytest.raises(ValidationError):
        TrainSpec(config=cfg, epochs=10, mode="minibatch")


def test_segment_shape_errors_before_device():
    net = g.init_weights(g.NetworkConfig(input_dim=4, seed=0))
    with pytest.raises(ShapeError):
        g.run_train_segment(net.w_ih2d, net.w_ho2d, np.zeros((3, 5), np.float32), np.zeros(3, np.float32), 1, 0.1,
                            g.cuda())
    with pytest.raises(ShapeError):
        g.run_train_segment(net.w_ih2d, net.w_ho2d, np.zeros((3, 4), np.float32), np.zeros(2, np.float32), 1, 0.1,
                            g.cuda())


def test_no_cpu_fallback(built):
    # on a box without a GPU every compute entry point must fail loudly
    import paper_1908_07847_b200._lib as L

    if L.load(require_device=False).glx_device_count() > 0:
        pytest.skip("a GPU is visible")
    net = g.init_weights(g.NetworkConfig(input_dim=4, seed=0))
    with pytest.raises(RuntimeError):
        g.run_train_segment(net.w_ih2d, net.w_ho2d, np.zeros((3, 4), np.float32), np.zeros(3, np.float32), 1, 0.1,
                            g.cuda())


def test_lpt_shards_balance_and_cover():
    hs, ss = g.sweep_grid(range(8, 513, 8), range(64))
    assert len(hs) == 4096
    spec = g.SweepSpec(input_dim=33, hidden_dims=hs, seeds=ss, epochs=1)
    costs = spec.costs()
    for n in (1, 2, 4, 8):
        shards = g.lpt_shards(costs, n)
        assert sorted(i for s in shards for i in s) == list(range(4096))
        loads = [costs[s].sum() for s in shards]
        assert max(loads) / (costs.sum() / n) < 1.001  # near-perfect balance on this grid
    assert g.lpt_shards([5, 1, 1, 1, 1, 1], 2) == [[0], [1, 2, 3, 4, 5]]


def test_sweep_pool_round_trip():
    from paper_1908_07847_b200.sweep import pack_pool, unpack_pool

    nets = [g.init_weights(g.NetworkConfig(input_dim=5, hidden_dim=h, seed=h)) for h in (3, 8, 1)]
    pool, H, off = pack_pool(nets)
    assert H.tolist() == [3, 8, 1] and off.tolist() == [0, 3 * 6 + 4, 3 * 6 + 4 + 8 * 6 + 9]
    copies = [n.copy() for n in nets]
    for n in copies:
        n.w_ih[:] = 0
        n.w_ho[:] = 0
    unpack_pool(pool, copies, off)
    assert all(a.w_ih.tobytes() == b.w_ih.tobytes() and a.w_ho.tobytes() == b.w_ho.tobytes()
               for a, b in zip(nets, copies))


@pytest.mark.parametrize("n,w", [(10, 3), (1, 4), (67_108_864, 8), (7, 7)])
def test_shard_bounds_partition(n, w):
    b = [dp.shard_bounds(n, w, r) for r in range(w)]
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
    assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1


@pytest.mark.parametrize("rows,cols,seed", [(120, 33, 7), (257, 5, 3), (11, 3, 5), (1000, 1, 2)])
def test_post_feature_generator_matches_reference_draws(rows, cols, seed):
    """The host half of synthetic_arrays_device: default_rng(seed) advanced past the
    float32 features (including the buffered 32-bit half when rows*cols is odd)
    draws the same planted columns and weights as synthetic_arrays."""
    from paper_1908_07847_b200.dataset import _post_feature_generator, _split128

    ref = np.random.default_rng(seed)
    ref.random((rows, cols), dtype=np.float32)
    pick = ref.choice(cols, size=min(5, cols), replace=False)
    coef = ref.normal(0.0, 1.0, size=pick.shape[0])
    gen = _post_feature_generator(seed, rows * cols)
    assert (gen.choice(cols, size=min(5, cols), replace=False) == pick).all()
    assert (gen.normal(0.0, 1.0, size=pick.shape[0]) == coef).all()
    hi, lo = _split128((1 << 127) + 5)
    assert hi == 1 << 63 and lo == 5


def test_parallel_workers_validated_and_clamped():
    """backend.py:45-62: workers >= 1, effective_workers clamped to max_workers()."""
    import pytest

    from paper_1908_07847_b200 import backend as B
    from paper_1908_07847_b200.errors import ValidationError

    assert B.max_workers() == B.hardware_parallelism()
    assert B.parallel(10 ** 6).effective_workers == B.max_workers()
    assert B.sequential().effective_workers == 1
    with pytest.raises(ValidationError):
        B.parallel(0)
    with pytest.raises(ValidationError):
        B.BackendKind("numba")


def test_wide_shard_rows_block_alignment():
    from paper_1908_07847_b200 import wide
    from paper_1908_07847_b200.errors import ShapeError

    for block in (32, 64):
        n = block * 37
        bounds = [wide.shard_rows(n, 4, r, block) for r in range(4)]
        assert bounds[0][0] == 0 and bounds[-1][1] == n
        assert all(a % block == 0 and b % block == 0 and a <= b for a, b in bounds)
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(3))
    import pytest

    with pytest.raises(ShapeError):
        wide.shard_rows(100, 2, 0, 32)


def test_glycemlp_import_surface():
    """pkg/src/glycemlp re-exports the reference's hot-path names
    (/root/reference/pkg/src/glycemlp/__init__.py:5-106) on this engine."""
    import glycemlp as G

    for name in ("train", "evaluate", "TrainSpec", "NetworkConfig", "init_weights", "sequential", "parallel",
                 "BackendKind", "forward", "predict", "backprop_update", "normalize_split", "synthetic_matrix",
                 "save_checkpoint", "load_checkpoint", "run_bench", "max_workers", "hardware_parallelism"):
        assert hasattr(G, name), name
    from glycemlp import kernels

    assert callable(kernels.train_segment_seq) and callable(kernels.eval_counts)
    import pytest

    with pytest.raises(AttributeError):
        G.parse_csv  # out of scope: host CSV plumbing
