"""Min-max normalisation (reference dataset.py:369-410).

CPU: the oracle restatement reproduces the reference's outputs recorded in
tests/golden/normalize_cases.npz bit for bit. GPU: glx_minmax_fit /
glx_minmax_apply / glx_pack_rows_minmax (csrc/glx_data.cu) reproduce them too,
and agree with the oracle at 1M rows.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = np.load(Path(__file__).parent / "golden" / "normalize_cases.npz")
CASES = ("paper", "cohort", "edge")


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_golden(case):
    mn, mx = O.normalize_fit(GOLD[f"{case}_train_raw"])
    assert mn.tobytes() == GOLD[f"{case}_col_min"].tobytes()
    assert mx.tobytes() == GOLD[f"{case}_col_max"].tobytes()
    for side in ("train", "test"):
        y = O.normalize_apply(GOLD[f"{case}_{side}_raw"], mn, mx)
        assert y.tobytes() == GOLD[f"{case}_{side}_norm"].tobytes()


def test_golden_covers_edges():
    assert (GOLD["edge_col_min"] == GOLD["edge_col_max"]).any()  # constant column -> 0
    te = GOLD["edge_test_norm"]
    assert (te == 1.5).any() and (te == -0.5).any()  # both clamps exercised


def _ds(m):
    import paper_1908_07847_b200 as g

    return g.Dataset(features=np.ascontiguousarray(m, dtype=np.float32).reshape(-1),
                     labels=np.zeros(m.shape[0], np.uint8), rows=m.shape[0], columns=m.shape[1],
                     subset_tag="synthetic", row_ids=tuple(range(m.shape[0])))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_device_normalize_matches_reference_golden(gpu, case):
    import paper_1908_07847_b200 as g

    tr, te = _ds(GOLD[f"{case}_train_raw"]), _ds(GOLD[f"{case}_test_raw"])
    pair = g.normalize_split(g.SplitPair(train=tr, test=te, seed=0, fraction=0.75))
    assert pair.train.norm_stats.col_min.tobytes() == GOLD[f"{case}_col_min"].tobytes()
    assert pair.train.norm_stats.col_max.tobytes() == GOLD[f"{case}_col_max"].tobytes()
    assert pair.train.features.tobytes() == GOLD[f"{case}_train_norm"].reshape(-1).tobytes()
    assert pair.test.features.tobytes() == GOLD[f"{case}_test_norm"].reshape(-1).tobytes()


@pytest.mark.gpu
def test_device_normalize_1M_rows_vs_oracle_and_fused_pack(gpu):
    import torch

    import paper_1908_07847_b200 as g
    import paper_1908_07847_b200._lib as L

    x, lab = g.synthetic_arrays(1_000_000, 33, 0, "planted-linear")
    x = (x * np.linspace(0.5, 400.0, 33, dtype=np.float32) - 7.0).astype(np.float32)
    x[:, 4] = 3.0
    fit_rows = 750_000
    mn, mx = O.normalize_fit(x[:fit_rows])
    ref = O.normalize_apply(x, mn, mx)
    lib = L.load()
    st = torch.cuda.current_stream().cuda_stream
    X = torch.from_numpy(x).cuda()
    dmn = torch.empty(33, device="cuda")
    dmx = torch.empty(33, device="cuda")
    L.check(lib.glx_minmax_fit(X.data_ptr(), fit_rows, 33, dmn.data_ptr(), dmx.data_ptr(), st))
    assert dmn.cpu().numpy().tobytes() == mn.tobytes() and dmx.cpu().numpy().tobytes() == mx.tobytes()
    # normalisation fused into the batch row packing
    ld = int(lib.glx_packed_ld(33))
    T = torch.from_numpy(lab.astype(np.float32)).cuda()
    Xp = torch.empty((x.shape[0], ld), device="cuda")
    L.check(lib.glx_pack_rows_minmax(X.data_ptr(), T.data_ptr(), None, x.shape[0], 33, dmn.data_ptr(),
                                     dmx.data_ptr(), Xp.data_ptr(), st))
    packed = Xp.cpu().numpy()
    assert packed[:, :33].tobytes() == np.ascontiguousarray(ref).tobytes()
    assert (packed[:, 33] == 1.0).all() and (packed[:, 34] == lab).all()
    # in place (Y aliases X)
    L.check(lib.glx_minmax_apply(X.data_ptr(), x.shape[0], 33, dmn.data_ptr(), dmx.data_ptr(), X.data_ptr(), st))
    assert X.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.gpu
def test_device_normalize_wide_and_ragged_columns(gpu):
    """D > 256 (several column slices of the fit kernel) and D not a multiple of 32."""
    import paper_1908_07847_b200 as g

    rng = np.random.default_rng(3)
    for rows, cols in ((517, 300), (64, 1), (3, 33), (1, 5)):
        m = (rng.normal(size=(rows, cols)) * 50).astype(np.float32)
        st = g.normalize_fit(_ds(m))
        mn, mx = O.normalize_fit(m)
        assert st.col_min.tobytes() == mn.tobytes() and st.col_max.tobytes() == mx.tobytes()
        y = g.normalize_apply(_ds(m), st)
        assert y.features.tobytes() == O.normalize_apply(m, mn, mx).reshape(-1).tobytes()


@pytest.mark.gpu
def test_normalize_column_mismatch_raises(gpu):
    import paper_1908_07847_b200 as g

    st = g.NormStats(col_min=np.zeros(3, np.float32), col_max=np.ones(3, np.float32))
    with pytest.raises(g.ShapeError):
        g.normalize_apply(_ds(np.zeros((4, 5), np.float32)), st)


@pytest.mark.gpu
@pytest.mark.parametrize("N,D", [(1, 1), (223, 7), (1000, 33), (4099, 33), (37, 250), (100_003, 15)])
def test_pack_rows_layout(gpu, N, D):
    """glx_pack_rows / glx_pack_rows_minmax: row r = [x_r (normalised or not), 1, target, 0...]
    of glx_packed_ld(D) floats, for ragged N (tile tails) and odd D."""
    import torch

    import paper_1908_07847_b200._lib as L

    rng = np.random.default_rng(N + D)
    x = (rng.normal(size=(N, D)) * 9).astype(np.float32)
    lab = (rng.random(N) < 0.5).astype(np.uint8)
    t = lab.astype(np.float32) * 0.75
    lib = L.load()
    ld = int(lib.glx_packed_ld(D))
    st = torch.cuda.current_stream().cuda_stream
    X, T, Lb = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda(), torch.from_numpy(lab).cuda()
    mn, mx = O.normalize_fit(x)
    dmn, dmx = torch.from_numpy(mn).cuda(), torch.from_numpy(mx).cuda()
    for norm in (False, True):
        for use_t in (True, False):
            Xp = torch.full((N, ld), float("nan"), device="cuda")
            if norm:
                L.check(lib.glx_pack_rows_minmax(X.data_ptr(), T.data_ptr() if use_t else None,
                                                 None if use_t else Lb.data_ptr(), N, D, dmn.data_ptr(),
                                                 dmx.data_ptr(), Xp.data_ptr(), st))
            else:
                L.check(lib.glx_pack_rows(X.data_ptr(), T.data_ptr() if use_t else None,
                                          None if use_t else Lb.data_ptr(), N, D, Xp.data_ptr(), st))
            want = np.zeros((N, ld), np.float32)
            want[:, :D] = O.normalize_apply(x, mn, mx) if norm else x
            want[:, D] = 1.0
            want[:, D + 1] = t if use_t else lab
            assert Xp.cpu().numpy().tobytes() == want.tobytes(), (norm, use_t)
