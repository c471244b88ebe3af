"""The C-ABI library loads and exports exactly what include/glycemlp_cuda.h declares."""

import ctypes
import re

from conftest import ROOT

import paper_1908_07847_b200._lib as L


def declared_symbols():
    text = (ROOT / "include" / "glycemlp_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(glx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("glx_run_train_segment", "glx_eval_counts", "glx_train_online", "glx_train_sweep",
                 "glx_train_batch", "glx_batch_grad", "glx_batch_apply", "glx_eval", "glx_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(str(L.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"
    # and the ctypes signature table covers the same set
    assert sorted(L.SIGNATURES) == declared_symbols()


def test_host_queries_without_device(built):
    lib = L.load(require_device=False)
    assert lib.glx_version() >= 100
    assert lib.glx_packed_ld(33) == 36 and lib.glx_packed_ld(7) == 12 and lib.glx_packed_ld(30) == 36
    assert lib.glx_batch_grad_len(33, 256) == 256 * 34 + 257 + 5
    assert lib.glx_device_count() >= 0


def test_error_codes_map_to_reference_exceptions(built):
    import pytest

    from paper_1908_07847_b200.errors import ShapeError, ValidationError

    lib = L.load(require_device=False)
    rc = lib.glx_train_online(None, None, None, None, 10, 0, 4, 1, 0.1, 0, None)  # input_dim 0
    assert rc == L.GLX_ERR_SHAPE
    with pytest.raises(ShapeError):
        L.check(rc)
    rc = lib.glx_train_online(None, None, None, None, 10, 4, 4, -1, 0.1, 0, None)  # negative epochs
    assert rc == L.GLX_ERR_INVALID
    with pytest.raises(ValidationError):
        L.check(rc)


def test_nccl_bound_at_run_time_to_the_loaded_copy(built):
    """The library has no link-time libnccl dependency (a system libnccl loaded first
    would shadow torch's newer one); glx_dp_unique_id binds the copy torch loaded."""
    import subprocess

    import numpy as np

    ldd = subprocess.run(["ldd", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    assert "nccl" not in ldd
    lib = L.load(require_device=False)
    uid = np.zeros(128, np.uint8)
    assert lib.glx_dp_unique_id(L.ptr(uid)) == 0 and uid.any()
    maps = [l for l in open("/proc/self/maps").read().splitlines() if "libnccl" in l]
    assert maps and all("nvidia/nccl" in l for l in maps), maps  # torch's bundled copy only
    assert lib.glx_dp_train_batch(None, None, None, None, 10, 10, 33, 256, 1, 0.1, None, None, None) == L.GLX_ERR_INVALID
