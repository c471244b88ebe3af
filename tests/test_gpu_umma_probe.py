"""The tcgen05 kind::tf32 operand forms glx_batchtc.cu relies on, checked on the
hardware with tools/umma_probe.cu (compiled here with nvcc): SS and TS (A from
TMEM) MMAs with K-major no-swizzle operands are exact, and the MN-major tf32 B
result is reported as a diagnostic (it produced zeros on sm_100a) -- the reason the backward GEMM
reads a transposed K-major copy of the x tile."""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_tf32_operand_forms(gpu, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "umma_probe"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                    str(ROOT / "tools" / "umma_probe.cu")], check=True, timeout=300)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=120).stdout
    rows = re.findall(r"bmode (\d) layout (\d) lbo +(\d+) sbo +(\d+) ts (\d) N (\d+): no error max err (\S+) poisoned (\d+)",
                      out)
    assert len(rows) == 7, out
    for bmode, layout, lbo, sbo, ts, n, err, poisoned in rows:
        assert int(poisoned) == 0, out  # every configuration wrote D
        if bmode == "0":
            assert float(err) == 0.0, out  # K-major B: exact (SS and TS)
        else:
            # MN-major B with tf32: a diagnostic only (the product never uses this form;
            # the probe's own operand layout may be what produces zeros)
            print(f"MN-major tf32 B (layout {layout}, N {n}): max err {err}")
