"""Build libglycemlp_cuda.so variants with different epoch-kernel knobs into variants/ (tuning only).

    python tools/build_variants.py NAME="-DKNOB=1 ..." ...

Only one source is recompiled per variant (glx_batchtc.cu, or GLX_VARIANT_SRC);
the other objects come from build/ (run the normal build first). Time a variant with
GLX_LIB=variants/lib_NAME.so python tools/batch_epoch_time.py.
"""
import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1908_07847_b200 import _build as B  # noqa: E402

VARIANTS = {name: flags for name, flags in (a.split("=", 1) for a in sys.argv[1:])}
out = ROOT / "variants"
out.mkdir(exist_ok=True)
B.build()


SRC = os.environ.get("GLX_VARIANT_SRC", "glx_batchtc.cu")


def one(name, flags):
    obj = out / f"{name}_{Path(SRC).stem}.o"
    cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *flags.split(), "-c", str(B.CSRC / SRC), "-o", str(obj)]
    subprocess.run(cmd, check=True, capture_output=True)
    objs = [str(obj) if src == SRC else str(B.BUILD / (Path(src).stem + ".o")) for src in B.SOURCES]
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out / f"lib_{name}.so"), *objs, *B.LINK], check=True)
    return name


with cf.ThreadPoolExecutor(4) as ex:
    for n in ex.map(lambda kv: one(*kv), VARIANTS.items()):
        print("built", n)
