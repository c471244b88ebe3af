"""Build libglycemlp_cuda.so variants with different batch-kernel knobs into variants/ (tuning only)."""
import subprocess, sys, concurrent.futures as cf
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1908_07847_b200 import _build as B

VARIANTS = {name: flags for name, flags in (a.split("=", 1) for a in sys.argv[1:])}
out = ROOT / "variants"; out.mkdir(exist_ok=True)

def one(name, flags):
    objs = []
    for src in B.SOURCES:
        obj = out / f"{name}_{Path(src).stem}.o"
        cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *flags.split(), "-c", str(B.CSRC / src), "-o", str(obj)]
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(str(obj))
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out / f"lib_{name}.so"), *objs], check=True)
    return name

with cf.ThreadPoolExecutor(4) as ex:
    for n in ex.map(lambda kv: one(*kv), VARIANTS.items()):
        print("built", n)
