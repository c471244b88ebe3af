"""Build libglycemlp_cuda.so in-tree for sm_100a (explicit nvcc, no JIT cache).

The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build"
LIB = PKG / "libglycemlp_cuda.so"
SOURCES = ("glx_online.cu", "glx_batch.cu", "glx_batch3.cu", "glx_batchtc.cu", "glx_eval.cu", "glx_tc.cu", "glx_data.cu", "glx_generic.cu", "glx_abi.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL is bound at run time (dlopen in glx_abi.cu), so the library never pins a
# libnccl.so.2 that could shadow the one torch loads
LINK = ["-ldl"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(exe).exists():
        raise RuntimeError("nvcc not found; cannot build libglycemlp_cuda.so")
    return exe


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    BUILD.mkdir(exist_ok=True)
    objs = []
    jobs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *headers]):
            cmd = [nvcc(), *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
            jobs.append((src, cmd, BUILD / (Path(src).stem + ".ptxas.log")))

    def run(job):
        src, cmd, log = job
        p = subprocess.run(cmd, capture_output=True, text=True)
        log.write_text(p.stdout + p.stderr)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr[-4000:]}")
        return src

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for src in ex.map(run, jobs):
                if verbose:
                    print(f"compiled {src}")
    if force or jobs or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), *LINK]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr[-4000:]}")
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
