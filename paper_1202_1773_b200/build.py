"""Build libffst.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libffst.so"
SOURCES = ["ffst_api.cu", "ffst_kern_f32.cu", "ffst_kern_f64.cu", "ffst_gen_f32.cu", "ffst_gen_f64.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> Path:
    """The NCCL that torch.distributed loads (nvidia-nccl wheel): headers and libnccl.so.2.  Found
    without importing torch; the library binds to the same SONAME torch has loaded."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = Path(base) / "nccl"
        if (d / "include" / "nccl.h").exists() and (d / "lib" / "libnccl.so.2").exists():
            return d
    raise RuntimeError("NCCL (nvidia-nccl wheel: include/nccl.h, lib/libnccl.so.2) not found")


NCCL = _nccl_dir()
FLAGS = ["-std=c++17", "-O3", "--expt-relaxed-constexpr", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}", f"-I{CSRC}",
         f"-I{NCCL / 'include'}"]
EXTRA = {}   # per-source extra flags (none)


def _stale(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "ffst.h"]
    jobs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        if force or _stale(obj, headers + [CSRC / src]):
            jobs.append([NVCC, *FLAGS, *EXTRA.get(src, []), "-c", str(CSRC / src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout, r.stderr, flush=True)
        return r

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    objs = [str(BUILD / (Path(s).stem + ".o")) for s in SOURCES]
    if force or jobs or not LIB.exists():
        run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(LIB),
             f"-L{NCCL / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={NCCL / 'lib'}"])
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
