"""Build librecd.so (in-tree) with nvcc for sm_100a.

    python -m paper_2211_05239_b200.build [--force]

The shared library is the product: a torch-free C ABI (`include/recd.h`)
loaded by `paper_2211_05239_b200._lib` through ctypes.  cudart is linked
statically so the library does not depend on torch's bundled runtime.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "librecd.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps(src: Path):
    return [src] + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "recd.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None,
          tag: str = "") -> Path:
    """Compile csrc/*.cu and link librecd.so (or `out` for a tuning variant
    built with extra -D `defines`, objects kept under build/obj<tag>)."""
    obj_dir = OBJ.parent / f"obj{tag}" if tag else OBJ
    lib = Path(out) if out else LIB
    obj_dir.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in sources():
        obj = obj_dir / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, _deps(src)):
            cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                print(err, file=sys.stderr)
    if force or jobs or _stale(lib, objs):
        lib.parent.mkdir(parents=True, exist_ok=True)
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)]
        run(cmd)
    return lib


def build_host(force: bool = False) -> Path:
    """Compile the native host-side packer (CPython C API, g++)."""
    import sysconfig
    src = CSRC / "host" / "recd_hostpack.cpp"
    out = PKG / ("_hostpack" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or _stale(out, [src]):
        cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared", "-fPIC",
               f"-I{sysconfig.get_paths()['include']}", str(src), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


def build_host_lib(force: bool = False) -> Path:
    """Compile librecd_host.so (plain C ABI, g++ + threads): the row-delta
    encoder of the H2D path (include/recd_host.h)."""
    src = CSRC / "host" / "recd_rowcode.cpp"
    out = PKG / "librecd_host.so"
    if force or _stale(out, [src, ROOT / "include" / "recd_host.h"]):
        cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared",
               "-fPIC", "-pthread", str(src), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    build_host(force="--force" in sys.argv)
    build_host_lib(force="--force" in sys.argv)
    lib = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(lib)
