"""Build libidconv.so (nvcc, sm_100a) in-tree.  Used by __graft_entry__.build()."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libidconv.so")
# debug library: the same sources with the transform counter compiled in
# (-DIDC_COUNT_FFT=1, fft_dev.cuh); used only by tests/test_transform_counts.py
OBJ_COUNT = os.path.join(HERE, "build_count")
LIB_COUNT = os.path.join(HERE, "libidconv_count.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _nccl_dirs():
    try:
        import nvidia.nccl as n  # torch's bundled NCCL (headers + libnccl.so.2)
        base = list(n.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return None, None


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "idconv.h"))
    return hs


def _deps(path, seen=None):
    """Transitive quoted #include dependencies of a source file."""
    import re
    seen = set() if seen is None else seen
    for inc in re.findall(r'^#include "([^"]+)"', open(path).read(), flags=re.M):
        dep = os.path.normpath(os.path.join(os.path.dirname(path), inc))
        if os.path.exists(dep) and dep not in seen:
            seen.add(dep)
            _deps(dep, seen)
    return seen


def _compile(src, extra, force, objdir=OBJ):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _deps(src)])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def _link(lib, objs, libdir, force):
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        link = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
        if libdir:
            link += ["-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")


def build(force: bool = False, verbose: bool = False, count_lib: bool = True) -> str:
    """Build libidconv.so (and the transform-counting debug library)."""
    inc, libdir = _nccl_dirs()
    extra = ["-I" + inc] if inc else []
    srcs = sources()
    jobs = [(s_, extra, OBJ) for s_ in srcs]
    if count_lib:
        jobs += [(s_, extra + ["-DIDC_COUNT_FFT=1"], OBJ_COUNT) for s_ in srcs]
    for d in {j[2] for j in jobs}:
        os.makedirs(d, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda j: _compile(j[0], j[1], force, j[2]), jobs))
    _link(LIB, objs[:len(srcs)], libdir, force)
    if count_lib:
        _link(LIB_COUNT, objs[len(srcs):], libdir, force)
    if verbose:
        print("built", LIB, "and", LIB_COUNT if count_lib else "")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
