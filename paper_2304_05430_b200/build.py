"""Build libtt_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2304_05430_b200.build [-v]

Each csrc/*.cu is compiled to an object in parallel (-gencode
arch=compute_100a,code=sm_100a -O3 -lineinfo), then linked into
paper_2304_05430_b200/libtt_b200.so (static cudart, no torch dependency).
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libtt_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (set NVCC or install CUDA 12.9)")


def _stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "tt_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if not _stale(src, obj):
        return obj
    cmd = [nvcc(), *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = obj + ".ptxas.txt"
    with open(log, "w") as fh:
        fh.write(r.stderr)
    if verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def _build_host_module(name: str, src_name: str, force: bool, numpy_inc: bool) -> str:
    import sysconfig

    src = os.path.join(CSRC, "host", src_name)
    out = os.path.join(PKG, name + sysconfig.get_config_var("EXT_SUFFIX"))
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    cc = os.environ.get("CC") or shutil.which("gcc") or "cc"
    cmd = [cc, "-O3", "-shared", "-fPIC", "-Wall", "-pthread", "-I", sysconfig.get_paths()["include"]]
    if numpy_inc:
        import numpy

        cmd += ["-I", numpy.get_include()]
    cmd += [src, "-o", out + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host module {name} build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(out + ".tmp", out)
    return out


def build_host(force: bool = False) -> str:
    """The CPython host modules: csrc/host/tt_pack.c -> _ttpack (K9 packer) and
    csrc/host/tt_jsonl.c -> _ttjsonl (dataset record codec), gcc -O3."""
    _build_host_module("_ttjsonl", "tt_jsonl.c", force, numpy_inc=False)
    return _build_host_module("_ttpack", "tt_pack.c", force, numpy_inc=True)


def build(verbose: bool = False, force: bool = False) -> str:
    build_host(force)
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if os.path.exists(LIB) and not force:
        lt = os.path.getmtime(LIB)
        if all(os.path.getmtime(o) <= lt for o in objs):
            return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
