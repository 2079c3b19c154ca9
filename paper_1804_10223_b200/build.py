"""Build libsrnn.so (the C-ABI library) in-tree for sm_100a.

Every .cu/.cpp under csrc/ is compiled with nvcc
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (objects in
parallel) and linked into ``paper_1804_10223_b200/libsrnn.so`` with the CUDA
runtime linked statically, so the library loads on a host without a GPU
(no CUDA call happens at load time).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsrnn.so")
# diagnostics build with the per-phase timestamps (SRNN_FLAG_PROFILE, scripts/timeline.py)
PROFILE_OBJ = os.path.join(PKG, "_build_profile")
PROFILE_LIB = os.path.join(PKG, "libsrnn_profile.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def _deps():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _flags_stamp(extra):
    """Sidecar recording the experiment flags an object was built with (A/B builds)."""
    return hashlib.sha1(" ".join(extra).encode()).hexdigest()[:16]


def _compile(src, verbose=False, obj_dir=OBJ, variant_flags=()):
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    extra = list(variant_flags)
    only = os.environ.get("SRNN_NVCC_FLAGS_ONLY", "")  # comma list of source-name substrings the flags apply to
    if not only or any(t and t in os.path.basename(src) for t in only.split(",")):
        extra += os.environ.get("SRNN_NVCC_FLAGS", "").split()  # A/B experiments (e.g. -DSRNN_LOADK_BT4=3)
    stamp = _flags_stamp(extra)
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(d) for d in _deps()])
    try:
        same_flags = open(obj + ".flags").read().strip() == stamp
    except OSError:
        same_flags = False
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep and same_flags:
        return obj, ""
    cmd = [nvcc()] + ARCH + extra + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                             "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj + ".tmp"]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    else:
        cmd += ["-x", "cu"] if False else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    with open(obj + ".flags", "w") as f:
        f.write(stamp)
    with open(obj + ".ptxas.log", "w") as f:
        f.write(r.stderr)
    return obj, r.stderr


def build(verbose: bool = False, jobs: int | None = None, profile: bool = False) -> str:
    """Compile and link libsrnn.so (profile=True: libsrnn_profile.so with -DSRNN_PROFILE)."""
    obj_dir, lib, vflags = (PROFILE_OBJ, PROFILE_LIB, ("-DSRNN_PROFILE",)) if profile else (OBJ, LIB, ())
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    jobs = jobs or max(1, os.cpu_count() or 1)
    logs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = []
        for obj, log in ex.map(lambda s: _compile(s, verbose, obj_dir, vflags), srcs):
            objs.append(obj)
            logs.append(log)
    with open(os.path.join(obj_dir, "ptxas.log"), "w") as f:
        for o in objs:
            if os.path.exists(o + ".ptxas.log"):
                f.write(open(o + ".ptxas.log").read())
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(lib) or os.path.getmtime(lib) < newest:
        cmd = [nvcc()] + ARCH + ["-shared", "-o", lib + ".tmp"] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(lib + ".tmp", lib)
    if verbose:
        print(lib)
    return lib


if __name__ == "__main__":
    build(verbose=True, profile="--profile" in sys.argv)
    sys.exit(0)
