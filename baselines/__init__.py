"""Comparators and measurement tools for bench.py -- NOT the product path.

* ``libbaseline_cublaslt.so`` (cublaslt_rnn.cu): the dense per-timestep cuBLASLt GEMM with
  a fused bias(b'_t, beta = 1) + ReLU epilogue, eager and CUDA-graph (SURVEY.md Sec. 8 d-v).
* ``mb_exchange`` (scripts/microbench_exchange.cu --floor): the all-to-all exchange floor of
  the product's exchange format with no compute (the latency term of the roofline).
"""
from __future__ import annotations

import ctypes
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LT_LIB = os.path.join(HERE, "libbaseline_cublaslt.so")
MB_EXCHANGE = os.path.join(HERE, "mb_exchange")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    return shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


def _stale(out, src):
    return not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src)


def build():
    src = os.path.join(HERE, "cublaslt_rnn.cu")
    if _stale(LT_LIB, src):
        subprocess.check_call([_nvcc()] + ARCH + ["-O2", "-shared", "-Xcompiler", "-fPIC", "-o", LT_LIB, src,
                                                  "-lcublasLt"])
    src = os.path.join(ROOT, "scripts", "microbench_exchange.cu")
    if _stale(MB_EXCHANGE, src):
        subprocess.check_call([_nvcc()] + ARCH + ["-O3", "-o", MB_EXCHANGE, src], stderr=subprocess.DEVNULL)
    return LT_LIB, MB_EXCHANGE


def cublaslt_rnn(H, B, T, reps=5):
    """Dense cuBLASLt per-step loop: dict(eager_us_per_timestep, graph_us_per_timestep, launches_per_step)."""
    lib = ctypes.CDLL(build()[0])
    e, g = ctypes.c_double(), ctypes.c_double()
    n = ctypes.c_int()
    rc = lib.lt_rnn_bench(H, B, T, reps, ctypes.byref(e), ctypes.byref(g), ctypes.byref(n))
    if rc != 0:
        raise RuntimeError(f"lt_rnn_bench failed ({rc})")
    return {"eager_us_per_timestep": e.value, "graph_us_per_timestep": g.value, "launches_per_step": n.value}


def exchange_floor(H, bt, ctas=148, threads=512):
    """Microbenchmarked per-step all-to-all of the product's fp16 exchange format (no compute)."""
    import json
    out = subprocess.run([build()[1], "--floor", str(H), str(bt), str(ctas), str(threads)], capture_output=True,
                         text=True, timeout=120, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])
