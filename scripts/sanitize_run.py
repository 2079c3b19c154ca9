"""Small end-to-end runs of the hot path for compute-sanitizer (SURVEY.md Sec. 5,
race detection / sanitizers): every kernel of the library (fp32 SIMT GEMM,
f32->f16 + tcgen05 GEMM, the opt-in 3xTF32 GEMM, sparse persistent kernel
RNN/LSTM/GRU in both precisions and batch tiles 1/4/8, the dense tensor-core
comparator) runs once through
srnn_forward_host (host buffers, no torch kernels), and is checked against the
oracle so an instrumented run that silently changes results also fails.

usage: compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SRNN_TIMEOUT_MS", "600000")  # instrumented kernels are slow: no watchdog trips

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1804_10223_b200 import FLAG_DENSE_TC, from_problem, inputs  # noqa: E402
from paper_1804_10223_b200._lib import FLAG_FP32_TC_GEMM  # noqa: E402

CASES = [
    (dict(H=256, I=256, B=1, T=6, density=0.10, act="relu"), "fp32", 0),
    (dict(H=300, I=200, B=4, T=5, density=0.05, act="tanh", h0="random"), "fp16", 0),
    (dict(H=333, I=333, B=8, T=4, density=0.10, act="relu"), "fp16", 0),
    (dict(H=128, I=96, B=3, T=4, density=0.125, cell="lstm", pattern="row_balanced", h0="random",
          c0="random"), "fp32", 0),
    (dict(H=160, I=160, B=4, T=4, density=0.125, cell="lstm", pattern="row_balanced"), "fp16", 0),
    (dict(H=300, I=300, B=4, T=4, density=0.2, act="tanh"), "fp16", FLAG_DENSE_TC),
    (dict(H=200, I=120, B=3, T=4, density=0.1, cell="gru", h0="random"), "fp32", 0),
    (dict(H=200, I=120, B=8, T=4, density=0.1, cell="gru"), "fp16", 0),
    (dict(H=256, I=200, B=2, T=4, density=0.1, act="tanh"), "fp32", FLAG_FP32_TC_GEMM),
]
TOL = {"fp32": 1e-5, "fp16": 2e-2}
TOL_FLAGS = {FLAG_FP32_TC_GEMM: 5e-5}  # the opt-in 3xTF32 projection's documented error

bad = 0
for cfg, prec, flags in CASES:
    prob = inputs.make_problem(**cfg)
    m = from_problem(prob, prec=prec, flags=flags)
    out = m.forward_host(prob["x"], prob["h0"], prob.get("c0"))
    m.status()
    m.close()
    ref = oracle.forward(prob)
    err = float(np.abs(out[0].astype(np.float64) - ref["y"]).max())
    ok = err <= TOL_FLAGS.get(flags, TOL[prec])
    bad += not ok
    print(f"sanitize {cfg} {prec} flags={flags}: max-abs err {err:.3e} {'ok' if ok else 'FAIL'}", flush=True)
sys.exit(1 if bad else 0)
