"""CPU fp64 oracle for the sparse persistent RNN hot path (arXiv 1804.10223).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1804_10223_b200`` never imports it and
shares no code with it; the C source ``srnn_oracle.c`` is compiled here with
plain ``gcc -O2`` (no fast-math) into ``oracle/_build/libsrnn_oracle.so``.

Functions follow PAPER.md Eq. 1/2 (lines 43-49, Sec. 3.1), the LSTM case
study (App. B) and the GRU cell extension (R15) -- see the header of ``srnn_oracle.c`` for the
exact definitions and DESIGN.md for the readings (R1..R8) they rely on.

Inputs are the user's fp32 arrays upcast exactly to float64 (SURVEY.md
Sec. 8(c) c1).  Parity pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "srnn_oracle.c")
_BUILD = os.path.join(_HERE, "_build")
_LIB_PATH = os.path.join(_BUILD, "libsrnn_oracle.so")
_lock = threading.Lock()
_lib = None

ACT = {"relu": 0, "tanh": 1, "identity": 2}


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, -O2, no fast-math). Returns the .so path."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-fno-fast-math",
                               "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            lib.oracle_input_projection.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, P, P]
            lib.oracle_input_projection.restype = None
            lib.oracle_rnn_forward.argtypes = [ctypes.c_int32] * 3 + [P, P, P, P, P, ctypes.c_int32, P, P, P]
            lib.oracle_rnn_forward.restype = None
            lib.oracle_lstm_forward.argtypes = [ctypes.c_int32] * 3 + [P] * 10
            lib.oracle_lstm_forward.restype = None
            lib.oracle_gru_forward.argtypes = [ctypes.c_int32] * 3 + [P] * 9
            lib.oracle_gru_forward.restype = None
            _lib = lib
    return _lib


def _d(a):
    """Exact upcast to a C-contiguous float64 array (None passes through)."""
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a), dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def input_projection(x, wx, bias):
    """b'[m][r] = bias[r] + sum_i Wx[r][i] x[m][i]   (Eq. 2).

    x: [..., I] (leading dims flattened to M rows), wx: [R, I], bias: [R] or None.
    Returns float64 [..., R].
    """
    x = _d(x)
    wx = _d(wx)
    bias = _d(bias)
    lead = x.shape[:-1]
    I = x.shape[-1]
    R = wx.shape[0]
    assert wx.shape[1] == I
    xm = x.reshape(-1, I)
    M = xm.shape[0]
    out = np.empty((M, R), dtype=np.float64)
    _load().oracle_input_projection(M, I, R, _p(xm), _p(wx), _p(bias), _p(out))
    return out.reshape(*lead, R)


def _csr(rowptr, col, val):
    return (np.ascontiguousarray(rowptr, dtype=np.int64), np.ascontiguousarray(col, dtype=np.int32), _d(val))


def rnn_forward(H, rowptr, col, val, bp, h0=None, act="relu"):
    """Vanilla RNN, Eq. 2: h_t = g(U h_{t-1} + b'_t).

    bp: [T, B, H]; h0: [B, H] or None (zeros). Returns (y [T,B,H], hT [B,H]) float64.
    """
    bp = _d(bp)
    T, B, Hb = bp.shape
    assert Hb == H
    rp, cl, vl = _csr(rowptr, col, val)
    assert rp.shape[0] == H + 1
    h0 = _d(h0)
    y = np.empty((T, B, H), dtype=np.float64)
    hT = np.empty((B, H), dtype=np.float64)
    work = np.empty(2 * H, dtype=np.float64)
    _load().oracle_rnn_forward(H, B, T, _p(rp), _p(cl), _p(vl), _p(bp), _p(h0), ACT[act],
                               _p(y), _p(hT), _p(work))
    return y, hT


def lstm_forward(H, rowptr, col, val, bp, h0=None, c0=None):
    """LSTM (gate equations DESIGN.md R3): 4H CSR rows [i;f;g;o].

    bp: [T, B, 4H]. Returns (y [T,B,H], hT [B,H], cT [B,H]) float64.
    """
    bp = _d(bp)
    T, B, R = bp.shape
    assert R == 4 * H
    rp, cl, vl = _csr(rowptr, col, val)
    assert rp.shape[0] == 4 * H + 1
    h0 = _d(h0)
    c0 = _d(c0)
    y = np.empty((T, B, H), dtype=np.float64)
    hT = np.empty((B, H), dtype=np.float64)
    cT = np.empty((B, H), dtype=np.float64)
    work = np.empty(6 * H, dtype=np.float64)
    _load().oracle_lstm_forward(H, B, T, _p(rp), _p(cl), _p(vl), _p(bp), _p(h0), _p(c0),
                                _p(y), _p(hT), _p(cT), _p(work))
    return y, hT, cT


def gru_forward(H, rowptr, col, val, bp, bhn=None, h0=None):
    """GRU (cell extension, R15): 3H CSR rows [r; z; n], n-gate recurrent bias bhn [H].

    bp: [T, B, 3H]. Returns (y [T,B,H], hT [B,H]) float64.
    """
    bp = _d(bp)
    T, B, R = bp.shape
    assert R == 3 * H
    rp, cl, vl = _csr(rowptr, col, val)
    assert rp.shape[0] == 3 * H + 1
    bhn = _d(bhn)
    h0 = _d(h0)
    y = np.empty((T, B, H), dtype=np.float64)
    hT = np.empty((B, H), dtype=np.float64)
    work = np.empty(4 * H, dtype=np.float64)
    _load().oracle_gru_forward(H, B, T, _p(rp), _p(cl), _p(vl), _p(bp), _p(bhn), _p(h0), _p(y), _p(hT), _p(work))
    return y, hT


def forward(prob, act=None, quantize_fp16=False):
    """Whole hot path on a problem dict from ``paper_1804_10223_b200.inputs``.

    Input projection (Eq. 2) followed by the recurrence (RNN or LSTM).
    ``quantize_fp16`` feeds the oracle fp16-RNE-rounded W_h / W_x / x values
    (numpy rounding, outside the oracle) -- the diagnostic "quantized oracle"
    of SURVEY.md Sec. 8(c) c1, never a gate.
    Returns dict(y, hT[, cT], bp) in float64.
    """
    cell = prob["cell"]
    act = act or prob.get("act", "relu")
    val, wx, x = prob["val"], prob["wx"], prob["x"]
    if quantize_fp16:
        val = np.asarray(val, np.float32).astype(np.float16).astype(np.float64)
        wx = np.asarray(wx, np.float32).astype(np.float16).astype(np.float64)
        x = np.asarray(x, np.float32).astype(np.float16).astype(np.float64)
    H = prob["H"]
    bias = prob["bias"]
    if cell == "gru":  # bias = [b_r; b_z; b_n; b_hn] (4H): the projection takes the first 3H
        bp = input_projection(x, wx, None if bias is None else np.asarray(bias)[:3 * H])
        y, hT = gru_forward(H, prob["rowptr"], prob["col"], val, bp,
                            None if bias is None else np.asarray(bias)[3 * H:], prob.get("h0"))
        return {"y": y, "hT": hT, "bp": bp}
    bp = input_projection(x, wx, bias)
    if cell == "rnn":
        y, hT = rnn_forward(H, prob["rowptr"], prob["col"], val, bp, prob.get("h0"), act)
        return {"y": y, "hT": hT, "bp": bp}
    y, hT, cT = lstm_forward(H, prob["rowptr"], prob["col"], val, bp, prob.get("h0"), prob.get("c0"))
    return {"y": y, "hT": hT, "cT": cT, "bp": bp}
