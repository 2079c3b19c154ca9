"""ctypes binding of libsrnn.so (include/srnn.h) -- argument marshalling only.

Every computation of the hot path runs in the library's CUDA kernels; this
module only converts Python/torch/numpy arguments into the plain pointers and
sizes the C ABI takes.  There is no fallback: if libsrnn.so is missing or a
call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SRNN_LIB") or os.path.join(_PKG, "libsrnn.so")  # SRNN_LIB: A/B experiments only

SRNN_OK = 0
STATUS = {0: "SRNN_OK", -1: "SRNN_ERR_INVALID_VALUE", -2: "SRNN_ERR_NOT_ON_CHIP", -3: "SRNN_ERR_BAD_WEIGHTS",
          -4: "SRNN_ERR_STATE", -5: "SRNN_ERR_CUDA", -6: "SRNN_ERR_TIMEOUT", -7: "SRNN_ERR_UNSUPPORTED"}
CELL = {"rnn": 0, "lstm": 1, "gru": 2}
ACT = {"relu": 0, "tanh": 1, "identity": 2}
PREC = {"fp32": 0, "fp16": 1}
FLAG_GRID_SYNC = 1 << 0
FLAG_NAIVE_LAYOUT = 1 << 1
FLAG_HOST_ONLY = 1 << 2
FLAG_SIMT_GEMM = 1 << 3
FLAG_DEBUG_JITTER = 1 << 4
FLAG_FP32_STAGING = 1 << 5
FLAG_PROFILE = 1 << 6
FLAG_RESERVE_SMS = 1 << 7
FLAG_DENSE_TC = 1 << 8
FLAG_DEBUG_DROP_PUBLISH = 1 << 9
FLAG_FP32_TC_GEMM = 1 << 10
FLAG_Y_BATCH_MAJOR = 1 << 11
FLAG_CLASS_BALANCE = 1 << 12
FLAG_COLUMN_SPLIT = 1 << 13
FLAG_STAGED = 1 << 14

EXPORTED = ["srnn_plan_create", "srnn_plan_query", "srnn_load_weights", "srnn_forward", "srnn_input_projection",
            "srnn_recurrence", "srnn_forward_host", "srnn_plan_status", "srnn_plan_export_layout",
            "srnn_status_string", "srnn_version", "srnn_destroy", "srnn_plan_debug_timeline"]


class SrnnError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")
        self.code = code


class Config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("input", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("max_steps", ctypes.c_int32), ("density", ctypes.c_float), ("cell", ctypes.c_int32),
                ("act", ctypes.c_int32), ("prec", ctypes.c_int32), ("device", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("num_ctas", ctypes.c_int32), ("lanes_per_row", ctypes.c_int32),
                ("batch_tile", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("sm_count", "num_ctas", "threads_per_cta", "lanes_per_row", "pairs_per_lane", "slots_used",
                 "batch_tile", "num_batch_tiles", "units_per_cta_max", "regs_per_thread", "packed_registers",
                 "fits")] + \
               [(n, ctypes.c_int64) for n in
                ("nnz", "slots_total", "smem_bytes_per_cta", "weight_image_bytes", "wavefronts_per_step_max",
                 "wavefronts_per_step_ideal", "conflict_wavefronts", "smem_weight_bytes_per_cta",
                 "image_slots_per_lane", "model_cycles_per_step")] + \
               [(n, ctypes.c_int32) for n in
                ("dense_m_tiles", "dense_kblocks_per_warp", "dense_frags_reg", "dense_frags_smem", "spill_bytes",
                 "column_split", "column_half", "staged", "early_chunks")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsrnn.so; raises (loudly) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_1804_10223_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "srnn_plan_create": ([ctypes.POINTER(Config), ctypes.POINTER(P)], I32),
        "srnn_plan_query": ([P, ctypes.POINTER(PlanInfo)], I32),
        "srnn_load_weights": ([P, P, P, P, I64, P, P], I32),
        "srnn_forward": ([P, I32, I32, P, P, P, P, P, P, P], I32),
        "srnn_input_projection": ([P, I32, I32, P, P, P], I32),
        "srnn_recurrence": ([P, I32, I32, P, P, P, P, P, P, P], I32),
        "srnn_forward_host": ([P, I32, I32, P, P, P, P, P, P], I32),
        "srnn_plan_status": ([P], I32),
        "srnn_plan_export_layout": ([P, P, P, P, I64], I32),
        "srnn_status_string": ([I32], ctypes.c_char_p),
        "srnn_version": ([], ctypes.c_char_p),
        "srnn_destroy": ([P], I32),
        "srnn_plan_debug_timeline": ([P, P, I64, ctypes.POINTER(I64)], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(fn, code):
    if code != SRNN_OK:
        raise SrnnError(fn, code)


def _ptr(t):
    """Device/host address of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class SparseRNN:
    """One plan (srnn_plan_t) for a pruned recurrent layer.

    Names follow include/srnn.h: ``load_weights`` -> srnn_load_weights,
    ``forward`` -> srnn_forward, ``input_projection`` -> srnn_input_projection,
    ``recurrence`` -> srnn_recurrence, ``forward_host`` -> srnn_forward_host.
    """

    def __init__(self, hidden, input, batch, max_steps, density, cell="rnn", act="relu", prec="fp16",
                 device=0, flags=0, num_ctas=0, lanes_per_row=0, batch_tile=0):
        self.lib = load_library()
        self.cfg = Config(hidden, input, batch, max_steps, float(density), CELL[cell], ACT[act], PREC[prec],
                          device, flags, num_ctas, lanes_per_row, batch_tile)
        self.H, self.I, self.B_max, self.T_max = hidden, input, batch, max_steps
        self.G = {"rnn": 1, "lstm": 4, "gru": 3}[cell]
        self.cell, self.prec = cell, prec
        self.device = device
        self.flags = flags
        h = ctypes.c_void_p()
        _check("srnn_plan_create", self.lib.srnn_plan_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self.handle = h

    # -- lifecycle -------------------------------------------------------
    def close(self):
        if getattr(self, "handle", None):
            self.lib.srnn_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- weights ---------------------------------------------------------
    def load_weights(self, rowptr, col, val, wx, bias=None):
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float32)
        wx = np.ascontiguousarray(wx, dtype=np.float32)
        bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
        assert rowptr.shape == (self.G * self.H + 1,), rowptr.shape
        assert wx.shape == (self.G * self.H, self.I), wx.shape
        if bias is not None:  # GRU: [b_r; b_z; b_n; b_hn]
            assert bias.shape == ((self.G + (1 if self.cell == "gru" else 0)) * self.H,), bias.shape
        _check("srnn_load_weights", self.lib.srnn_load_weights(
            self.handle, _ptr(rowptr), _ptr(col), _ptr(val), int(col.shape[0]), _ptr(wx), _ptr(bias)))
        return self

    def info(self):
        inf = PlanInfo()
        _check("srnn_plan_query", self.lib.srnn_plan_query(self.handle, ctypes.byref(inf)))
        return inf.as_dict()

    def export_layout(self):
        inf = self.info()
        n = inf["num_ctas"] * inf["image_slots_per_lane"] * inf["threads_per_cta"]
        col = np.empty(n, np.int32)
        val = np.empty(n, np.float32)
        row = np.empty(n, np.int32)
        _check("srnn_plan_export_layout",
               self.lib.srnn_plan_export_layout(self.handle, _ptr(col), _ptr(val), _ptr(row), n))
        shape = (inf["num_ctas"], inf["image_slots_per_lane"], inf["threads_per_cta"])
        return col.reshape(shape), val.reshape(shape), row.reshape(shape)

    # -- device calls (torch tensors; stream = torch's current stream) ----
    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def _check_dev(self, t, shape, name):
        import torch
        if t is None:
            return
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")

    def _yshape(self, T, B):
        return (B, T, self.H) if self.flags & FLAG_Y_BATCH_MAJOR else (T, B, self.H)

    def forward(self, x, h0=None, c0=None, y=None, hT=None, cT=None, stream=None):
        """srnn_forward: x [T,B,I] -> y [T,B,H] ([B,T,H] with FLAG_Y_BATCH_MAJOR; allocated if None), hT [B,H]."""
        import torch
        T, B = int(x.shape[0]), int(x.shape[1])
        dev = x.device
        if y is None:
            y = torch.empty(self._yshape(T, B), dtype=torch.float32, device=dev)
        if hT is None:
            hT = torch.empty((B, self.H), dtype=torch.float32, device=dev)
        if self.G == 4 and cT is None:
            cT = torch.empty((B, self.H), dtype=torch.float32, device=dev)
        self._check_dev(x, (T, B, self.I), "x")
        self._check_dev(h0, (B, self.H), "h0")
        self._check_dev(c0, (B, self.H), "c0")
        self._check_dev(y, self._yshape(T, B), "y")
        self._check_dev(hT, (B, self.H), "hT")
        self._check_dev(cT, (B, self.H), "cT")
        _check("srnn_forward", self.lib.srnn_forward(self.handle, T, B, _ptr(x), _ptr(h0), _ptr(c0), _ptr(y),
                                                     _ptr(hT), _ptr(cT), self._stream(stream)))
        return (y, hT, cT) if self.G == 4 else (y, hT)

    def input_projection(self, x, bprime=None, stream=None):
        import torch
        T, B = int(x.shape[0]), int(x.shape[1])
        if bprime is None:
            bprime = torch.empty((T, B, self.G * self.H), dtype=torch.float32, device=x.device)
        self._check_dev(x, (T, B, self.I), "x")
        self._check_dev(bprime, (T, B, self.G * self.H), "bprime")
        _check("srnn_input_projection", self.lib.srnn_input_projection(
            self.handle, T, B, _ptr(x), _ptr(bprime), self._stream(stream)))
        return bprime

    def recurrence(self, bprime, h0=None, c0=None, y=None, hT=None, cT=None, stream=None):
        import torch
        T, B = int(bprime.shape[0]), int(bprime.shape[1])
        dev = bprime.device
        if y is None:
            y = torch.empty(self._yshape(T, B), dtype=torch.float32, device=dev)
        if hT is None:
            hT = torch.empty((B, self.H), dtype=torch.float32, device=dev)
        if self.G == 4 and cT is None:
            cT = torch.empty((B, self.H), dtype=torch.float32, device=dev)
        self._check_dev(bprime, (T, B, self.G * self.H), "bprime")
        self._check_dev(y, self._yshape(T, B), "y")
        _check("srnn_recurrence", self.lib.srnn_recurrence(self.handle, T, B, _ptr(bprime), _ptr(h0), _ptr(c0),
                                                           _ptr(y), _ptr(hT), _ptr(cT), self._stream(stream)))
        return (y, hT, cT) if self.G == 4 else (y, hT)

    def forward_host(self, x, h0=None, c0=None, y=None, hT=None, cT=None):
        """srnn_forward_host on numpy (or pinned torch CPU) buffers; synchronous."""
        T, B = int(x.shape[0]), int(x.shape[1])
        if y is None:
            y = np.empty(self._yshape(T, B), np.float32)
        if hT is None:
            hT = np.empty((B, self.H), np.float32)
        if self.G == 4 and cT is None:
            cT = np.empty((B, self.H), np.float32)
        for a in (x, h0, c0, y, hT, cT):
            if isinstance(a, np.ndarray):
                assert a.dtype == np.float32 and a.flags.c_contiguous
        _check("srnn_forward_host", self.lib.srnn_forward_host(self.handle, T, B, _ptr(x), _ptr(h0), _ptr(c0),
                                                               _ptr(y), _ptr(hT), _ptr(cT)))
        return (y, hT, cT) if self.G == 4 else (y, hT)

    def debug_timeline(self):
        """[num_ctas, T, n_tiles, 4] clock64 stamps of the last forward (SRNN_FLAG_PROFILE)."""
        n = ctypes.c_int64()
        _check("srnn_plan_debug_timeline", self.lib.srnn_plan_debug_timeline(self.handle, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, np.int64)
        _check("srnn_plan_debug_timeline",
               self.lib.srnn_plan_debug_timeline(self.handle, _ptr(out), n.value, ctypes.byref(n)))
        return out

    def status(self):
        """srnn_plan_status after a stream sync; raises on a device-side error."""
        code = self.lib.srnn_plan_status(self.handle)
        _check("srnn_plan_status", code)


def from_problem(prob, prec="fp16", device=0, flags=0, num_ctas=0, lanes_per_row=0, batch=None, max_steps=None,
                 batch_tile=0):
    """Plan + load for a problem dict of ``paper_1804_10223_b200.inputs``."""
    m = SparseRNN(prob["H"], prob["I"], batch or prob["B"], prob["T"] if max_steps is None else max_steps,
                  prob["density"], prob["cell"], prob.get("act", "relu"), prec, device, flags, num_ctas,
                  lanes_per_row, batch_tile)
    m.load_weights(prob["rowptr"], prob["col"], prob["val"], prob["wx"], prob["bias"])
    return m
