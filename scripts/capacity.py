"""Capacity frontier (SURVEY.md Sec. 8 d-iv, a10): largest hidden size that plans fully on-chip.

Dense persistent capacity := largest H whose density-1 (dense) layer plans with this
library's register-resident format (fp16 mode: one register per weight).  Then checks
that a hidden size >= 5x that still plans on-chip at low density.
usage: python scripts/capacity.py [--B 4] [--prec fp16] [--device]  (--device: real register counts)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1804_10223_b200 import FLAG_HOST_ONLY, SparseRNN, SrnnError, inputs  # noqa: E402


def fits(H, d, B, prec, device, pattern="unstructured"):
    rowptr, col = inputs.sparse_pattern(H, H, d, pattern)
    val = np.full(len(col), 0.01, np.float32)
    try:
        m = SparseRNN(H, 8, B, 4, d, prec=prec, flags=0 if device else FLAG_HOST_ONLY)
        m.load_weights(rowptr, col, val, np.zeros((H, 8), np.float32))
        inf = m.info()
        m.close()
        return inf
    except SrnnError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=4)
    ap.add_argument("--prec", default="fp16")
    ap.add_argument("--device", action="store_true")
    ap.add_argument("--curve", action="store_true",
                    help="Fig. 2b analogue (PAPER.md:151): largest on-chip H per density, one JSON line each")
    a = ap.parse_args()
    if a.curve:
        for d in (0.0025, 0.005, 0.01, 0.02, 0.05, 0.10, 0.20, 0.30, 0.50, 1.0):
            lo, hi = 256, 65536
            if not fits(lo, d, a.B, a.prec, a.device):
                print(json.dumps({"density": d, "H_max": None}), flush=True)
                continue
            while hi - lo > 64:
                mid = (lo + hi) // 2
                if fits(mid, d, a.B, a.prec, a.device):
                    lo = mid
                else:
                    hi = mid
            print(json.dumps({"density": d, "B": a.B, "prec": a.prec, "device_checked": a.device, "H_max": lo,
                              "nnz_at_max": int(round(d * lo * lo))}), flush=True)
        return
    lo, hi = 256, 8192
    while hi - lo > 16:
        mid = (lo + hi) // 2
        if fits(mid, 1.0, a.B, a.prec, a.device):
            lo = mid
        else:
            hi = mid
    h_dense = lo
    out = {"B": a.B, "prec": a.prec, "device_checked": a.device, "H_dense_max": h_dense}
    target = 5 * h_dense
    for d in (0.02, 0.01, 0.005, 0.0025):
        inf = fits(target, d, a.B, a.prec, a.device)
        out[f"H={target} d={d}"] = None if inf is None else {k: inf[k] for k in (
            "num_ctas", "threads_per_cta", "lanes_per_row", "pairs_per_lane", "batch_tile", "regs_per_thread",
            "smem_bytes_per_cta", "nnz")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
