"""Quick timing of the recurrent kernel and the whole forward (dev tool).

usage: python scripts/quick_time.py [H B d T prec] [--L l] [--C c] [--flags f]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=2304)
    ap.add_argument("--B", type=int, default=4)
    ap.add_argument("--d", type=float, default=0.3)
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--cell", default="rnn")
    ap.add_argument("--pattern", default="unstructured")
    ap.add_argument("--prec", default="fp16")
    ap.add_argument("--L", type=int, default=0)
    ap.add_argument("--C", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--bt", type=int, default=0, help="SRNN_BT override (batch tile)")
    ap.add_argument("--delay", type=int, default=-1, help="SRNN_POLL_DELAY_NS")
    a = ap.parse_args()
    if a.bt:
        os.environ["SRNN_BT"] = str(a.bt)
    if a.delay >= 0:
        os.environ["SRNN_POLL_DELAY_NS"] = str(a.delay)
    prob = inputs.make_problem(a.H, a.H, a.B, a.T, a.d, cell=a.cell, pattern=a.pattern)
    m = from_problem(prob, prec=a.prec, flags=a.flags, num_ctas=a.C, lanes_per_row=a.L)
    x = torch.from_numpy(prob["x"]).cuda()
    bp = m.input_projection(x)
    y = torch.empty(a.T, a.B, a.H, device="cuda")
    for _ in range(3):
        m.recurrence(bp, y=y)
        m.forward(x, y=y)
    torch.cuda.synchronize()
    m.status()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    rec, fwd, gem = [], [], []
    for _ in range(a.reps):
        ev[0].record()
        m.recurrence(bp, y=y)
        ev[1].record()
        m.forward(x, y=y)
        ev[2].record()
        m.input_projection(x, bp)
        ev[3].record()
        torch.cuda.synchronize()
        rec.append(ev[0].elapsed_time(ev[1]))
        fwd.append(ev[1].elapsed_time(ev[2]))
        gem.append(ev[2].elapsed_time(ev[3]))
    m.status()
    rec.sort(); fwd.sort(); gem.sort()
    r = rec[len(rec) // 2]
    out = {"cfg": vars(a), "info": m.info(), "rec_ms": r, "us_per_step": 1000 * r / a.T,
           "fwd_ms": fwd[len(fwd) // 2], "gemm_ms": gem[len(gem) // 2],
           "eff_gflops": 2 * prob["nnz"] * a.B * a.T / (r * 1e-3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
