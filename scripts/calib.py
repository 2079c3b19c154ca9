"""Planner cost-model calibration (GPU): for a grid of problems and every forced
lanes-per-row L, record the planner's cost-model components (SRNN_PLAN_LOG) and
the measured recurrence time per step.  Used to fit the constants in
cost_model() (srnn_api.cpp); results under profiles/calib_r*.jsonl.

usage: python scripts/calib.py [--quick] > gpurun_out/calib.jsonl
"""
import argparse
import json
import os
import re
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SRNN_PLAN_LOG"] = "1"
import torch  # noqa: E402

from paper_1804_10223_b200 import SrnnError, from_problem, inputs  # noqa: E402

COST = re.compile(r"srnn cost: (.*)")


def capture_stderr(fn):
    """Run fn() with C-level stderr redirected to a temp file; return (result, text)."""
    sys.stderr.flush()
    saved = os.dup(2)
    with tempfile.TemporaryFile(mode="w+b") as f:
        os.dup2(f.fileno(), 2)
        try:
            r = fn()
        finally:
            os.dup2(saved, 2)
            os.close(saved)
        f.seek(0)
        return r, f.read().decode(errors="replace")


def t_events(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    T = 128
    probs = [(1152, 0.1, 4, "rnn"), (2304, 0.25, 4, "rnn"), (2304, 0.1, 1, "rnn"), (3072, 0.140625, 4, "rnn"),
             (4096, 0.0791, 4, "rnn"), (4096, 0.3, 4, "rnn"), (5760, 0.04, 4, "rnn"), (5760, 0.3, 1, "rnn"),
             (5760, 0.1, 4, "rnn"), (2304, 0.1, 16, "rnn"), (9216, 0.0156, 4, "rnn"), (1792, 0.3, 8, "rnn"),
             (1024, 0.1, 4, "lstm"), (2048, 0.05, 4, "lstm"), (1536, 0.1, 1, "lstm")]
    if a.quick:
        probs = probs[:3]
    for H, d, B, cell in probs:
        prob = inputs.make_problem(H, H, B, T, d, cell=cell)
        for L in (32, 16, 8, 4, 2):
            rec = {"H": H, "density": d, "B": B, "cell": cell, "L": L}
            try:
                m, log = capture_stderr(lambda: from_problem(prob, prec="fp16", lanes_per_row=L))
            except SrnnError as e:
                rec["error"] = str(e)[:120]
                print(json.dumps(rec), flush=True)
                continue
            inf = m.info()
            comps = []
            for line in log.splitlines():
                mm = COST.search(line)
                if not mm:
                    continue
                kv = dict(x.split("=") for x in mm.group(1).split())
                kv = {k: float(v) for k, v in kv.items()}
                if (int(kv["C"]) == inf["num_ctas"] and int(kv["threads"]) == inf["threads_per_cta"]
                        and int(kv["inst"]) == inf["pairs_per_lane"]):
                    comps.append(kv)
            rec["plan"] = {k: inf[k] for k in ("num_ctas", "threads_per_cta", "pairs_per_lane", "image_slots_per_lane",
                                               "slots_used", "batch_tile", "num_batch_tiles", "units_per_cta_max",
                                               "wavefronts_per_step_max", "model_cycles_per_step", "regs_per_thread")}
            rec["cost"] = min(comps, key=lambda c: c["wf"]) if comps else None
            x = torch.from_numpy(prob["x"]).cuda()
            bp = m.input_projection(x)
            y = torch.empty(T, B, H, device="cuda")
            hT = torch.empty(B, H, device="cuda") if cell == "lstm" else None
            m.recurrence(bp, y=y)
            torch.cuda.synchronize()
            ms = t_events(lambda: m.recurrence(bp, y=y))
            m.status()
            rec["us_per_step"] = 1000 * ms / T
            rec["cycles_per_step_at_1965"] = rec["us_per_step"] * 1965
            m.close()
            del hT
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
