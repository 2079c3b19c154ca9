"""A/B of the staged (partial-progress) plan vs the one-stage plan on one box.

usage: python scripts/staged_ab.py [--rounds 3] [--early 0,384,448,512,576]
Prints one JSON line per (config, variant, round): recurrence µs/step (median of 10 launches)
and the max-abs difference of y vs the one-stage plan."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

CONFIGS = [
    dict(name="C2", H=2304, B=4, d=0.30, T=256),
    dict(name="2304@10%", H=2304, B=4, d=0.10, T=256),
    dict(name="1152@10%", H=1152, B=4, d=0.10, T=256),
    dict(name="C4-lstm", H=1024, B=4, d=0.125, T=256, cell="lstm", pattern="row_balanced"),
    dict(name="B8", H=2304, B=8, d=0.30, T=256),
    dict(name="4096@5%", H=4096, B=4, d=0.05, T=256),
]


def run(cfg, staged, early, reps=10):
    os.environ["SRNN_STAGED"] = "1" if staged else "0"
    if early:
        os.environ["SRNN_EARLY_CHUNKS"] = str(early)
    else:
        os.environ.pop("SRNN_EARLY_CHUNKS", None)
    prob = inputs.make_problem(cfg["H"], cfg["H"], cfg["B"], cfg["T"], cfg["d"], cell=cfg.get("cell", "rnn"),
                               pattern=cfg.get("pattern", "unstructured"))
    m = from_problem(prob, prec="fp16")
    inf = m.info()
    x = torch.from_numpy(prob["x"]).cuda()
    bp = m.input_projection(x)
    y = torch.empty(cfg["T"], cfg["B"], cfg["H"], device="cuda")
    for _ in range(3):
        m.recurrence(bp, y=y)
    torch.cuda.synchronize()
    m.status()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.recurrence(bp, y=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / cfg["T"])
    m.status()
    ts.sort()
    out = y.clone()
    m.close()
    return ts[len(ts) // 2], out, inf


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--early", default="0")
    ap.add_argument("--configs", default="")
    a = ap.parse_args()
    earlies = [int(e) for e in a.early.split(",")]
    cfgs = [c for c in CONFIGS if not a.configs or c["name"] in a.configs.split(",")]
    for r in range(a.rounds):
        for cfg in cfgs:
            t0, y0, i0 = run(cfg, False, 0)
            print(json.dumps(dict(cfg=cfg["name"], variant="one-stage", round=r, us=t0, slots=i0["slots_used"],
                                  wf=i0["wavefronts_per_step_max"], inst=i0["pairs_per_lane"])), flush=True)
            for e in earlies:
                t1, y1, i1 = run(cfg, True, e)
                d = float((y1 - y0).abs().max())
                print(json.dumps(dict(cfg=cfg["name"], variant=f"staged{e or ''}", round=r, us=t1, staged=i1["staged"],
                                      early=i1["early_chunks"], slots=i1["slots_used"], wf=i1["wavefronts_per_step_max"],
                                      inst=i1["pairs_per_lane"], regs=i1["regs_per_thread"], maxdiff=d)), flush=True)


if __name__ == "__main__":
    main()
