"""Per-phase timeline of the persistent kernel (SRNN_FLAG_PROFILE): where a step goes.

usage: python scripts/timeline.py [--H 2304 --B 4 --d 0.3 --T 256 --prec fp16 --L 0 --bt 0 --flags 0]
Prints median / p90 cycles per phase over CTAs and steps (skipping the first 8 steps).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the phase timestamps live in the diagnostics build only (-DSRNN_PROFILE): point the binding
# at libsrnn_profile.so before it is imported, then make sure that build is current
if not os.environ.get("SRNN_LIB"):
    _root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.environ["SRNN_LIB"] = os.path.join(_root, "paper_1804_10223_b200", "libsrnn_profile.so")
    from paper_1804_10223_b200 import build as _b  # noqa: E402
    _b.build(profile=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1804_10223_b200 import FLAG_PROFILE, from_problem, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=2304)
ap.add_argument("--B", type=int, default=4)
ap.add_argument("--d", type=float, default=0.3)
ap.add_argument("--T", type=int, default=256)
ap.add_argument("--prec", default="fp16")
ap.add_argument("--cell", default="rnn")
ap.add_argument("--pattern", default="unstructured")
ap.add_argument("--L", type=int, default=0)
ap.add_argument("--C", type=int, default=0)
ap.add_argument("--bt", type=int, default=0)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
if a.bt:
    os.environ["SRNN_BT"] = str(a.bt)
prob = inputs.make_problem(a.H, a.H, a.B, a.T, a.d, cell=a.cell, pattern=a.pattern)
m = from_problem(prob, prec=a.prec, flags=a.flags | FLAG_PROFILE, num_ctas=a.C, lanes_per_row=a.L)
x = torch.from_numpy(prob["x"]).cuda()
for _ in range(3):
    m.forward(x)
torch.cuda.synchronize()
m.status()
inf = m.info()
tl = m.debug_timeline().reshape(inf["num_ctas"], a.T, -1, 16)
nt = tl.shape[2]
flat = tl.reshape(inf["num_ctas"], a.T * nt, 16).astype(np.float64)
load = flat[:, :, 1] - flat[:, :, 0]
oper = flat[:, :, 2] - flat[:, :, 1]
op_loop = flat[:, :, 4] - flat[:, :, 1]
butterfly = flat[:, :, 5] - flat[:, :, 4]
bwait = flat[:, :, 6] - flat[:, :, 5]
bar2 = flat[:, :, 2] - flat[:, :, 6]
epi = flat[:, :, 3] - flat[:, :, 2]
gap = flat[:, 1:, 0] - flat[:, :-1, 3]
bar3 = flat[:, :, 7] - flat[:, :, 3]
loop = flat[:, 1:, 0] - flat[:, :-1, 7]
first_round = flat[:, :, 10] - flat[:, :, 0]
rounds0 = flat[:, :, 8]
rounds_max = flat[:, :, 9]
# cross-CTA skew of the publish time (globaltimer ns): per step, publish time minus the step's earliest publish
pub = flat[:, :, 11]
skew = pub - pub.min(axis=0, keepdims=True)
# per step: latest publish of step s-1 -> this CTA's load end of step s
lat = flat[:, 1:, 12] - pub.max(axis=0, keepdims=True)[:, :-1]
period = flat[:, 1:, 0] - flat[:, :-1, 0]
# staged plans (SRNN_FLAG_STAGED): early chunks staged (13), early slots operated (14)
early_load = flat[:, :, 13] - flat[:, :, 0]
early_op = flat[:, :, 14] - flat[:, :, 13]
late_wait = flat[:, :, 1] - flat[:, :, 14]
sk = 8 * nt
res = {"cfg": vars(a), "plan": {k: inf[k] for k in ("num_ctas", "threads_per_cta", "lanes_per_row", "pairs_per_lane",
                                                     "slots_used", "batch_tile", "wavefronts_per_step_max")}}
for name, v in (("load", load[:, sk:]), ("operate", oper[:, sk:]), ("op_loop", op_loop[:, sk:]),
                ("butterfly", butterfly[:, sk:]), ("bprime_wait", bwait[:, sk:]), ("barrier2", bar2[:, sk:]), ("epilogue", epi[:, sk:]), ("gap", gap[:, sk:]), ("bar3", bar3[:, sk:]), ("loop", loop[:, sk:]),
                ("first_round", first_round[:, sk:]), ("rounds0", rounds0[:, sk:]), ("rounds_max", rounds_max[:, sk:]),
                ("pub_skew_ns", skew[:, sk:]), ("lastpub_to_loaded_ns", lat[:, sk:]),
                ("tile_period", period[:, sk:])) + (
                (("early_load", early_load[:, sk:]), ("early_operate", early_op[:, sk:]), ("late_wait", late_wait[:, sk:]))
                if inf.get("staged") else ()):
    res[name] = {"median": float(np.median(v)), "p10": float(np.percentile(v, 10)), "p90": float(np.percentile(v, 90))}
print(json.dumps(res))
