"""B200 re-run of the paper's Table 1 optimisation ladder:
H = 1152, B = 4, density 10%, T = 256 -- naive -> wide loads -> bank-aware layout ->
Lamport-style flags (here: timestep-tagged words), as speedups over a per-step dense
cuBLAS loop (CUDA graph, fp16 GEMM + bias/ReLU).  The paper's "bank conflict penalty" is
undefined; the packer's predicted extra shared-memory wavefronts per step of
the busiest CTA stand in for it (they match ncu's wavefront counts).

usage: python scripts/table1.py > table1.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from paper_1804_10223_b200 import FLAG_GRID_SYNC, FLAG_NAIVE_LAYOUT, from_problem, inputs  # noqa: E402
from sweep import dense_graph_us, t_events  # noqa: E402

H, B, d, T = 1152, 4, 0.10, 256
prob = inputs.make_problem(H, H, B, T, d)
dense = dense_graph_us(H, B, T)
RUNGS = [  # (name, batch tile, flags) -- the paper's Table 1 columns, in order
    ("naive (scalar loads, CSR-order layout, grid barrier)", 1, FLAG_NAIVE_LAYOUT | FLAG_GRID_SYNC),
    ("wide loads (4 samples per LDS)", 4, FLAG_NAIVE_LAYOUT | FLAG_GRID_SYNC),
    ("bank-aware layout", 4, FLAG_GRID_SYNC),
    ("Lamport -> timestep-tagged words", 4, 0),
]
for prec in ("fp32", "fp16"):
    for name, bt, flags in RUNGS:
        m = from_problem(prob, prec=prec, flags=flags, batch_tile=bt)
        x = torch.from_numpy(prob["x"]).cuda()
        bp = m.input_projection(x)
        y = torch.empty(T, B, H, device="cuda")
        m.recurrence(bp, y=y)
        torch.cuda.synchronize()
        us = 1000 * t_events(lambda: m.recurrence(bp, y=y), reps=10) / T
        m.status()
        inf = m.info()
        print(json.dumps({"prec": prec, "rung": name, "batch_tile": inf["batch_tile"], "flags": flags,
                          "us_per_step": us, "dense_cublas_graph_us_per_step": dense, "speedup_vs_dense": dense / us,
                          "wavefronts_per_step_max": inf["wavefronts_per_step_max"] * inf["num_batch_tiles"],
                          "conflict_wavefronts": inf["conflict_wavefronts"] * inf["num_batch_tiles"]}), flush=True)
        m.close()
