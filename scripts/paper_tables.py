"""The paper's application shapes on B200 (shapes only; context, not
targets -- the paper's numbers are V100 and its batch / sequence length for Table 2 are not
stated): Table 2 NMT LSTM layers (row-balanced) and Table 3 DS2 RNN
layers (B = 1, T = 256, 12% unstructured).  Recurrent kernel only.

usage: python scripts/paper_tables.py > paper_tables.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402
from sweep import t_events  # noqa: E402

# (table, cell, H, per-row nnz or density, B, T, paper persistent ms on V100)
CASES = [("T2", "lstm", 256, 32, 4, 100, 0.33), ("T2", "lstm", 512, 32, 4, 100, 0.37),
         ("T2", "lstm", 768, 32, 4, 100, 0.48), ("T2", "lstm", 1024, 48, 4, 100, 0.55),
         ("T2", "lstm", 1024, 128, 4, 100, 0.63), ("T2", "lstm", 1448, 68, 4, 100, 0.78),
         ("T3", "rnn", 1760, 0.12, 1, 256, 0.72), ("T3", "rnn", 2560, 0.12, 1, 256, 0.89),
         ("T3", "rnn", 3072, 0.12, 1, 256, 0.94)]
for table, cell, H, dens, B, T, paper_ms in CASES:
    if table == "T2":
        d, pattern = dens / H, "row_balanced"
    else:
        d, pattern = dens, "unstructured"
    prob = inputs.make_problem(H, H, B, T, d, cell=cell, pattern=pattern)
    m = from_problem(prob, prec="fp16")
    x = torch.from_numpy(prob["x"]).cuda()
    bp = m.input_projection(x)
    y = torch.empty(T, B, H, device="cuda")
    m.recurrence(bp, y=y)
    torch.cuda.synchronize()
    ms = t_events(lambda: m.recurrence(bp, y=y), reps=10)
    m.status()
    print(json.dumps({"table": table, "cell": cell, "H": H, "density": d, "pattern": pattern, "B": B, "T": T,
                      "ours_ms": ms, "ours_us_per_step": 1000 * ms / T, "paper_v100_persistent_ms": paper_ms,
                      "paper_us_per_step_if_same_T": 1000 * paper_ms / T}), flush=True)
    m.close()
