"""Debug helper: one forward of a small problem (python scripts/dbg_tma.py H B T d prec)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

H, B, T, d, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), sys.argv[5]
flags = int(sys.argv[6]) if len(sys.argv) > 6 else 0
prob = inputs.make_problem(H, H, B, T, d, act="relu")
m = from_problem(prob, prec=prec, flags=flags)
print(m.info())
out = m.forward(torch.from_numpy(prob["x"]).cuda())
torch.cuda.synchronize()
m.status()
ref = oracle.forward(prob)
print("err", float(np.abs(out[0].cpu().numpy() - ref["y"]).max()))
