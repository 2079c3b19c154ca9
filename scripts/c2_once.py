"""One C2 forward (recurrence only) for ncu source-level captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

cfg = dict(H=2304, B=4, d=0.3, T=256)
if len(sys.argv) > 1 and sys.argv[1] == "C5":
    cfg = dict(H=5760, B=64, d=0.1, T=64)
prob = inputs.make_problem(cfg["H"], cfg["H"], cfg["B"], cfg["T"], cfg["d"])
m = from_problem(prob, prec="fp16")
x = torch.from_numpy(prob["x"]).cuda()
bp = m.input_projection(x)
y = torch.empty(cfg["T"], cfg["B"], cfg["H"], device="cuda")
for _ in range(2):
    m.recurrence(bp, y=y)
torch.cuda.synchronize()
m.status()
print(m.info())
