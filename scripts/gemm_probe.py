"""Input-projection kernel times by tile width and grid cap (run under ncu for per-kernel times):
ncu --metrics gpu__time_duration.sum python scripts/gemm_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

prob = inputs.make_problem(2304, 2304, 4, 256, 0.01)
m = from_problem(prob, prec="fp16")
for steps in (32, 256):
    xc = torch.from_numpy(prob["x"][:steps]).cuda()
    for bn in ("128", "192", "256"):
        for sms in ("4", "8", "148"):
            os.environ["SRNN_GEMM_BN"] = bn
            os.environ["SRNN_GEMM_SMS"] = sms
            for _ in range(2):
                m.input_projection(xc)
            torch.cuda.synchronize()
            print(f"M={steps * 4} BN={bn} sms={sms}", flush=True)
