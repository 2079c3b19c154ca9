"""Input projection (f32->f16 + tcgen05 GEMM) at C2 (M = T*B = 1024, N = K = 2304) by W_x multicast
cluster size (SRNN_GEMM_CM = 1 / 2 / 4): CUDA-event medians of 30 launches, L2 flushed between."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

prob = inputs.make_problem(2304, 2304, 4, 256, 0.01)
m = from_problem(prob, prec="fp16")
x = torch.from_numpy(prob["x"]).cuda()
bp = m.input_projection(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rnd in range(3):
    for cm in sys.argv[1:] or ["1", "2", "4", "auto"]:
        if cm == "auto":
            os.environ.pop("SRNN_GEMM_CM", None)  # the default: 144-wide tiles in 4-CTA clusters
        else:
            os.environ["SRNN_GEMM_CM"] = cm
        for _ in range(3):
            m.input_projection(x, bp)
        ts = []
        for _ in range(30):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m.input_projection(x, bp)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(json.dumps({"cm": cm, "round": rnd, "us_median": ts[15], "us_min": ts[0]}), flush=True)
