"""Stage timeline of the pipelined srnn_forward_host (SRNN_PIPE_TRACE=1 events, printed by the library)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import FLAG_RESERVE_SMS, from_problem, inputs  # noqa: E402

prob = inputs.make_problem(2304, 2304, 4, 256, 0.3)
m = from_problem(prob, prec="fp16", flags=FLAG_RESERVE_SMS)
xh = torch.from_numpy(prob["x"]).pin_memory()
yh = torch.empty(256, 4, 2304).pin_memory()
hh = torch.empty(4, 2304).pin_memory()
for i in range(4):
    t0 = time.perf_counter()
    m.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())
    print(f"--- call {i}: wall {1e6 * (time.perf_counter() - t0):.1f} us", file=sys.stderr, flush=True)
