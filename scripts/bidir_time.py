"""Bidirectional layer timing: two directions sequentially on all SMs vs concurrently on
half the SMs each (two persistent kernels side by side).  usage: python scripts/bidir_time.py [H B d T]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import inputs  # noqa: E402
from paper_1804_10223_b200.layers import BiSparseRNN  # noqa: E402

H, B, d, T = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 \
    else (2304, 4, 0.3, 256)
pf = inputs.make_problem(H, H, B, T, d, seed_offset=1)
pb = inputs.make_problem(H, H, B, T, d, seed_offset=2)
x = torch.from_numpy(pf["x"]).cuda()
res = {"H": H, "B": B, "density": d, "T": T}
for conc in (False, True):
    n = torch.cuda.get_device_properties(0).multi_processor_count // 2 if conc else 0
    bi = BiSparseRNN.from_problems(pf, pb, prec="fp16", num_ctas=n)
    st = (torch.cuda.Stream(), torch.cuda.Stream()) if conc else None
    for _ in range(3):
        bi.forward(x, streams=st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bi.forward(x, streams=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    bi.status()
    res["concurrent_half_sms_ms" if conc else "sequential_all_sms_ms"] = statistics.median(ts)
    res[("concurrent" if conc else "sequential") + "_ctas"] = bi.fwd.info()["num_ctas"]
    bi.close()
print(json.dumps(res))
