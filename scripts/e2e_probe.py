"""Where the end-to-end (host buffer) time goes at C2: copy bandwidths, the
plain and the pipelined srnn_forward_host, and the device-only forward of the
same plans.  usage: python scripts/e2e_probe.py [--H 2304 --B 4 --d 0.3 --T 256]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import FLAG_RESERVE_SMS, from_problem, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=2304)
ap.add_argument("--B", type=int, default=4)
ap.add_argument("--d", type=float, default=0.3)
ap.add_argument("--T", type=int, default=256)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()


def wall(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)


prob = inputs.make_problem(a.H, a.H, a.B, a.T, a.d)
T, B, H = a.T, a.B, a.H
xh = torch.from_numpy(prob["x"]).pin_memory()
yh = torch.empty(T, B, H).pin_memory()
hh = torch.empty(B, H).pin_memory()
xd = torch.empty_like(xh, device="cuda")
yd = torch.empty(T, B, H, device="cuda")
print(f"bytes x {xh.numel() * 4}  y {yh.numel() * 4}")
print(f"H2D x pinned            {wall(lambda: xd.copy_(xh, non_blocking=True), a.reps):8.1f} us")
print(f"D2H y pinned            {wall(lambda: yh.copy_(yd, non_blocking=True), a.reps):8.1f} us")
s2 = torch.cuda.Stream()


def both():
    xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
    s2.synchronize()


print(f"H2D || D2H              {wall(both, a.reps):8.1f} us")
for name, flags, res in (("full plan (plain path)", 0, 0), ("reserve 4 (pipelined)", FLAG_RESERVE_SMS, 4),
                         ("reserve 8 (pipelined)", FLAG_RESERVE_SMS, 8)):
    os.environ["SRNN_RESERVE_SMS"] = str(max(res, 1))
    m = from_problem(prob, prec="fp16", flags=flags)
    inf = m.info()
    xdev = torch.from_numpy(prob["x"]).cuda()

    def dev_fwd():
        m.forward(xdev, y=yd)

    def host_fwd():
        m.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())

    print(f"{name}: ctas {inf['num_ctas']}")
    print(f"   device forward (x resident)   {wall(dev_fwd, a.reps):8.1f} us")
    print(f"   forward_host (x in, y out)    {wall(host_fwd, a.reps):8.1f} us")
    m.close()

# per-chunk input projection (M = steps x B rows), all SMs free: one 128 x 128 tile per CTA
m = from_problem(prob, prec="fp16")
for steps, bn in ((32, "128"), (32, "256"), (64, "128"), (64, "256"), (256, "128"), (256, "256")):
    os.environ["SRNN_GEMM_BN"] = bn
    xc = torch.from_numpy(prob["x"][:steps]).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m.input_projection(xc)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0.record()
        m.input_projection(xc)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    print(f"input_projection M={steps * B:5d} BN={bn}: {statistics.median(ts):7.1f} us")
m.close()
