"""C3 sweep (BASELINE.json configs[2]; the paper's Fig. 2/3 axes):
hidden x density x batch at T = 256, our persistent kernel vs the per-step
dense cuBLAS loop (CUDA graph) and the per-step cuSPARSE SpMM loop (eager),
plus the largest on-chip points.  Writes one JSON line per point.

usage: python scripts/sweep.py [--quick] > gpurun_out/sweep.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10223_b200 import FLAG_DENSE_TC, SrnnError, from_problem, inputs  # noqa: E402


def t_events(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def dense_graph_us(H, B, T):
    W = (torch.rand(H, H, device="cuda") - 0.5).half()
    bp = torch.rand(T, H, B, device="cuda")
    h = torch.zeros(H, B, device="cuda", dtype=torch.float16)
    z = torch.empty(H, B, device="cuda", dtype=torch.float16)

    def loop():
        hh = h
        for t in range(T):
            torch.mm(W, hh, out=z)
            hh = torch.relu(z.float() + bp[t]).half()
    loop()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        loop()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        loop()
    return 1000 * t_events(g.replay) / T


def cudnn_rnn_us(H, B, T):
    """torch.nn.RNN (cuDNN, fp16, ReLU, dense): the library's per-layer RNN, which may use
    cuDNN's persistent kernels -- the paper's 'dense persistent' comparator."""
    rnn = torch.nn.RNN(H, H, nonlinearity="relu").cuda().half()
    x = torch.rand(T, B, H, device="cuda", dtype=torch.float16)
    with torch.no_grad():
        rnn(x)
        ms = t_events(lambda: rnn(x), reps=3)
    # the layer includes the input projection: report it separately-timed GEMM-free estimate is not
    # possible through the module, so this is the whole layer (an upper bound for its recurrence)
    return 1000 * ms / T


def cusparse_us(prob, B, T):
    H = prob["H"]
    crow = torch.from_numpy(prob["rowptr"]).long()
    col = torch.from_numpy(prob["col"]).long()
    val = torch.from_numpy(prob["val"])
    W = torch.sparse_csr_tensor(crow, col, val, (H, H)).cuda()
    bp = torch.rand(T, H, B, device="cuda")
    h = torch.zeros(H, B, device="cuda")

    def loop():
        hh = h
        for t in range(T):
            hh = torch.relu(torch.sparse.mm(W, hh) + bp[t])
    loop()
    return 1000 * t_events(loop, reps=3) / T


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--experiment", default="c3", choices=["c3", "e4", "e5", "f1"],
                    help="c3: hidden x batch x density grid; e4: constant nnz 1.32M (PAPER.md:161); "
                         "e5: load-balanced vs unbalanced pruning at 2304 @ 25% (PAPER.md:188); "
                         "f1: sparse vs the dense tensor-core persistent comparator (SURVEY.md 8(f)1)")
    a = ap.parse_args()
    T = 256
    if a.experiment == "c3":
        Hs = [1152, 1792, 2304, 4096, 5760] if not a.quick else [1792, 2304]
        ds = [0.01, 0.05, 0.10, 0.30]
        Bs = [1, 4, 16] if not a.quick else [4]
        points = [(H, B, d, "unstructured") for H in Hs for B in Bs for d in ds]
    elif a.experiment == "e4":  # constant nnz = 2304^2 * 0.25 = 11520^2 * 0.01 = 1,327,104
        points = [(H, 4, 1327104 / (H * H), "unstructured") for H in (2304, 3072, 4096, 5760, 7168, 9216, 11520)]
    elif a.experiment == "f1":  # where does sparse stop winning against a dense persistent kernel on B200?
        points = [(H, B, d, "unstructured") for H in (1152, 2304, 3584) for B in (1, 4, 8)
                  for d in (0.01, 0.1, 0.3, 0.5, 1.0)]
    else:  # E5: row-balanced vs unbalanced at 2304 @ 25%, B = 4
        points = [(2304, 4, 0.25, "unstructured"), (2304, 4, 0.25, "row_balanced"),
                  (1024, 4, 0.125, "unstructured"), (1024, 4, 0.125, "row_balanced")]
    dense_cache = {}
    cudnn_cache = {}
    dtc_cache = {}
    for H, B, d, pattern in points:
                rec = {"H": H, "B": B, "density": d, "T": T, "pattern": pattern, "experiment": a.experiment}
                try:
                    t0 = time.time()
                    prob = inputs.make_problem(H, H, B, T, d, pattern=pattern)
                    m = from_problem(prob, prec="fp16")
                    rec["plan_s"] = round(time.time() - t0, 2)
                    x = torch.from_numpy(prob["x"]).cuda()
                    bp = m.input_projection(x)
                    y = torch.empty(T, B, H, device="cuda")
                    m.recurrence(bp, y=y)
                    torch.cuda.synchronize()
                    ms = t_events(lambda: m.recurrence(bp, y=y))
                    m.status()
                    inf = m.info()
                    rec["ours_us_per_step"] = 1000 * ms / T
                    rec["ours_eff_gflops"] = 2 * prob["nnz"] * B * T / (ms * 1e-3) / 1e9
                    rec["plan"] = {k: inf[k] for k in ("num_ctas", "threads_per_cta", "lanes_per_row", "pairs_per_lane",
                                                       "image_slots_per_lane", "batch_tile", "num_batch_tiles", "column_split")}
                    rec["no_auto_split"] = os.environ.get("SRNN_NO_AUTO_SPLIT") is not None
                    m.close()
                except SrnnError as e:
                    rec["ours"] = f"not on chip / unsupported: {e}"
                if a.experiment == "f1":
                    try:
                        key = (H, B)
                        if key not in dtc_cache:
                            dm = from_problem(prob, prec="fp16", flags=FLAG_DENSE_TC)
                            bpd = dm.input_projection(torch.from_numpy(prob["x"]).cuda())
                            yd = torch.empty(T, B, H, device="cuda")
                            dm.recurrence(bpd, y=yd)
                            torch.cuda.synchronize()
                            dtc_cache[key] = 1000 * t_events(lambda: dm.recurrence(bpd, y=yd)) / T
                            dm.status()
                            dm.close()
                        rec["dense_tc_persistent_us_per_step"] = dtc_cache[key]
                        if "ours_us_per_step" in rec:
                            rec["speedup_vs_dense_tc"] = dtc_cache[key] / rec["ours_us_per_step"]
                    except SrnnError as e:
                        rec["dense_tc"] = f"not on chip / unsupported: {e}"
                    print(json.dumps(rec), flush=True)
                    continue
                try:
                    key = (H, B)
                    if key not in dense_cache:
                        dense_cache[key] = dense_graph_us(H, B, T)
                    rec["cublas_dense_graph_us_per_step"] = dense_cache[key]
                    if key not in cudnn_cache:
                        try:
                            cudnn_cache[key] = cudnn_rnn_us(H, B, T)
                        except Exception as e:  # noqa: BLE001
                            cudnn_cache[key] = None
                    rec["cudnn_rnn_layer_us_per_step"] = cudnn_cache[key]
                    rec["cusparse_us_per_step"] = cusparse_us(prob, B, T)
                except Exception as e:  # noqa: BLE001
                    rec["baseline_error"] = str(e)[:200]
                if "ours_us_per_step" in rec and "cublas_dense_graph_us_per_step" in rec:
                    rec["speedup_vs_dense_graph"] = rec["cublas_dense_graph_us_per_step"] / rec["ours_us_per_step"]
                    if "cusparse_us_per_step" in rec:
                        rec["speedup_vs_cusparse"] = rec["cusparse_us_per_step"] / rec["ours_us_per_step"]
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
