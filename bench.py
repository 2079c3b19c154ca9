#!/usr/bin/env python
"""Benchmark of the sparse persistent RNN hot path (arXiv 1804.10223) on B200.

One bench "step" = one pass of the whole hot path over one batch of
synthetic input: the input-projection GEMM for all T timesteps (a1) followed
by the persistent recurrent kernel over T timesteps (a3-a9) -- exactly the
launches of srnn_forward, issued through the C ABI -- and, at N > 1 GPUs, the
all-gather of y.

Workloads (BASELINE.json configs; SURVEY.md Sec. 8 shorthand):
  --config C2 (default, N = 1 headline): vanilla ReLU RNN, H = I = 2304, B = 4,
      density 30% unstructured, T = 256, fp16 weights / fp32 accumulate.  At N > 1
      every rank runs its own B = 4 (weak scaling).
  --config C5: H = I = 5760, density 10%, global B = 64 split over the N ranks
      (B/N each, strong scaling), T = 512, y batch-major ([B][T][H],
      SRNN_FLAG_Y_BATCH_MAJOR) and all-gathered over NCCL with no re-layout;
      compute-only and final-state-only (h_T all-gather) times reported alongside.

Metric: effective GFLOP/s = 2 * nnz(U_r) * B * T / t_step (the recurrence's
algorithmic flops -- padding and the input GEMM excluded -- over the whole
step's time), whole job over all ranks; us_per_timestep = t_step / T.

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "µs/timestep & effective GFLOP/s, h=2304 b=4 d=30%, vs oracle and dense cuBLAS"
SMEM_BYTES_PER_CLK = 128  # per SM (B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM")
TOL = {"fp32": 1e-5, "fp16": 2e-2}  # BASELINE.json north_star parity tolerances


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--prec", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the comparator / ablation legs")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the host-buffer leg (profilers that serialise kernels stall its pipelined plan)")
    ap.add_argument("--flags", type=int, default=0)
    return ap.parse_args()


def workload(cfg_name, prec_override=None):
    from paper_1804_10223_b200 import inputs
    cfg = dict(inputs.CONFIGS[cfg_name])
    prec = prec_override or cfg.pop("prec")
    cfg.pop("prec", None)
    return cfg, prec


def describe(cfg, prec, name):
    cell = cfg.get("cell", "rnn")
    return (f"{name}: {'LSTM' if cell == 'lstm' else 'vanilla ' + cfg.get('act', 'relu') + ' RNN'} "
            f"H={cfg['H']} I={cfg['I']} B={cfg['B']} density={cfg['density']:.4g} "
            f"{cfg.get('pattern', 'unstructured')} T={cfg['T']} {prec}")


def measured_peaks():
    """Driver-written MEASURED_PEAKS.json (HBM GB/s, dense bf16 TFLOP/s on this pool's B200s)."""
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def host_cpu():
    """lscpu model name and nproc of the host the CPU legs run on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) during the timed region."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                         pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
                except Exception:
                    pass
                self._stop.wait(0.005)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        mhz = [m for m, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML every 5 ms during the timed steps"}


# ---------------------------------------------------------------------------
# CPU legs: the oracle (test infrastructure) as it stands
# ---------------------------------------------------------------------------

def oracle_samples(prob, samples, threads):
    """The fp64 oracle on the given batch samples, `threads` host threads in parallel
    (samples are independent sequences; the oracle's C calls release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    def one(b):
        q = dict(prob)
        q["x"] = np.ascontiguousarray(prob["x"][:, b:b + 1])
        q["B"] = 1
        for k in ("h0", "c0"):
            if prob.get(k) is not None:
                q[k] = np.ascontiguousarray(prob[k][b:b + 1])
        return b, oracle.forward(q)

    with ThreadPoolExecutor(max(1, threads)) as ex:
        return dict(ex.map(one, samples))


def cpu_oracle_leg(prob, samples, threads):
    """(seconds, algorithmic flops, {b: oracle output}) of the oracle on `samples` of `prob`."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    outs = oracle_samples(prob, samples, threads)
    dt = time.perf_counter() - t0
    return dt, 2.0 * prob["nnz"] * len(samples) * prob["T"], outs


def run_reference(args):
    """--impl reference: the oracle (C, fp64) on the host cores, on this arm's workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1804_10223_b200 import inputs
    cfg, prec = workload(args.config, args.prec)
    # each step: one sequence of T/4 steps of the same layer (bounded: ~0.3-2 s per step)
    c = dict(cfg)
    c["B"], c["T"] = 1, max(1, cfg["T"] // 4)
    prob = inputs.make_problem(**c)
    for _ in range(args.warmup):
        cpu_oracle_leg(prob, [0], 1)
    times = [cpu_oracle_leg(prob, [0], 1)[0] for _ in range(args.steps)]
    t = statistics.median(times)
    val = 2.0 * prob["nnz"] * c["T"] / t / 1e9
    cpu = host_cpu()
    sample = (f"oracle (C, fp64, 1 thread) on B=1 of {cfg['B']} sequences, T={c['T']} of {cfg['T']} steps "
              f"per step; host {cpu['model']}, nproc {cpu['nproc']}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t,
        "us_per_timestep": 1e6 * t / c["T"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded PCG64, paper-shaped)",
        "config": {"workload": describe(cfg, prec, args.config), "sample": sample},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu["model"], "nproc": cpu["nproc"]},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------
# GPU comparators
# ---------------------------------------------------------------------------

def cublas_dense_torch(H, B, T, device, reps=5):
    """Dense per-timestep loop through torch: z = W_h h (cuBLAS, fp16 in / fp32 acc) then
    +b', ReLU, cast -- eager and CUDA-graph captured over T steps (5 launches per step)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(0)
    W = (torch.rand(H, H, generator=g) - 0.5).to(device=device, dtype=torch.float16)
    bp = torch.rand(T, H, B, generator=g).to(device)
    h = torch.zeros(H, B, device=device, dtype=torch.float16)
    z = torch.empty(H, B, device=device, dtype=torch.float16)

    def loop():
        hh = h
        for t in range(T):
            torch.mm(W, hh, out=z)
            hh = torch.relu(z.float() + bp[t]).half()
        return hh

    for _ in range(2):
        loop()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        loop()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    eager = statistics.median(ts) * 1000 / T
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        loop()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        loop()
    graph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return {"eager_us_per_timestep": eager, "graph_us_per_timestep": statistics.median(ts) * 1000 / T,
            "launches_per_step": 5}


def time_recurrence(m, bp, y, hT, reps=7, flush=None):
    """Median recurrence-kernel time (ms) of a plan over a resident b' (CUDA events)."""
    import torch
    m.recurrence(bp, y=y, hT=hT)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        ev[0].record()
        m.recurrence(bp, y=y, hT=hT)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    m.status()
    return statistics.median(ts)


def launch_list_kernel_us(substr):
    """Median duration (µs) of a kernel in the committed ncu launch list (cold, serialised), if any."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "launches_r*.csv")))
    if not files:
        return None, None
    vals, hdr = [], None
    try:
        for r in csv.reader(open(files[-1])):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if substr in d["Kernel Name"] and d.get("Metric Name") == "gpu__time_duration.sum":
                    vals.append(float(d["Metric Value"]) / 1000.0)  # ns -> µs
    except Exception:
        return None, None
    return (statistics.median(vals) if vals else None), os.path.relpath(files[-1], ROOT)


def load_traffic():
    """dram bytes per launch of the recurrent kernel from the committed ncu summary, if any."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")))
    if not files:
        return None, None
    try:
        d = json.load(open(files[-1]))
        return d.get("recurrent_dram_bytes_per_launch"), os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# main (our arm)
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1804_10223_b200 import FLAG_Y_BATCH_MAJOR, from_problem, inputs
    from paper_1804_10223_b200.multigpu import gather_batch_major, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg, prec = workload(args.config, args.prec)
    H, T = cfg["H"], cfg["T"]
    strong = args.config == "C5"  # global batch split over ranks (BASELINE configs[4])
    flags = args.flags | (FLAG_Y_BATCH_MAJOR if strong else 0)
    if strong:
        B_glob = cfg["B"]
        s0, B = shard(B_glob, world, rank)
        prob_g = inputs.make_problem(**cfg)
        prob = dict(prob_g)
        prob["x"] = np.ascontiguousarray(prob_g["x"][:, s0:s0 + B])
        prob["B"] = B
    else:
        B = cfg["B"]
        B_glob = B * world
        prob = inputs.make_problem(**cfg, seed_offset=rank)  # weak scaling: each rank its own sequences
    m = from_problem(prob, prec=prec, device=local, flags=flags)
    info = m.info()
    G = prob["G"]
    x = torch.from_numpy(prob["x"]).to(dev)
    bp = torch.empty(T, B, G * H, device=dev)
    y = torch.empty((B, T, H) if strong else (T, B, H), device=dev)
    hT = torch.empty(B, H, device=dev)
    yall = torch.empty((B_glob, T, H) if strong else (world, T, B, H), device=dev) if world > 1 else None
    hall = torch.empty(world * B, H, device=dev) if world > 1 else None
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(ev=None, gather="y"):
        if ev:
            ev[0].record(stream)
        m.input_projection(x, bp)
        if ev:
            ev[1].record(stream)
        m.recurrence(bp, y=y, hT=hT)
        if ev:
            ev[2].record(stream)
        if world > 1 and gather == "y":
            if strong:
                gather_batch_major(y, global_batch=B_glob, out=yall)
            else:
                dist.all_gather_into_tensor(yall, y)
        elif world > 1 and gather == "hT":
            dist.all_gather_into_tensor(hall, hT)
        if ev:
            ev[3].record(stream)

    def timed(gather, n):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(n):
            flush.fill_(float(k))  # L2 flush between timed steps (outside the events)
            step(evs[k], gather)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        m.status()
        tot = torch.tensor([sum(e[0].elapsed_time(e[3]) for e in evs), sum(e[1].elapsed_time(e[2]) for e in evs),
                            sum(e[0].elapsed_time(e[1]) for e in evs)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        return [v / n / 1000.0 for v in tot.tolist()]  # s: step, recurrence, projection (max over ranks)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    m.status()
    with ClockSampler(local) as clk:
        t_step, t_rec, t_gemm = timed("y", args.steps)
    eff_flops_rank = 2.0 * prob["nnz"] * B * T
    value = eff_flops_rank * world / t_step / 1e9
    y_ref = y.clone()  # output of the timed step (self-check below)
    extra_scaling = {}
    if world > 1:  # compute-only and final-state-only variants of the same step
        t_c = timed("none", max(3, args.steps // 2))[0]
        t_h = timed("hT", max(3, args.steps // 2))[0]
        extra_scaling = {
            "compute_only": {"value": eff_flops_rank * world / t_c / 1e9, "ms_per_step": 1000 * t_c},
            "final_state_only": {"value": eff_flops_rank * world / t_h / 1e9, "ms_per_step": 1000 * t_h,
                                 "gathered_bytes": int(hall.numel() * 4)},
            "y_allgather_bytes": int(yall.numel() * 4),
        }

    # ---- e2e: the public host-buffer call srnn_forward_host, pinned memory ----
    e2e_val = None
    xh = torch.from_numpy(prob["x"]).pin_memory()
    yh = torch.empty(tuple(y.shape)).pin_memory()
    hh = torch.empty(B, H).pin_memory()
    if not args.no_e2e:
        from paper_1804_10223_b200 import FLAG_RESERVE_SMS
        me = from_problem(prob, prec=prec, device=local, flags=flags | FLAG_RESERVE_SMS)
        for _ in range(2):
            me.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())
        if world > 1:
            dist.barrier()
        e2e_t = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            me.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())
            e2e_t.append(time.perf_counter() - t0)
        e2e_s = torch.tensor([sum(e2e_t) / len(e2e_t)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e_val = eff_flops_rank * world / e2e_s.item() / 1e9
        me.close()

    if rank == 0:
        peaks = measured_peaks()
        clocks = clk.summary()
        f_hz = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0) * 1e6
        f_peak_hz = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
        smem_peak = info["sm_count"] * SMEM_BYTES_PER_CLK * f_peak_hz / 1e9  # GB/s
        fp32_h = prec == "fp32" or (args.flags & (1 << 5))
        h_bytes = 4.0 if fp32_h else 2.0
        gather_bytes = h_bytes * prob["nnz"] * B * T
        achieved = gather_bytes / t_rec / 1e9
        traffic, traffic_src = load_traffic()
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t_step * 1000, "us_per_timestep": t_step * 1e6 / T,
            "us_per_timestep_recurrence": t_rec * 1e6 / T, "ms_input_gemm": t_gemm * 1000,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f16" if prec == "fp16" else "f32",
            "dtype_note": ("fp16 multiplies (W_h, W_x, x and the exchanged h rounded RNE; h keeps 10 significant bits "
                           "plus the 1-bit step tag, DESIGN.md R9/R16), fp32 accumulate; b', activations, c and y fp32"
                           if prec == "fp16" else "fp32 throughout, no TF32 (exchanged h: 23 significant bits, R16)"),
            "data": "synthetic (seeded PCG64: uniform unstructured pattern, U(-a,a) weights)",
            "config": {"workload": describe(cfg, prec, args.config), "H": H, "I": cfg["I"], "B_per_rank": B,
                       "global_batch": B_glob, "T": T, "density": cfg["density"], "nnz": prob["nnz"],
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "y_layout": "[B][T][H] batch-major" if strong else "[T][B][H]",
                       "parallelism": (f"batch-partitioned x{world}" + (", y all-gathered (NCCL)" if world > 1 else "")),
                       "plan": {k: info[k] for k in ("num_ctas", "threads_per_cta", "lanes_per_row", "batch_tile",
                                                     "num_batch_tiles", "pairs_per_lane", "slots_used",
                                                     "regs_per_thread", "spill_bytes", "wavefronts_per_step_max",
                                                     "wavefronts_per_step_ideal", "conflict_wavefronts")
                                if k in info}},
            "roofline": {"bound": "smem", "kernel": "srnn_persistent_kernel",
                         "achieved": achieved, "peak": smem_peak, "unit": "GB/s", "frac": achieved / smem_peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": f"derived: {info['sm_count']} SMs x 128 B/clk shared-memory crossbar x "
                                        f"{f_peak_hz / 1e6:.0f} MHz (B300_MICROARCH.md smem BW; MEASURED_PEAKS.json "
                                        "sm_max_mhz)",
                         "note": f"achieved = algorithmic h-gather bytes ({h_bytes:g} B x nnz x B x T) / recurrent kernel "
                                 "time (CUDA events); the per-step exchange latency is not in this bound (see "
                                 "roofline_latency)"},
            "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": int(xh.numel() * 4),
                    "d2h_bytes_per_step": int(yh.numel() * 4 + hh.numel() * 4),
                    "api": "srnn_forward_host (pinned host buffers, H2D + forward + D2H + sync; plan with "
                           "SRNN_FLAG_RESERVE_SMS: x chunks projected on 4 free SMs and y chunks copied back "
                           "while the persistent kernel runs)"},
            "gpu_launches": (3 if prec == "fp16" else 2) * args.steps,
            "gpu_launches_note": "per step: f32->f16 convert + tcgen05 GEMM + persistent recurrent kernel (fp16 mode)",
            "clocks": clocks,
        }
        out.update({"scaling_detail": extra_scaling} if extra_scaling else {})
        # ---- input projection (tensor cores) against the measured dense peak ----
        gemm_flops = 2.0 * T * B * cfg["I"] * G * H
        bf16_peak = peaks.get("bf16_tflops") or 1663.3
        out["input_gemm"] = {"kernel": "gemm_tc_f16_kernel (tcgen05) + f32_to_f16" if prec == "fp16" else
                             "gemm_f32_nt_kernel (SIMT fp32)", "ms": t_gemm * 1000,
                             "achieved_tflops": gemm_flops / t_gemm / 1e12,
                             "peak_tflops": bf16_peak if prec == "fp16" else None,
                             "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; fp16 has the same dense rate)",
                             "frac": (gemm_flops / t_gemm / 1e12) / bf16_peak if prec == "fp16" else None,
                             "note": "ms covers the whole srnn_input_projection call (conversion + GEMM + gaps)"}
        if prec == "fp16":
            k_us, k_src = launch_list_kernel_us("gemm_tc_f16_kernel")
            if k_us:
                out["input_gemm"].update({"gemm_kernel_only_us": k_us,
                                          "gemm_kernel_only_frac": gemm_flops / (k_us * 1e-6) / 1e12 / bf16_peak,
                                          "gemm_kernel_only_source": k_src + " (ncu launch list, cold L2, serialised)"})
        t_us = t_rec * 1e6 / T
        if world == 1 and not args.no_extras:
            extras(out, args, prob, prec, info, m, bp, y, hT, flush, dev, t_us, f_hz)
        # ---- CPU legs + self-check of this run's y against the oracle ----
        if not args.no_cpu_baseline and world == 1:
            cpu = host_cpu()
            samples = list(range(min(B, 8))) if not strong else [0, B - 1]
            dt1, fl1, outs = cpu_oracle_leg(prob, samples[:1], 1)
            par = min(len(samples), cpu["nproc"] or 1)
            dtp, flp, outs_p = cpu_oracle_leg(prob, samples, par)
            outs.update(outs_p)
            yc = y_ref.cpu().numpy().astype(np.float64)
            errs, mx = [], 0.0
            for b, o in outs.items():
                yb = yc[b] if strong else yc[:, b]
                errs.append(float(np.abs(yb - o["y"][:, 0]).max()))
                mx = max(mx, float(np.abs(o["y"]).max()))
            out["cpu_baseline"] = {
                "value": fl1 / dt1 / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                "sample": f"{args.config} sequence {samples[0]} (T={T}) through the C fp64 oracle, "
                          f"{dt1:.2f} s on one core",
                "cpu_model": cpu["model"], "nproc": cpu["nproc"],
                "host_parallel": {"value": flp / dtp / 1e9, "unit": "GFLOP/s", "cores": par,
                                  "sample": f"{len(samples)} independent sequences (T={T}) in {par} threads, "
                                            f"{dtp:.2f} s"}}
            out["parity"] = {"max_abs_err": max(errs), "max_abs_h": mx, "tolerance": TOL[prec],
                             "ok": max(errs) <= TOL[prec],
                             "checked": f"every output of batch samples {sorted(outs)} of the timed step vs the "
                                        "fp64 oracle (unquantised weights)"}
        print(json.dumps(out))
    m.close()
    if world > 1:
        dist.destroy_process_group()


def extras(out, args, prob, prec, info, m, bp, y, hT, flush, dev, t_us, f_hz):
    """Single-GPU comparators and ablations added to the JSON line (rank 0, N = 1)."""
    import torch

    from paper_1804_10223_b200 import FLAG_DENSE_TC, FLAG_FP32_STAGING, from_problem
    H, B, T = prob["H"], prob["B"], prob["T"]
    # ---- latency roofline: the measured exchange floor of this format vs the smem time ----
    try:
        import baselines
        fl = baselines.exchange_floor(H, info["batch_tile"], info["num_ctas"], info["threads_per_cta"])
        floor_us = fl["a2a_lsb_us_per_step"] * info["num_batch_tiles"]
        smem_us = info["wavefronts_per_step_max"] * info["num_batch_tiles"] / f_hz * 1e6
        out["roofline_latency"] = {
            "exchange_floor_us_per_step": floor_us, "smem_us_per_step": smem_us, "t_us_per_step": t_us,
            "frac_serial": (floor_us + smem_us) / t_us, "frac_overlap": max(floor_us, smem_us) / t_us,
            "floor_source": "baselines/mb_exchange --floor (scripts/microbench_exchange.cu k_a2a_lsb): all-to-all "
                            f"of the product's fp16 exchange format, {fl['bytes_per_cta']} B per CTA, "
                            f"{fl['ctas']} CTAs x {fl['threads']} threads, no compute",
            "note": "frac_serial: floor + smem as a fraction of the measured step (the kernel runs them back to "
                    "back); frac_overlap: max(floor, smem), the bound if the operate fully overlapped the "
                    "exchange (PAPER.md:103 partial progress)"}
    except Exception as ex:  # noqa: BLE001
        out["roofline_latency"] = {"error": str(ex)[:200]}
    if not args.no_cublas:
        cb = cublas_dense_torch(H, B, T, dev)
        cb["speedup_vs_graph"] = cb["graph_us_per_timestep"] / t_us
        cb["speedup_vs_eager"] = cb["eager_us_per_timestep"] / t_us
        out["baseline_cublas_dense"] = cb
        try:
            import baselines
            lt = baselines.cublaslt_rnn(H, B, T)
            lt["speedup_vs_graph"] = lt["graph_us_per_timestep"] / t_us
            lt["speedup_vs_eager"] = lt["eager_us_per_timestep"] / t_us
            lt["note"] = ("one cublasLtMatmul per step: fp16 W_h x fp16 h, fp32 accumulate, beta = 1 with C = b'_t "
                          "(fp16), RELU epilogue, D = h_{t+1} fp16 (baselines/cublaslt_rnn.cu)")
            out["baseline_cublaslt_fused"] = lt
        except Exception as ex:  # noqa: BLE001
            out["baseline_cublaslt_fused"] = {"error": str(ex)[:200]}
    if prec == "fp16":
        # SURVEY.md Sec. 8(f)1 comparator: the dense persistent RNN on tensor cores
        try:
            dm = from_problem(prob, prec=prec, flags=args.flags | FLAG_DENSE_TC)
            d_us = time_recurrence(dm, bp, y, hT, 10, flush) * 1000 / T
            dinf = dm.info()
            dm.close()
            out["baseline_dense_tc_persistent"] = {
                "us_per_timestep": d_us, "speedup_sparse_vs_dense_tc": d_us / t_us,
                "plan": {k: dinf[k] for k in ("num_ctas", "batch_tile", "dense_m_tiles", "dense_kblocks_per_warp",
                                              "dense_frags_reg", "dense_frags_smem")},
                "note": "same library, SRNN_FLAG_DENSE_TC: dense fp16 U_r in mma.sync m16n8k16 fragments, same "
                        "exchange and epilogue (recurrence only, median of 10)"}
        except Exception as ex:  # noqa: BLE001
            out["baseline_dense_tc_persistent"] = {"error": str(ex)[:200]}
        # precision ablations of the same workload (recurrence only, median of 7)
        abl = {}
        for name, pr, fl in (("fp32_mode", "fp32", 0), ("fp16_weights_fp32_h", "fp16", FLAG_FP32_STAGING)):
            try:
                am = from_problem(prob, prec=pr, flags=args.flags | fl)
                a_us = time_recurrence(am, bp, y, hT, 7, flush) * 1000 / T
                abl[name] = {"us_per_timestep": a_us, "effective_gflops": 2.0 * prob["nnz"] * B / (a_us * 1e3),
                             "plan": {k: am.info()[k] for k in ("batch_tile", "pairs_per_lane", "regs_per_thread")}}
                am.close()
            except Exception as ex:  # noqa: BLE001
                abl[name] = {"error": str(ex)[:200]}
        abl["note"] = ("same workload, recurrence only: fp32_mode = fp32 weights / h / accumulate (1e-5 parity); "
                       "fp16_weights_fp32_h = SRNN_FLAG_FP32_STAGING (fp16 weights, fp32 h exchange)")
        out["precision_ablations"] = abl


if __name__ == "__main__":
    main()
