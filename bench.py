#!/usr/bin/env python
"""Benchmark of the sparse persistent RNN hot path (arXiv 1804.10223) on B200.

One bench "step" = one pass of the whole hot path over one batch of
synthetic input: the input-projection GEMM for all T timesteps (a1) followed
by the persistent recurrent kernel over T timesteps (a3-a9), i.e. exactly the
two launches of srnn_forward, issued through the C ABI.

Default workload (BASELINE.json configs[1]): vanilla ReLU RNN,
H = I = 2304, B = 4, density 30% unstructured, T = 256, fp16 weights / fp32
accumulate.  Inputs are seeded synthetic (paper_1804_10223_b200.inputs).

Metric: effective GFLOP/s = 2 * nnz(U_r) * B * T / t_step (the recurrence's
algorithmic flops -- padding and the input GEMM excluded -- divided by the
whole step's time), whole job over all ranks.  us_per_timestep = t_step / T
is reported alongside.

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       (N > 1: launched by torch.distributed.run, one rank per GPU; each rank
        runs its own batch of sequences -- weak scaling -- and y is
        all-gathered over NCCL at the end of every step)
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
SM_COUNT_B200 = 148
SMEM_BYTES_PER_CLK = 128  # per SM (B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--prec", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the host-buffer leg (profilers that serialise kernels stall its pipelined plan)")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--gather", default="y", choices=["y", "hT", "none"])
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


def cpu_oracle_run(cfg, B, T, seed_offset=0):
    """The oracle (as it stands) on a sample of the workload; returns (seconds, flops_effective)."""
    import oracle
    from paper_1804_10223_b200 import inputs
    c = dict(cfg)
    c["B"], c["T"] = B, T
    prob = inputs.make_problem(**c, seed_offset=seed_offset)
    oracle.build()
    t0 = time.perf_counter()
    oracle.forward(prob)
    dt = time.perf_counter() - t0
    return dt, 2.0 * prob["nnz"] * B * T


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, prec = workload(args.config, args.prec)
    # each step: the oracle on one sequence of T/4 steps of the same layer
    B, T = 1, max(1, cfg["T"] // 4)
    for _ in range(args.warmup):
        cpu_oracle_run(cfg, B, T)
    times, flops = [], 0.0
    for k in range(args.steps):
        dt, fl = cpu_oracle_run(cfg, B, T, seed_offset=0)
        times.append(dt)
        flops = fl
    t = statistics.median(times)
    val = flops / t / 1e9
    sample = f"oracle (C, fp64, 1 thread) on B={B} of {cfg['B']} sequences, T={T} of {cfg['T']} steps per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t,
        "us_per_timestep": 1e6 * t / T, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded PCG64, paper-shaped)",
        "config": {"workload": describe(cfg, prec, args.config), "sample": sample},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cublas_dense_baseline(H, B, T, device, reps=5):
    """Dense per-timestep cuBLAS loop: z = W_h h (fp16 in, fp32 acc) then +b', ReLU, cast --
    eager and CUDA-graph captured over T steps (SURVEY.md Sec. 8 d-v)."""
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
    graphed = statistics.median(ts) * 1000 / T
    return {"eager_us_per_timestep": eager, "graph_us_per_timestep": graphed}


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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1804_10223_b200 import from_problem, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg, prec = workload(args.config, args.prec)
    H, B, T = cfg["H"], cfg["B"], cfg["T"]
    # weak scaling: each rank owns its own B sequences (independent samples)
    prob = inputs.make_problem(**cfg, seed_offset=rank)
    m = from_problem(prob, prec=prec, device=local, flags=args.flags)
    info = m.info()
    x = torch.from_numpy(prob["x"]).to(dev)
    bp = torch.empty(T, B, prob["G"] * H, device=dev)
    y = torch.empty(T, B, H, device=dev)
    hT = torch.empty(B, H, device=dev)
    yall = torch.empty(world, T, B, H, device=dev) if world > 1 else None
    hall = torch.empty(world, B, H, device=dev) if world > 1 else None
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        m.input_projection(x, bp)
        if ev:
            ev[1].record(stream)
        m.recurrence(bp, y=y, hT=hT)
        if ev:
            ev[2].record(stream)
        if world > 1 and args.gather != "none":
            if args.gather == "y":
                dist.all_gather_into_tensor(yall, y)
            else:
                dist.all_gather_into_tensor(hall, hT)
        if ev:
            ev[3].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    m.status()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(float(k))  # L2 flush between timed steps (outside the events)
            step(evs[k])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    m.status()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    rec_ms = [e[1].elapsed_time(e[2]) for e in evs]
    gemm_ms = [e[0].elapsed_time(e[1]) for e in evs]
    tot = torch.tensor([sum(step_ms), sum(rec_ms), sum(gemm_ms)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    t_step = tot[0].item() / args.steps / 1000.0   # s, max over ranks
    t_rec = tot[1].item() / args.steps / 1000.0
    t_gemm = tot[2].item() / args.steps / 1000.0
    eff_flops_rank = 2.0 * prob["nnz"] * B * T
    value = eff_flops_rank * world / t_step / 1e9

    # ---- e2e: the public host-buffer call srnn_forward_host, pinned memory ----
    # (a plan that leaves 4 SMs free pipelines the copies/projection with the kernel)
    e2e_val = None
    xh = torch.empty(T, B, prob["I"])
    yh = torch.empty(T, B, H)
    hh = torch.empty(B, H)
    if not args.no_e2e:
        from paper_1804_10223_b200 import FLAG_RESERVE_SMS
        m_dev = m
        m = from_problem(prob, prec=prec, device=local, flags=args.flags | FLAG_RESERVE_SMS)
        xh = torch.from_numpy(prob["x"]).pin_memory()
        yh = torch.empty(T, B, H).pin_memory()
        hh = torch.empty(B, H).pin_memory()
        for _ in range(2):
            m.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())
        if world > 1:
            dist.barrier()
        e2e_t = []
        for k in range(args.steps):
            t0 = time.perf_counter()
            m.forward_host(xh.numpy(), y=yh.numpy(), hT=hh.numpy())
            e2e_t.append(time.perf_counter() - t0)
        e2e_s = torch.tensor([sum(e2e_t) / len(e2e_t)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e_val = eff_flops_rank * world / e2e_s.item() / 1e9
        m.close()
        m = m_dev

    if rank == 0:
        clocks = clk.summary()
        f_peak_hz = 1965e6
        smem_peak = info["sm_count"] * SMEM_BYTES_PER_CLK * f_peak_hz / 1e9  # GB/s
        # algorithmic: one staged h element per (nonzero, sample, step) -- fp16 (2 B) in fp16 mode
        # (h is staged and exchanged in fp16, R9), fp32 (4 B) in fp32 mode
        h_bytes = 2.0 if (prec == "fp16" and not (args.flags & (1 << 5))) else 4.0
        gather_bytes = h_bytes * prob["nnz"] * B * T
        achieved = gather_bytes / t_rec / 1e9
        traffic, traffic_src = load_traffic()
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t_step * 1000, "us_per_timestep": t_step * 1e6 / T,
            "us_per_timestep_recurrence": t_rec * 1e6 / T, "ms_input_gemm": t_gemm * 1000,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16" if prec == "fp16" else "f32",
            "dtype_note": "fp16 multiplies (W_h, W_x, x and the staged h rounded RNE), fp32 accumulate; b', "
                          "activations, LSTM c and y in fp32" if prec == "fp16" else "fp32 throughout, no TF32",
            "data": "synthetic (seeded PCG64: uniform unstructured pattern, U(-a,a) weights)",
            "config": {"workload": describe(cfg, prec, args.config), "H": H, "I": cfg["I"], "B_per_rank": B,
                       "global_batch": B * world, "T": T, "density": cfg["density"], "nnz": prob["nnz"],
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": f"batch-partitioned x{world}" + (f", all-gather {args.gather}" if world > 1 else ""),
                       "plan": {k: info[k] for k in ("num_ctas", "threads_per_cta", "lanes_per_row",
                                                     "pairs_per_lane", "slots_used", "regs_per_thread",
                                                     "wavefronts_per_step_max", "wavefronts_per_step_ideal",
                                                     "conflict_wavefronts")}},
            "roofline": {"bound": "smem", "kernel": "srnn_persistent_kernel",
                         "achieved": achieved, "peak": smem_peak, "unit": "GB/s", "frac": achieved / smem_peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "derived: 148 SMs x 128 B/clk shared-memory crossbar x 1965 MHz "
                                        "(B300_MICROARCH.md smem BW, B200_PROFILING.md clocks)",
                         "note": f"achieved = algorithmic h-gather bytes ({h_bytes:g} B x nnz x B x T) / recurrent kernel "
                                 "time (CUDA events); the per-step exchange latency is not in this bound"},
            "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": int(xh.numel() * 4),
                    "d2h_bytes_per_step": int(yh.numel() * 4 + hh.numel() * 4),
                    "api": "srnn_forward_host (pinned host buffers, H2D + forward + D2H + sync; plan with "
                           "SRNN_FLAG_RESERVE_SMS: x chunks projected on 4 free SMs and y chunks copied back "
                           "while the persistent kernel runs)"},
            "gpu_launches": (3 if prec == "fp16" else 2) * args.steps,
            "gpu_launches_note": "per step: f32->f16 convert + tcgen05 GEMM + persistent recurrent kernel (fp16 mode)",
            "clocks": clocks,
        }
        gemm_flops = 2.0 * T * B * cfg["I"] * prob["G"] * H
        out["input_gemm"] = {"kernel": "gemm_tc_f16_kernel (tcgen05) + f32_to_f16" if prec == "fp16" else
                             "gemm_f32_nt_kernel (SIMT fp32)", "ms": t_gemm * 1000,
                             "achieved_tflops": gemm_flops / t_gemm / 1e12,
                             "peak_tflops": 1663.3 if prec == "fp16" else None,
                             "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; fp16 has the same dense rate)",
                             "frac": (gemm_flops / t_gemm / 1e12) / 1663.3 if prec == "fp16" else None,
                             "note": "ms covers the whole srnn_input_projection call (x f32->f16 conversion + GEMM + "
                                     "launch gaps)"}
        if prec == "fp16":
            k_us, k_src = launch_list_kernel_us("gemm_tc_f16_kernel")
            if k_us:
                out["input_gemm"].update({"gemm_kernel_only_us": k_us,
                                          "gemm_kernel_only_frac": gemm_flops / (k_us * 1e-6) / 1e12 / 1663.3,
                                          "gemm_kernel_only_source": k_src + " (ncu launch list, cold L2, serialised)"})
        # Latency roofline of the recurrent kernel: the measured exchange/sync floor (same
        # H, B, plan shape, density 0: no pairs, everything else identical) plus the
        # shared-memory time of the packer's predicted wavefronts (busiest CTA, per step).
        try:
            zprob = dict(prob)
            zprob["rowptr"] = np.zeros_like(prob["rowptr"])
            zprob["col"] = np.zeros(0, np.int32)
            zprob["val"] = np.zeros(0, np.float32)
            zm = from_problem(zprob, prec=prec, device=local, flags=args.flags, num_ctas=info["num_ctas"],
                              lanes_per_row=info["lanes_per_row"])
            zm.recurrence(bp, y=y, hT=hT)
            torch.cuda.synchronize()
            ze = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            zts = []
            for _ in range(5):
                ze[0].record(stream)
                zm.recurrence(bp, y=y, hT=hT)
                ze[1].record(stream)
                torch.cuda.synchronize()
                zts.append(ze[0].elapsed_time(ze[1]))
            zm.status()
            zm.close()
            f_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
            floor_us = statistics.median(zts) * 1000 / T
            smem_us = info["wavefronts_per_step_max"] * info["num_batch_tiles"] / f_hz * 1e6
            out["roofline_latency"] = {
                "sync_floor_us_per_step": floor_us, "smem_us_per_step": smem_us,
                "t_roof_us_per_step": floor_us + smem_us, "t_us_per_step": t_rec * 1e6 / T,
                "frac": (floor_us + smem_us) / (t_rec * 1e6 / T),
                "note": "sync floor = same plan shape at density 0 (exchange + barriers + epilogue, no "
                        "pairs), measured here; smem = predicted wavefronts of the busiest CTA / SM clock"}
        except Exception as ex:  # noqa: BLE001
            out["roofline_latency"] = {"error": str(ex)[:200]}
        if not args.no_cublas and world == 1:
            cb = cublas_dense_baseline(H, B, T, dev)
            cb["speedup_vs_graph"] = cb["graph_us_per_timestep"] / (t_rec * 1e6 / T)
            cb["speedup_vs_eager"] = cb["eager_us_per_timestep"] / (t_rec * 1e6 / T)
            out["baseline_cublas_dense"] = cb
        if not args.no_cublas and world == 1 and prec == "fp16":
            # SURVEY.md Sec. 8(f)1 comparator: the dense persistent RNN on tensor cores
            # (SRNN_FLAG_DENSE_TC: same exchange/epilogue, U_r as mma.sync fragments)
            try:
                from paper_1804_10223_b200 import FLAG_DENSE_TC
                dm = from_problem(prob, prec=prec, device=local, flags=args.flags | FLAG_DENSE_TC)
                dm.recurrence(bp, y=y, hT=hT)
                torch.cuda.synchronize()
                de = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                dts = []
                for _ in range(10):
                    flush.fill_(1.0)
                    de[0].record(stream)
                    dm.recurrence(bp, y=y, hT=hT)
                    de[1].record(stream)
                    torch.cuda.synchronize()
                    dts.append(de[0].elapsed_time(de[1]))
                dm.status()
                dinf = dm.info()
                dm.close()
                d_us = statistics.median(dts) * 1000 / T
                out["baseline_dense_tc_persistent"] = {
                    "us_per_timestep": d_us, "speedup_sparse_vs_dense_tc": d_us / (t_rec * 1e6 / T),
                    "plan": {k: dinf[k] for k in ("num_ctas", "batch_tile", "dense_m_tiles",
                                                  "dense_kblocks_per_warp", "dense_frags_reg", "dense_frags_smem")},
                    "note": "same library, SRNN_FLAG_DENSE_TC: dense fp16 U_r in mma.sync m16n8k16 fragments, "
                            "same tagged exchange and epilogue (recurrence only, median of 10)"}
            except Exception as ex:  # noqa: BLE001
                out["baseline_dense_tc_persistent"] = {"error": str(ex)[:200]}
        if not args.no_cpu_baseline and world == 1:
            dt, fl = cpu_oracle_run(cfg, B, T)
            out["cpu_baseline"] = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                                   "sample": f"full {args.config} workload (B={B}, T={T}) through the C fp64 oracle, "
                                             f"{dt:.1f} s single-threaded"}
        print(json.dumps(out))
    m.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
