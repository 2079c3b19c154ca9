"""Summarise ncu --set full captures into profiles/ncu_summary_<round>.json (+ .md).

usage: python scripts/ncu_summary.py r01 gpurun_out/prof_rec.ncu-rep gpurun_out/prof_gemm.ncu-rep [launches.csv]
"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_elapsed",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "local_load", "lsu_mem_local",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_requests.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if any(h.startswith(w) for w in WANT) or h in (
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"):
                try:
                    d[h] = [float(v.replace(",", "")), u]
                except ValueError:
                    pass
        res.append(d)
    return res


def to_bytes(v):
    x, u = v
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    out = {"round": tag, "captures": {}}
    for rep in reps:
        for d in raw(rep):
            name = d["kernel"]
            key = "recurrent" if "persistent" in name else ("gemm_tc" if "gemm_tc" in name else name[:40])
            if key == "recurrent" and ", 0>(" not in name:  # template MT > 0: dense tensor-core comparator
                key = "recurrent_dense_tc"
            out["captures"][key] = d
            if key == "recurrent":
                out["recurrent_dram_bytes_per_launch"] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
            if key == "gemm_tc":
                out["gemm_dram_bytes_per_launch"] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
    json.dump(out, open(f"profiles/ncu_summary_{tag}.json", "w"), indent=1)
    with open(f"profiles/ncu_summary_{tag}.md", "w") as f:
        f.write(f"# ncu --set full summaries ({tag})\n\n")
        for k, d in out["captures"].items():
            f.write(f"## {k}: `{d['kernel'][:100]}`\n\n| metric | value | unit |\n|---|---|---|\n")
            for m, (v, u) in sorted(d.items() if False else [(a, b) for a, b in d.items() if a != "kernel"]):
                f.write(f"| {m} | {v:g} | {u} |\n")
            f.write("\n")
    print(json.dumps({k: v for k, v in out.items() if k != "captures"}))


if __name__ == "__main__":
    main()
