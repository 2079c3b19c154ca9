"""Markdown table from scripts/sweep.py JSONL output (c3 / e4 / e5 rows).

usage: python scripts/sweep_md.py sweep.jsonl > table.md
"""
import json
import sys


def fmt(v):
    return "–" if v is None else f"{v:.2f}"


rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
print("| H | B | density | pattern | ours | dense cuBLAS (graph) | cuDNN RNN layer | cuSPARSE | speedup vs dense | "
      "vs cuDNN | vs cuSPARSE |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    ours = r.get("ours_us_per_step")
    dense, cud, csp = r.get("cublas_dense_graph_us_per_step"), r.get("cudnn_rnn_layer_us_per_step"), \
        r.get("cusparse_us_per_step")
    sp = lambda b: fmt(b / ours) if (b is not None and ours) else "–"  # noqa: E731
    print(f"| {r['H']} | {r['B']} | {r['density'] * 100:g}% | {r['pattern']} | "
          f"{fmt(ours) if ours else 'not on chip'} | {fmt(dense)} | {fmt(cud)} | {fmt(csp)} | {sp(dense)} | "
          f"{sp(cud)} | {sp(csp)} |")
