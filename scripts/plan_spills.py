"""Chosen compiled instance (NP, BT, k8) and its spill bytes for the BASELINE configs and a
few k8 / wide-tile plans (SURVEY Sec. 8 d-vi: 0 spill bytes).  Needs a GPU (compiled query)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_10223_b200 import from_problem, inputs  # noqa: E402

cases = []
for name, c in inputs.CONFIGS.items():
    c = dict(c)
    prec = c.pop("prec")
    c["T"] = 4
    cases.append((name, c, prec))
    if name in ("C2", "C4_speech"):
        cases.append((name + "_fp32", c, "fp32"))
for H, B, d in ((512, 8, 0.1), (768, 8, 0.1), (2304, 16, 0.3), (3584, 4, 0.1), (1152, 32, 0.5)):
    cases.append((f"H{H}_B{B}_d{d}", dict(H=H, I=H, B=B, T=4, density=d), "fp16"))
rows = []
for name, c, prec in cases:
    prob = inputs.make_problem(**c)
    m = from_problem(prob, prec=prec)
    i = m.info()
    rows.append({"case": name, "prec": prec, "NP": i["pairs_per_lane"], "BT": i["batch_tile"],
                 "threads": i["threads_per_cta"], "regs": i["regs_per_thread"], "spill_bytes": i["spill_bytes"],
                 "smem_slots": i["image_slots_per_lane"] - i["pairs_per_lane"]})
    m.close()
    print(json.dumps(rows[-1]))
print(json.dumps({"all_spill_free": all(r["spill_bytes"] == 0 for r in rows)}))
