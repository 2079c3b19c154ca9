"""Print one line per quick_time / timeline JSON record in the given logs."""
import json
import sys

for fn in sys.argv[1:]:
    for line in open(fn):
        try:
            d = json.loads(line)
        except Exception:
            if line.strip():
                print("  !", line.rstrip()[:200])
            continue
        c = d["cfg"]
        key = f"H={c['H']} B={c['B']} d={c['d']} {c['prec']} {c.get('cell','rnn')} {c.get('pattern','')} flags={c.get('flags',0)}"
        if "us_per_step" in d:
            print(f"{key:55s} us/step {d['us_per_step']:.3f} fwd {d['fwd_ms']:.3f} ms gemm {d['gemm_ms']*1e3:.1f} us")
        else:
            ph = {k: round(v["median"]) for k, v in d.items() if isinstance(v, dict) and "median" in v}
            print(f"{key:55s} {ph}")
