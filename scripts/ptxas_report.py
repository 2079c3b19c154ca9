"""Summarise registers / stack / spills per kernel instance from the build's ptxas log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1804_10223_b200/_build/ptxas.log").read().splitlines()
cur = None
rows = []
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur, st, sp = m.group(1), 0, 0
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        st, sp = int(m.group(1)), int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        k = re.search(r"srnn_persistent_kernelILi(\d+)ELi(\d+)ELi(\d+)ELb(\d)ELi(n?\d+)E", cur)
        name = (f"rec NP={k.group(1)} BT={k.group(2)} G={k.group(3)} f16={k.group(4)} MT={k.group(5).replace('n', '-')}"
                if k else cur[:60])
        rows.append((name, int(m.group(1)), st, sp))
        cur = None
bad = [r for r in rows if r[2] or r[3]]
for r in rows:
    print(f"{r[0]:40s} regs={r[1]:3d} stack={r[2]:3d} spill={r[3]:3d}")
print(f"{len(rows)} kernels, {len(bad)} with stack/spill")
