"""Warp-stall samples of an ncu source page (csv) summed between synchronisation points."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
S = idx['Warp Stall Sampling (All Samples)']
E = idx['Instructions Executed']
tot = sum(int(r[S] or 0) for r in data)
print('total samples', tot)
acc = seg = 0
start = data[0][0][-5:]
for r in data:
    n = int(r[S] or 0)
    acc += n
    seg += n
    src = r[1]
    if any(k in src for k in ('BAR.SYNC', 'EXIT', 'LDGDEPBAR', 'DEPBAR', 'LDG.E.128', 'SHFL.BFLY', 'STG.E')) and int(r[E] or 0) > 0:
        print(f"{start}-{r[0][-5:]} seg {100 * seg / tot:5.1f}%  cum {100 * acc / tot:5.1f}%  {src.strip()[:58]} exec={r[E]}")
        seg = 0
        start = r[0][-5:]
