import json, sys
tag = None
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/ab.log'):
    if l.startswith('## '):
        tag = l[3:].strip(); continue
    if l.startswith('{'):
        d = json.loads(l)
        if 'us_per_step' in d:
            i = d['info']
            print(f"{tag:40s} BT={i['batch_tile']} NP={i['pairs_per_lane']} regs={i['regs_per_thread']} us/step={d['us_per_step']:.3f}")
        elif 'load' in d:
            print(f"{tag:40s}   " + ' | '.join(f"{k}: {d[k]['median']:.0f}" for k in ['load', 'op_loop', 'butterfly', 'bprime_wait', 'epilogue', 'gap', 'bar3', 'loop', 'tile_period', 'first_round', 'rounds0', 'rounds_max', 'pub_skew_ns', 'lastpub_to_loaded_ns'] if k in d))
    elif 'Error' in l or 'error' in l:
        print(tag, l.strip()[:160])

# medians per (tag) over rounds
import collections, statistics
agg = collections.defaultdict(list)
tag = None
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/ab.log'):
    if l.startswith('## '):
        tag = l[3:].strip(); continue
    if l.startswith('{'):
        d = json.loads(l)
        if 'us_per_step' in d:
            agg[tag].append(d['us_per_step'])
print("---- medians ----")
for k in sorted(agg, key=lambda t: (t.split(' ', 1)[1] if ' ' in t else '', t)):
    v = agg[k]
    print(f"{k:50s} n={len(v)} median={statistics.median(v):.3f} min={min(v):.3f} max={max(v):.3f}")
