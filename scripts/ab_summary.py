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
            print(f"{tag:40s}   " + ' | '.join(f"{k}: {d[k]['median']:.0f}" for k in ['load', 'operate', 'epilogue', 'gap', 'tile_period']))
    elif 'Error' in l or 'error' in l:
        print(tag, l.strip()[:160])
