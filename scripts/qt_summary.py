import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/qt.log'):
    if l.startswith('{'):
        d = json.loads(l); i = d['info']; c = d['cfg']
        print(f"H={c['H']} B={c['B']} d={c['d']} {c['cell']} {c['prec']} flags={c['flags']} | C={i['num_ctas']} L={i['lanes_per_row']} NP={i['pairs_per_lane']}/{i['slots_used']} thr={i['threads_per_cta']} regs={i['regs_per_thread']} wf={i['wavefronts_per_step_max']} | us/step={d['us_per_step']:.3f} gemm_ms={d['gemm_ms']:.3f}")
    elif 'Error' in l:
        print(l.strip()[:200])
