import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_1804_10223_b200 import from_problem, inputs
cases = [(64,4,3,0.3,'fp32',1), (64,4,3,0.3,'fp32',0), (1000,4,12,0.3,'fp32',0), (1000,2,12,0.3,'fp32',0), (1000,4,12,0.3,'fp16',0), (257,4,5,0.3,'fp32',2)]
for H,B,T,d,prec,C in cases:
    prob = inputs.make_problem(H,H,B,T,d,act='relu',h0='random',seed_offset=H)
    m = from_problem(prob, prec=prec, num_ctas=C)
    x = torch.from_numpy(prob['x']).cuda(); h0 = torch.from_numpy(prob['h0']).cuda()
    out = m.forward(x, h0); torch.cuda.synchronize()
    try: m.status()
    except Exception as e: print('status', e)
    o = oracle.forward(prob)
    y = out[0].cpu().numpy().astype(np.float64)
    err = np.abs(y - o['y'])
    inf = m.info()
    bad = np.argwhere(err > 1e-3)
    print(H,B,T,d,prec,C, 'err %.3g'%err.max(), 'plan', inf['num_ctas'], inf['threads_per_cta'], inf['batch_tile'], 'first bad', bad[:3].tolist(), 'per-step', [float('%.2g'%err[t].max()) for t in range(T)])
    m.close()
