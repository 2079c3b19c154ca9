import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys
from paper_1804_10223_b200 import inputs, from_problem, FLAG_HOST_ONLY
H=int(sys.argv[1]); d=float(sys.argv[2]); B=int(sys.argv[3]) if len(sys.argv)>3 else 4
prob=inputs.make_problem(H,H,B,4,d)
m=from_problem(prob,prec="fp16",flags=FLAG_HOST_ONLY)
print(m.info())
