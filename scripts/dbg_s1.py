import numpy as np, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, 'tests')
from rbc_testutil import uniform
import paper_1103_2635_b200 as rbc
g = np.load('tests/golden/golden.npz')
data = uniform(2000, 8, 101)
idx = rbc.build_exact(rbc.DataMatrix(data), 50, rbc.MetricSpec("l2", 8), seed=0)
q = g['bx_u8s0_queries']
out = rbc.exact_query_arrays(idx, q, 3)
print("gamma", out[2][:4], "want", g['xq_u8s0_k3_gamma'][:4])
