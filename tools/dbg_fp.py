import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1311_0089_b200 import *
g=np.load('tests/golden/generic3d.npz')
a=CoefficientField(GridSpec(tuple(g['Y']), tuple(int(s) for s in g['shape'])), g['packed'])
ref=ReferenceTensor(np.diag([3.0,2.0,2.5]))
rep=solve_neumann(a, LoadCase((0.3,-1.0,0.5)), SolverConfig(method='neumann', tol=1e-7, max_iter=5000, reference=ref))
h=np.array(rep.residual_history); hr=g['fp_history']
for x,y in zip(h,hr): print(f"{x:.17e} {y:.17e} {abs(x-y)/y:.2e}")
