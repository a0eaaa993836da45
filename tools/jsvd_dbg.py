import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
a = np.random.Generator(np.random.PCG64(31)).standard_normal((15, 9))
f = P.dense.jacobi_svd(a)
print(f.sigma)
