import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A
rng = np.random.default_rng(0)
for n in [5, 40, 80, 81, 100, 130, 257, 700]:
    M = rng.standard_normal((n, n)) + 0.1*np.eye(n)
    Mi = A.debug_inverse(torch.from_numpy(M).cuda()).cpu().numpy()
    print(n, np.abs(Mi @ M - np.eye(n)).max(), np.linalg.cond(M))
