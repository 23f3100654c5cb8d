import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2104_01101_b200.linalg import chol_inv_upper_dev
for n in (401, 450, 512):
    g = np.random.default_rng(n)
    z = g.standard_normal((2 * n + 8, n)) @ np.diag(np.logspace(0, -2, n))
    gram = torch.from_numpy(z.T @ z).cuda()
    os.environ["SKX_CHOL_ONE_CTA"] = "1"
    r1, i1, f1 = (x.cpu().numpy() for x in chol_inv_upper_dev(gram))
    del os.environ["SKX_CHOL_ONE_CTA"]
    r2, i2, f2 = (x.cpu().numpy() for x in chol_inv_upper_dev(gram))
    dr = np.abs(r1 - r2); di = np.abs(i1 - i2)
    print(n, 'info', f1, f2, 'R maxdiff', dr.max(), 'Rinv maxdiff', di.max())
    bad = np.argwhere(di > 1e-9 * np.abs(i1).max())
    if len(bad):
        rows = np.unique(bad[:, 0] // 32); cols = np.unique(bad[:, 1] // 32)
        print('   bad row blocks', rows[:20], 'col blocks', cols[:20], 'count', len(bad))
        print('   first', bad[:5].tolist(), 'lower?', (bad[:, 0] > bad[:, 1]).sum())
