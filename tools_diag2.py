import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2010_05872_b200 as mg
from oracle.oracle import Oracle
o = Oracle()
for shape in [(33, 33, 33), (33, 33, 65)]:
    x = np.random.default_rng(1).uniform(-10, 10, shape)
    h = mg.GridHierarchy.create(shape); L = h.num_levels()
    ws = mg.SolverWorkspace()
    got = mg.decompose(torch.from_numpy(x).cuda(), h, L - 1, ws).buffer.cpu().numpy()
    want = o.decompose(x, L - 1)
    cd = h.level_dims(L - 1); nc = h.node_count(L - 1)
    nodal = x[::2, ::2, ::2].ravel()
    zg = got[:nc] - nodal; zw = want[:nc] - nodal
    print(shape, "|z_ref| max", np.abs(zw).max(), "|z_gpu| max", np.abs(zg).max())
    zg3 = zg.reshape(cd); zw3 = zw.reshape(cd)
    np.set_printoptions(precision=4, linewidth=200)
    print(" ref z[0,0,:6]", zw3[0, 0, :6]); print(" gpu z[0,0,:6]", zg3[0, 0, :6])
    print(" ref z[5,7,:6]", zw3[5, 7, :6]); print(" gpu z[5,7,:6]", zg3[5, 7, :6])
    r = zg3 / np.where(np.abs(zw3) > 1e-9, zw3, np.nan)
    print(" ratio gpu/ref median", np.nanmedian(r), "p10/p90", np.nanpercentile(r, 10), np.nanpercentile(r, 90))
    # per-axis-0 plane error
    e = np.abs(zg3 - zw3).max(axis=(1, 2)); print(" err by i0", e[:8], "...")
    e = np.abs(zg3 - zw3).max(axis=(0, 2)); print(" err by i1", e[:8], "...")
