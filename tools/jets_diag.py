import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_08271_b200 as rg
from oracle.oracle import Oracle
from tests.scenes import pair
ctx = rg.Context(0); orc = Oracle("C")
K = rg.simple_intrinsics(80, 60, 60.0)
fa, fb, T = pair(K, 8, "noisy", holes=True)
wp = rg.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth, T, K, ctx)
j, f = rg.residuals_and_jacobians(fa, wp, K, ctx=ctx, as_array=True)
jo, fo = orc.residuals_and_jacobians(fa.intensity, fa.inverse_depth, wp.intensity, wp.inverse_depth, K.to_c())
print(j.shape, jo.shape, np.array_equal(f, fo))
for c in range(17):
    d = np.abs(j[:, c] - jo[:, c]); rel = d / np.maximum(np.abs(jo[:, c]), 1e-300)
    print(c, "maxabs", d.max(), "maxrel", np.nanmax(np.where(np.abs(jo[:, c]) > 0, rel, 0)), "n_diff", int((j[:, c] != jo[:, c]).sum()))
