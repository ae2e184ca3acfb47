"""Debug probe for the tensor-core BWW (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_1911_10175_b200 as sp

V = 16
N, C, K, H, W = 16, 128, 128, 16, 16
for R in (1, 3):
    sh = sp.ConvShape.make(N, C, K, H, W, R, R, 1, 1)
    rng = np.random.default_rng(0)
    d = rng.standard_normal((N, C, H, W)).astype(np.float32)
    dy = rng.standard_normal((N, K, H, W)).astype(np.float32)
    ref = O.dense(2, sh.astuple(), d, dy)
    ba, bb = sp.pack_act_chwnn(d, V).to("cuda"), sp.pack_act_nchwc(dy, V).to("cuda")
    pl = sp.plan(sh, sp.Component.bww, V)
    with sp.math_mode(sp.Math.tf32x3):
        res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
    got = sp.unpack(res.out).cpu().numpy()
    print(f"R={R} LBO={os.environ.get('SPC_TC_LBO')} SBO={os.environ.get('SPC_TC_SBO')} max|got|={np.abs(got).max():.4g} "
          f"max|ref|={np.abs(ref).max():.4g} err={O.max_abs_rel(got, ref):.3g} "
          f"corr={np.corrcoef(got.ravel(), ref.ravel())[0, 1]:.4f}")
    if R == 1:
        # k (rows) x c (cols) structure of the error
        e = np.abs(got[:, :, 0, 0] - ref[:, :, 0, 0])
        print("  err by k-block:", np.round(e.reshape(8, 16, 8, 16).max(axis=(1, 2, 3)), 3))
        print("  err by c-block:", np.round(e.reshape(8, 16, 8, 16).max(axis=(0, 1, 3)), 3))
