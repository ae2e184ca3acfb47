"""Accuracy probe of the 3xTF32 tensor-core variant vs the 64-bit oracle
(development tool): prints max|got-ref|/max|ref| per shape and pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_1911_10175_b200 as sp

V = 16
SHAPES = [(1, 256, 128, 14, 14, 3, 3), (1, 512, 512, 14, 14, 3, 3), (2, 512, 256, 28, 28, 3, 3),
          (2, 64, 64, 56, 56, 3, 3), (1, 1024, 256, 14, 14, 1, 1)]
rng = np.random.default_rng(0)
sp.set_math(sp.Math.tf32x3)
for shape in SHAPES:
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 1, 1)
    t = sh.astuple()
    g = (rng.standard_normal((K, C, S, R)) * np.sqrt(2.0 / (C * R * S))).astype(np.float32)
    out = []
    for comp in (0, 1):
        shp = (N, C, H, W) if comp == 0 else (N, K, sh.out_h(), sh.out_w())
        a = np.maximum(rng.standard_normal(shp).astype(np.float32), 0)
        ref = O.dense(comp, t, a, g)
        ba = sp.pack_act_nchwc(a, V).to("cuda")
        bb = (sp.pack_filter(g, V) if comp == 0 else sp.pack_filter(g, V, True)).to("cuda")
        res = sp.run_parallel(ba, bb, sh, sp.plan(sh, sp.Component(comp), V), sp.RunMode.sparse)
        got = sp.unpack(res.out).cpu().numpy()
        out.append(f"{['fwd', 'bwi'][comp]} {O.max_abs_rel(got, ref):.2e}")
    print(f"SEG={os.environ.get('SPC_TC_SEG', 'default')} {shape}: " + "  ".join(out), flush=True)
