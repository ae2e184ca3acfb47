"""Shared GPU-vs-reference parity helpers (test infrastructure).

``ref_vs_gpu`` runs one pass of the UNMODIFIED reference library
(``oracle.RefRun`` -> ``spconv::run_parallel``, P/src/kernels.cpp:304-313,
backend automatic, all host threads) and the product's device path
(``spc_sparse_*`` through the C ABI -- the same entry ``PreparedPass`` and
``bench.py`` launch, so the same per-shape dispatch: split counts, kernel
pairs, block order) on the byte-identical blocked operands the reference
packed, and returns the north-star error and both counter sets.
"""
from __future__ import annotations

import os

import numpy as np

import oracle as O

TOL = 1e-5  # max|got-ref| / max|ref| (BASELINE.json north_star)


def blocked_operands(sp, sh, comp, check, ta, tb, V=16):
    """Wrap the reference's packed operands (device tensors) as BlockedTensors."""
    if comp == 0:
        ba = sp.BlockedTensor(sp.Layout.act_nchwc, V, sh.N, sh.C, sh.H, sh.W, data=ta)
        bb = sp.BlockedTensor(sp.Layout.filter_kcrs_blk, V, k=sh.K, c=sh.C, s=sh.S, r=sh.R, data=tb)
    elif comp == 1:
        ba = sp.BlockedTensor(sp.Layout.act_nchwc, V, sh.N, sh.K, sh.out_h(), sh.out_w(), data=ta)
        bb = sp.BlockedTensor(sp.Layout.filter_kcrs_blk, V, k=sh.C, c=sh.K, s=sh.S, r=sh.R, data=tb)
    else:
        la = sp.Layout.act_chwnn if check == 0 else sp.Layout.act_nchwc
        lb = sp.Layout.act_nchwc if check == 0 else sp.Layout.act_chwnn
        ba = sp.BlockedTensor(la, V, sh.N, sh.C, sh.H, sh.W, data=ta)
        bb = sp.BlockedTensor(lb, V, sh.N, sh.K, sh.out_h(), sh.out_w(), data=tb)
    return ba, bb


def ref_vs_gpu(sp, sh, comp, check, a, b, V=16, workers=None, mode=0, keep_gpu=False):
    """One pass on both sides.  a, b: plain operands in the reference's
    argument order ((D, G) fwd, (dY, G) bwi, (D, dY) bww).  Returns a dict with
    ``err`` (north-star metric vs the reference CPU fp32 result), both counter
    sets, and optionally the GPU output (plain layout, numpy)."""
    import torch
    workers = workers or os.cpu_count() or 1
    r = O.RefRun(comp, check, sh.astuple(), V, a, b)
    try:
        r.exec(mode, workers)
        ref_out, ref_cnt, _ = r.result()
        ta = torch.from_numpy(r.operand(0)).cuda()
        tb = torch.from_numpy(r.operand(1)).cuda()
    finally:
        r.close()
    ba, bb = blocked_operands(sp, sh, comp, check, ta, tb, V)
    pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
    res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode(mode))
    got = sp.unpack(res.out).cpu().numpy()
    del ta, tb, ba, bb
    out = {"err": O.max_abs_rel(got, ref_out), "ref": ref_cnt, "gpu": res.counters,
           "finite": bool(np.isfinite(got).all())}
    if keep_gpu:
        out["out"] = got
    return out


def assert_counts_equal(res, ctx):
    g, r = res["gpu"], res["ref"]
    assert g.executed_vector_fmas == r["executed_vector_fmas"], (ctx, g, r)
    assert g.checked_vectors == r["checked_vectors"], (ctx, g, r)
    assert g.output_vector_loads == r["output_vector_loads"], (ctx, g, r)
    assert g.output_vector_stores == r["output_vector_stores"], (ctx, g, r)
