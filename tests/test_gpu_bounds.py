"""Out-of-bounds access checks without compute-sanitizer (closed on this GPU
pool: "runs under it have left GPUs needing a reset").

Every operand and output of a pass is placed in the middle of a larger device
buffer whose guard zones (64 KiB each side) hold a sentinel:

* WRITES: the output's guard zones must be bit-identical after the pass, and
  the counters' neighbours untouched;
* READS that matter: the pass runs twice, once with the operands' guard zones
  filled with 0 and once with NaN.  A kernel that reads outside its operands
  and lets the value reach an output (or a zero/nonzero decision) shows up as
  a NaN / a differing bit / a differing counter.

Covered: every kernel family of the FP32 path (tile FWD/BWI branch + jump-table
pairs, KK=2 and KK=4, 3x3 stride 1 and 2, 1x1 GEMM, BWW tile/row/1x1/generic,
the non-finite fallbacks) and the 3xTF32 tcgen05/TMA kernels, sparse and dense,
on ragged shapes with partial tiles.
"""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
GUARD = 16384  # floats (64 KiB) each side


def _guarded(t: torch.Tensor, fill: float):
    buf = torch.full((t.numel() + 2 * GUARD,), fill, dtype=torch.float32, device="cuda")
    buf[GUARD:GUARD + t.numel()] = t.reshape(-1)
    return buf, buf[GUARD:GUARD + t.numel()]


def _run(sp, comp, check, sh, a, b, mode, fill, V=16):
    ga, va = _guarded(a.data, fill)
    gb, vb = _guarded(b.data, fill)
    A = sp.BlockedTensor(**{**a.header(), "data": va})
    B = sp.BlockedTensor(**{**b.header(), "data": vb})
    pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
    desc, numel = sp.api.output_desc(sh, pl)
    sentinel = -123.25
    out_buf = torch.full((numel + 2 * GUARD,), sentinel, device="cuda")
    cnt_buf = torch.full((12,), 7, dtype=torch.int64, device="cuda")
    pp = sp.PreparedPass(A, B, sh, pl, sp.RunMode(mode), out=out_buf[GUARD:GUARD + numel], counters=cnt_buf[4:8])
    pp.counters.zero_()
    pp.launch(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ob = out_buf.cpu().numpy()
    assert np.all(ob[:GUARD] == sentinel) and np.all(ob[GUARD + numel:] == sentinel), "write outside the output"
    cb = cnt_buf.cpu().numpy()
    assert np.all(cb[:4] == 7) and np.all(cb[8:] == 7), "write outside the counters"
    # operand guard zones are read-only too
    for g in (ga, gb):
        h = g.cpu().numpy()
        assert np.array_equal(h[:GUARD], np.full(GUARD, fill, np.float32), equal_nan=True)
        assert np.array_equal(h[-GUARD:], np.full(GUARD, fill, np.float32), equal_nan=True)
    return ob[GUARD:GUARD + numel].copy(), cb[4:8].copy()


CASES = [  # (N, C, K, H, W, R, stride)
    (3, 64, 64, 13, 11, 3, 1), (2, 128, 128, 9, 15, 3, 1), (2, 64, 128, 10, 7, 3, 2), (3, 128, 256, 7, 9, 3, 2),
    (2, 64, 128, 9, 10, 1, 1), (3, 128, 64, 7, 6, 1, 2), (2, 32, 48, 7, 9, 3, 1), (19, 64, 128, 5, 6, 3, 1),
]


@pytest.mark.parametrize("math", ["fp32", "tf32x3"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_no_out_of_bounds_reads_or_writes(sp, case, math):
    N, C, K, H, W, R, st = case
    V = 16
    sh = sp.ConvShape.make(N, C, K, H, W, R, R, st, st)
    for s in (0.5, 0.93):
        D = O.gen_sparse(N, C, H, W, s, 3)
        G = O.gen_sparse(K, C, R, R, 0.0, 4)
        dY = O.gen_sparse(N, K, sh.out_h(), sh.out_w(), s, 5)
        ops = [(0, 0, sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)),
               (1, 0, sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)),
               (2, 0, sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V)),
               (2, 1, sp.pack_act_nchwc(D, V), sp.pack_act_chwnn(dY, V))]
        with sp.math_mode(sp.Math[math]):
            for comp, check, a, b in ops:
                a, b = a.to("cuda"), b.to("cuda")
                for mode in (0, 1):
                    o0, c0 = _run(sp, comp, check, sh, a, b, mode, 0.0)
                    o1, c1 = _run(sp, comp, check, sh, a, b, mode, float("nan"))
                    assert np.isfinite(o0).all() and np.isfinite(o1).all(), (case, comp, check, mode)
                    assert np.array_equal(o0.view(np.uint32), o1.view(np.uint32)), (case, comp, check, mode)
                    assert np.array_equal(c0, c1)
