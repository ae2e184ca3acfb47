"""GPU parity of the 3xTF32 tensor-core variant (spc_set_math(SPC_MATH_TF32X3),
SURVEY.md 8(f)4) against the 64-bit oracle.

Stated tolerance of the variant: max|got - ref| / max|ref|
<= TC_TOL = 1e-5 -- the north-star fp32 gate itself; 3xTF32 products carry
~2^-21 relative error, measured ~1e-7 here.  Counters (executed_vector_fmas,
checked_vectors) stay integer-exact; Inf/NaN inputs take the exact FFMA path.
"""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
TC_TOL = 1e-5
V = 16


def _gauss_relu(rng, shape, s):
    x = rng.standard_normal(shape).astype(np.float32)
    x[rng.random(shape) < s] = 0.0
    return x


def _run(sp, sh, comp, a, b, mode=0, math=None, epi=None):
    math = sp.Math.tf32x3 if math is None else math
    if comp == 0:
        ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V)
    else:
        ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V, True)
    ba, bb = ba.to("cuda"), bb.to("cuda")
    pl = sp.plan(sh, sp.Component(comp), V)
    with sp.math_mode(math):
        res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode(mode))
    return pl, res, sp.unpack(res.out).cpu().numpy()


SHAPES = [
    (2, 64, 64, 56, 56, 3, 3),
    (2, 128, 256, 28, 28, 3, 3),
    (1, 256, 128, 14, 14, 3, 3),
    (3, 64, 128, 13, 9, 3, 3),
    (2, 512, 512, 7, 7, 3, 3),
    (2, 128, 64, 20, 36, 1, 1),
    (1, 256, 512, 14, 14, 1, 1),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("comp", [0, 1])
def test_tc_matches_oracle(sp, shape, comp):
    rng = np.random.default_rng(hash((shape, comp)) & 0xFFFF)
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 1, 1)
    t = sh.astuple()
    if comp == 0:
        a = _gauss_relu(rng, (N, C, H, W), 0.6)
    else:
        a = _gauss_relu(rng, (N, K, sh.out_h(), sh.out_w()), 0.5)
    g = (rng.standard_normal((K, C, S, R)) * np.sqrt(2.0 / (C * R * S))).astype(np.float32)
    ref = O.dense(comp, t, a, g)
    pl, res, got = _run(sp, sh, comp, a, g)
    err = O.max_abs_rel(got, ref)
    assert err <= TC_TOL, (shape, comp, err)
    want = O.expected_counts(t, O.plan(t, comp, V, 30, 0), a)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    assert res.counters.checked_vectors == want["checked_vectors"]
    # dense mode: same arithmetic, analytic dense total
    _, dres, dgot = _run(sp, sh, comp, a, g, mode=1)
    assert np.array_equal(dgot, got)
    assert dres.counters.executed_vector_fmas == want["dense_total"]


def test_tc_is_deterministic_and_close_to_fp32_path(sp):
    rng = np.random.default_rng(3)
    sh = sp.ConvShape.make(2, 128, 128, 28, 28, 3, 3, 1, 1)
    a = _gauss_relu(rng, (2, 128, 28, 28), 0.5)
    g = (rng.standard_normal((128, 128, 3, 3)) * 0.04).astype(np.float32)
    _, _, g1 = _run(sp, sh, 0, a, g)
    _, _, g2 = _run(sp, sh, 0, a, g)
    _, _, f32 = _run(sp, sh, 0, a, g, math=sp.Math.fp32)
    assert np.array_equal(g1, g2)
    assert O.max_abs_rel(g1, f32) <= TC_TOL


@pytest.mark.parametrize("where", ["src_nan", "src_inf", "filt_inf"])
def test_tc_nonfinite_inputs_take_exact_path(sp, where):
    rng = np.random.default_rng(11)
    sh = sp.ConvShape.make(1, 64, 128, 12, 12, 3, 3, 1, 1)
    a = _gauss_relu(rng, (1, 64, 12, 12), 0.5)
    g = (rng.standard_normal((128, 64, 3, 3)) * 0.05).astype(np.float32)
    if where == "src_nan":
        a[0, 3, 4, 5] = np.nan
    elif where == "src_inf":
        a[0, 7, 0, 0] = np.inf
    else:
        a[0, 9, :, :] = 0.0  # an all-zero channel: the reference skips it, so Inf taps there stay harmless
        g[5, 9, 1, 1] = np.inf
    _, r32, f32 = _run(sp, sh, 0, a, g, math=sp.Math.fp32)
    _, rtc, tc = _run(sp, sh, 0, a, g)
    assert np.array_equal(np.isnan(tc), np.isnan(f32))
    assert np.array_equal(np.isinf(tc), np.isinf(f32))
    assert np.array_equal(tc, f32) or O.max_abs_rel(np.nan_to_num(tc), np.nan_to_num(f32)) <= TC_TOL
    assert rtc.counters.executed_vector_fmas == r32.counters.executed_vector_fmas


def test_tc_fused_epilogue(sp):
    import torch
    rng = np.random.default_rng(5)
    sh = sp.ConvShape.make(2, 64, 128, 14, 14, 3, 3, 1, 1)
    a = _gauss_relu(rng, (2, 64, 14, 14), 0.5)
    g = (rng.standard_normal((128, 64, 3, 3)) * 0.06).astype(np.float32)
    add = _gauss_relu(rng, (2, 128, 14, 14), 0.0)
    mask = _gauss_relu(rng, (2, 128, 14, 14), 0.5)
    ba, bb = sp.pack_act_nchwc(a, V).to("cuda"), sp.pack_filter(g, V).to("cuda")
    badd, bmask = sp.pack_act_nchwc(add, V).to("cuda"), sp.pack_act_nchwc(mask, V).to("cuda")
    pl = sp.plan(sh, sp.Component.fwd, V)
    epi = sp.Epilogue(alpha=0.25, add=badd.data, mask=bmask.data, relu=True)
    outs = []
    for m in (sp.Math.fp32, sp.Math.tf32x3):
        with sp.math_mode(m):
            p = sp.PreparedPass(ba, bb, sh, pl, epilogue=epi)
            p.launch(torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            outs.append(p.out.cpu().numpy().copy())
    f32, tc = outs
    assert np.array_equal(f32 == 0, tc == 0) or np.mean((f32 == 0) != (tc == 0)) < 1e-4
    assert O.max_abs_rel(tc, f32) <= TC_TOL


BWW_SHAPES = [
    (3, 64, 128, 13, 9, 3, 3),      # ragged 16-image block, odd extents
    (16, 128, 256, 28, 28, 3, 3),
    (4, 256, 128, 14, 14, 3, 3),
    (2, 512, 512, 7, 7, 3, 3),
    (20, 64, 64, 30, 17, 3, 3),
    (8, 128, 256, 14, 14, 1, 1),
    (20, 256, 256, 13, 11, 3, 3),  # CTA-pair BWW (C >= 256, two k tiles), ragged images
]


@pytest.mark.parametrize("shape", BWW_SHAPES)
@pytest.mark.parametrize("check", [0, 1])
def test_tc_bww_matches_oracle(sp, shape, check):
    rng = np.random.default_rng((hash(shape) + check) & 0xFFFF)
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 1, 1)
    t = sh.astuple()
    d = _gauss_relu(rng, (N, C, H, W), 0.6)
    dy = _gauss_relu(rng, (N, K, sh.out_h(), sh.out_w()), 0.5)
    ref = O.dense(2, t, d, dy)
    if check == 0:
        ba, bb = sp.pack_act_chwnn(d, V), sp.pack_act_nchwc(dy, V)
    else:
        ba, bb = sp.pack_act_nchwc(d, V), sp.pack_act_chwnn(dy, V)
    ba, bb = ba.to("cuda"), bb.to("cuda")
    pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck(check))
    with sp.math_mode(sp.Math.tf32x3):
        res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
        dres = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.dense)
    got = sp.unpack(res.out).cpu().numpy()
    err = O.max_abs_rel(got, ref)
    assert err <= TC_TOL, (shape, check, err)
    want = O.expected_counts(t, O.plan(t, 2, V, 30, check), d if check == 0 else dy)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    assert res.counters.checked_vectors == want["checked_vectors"]
    assert np.array_equal(sp.unpack(dres.out).cpu().numpy(), got)
    assert dres.counters.executed_vector_fmas == want["dense_total"]


def test_tc_bww_nonfinite_takes_exact_path(sp):
    rng = np.random.default_rng(21)
    sh = sp.ConvShape.make(4, 64, 128, 10, 10, 3, 3, 1, 1)
    d = _gauss_relu(rng, (4, 64, 10, 10), 0.5)
    dy = _gauss_relu(rng, (4, 128, 10, 10), 0.5)
    dy[1, 5, 3, 3] = np.inf
    d[2, 7, 4, 4] = np.nan
    ba, bb = sp.pack_act_chwnn(d, V).to("cuda"), sp.pack_act_nchwc(dy, V).to("cuda")
    pl = sp.plan(sh, sp.Component.bww, V)
    outs = []
    for m in (sp.Math.fp32, sp.Math.tf32x3):
        with sp.math_mode(m):
            r = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
            outs.append((sp.unpack(r.out).cpu().numpy(), r.counters.executed_vector_fmas))
    (f32, c32), (tc, ctc) = outs
    assert np.array_equal(np.isnan(tc), np.isnan(f32)) and np.array_equal(np.isinf(tc), np.isinf(f32))
    fin = np.isfinite(f32)
    if os.environ.get("SPC_FORCE_GENERIC") == "1":
        # A/B knob: the FP32 run took the shape-general kernel, whose reduction
        # order differs from the tile BWW behind the tensor-core fallback
        assert O.max_abs_rel(tc[fin], f32[fin]) <= TC_TOL
    else:
        assert np.array_equal(tc[fin], f32[fin])
    assert ctc == c32


@pytest.mark.parametrize("comp", [0, 1])
@pytest.mark.parametrize("shape", [(2, 128, 256, 28, 28, 3, 3), (3, 64, 64, 40, 40, 3, 3), (2, 256, 128, 14, 14, 1, 1)])
def test_tc_skips_all_zero_tiles_exactly(sp, shape, comp):
    """Spatially structured zeros (whole channel blocks, half images): the
    variant's all-zero tile skip (north_star: "skips all-zero tiles") leaves
    outputs and exact counters unchanged, and sparse == dense bit for bit."""
    rng = np.random.default_rng(17 + comp)
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 1, 1)
    t = sh.astuple()
    chans = C if comp == 0 else K
    hh, ww = (H, W) if comp == 0 else (sh.out_h(), sh.out_w())
    a = _gauss_relu(rng, (N, chans, hh, ww), 0.5)
    a[:, 16:48] = 0.0                  # two whole 16-channel blocks
    a[0, :, : hh // 2] = 0.0           # top half of image 0
    a[-1, :, :, ww // 3:] = 0.0        # right two thirds of the last image
    g = (rng.standard_normal((K, C, S, R)) * np.sqrt(2.0 / (C * R * S))).astype(np.float32)
    ref = O.dense(comp, t, a, g)
    _, res, got = _run(sp, sh, comp, a, g)
    assert O.max_abs_rel(got, ref) <= TC_TOL
    want = O.expected_counts(t, O.plan(t, comp, V, 30, 0), a)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    _, _, dgot = _run(sp, sh, comp, a, g, mode=1)
    assert np.array_equal(dgot, got)


S2_SHAPES = [
    (2, 64, 128, 56, 56, 3, 3),     # ResNet stage-transition 3x3 s2
    (3, 128, 128, 15, 13, 3, 3),    # odd extents: ragged parity classes
    (2, 256, 512, 28, 28, 1, 1),    # 1x1 s2 projection
    (2, 64, 256, 13, 11, 1, 1),
]


@pytest.mark.parametrize("shape", S2_SHAPES)
@pytest.mark.parametrize("comp", [0, 1])
def test_tc_stride2_matches_oracle(sp, shape, comp):
    """Stride 2 on the tensor cores: FWD with TMA traversal stride 2, BWI as
    its 4 output parity classes (gap columns exactly 0 for 1x1)."""
    rng = np.random.default_rng((hash(shape) + 7 * comp) & 0xFFFF)
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 2, 2)
    t = sh.astuple()
    a = _gauss_relu(rng, (N, C, H, W) if comp == 0 else (N, K, sh.out_h(), sh.out_w()), 0.6)
    g = (rng.standard_normal((K, C, S, R)) * np.sqrt(2.0 / (C * R * S))).astype(np.float32)
    ref = O.dense(comp, t, a, g)
    _, res, got = _run(sp, sh, comp, a, g)
    assert O.max_abs_rel(got, ref) <= TC_TOL, (shape, comp, O.max_abs_rel(got, ref))
    if comp == 1 and R == 1:
        assert not got[:, :, 1::2, :].any() and not got[:, :, :, 1::2].any()  # stride gaps exactly 0
    want = O.expected_counts(t, O.plan(t, comp, V, 30, 0), a)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    _, _, dgot = _run(sp, sh, comp, a, g, mode=1)
    assert np.array_equal(dgot, got)


@pytest.mark.parametrize("shape", [(16, 64, 128, 56, 56, 3, 3), (20, 128, 256, 14, 14, 1, 1)])
@pytest.mark.parametrize("check", [0, 1])
def test_tc_bww_stride2_matches_oracle(sp, shape, check):
    rng = np.random.default_rng((hash(shape) + check) & 0xFFFF)
    N, C, K, H, W, R, S = shape
    sh = sp.ConvShape.make(N, C, K, H, W, R, S, 2, 2)
    t = sh.astuple()
    d = _gauss_relu(rng, (N, C, H, W), 0.6)
    dy = _gauss_relu(rng, (N, K, sh.out_h(), sh.out_w()), 0.5)
    ref = O.dense(2, t, d, dy)
    if check == 0:
        ba, bb = sp.pack_act_chwnn(d, V), sp.pack_act_nchwc(dy, V)
    else:
        ba, bb = sp.pack_act_nchwc(d, V), sp.pack_act_chwnn(dy, V)
    pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck(check))
    with sp.math_mode(sp.Math.tf32x3):
        res = sp.run_parallel(ba.to("cuda"), bb.to("cuda"), sh, pl, sp.RunMode.sparse)
    got = sp.unpack(res.out).cpu().numpy()
    assert O.max_abs_rel(got, ref) <= TC_TOL, (shape, check, O.max_abs_rel(got, ref))
    want = O.expected_counts(t, O.plan(t, 2, V, 30, check), d if check == 0 else dy)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]


@pytest.mark.parametrize("R", [1, 3])
@pytest.mark.parametrize("comp", [0, 1, 2])
def test_tc_stride2_nonfinite_takes_exact_path(sp, R, comp):
    """Inf/NaN with stride 2: the tensor-core kernels exit and the gated FFMA
    stride-2 kernels produce the reference's exact skip semantics."""
    rng = np.random.default_rng(31 + R + 5 * comp)
    sh = sp.ConvShape.make(4, 64, 128, 12, 12, R, R, 2, 2)
    hp, wp = sh.out_h(), sh.out_w()
    d = _gauss_relu(rng, (4, 64, 12, 12), 0.5)
    dy = _gauss_relu(rng, (4, 128, hp, wp), 0.5)
    g = (rng.standard_normal((128, 64, R, R)) * 0.05).astype(np.float32)
    if comp == 0:
        d[1, 2, 4, 4] = np.nan
        ba, bb = sp.pack_act_nchwc(d, V), sp.pack_filter(g, V)
    elif comp == 1:
        dy[2, 3, 1, 2] = np.inf
        ba, bb = sp.pack_act_nchwc(dy, V), sp.pack_filter(g, V, True)
    else:
        dy[0, 5, 2, 2] = -np.inf
        ba, bb = sp.pack_act_chwnn(d, V), sp.pack_act_nchwc(dy, V)
    ba, bb = ba.to("cuda"), bb.to("cuda")
    pl = sp.plan(sh, sp.Component(comp), V)
    outs = []
    for m in (sp.Math.fp32, sp.Math.tf32x3):
        with sp.math_mode(m):
            r = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
            outs.append((sp.unpack(r.out).cpu().numpy(), r.counters.executed_vector_fmas))
    (f32, c32), (tc, ctc) = outs
    assert np.array_equal(np.isnan(tc), np.isnan(f32)) and np.array_equal(np.isinf(tc), np.isinf(f32))
    fin = np.isfinite(f32)
    # the fallback is an FFMA kernel (the tile kernel), the FP32 default for
    # 1x1 BWW is the GEMM kernel: same products, possibly another summation order
    assert O.max_abs_rel(tc[fin], f32[fin]) <= TC_TOL
    assert ctc == c32


def test_tc_random_geometries_match_oracle(sp):
    """Randomised sweep of the geometries the variant covers (odd and tiny
    extents, 1..20 images, 64..256 channels, 3x3 / 1x1, stride 1 / 2), every
    pass and both BWW check sides against the 64-bit oracle, counters exact."""
    rng = np.random.default_rng(2024)
    for trial in range(48):
        N = int(rng.integers(1, 21))
        C, K = (int(x) for x in rng.choice([64, 128, 192, 256], 2))
        R = int(rng.choice([1, 3]))
        O_ = int(rng.choice([1, 2]))
        H, W = (int(x) for x in rng.integers(1, 21, 2))
        sh = sp.ConvShape.make(N, C, K, H, W, R, R, O_, O_)
        t = sh.astuple()
        d = _gauss_relu(rng, (N, C, H, W), float(rng.uniform(0.3, 0.9)))
        dy = _gauss_relu(rng, (N, K, sh.out_h(), sh.out_w()), float(rng.uniform(0.3, 0.9)))
        g = (rng.standard_normal((K, C, R, R)) * np.sqrt(2.0 / (C * R * R))).astype(np.float32)
        cases = [(0, 0, sp.pack_act_nchwc(d, V), sp.pack_filter(g, V), d, O.dense(0, t, d, g)),
                 (1, 0, sp.pack_act_nchwc(dy, V), sp.pack_filter(g, V, True), dy, O.dense(1, t, dy, g))]
        ref2 = O.dense(2, t, d, dy)
        cases += [(2, 0, sp.pack_act_chwnn(d, V), sp.pack_act_nchwc(dy, V), d, ref2),
                  (2, 1, sp.pack_act_nchwc(d, V), sp.pack_act_chwnn(dy, V), dy, ref2)]
        for comp, check, a, b, mask, ref in cases:
            pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
            with sp.math_mode(sp.Math.tf32x3):
                res = sp.run_parallel(a.to("cuda"), b.to("cuda"), sh, pl, sp.RunMode.sparse)
            got = sp.unpack(res.out).cpu().numpy()
            err = O.max_abs_rel(got, ref) if np.abs(ref).max() > 0 else float(np.abs(got).max())
            assert err <= TC_TOL, (trial, t, comp, check, err)
            want = O.expected_counts(t, O.plan(t, comp, V, 30, check), mask)
            assert res.counters.executed_vector_fmas == want["executed_vector_fmas"], (trial, t, comp, check)


def test_tc_host_buffer_path_matches_device_path(sp):
    """The host-buffer drop-in (spc_run_parallel_host: chunked H2D / kernels /
    D2H) under the tensor-core variant: FWD/BWI bitwise equal to the device
    path (per-image tiles do not depend on the chunking), BWW (chunk partials
    summed in fixed order) within the stated tolerance, counters equal."""
    rng = np.random.default_rng(41)
    sh = sp.ConvShape.make(40, 128, 256, 20, 18, 3, 3, 1, 1)
    d = _gauss_relu(rng, (40, 128, 20, 18), 0.6)
    dy = _gauss_relu(rng, (40, 256, 20, 18), 0.5)
    g = (rng.standard_normal((256, 128, 3, 3)) * 0.03).astype(np.float32)
    cases = [(0, 0, sp.pack_act_nchwc(d, V), sp.pack_filter(g, V)),
             (1, 0, sp.pack_act_nchwc(dy, V), sp.pack_filter(g, V, True)),
             (2, 0, sp.pack_act_chwnn(d, V), sp.pack_act_nchwc(dy, V))]
    with sp.math_mode(sp.Math.tf32x3):
        for comp, check, a, b in cases:
            pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
            rd = sp.run_parallel(a.to("cuda"), b.to("cuda"), sh, pl, sp.RunMode.sparse)
            rh = sp.run_parallel(a, b, sh, pl, sp.RunMode.sparse)
            gd = rd.out.data.cpu().numpy()
            if comp < 2:
                assert np.array_equal(rh.out.data, gd), comp
            else:
                assert O.max_abs_rel(rh.out.data, gd) <= TC_TOL
            assert rh.counters == rd.counters
