"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Mirrors the reference's hot-path suite P/tests/test_kernels.cpp case for case.
Bars (BASELINE.json north_star):
  * fp32 outputs: max|got - ref| / max|ref| <= 1e-5 (TOL below) against the
    64-bit oracle, and the reference's own elementwise metric <= 1e-4 on the
    all-positive gen_sparse inputs its tests use;
  * zero/nonzero indexing: executed_vector_fmas and checked_vectors equal the
    reference's exact counts (integer equality);
  * bitwise determinism run to run.
"""
import glob
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5  # max-abs-normalised fp32 tolerance (north_star)
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
ALL = [(0, 0), (1, 0), (2, 0), (2, 1)]  # (comp, check)


def rng_tiny_shape(rng, V):
    from test_oracle import rng_tiny_shape as f
    return f(rng, V)


def make_inputs(sp, sh, comp, check, s, V, seed):
    """testutil::make_inputs (P/tests/testutil.hpp:43-78) with the oracle's
    bit-identical gen_sparse; returns plain operands + blocked device operands."""
    t = sh.astuple()
    N, C, K, H, W, R, S = t[:7]
    hp, wp = sh.out_h(), sh.out_w()
    if comp == 0:
        a, b = O.gen_sparse(N, C, H, W, s, seed), O.gen_sparse(K, C, S, R, 0.0, seed + 1)
        ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V)
    elif comp == 1:
        a, b = O.gen_sparse(N, K, hp, wp, s, seed), O.gen_sparse(K, C, S, R, 0.0, seed + 1)
        ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V, True)
    elif check == 0:
        a, b = O.gen_sparse(N, C, H, W, s, seed), O.gen_sparse(N, K, hp, wp, 0.0, seed + 2)
        ba, bb = sp.pack_act_chwnn(a, V), sp.pack_act_nchwc(b, V)
    else:
        a, b = O.gen_sparse(N, C, H, W, 0.0, seed), O.gen_sparse(N, K, hp, wp, s, seed + 2)
        ba, bb = sp.pack_act_nchwc(a, V), sp.pack_act_chwnn(b, V)
    return a, b, ba.to("cuda"), bb.to("cuda")


def run(sp, sh, comp, check, V, ba, bb, mode=0):
    pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
    res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode(mode))
    return pl, res, sp.unpack(res.out).cpu().numpy()


def mask_of(comp, check, a, b):
    return b if (comp == 2 and check == 1) else a


def test_kernels_match_oracle_across_sparsities_and_modes(sp):  # test_kernels.cpp:26-47
    rng = np.random.default_rng(101)
    for trial in range(24):
        V = [4, 8, 16][trial % 3]
        sh = sp.ConvShape(*rng_tiny_shape(rng, V))
        s = float(rng.choice([0.0, 0.3, 0.5, 0.8, 0.9, 1.0]))
        for comp, check in ALL:
            a, b, ba, bb = make_inputs(sp, sh, comp, check, s, V, trial * 7 + 1)
            ref = O.dense(comp, sh.astuple(), a, b)
            for mode in (0, 1):
                _, res, got = run(sp, sh, comp, check, V, ba, bb, mode)
                assert O.max_abs_rel(got, ref) <= TOL, (sh, comp, check, s, mode)
                assert O.max_rel_error(got, ref) <= 1e-4, (sh, comp, check, s, mode)


def test_sparse_and_dense_modes_agree(sp):  # test_kernels.cpp:49-65
    rng = np.random.default_rng(55)
    for trial in range(9):
        V = [4, 8, 16][trial % 3]
        sh = sp.ConvShape(*rng_tiny_shape(rng, V))
        for comp, check in ALL:
            _, _, ba, bb = make_inputs(sp, sh, comp, check, 0.5, V, trial + 40)
            _, _, g0 = run(sp, sh, comp, check, V, ba, bb, 0)
            _, _, g1 = run(sp, sh, comp, check, V, ba, bb, 1)
            assert O.max_rel_error(g0, g1) <= 1e-4


def test_executed_fma_counters_match_simulation_exactly(sp):  # test_kernels.cpp:67-95
    rng = np.random.default_rng(77)
    for trial in range(30):
        V = [4, 8, 16][trial % 3]
        sh = sp.ConvShape(*rng_tiny_shape(rng, V))
        s = float(rng.choice([0.0, 0.3, 0.5, 0.8, 0.9, 1.0]))
        for comp, check in ALL:
            a, b, ba, bb = make_inputs(sp, sh, comp, check, s, V, trial * 13 + 3)
            pl, res, _ = run(sp, sh, comp, check, V, ba, bb, 0)
            want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), comp, V, 30, check),
                                     mask_of(comp, check, a, b))
            assert res.counters.executed_vector_fmas == want["executed_vector_fmas"], (sh, comp, check, s)
            assert res.counters.checked_vectors == want["checked_vectors"]
            _, dres, _ = run(sp, sh, comp, check, V, ba, bb, 1)
            assert dres.counters.executed_vector_fmas == want["dense_total"]
            assert dres.counters.checked_vectors == 0


def test_single_interior_nonzero_skips_everything_else(sp):  # test_kernels.cpp:97-110
    V = 8
    sh = sp.ConvShape.make(1, 32, 32, 8, 8, 3, 3, 1, 1)
    D = np.zeros((1, 32, 8, 8), np.float32)
    D[0, 5, 4, 4] = 0.7
    G = O.gen_sparse(32, 32, 3, 3, 0.0, 2)
    pl = sp.plan(sh, sp.Component.fwd, V)
    res = sp.sparse_fwd(sp.pack_act_nchwc(D, V).to("cuda"), sp.pack_filter(G, V).to("cuda"), sh, pl)
    assert res.counters.executed_vector_fmas == 36
    got = sp.unpack(res.out).cpu().numpy()
    assert O.max_rel_error(got, O.dense(0, sh.astuple(), D, G)) <= 1e-4


def test_all_zero_input_runs_zero_fmas(sp):  # test_kernels.cpp:112-123
    V = 8
    sh = sp.ConvShape.make(2, 16, 16, 6, 6, 3, 3, 1, 1)
    for comp, check in ALL:
        _, _, ba, bb = make_inputs(sp, sh, comp, check, 1.0, V, 9)
        _, res, got = run(sp, sh, comp, check, V, ba, bb, 0)
        assert res.counters.executed_vector_fmas == 0
        assert not got.any()


def test_bww_single_image_outer_product(sp):  # test_kernels.cpp:125-148
    V = 8
    sh = sp.ConvShape.make(8, 8, 8, 1, 1, 1, 1, 1, 1)
    D = np.zeros((8, 8, 1, 1), np.float32)
    D[3, :, 0, 0] = np.arange(1, 9)
    dY = O.gen_sparse(8, 8, 1, 1, 0.0, 4)
    pl = sp.plan(sh, sp.Component.bww, V)
    res = sp.sparse_bww(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh, pl)
    assert res.counters.executed_vector_fmas == sh.C * (sh.K // pl.Q) * (pl.Q // V)
    dG = sp.unpack(res.out).cpu().numpy()
    np.testing.assert_allclose(dG[:, :, 0, 0], np.outer(dY[3, :, 0, 0], D[3, :, 0, 0]), rtol=1e-6)


def test_adding_zeros_never_increases_executed_fmas(sp):  # test_kernels.cpp:227-253
    rng = np.random.default_rng(404)
    V = 8
    for trial in range(6):
        sh = sp.ConvShape(*rng_tiny_shape(rng, V))
        for comp, check in ALL[:3]:
            a, b, _, bb = make_inputs(sp, sh, comp, check, 0.3, V, trial)
            masked = a.copy()
            prev = None
            for step in range(4):
                flat = masked.reshape(-1)
                flat[rng.integers(0, flat.size, flat.size // 8)] = 0.0
                ba = (sp.pack_act_chwnn(masked, V) if comp == 2 else sp.pack_act_nchwc(masked, V)).to("cuda")
                _, res, _ = run(sp, sh, comp, check, V, ba, bb, 0)
                if prev is not None:
                    assert res.counters.executed_vector_fmas <= prev
                prev = res.counters.executed_vector_fmas


def test_results_are_bitwise_deterministic(sp):  # test_kernels.cpp:255-275
    rng = np.random.default_rng(505)
    for trial in range(8):
        V = [4, 8, 16][trial % 3]
        sh = sp.ConvShape(*rng_tiny_shape(rng, V))
        for comp, check in ALL:
            _, _, ba, bb = make_inputs(sp, sh, comp, check, 0.5, V, trial + 7)
            _, r0, g0 = run(sp, sh, comp, check, V, ba, bb, 0)
            for workers in (2, 4):
                pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
                r1 = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse, workers)
                assert np.array_equal(sp.unpack(r1.out).cpu().numpy(), g0)
                assert r1.counters == r0.counters


def test_bww_check_side_selection_stays_correct(sp):  # test_kernels.cpp:300-326
    V = 8
    sh = sp.ConvShape.make(5, 16, 24, 6, 7, 3, 3, 1, 1)
    D = O.gen_sparse(5, 16, 6, 7, 0.2, 1)
    dY = O.gen_sparse(5, 24, 6, 7, 0.8, 2)
    ref = O.dense(2, sh.astuple(), D, dY)
    pi = sp.plan(sh, sp.Component.bww, V)
    r = sp.sparse_bww(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh, pi)
    assert O.max_rel_error(sp.unpack(r.out).cpu().numpy(), ref) <= 1e-4
    po = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.output_grad)
    r2 = sp.sparse_bww(sp.pack_act_nchwc(D, V).to("cuda"), sp.pack_act_chwnn(dY, V).to("cuda"), sh, po)
    assert O.max_rel_error(sp.unpack(r2.out).cpu().numpy(), ref) <= 1e-4
    assert r2.counters.executed_vector_fmas < r.counters.executed_vector_fmas


def test_stride_wider_than_filter_leaves_gap_columns_zero(sp):  # test_kernels.cpp:354-385
    V = 8
    sh = sp.ConvShape.make(2, 16, 16, 7, 7, 1, 1, 2, 2)
    for comp, check in ALL:
        a, b, ba, bb = make_inputs(sp, sh, comp, check, 0.4, V, 61)
        pl, res, got = run(sp, sh, comp, check, V, ba, bb, 0)
        assert O.max_rel_error(got, O.dense(comp, sh.astuple(), a, b)) <= 1e-4
        want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), comp, V, 30, check), mask_of(comp, check, a, b))
        assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    _, _, ba, bb = make_inputs(sp, sh, 1, 0, 0.0, V, 62)
    pl, res, dD = run(sp, sh, 1, 0, V, ba, bb, 0)
    assert not dD[:, :, :, 1::2].any() and not dD[:, :, 1::2, :].any()
    sweeps = 4 * (sh.K // V) * sh.N * (sh.C // pl.Q)
    assert res.counters.output_vector_loads == sweeps * 4 * (pl.Q // V)
    assert res.counters.output_vector_stores == sweeps * 4 * (pl.Q // V)


def test_strided_geometries_match_oracle(sp):  # test_kernels.cpp:407-422
    V = 8
    sh = sp.ConvShape.make(2, 16, 16, 14, 14, 3, 3, 2, 2)
    for comp, check in ALL:
        a, b, ba, bb = make_inputs(sp, sh, comp, check, 0.5, V, 21)
        _, res, got = run(sp, sh, comp, check, V, ba, bb, 0)
        assert O.max_rel_error(got, O.dense(comp, sh.astuple(), a, b)) <= 1e-4
        want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), comp, V, 30, check), mask_of(comp, check, a, b))
        assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]


def test_negative_zero_is_skipped_nan_inf_participate(sp):  # vec.hpp:120-128, README "Notes"
    V = 16
    sh = sp.ConvShape.make(1, 16, 16, 4, 4, 3, 3, 1, 1)
    D = np.zeros((1, 16, 4, 4), np.float32)
    D[0, 0, 1, 1] = -0.0
    D[0, 3, 2, 2] = 1.5
    G = O.gen_sparse(16, 16, 3, 3, 0.0, 5)
    pl = sp.plan(sh, sp.Component.fwd, V)
    r = sp.sparse_fwd(sp.pack_act_nchwc(D, V).to("cuda"), sp.pack_filter(G, V).to("cuda"), sh, pl)
    assert r.counters.executed_vector_fmas == O.expected_counts(sh.astuple(), O.plan(sh.astuple(), 0, V), D)[
        "executed_vector_fmas"] == 9  # only the 1.5 (9 taps x K/V=1)
    D[0, 7, 0, 0] = math.nan
    D[0, 8, 3, 3] = math.inf
    r = sp.sparse_fwd(sp.pack_act_nchwc(D, V).to("cuda"), sp.pack_filter(G, V).to("cuda"), sh, pl)
    y = sp.unpack(r.out).cpu().numpy()
    ref = O.dense(0, sh.astuple(), D, G)
    assert np.array_equal(np.isnan(y), np.isnan(ref))
    assert np.array_equal(np.isinf(y), np.isinf(ref))
    fin = np.isfinite(ref)
    assert O.max_abs_rel(y[fin], ref[fin]) <= TOL


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_golden_fixtures_from_reference(sp, path):
    """Byte-identical operands the reference packed -> our kernels -> compare
    with the reference CPU kernel's output, its counters and the 64-bit oracle."""
    import torch
    z = np.load(path)
    sh = sp.ConvShape(*[int(v) for v in z["shape"]])
    V = int(z["V"])
    for comp, check, tag in [(0, 0, "fwd"), (1, 0, "bwi"), (2, 0, "bww_in"), (2, 1, "bww_og")]:
        a, b = z[f"{tag}_a"], z[f"{tag}_b"]
        if comp == 0:
            ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V)
        elif comp == 1:
            ba, bb = sp.pack_act_nchwc(a, V), sp.pack_filter(b, V, True)
        elif check == 0:
            ba, bb = sp.pack_act_chwnn(a, V), sp.pack_act_nchwc(b, V)
        else:
            ba, bb = sp.pack_act_nchwc(a, V), sp.pack_act_chwnn(b, V)
        assert np.array_equal(ba.data, z[f"{tag}_a_blk"]) and np.array_equal(bb.data, z[f"{tag}_b_blk"])
        ba.data, bb.data = torch.from_numpy(z[f"{tag}_a_blk"]).cuda(), torch.from_numpy(z[f"{tag}_b_blk"]).cuda()
        for mode, ckey in ((0, "sparse"), (1, "dense")):
            _, res, got = run(sp, sh, comp, check, V, ba, bb, mode)
            assert O.max_abs_rel(got, z[f"{tag}_oracle64"]) <= TOL, (tag, mode)
            assert O.max_abs_rel(got, z[f"{tag}_ref_{'sparse' if mode == 0 else 'dense_mode'}"]) <= 2 * TOL
            c = z[f"{tag}_counters_{ckey}"]
            assert [res.counters.checked_vectors, res.counters.executed_vector_fmas,
                    res.counters.output_vector_loads, res.counters.output_vector_stores] == [int(v) for v in c], tag


def test_host_buffer_dropin_matches_device_path(sp):
    """spc_run_parallel_host (numpy in, numpy out) == the device path, bitwise."""
    V = 16
    sh = sp.ConvShape.make(3, 32, 48, 9, 11, 3, 3, 1, 1)
    for comp, check in ALL:
        a, b, ba, bb = make_inputs(sp, sh, comp, check, 0.5, V, 5)
        pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
        rd = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
        rh = sp.run_parallel(ba.to(None), bb.to(None), sh, pl, sp.RunMode.sparse)
        assert isinstance(rh.out.data, np.ndarray)
        assert np.array_equal(rh.out.data, rd.out.data.cpu().numpy())
        assert rh.counters == rd.counters


def test_relu_and_grad_mask_bit_exact(sp):
    import torch
    x = np.array([-1.0, -0.0, 0.0, 2.5, math.nan, math.inf, -math.inf, 1e-38, -1e-45, 3.0], np.float32)
    x = np.tile(x, 1000)
    up = np.arange(x.size, dtype=np.float32) - 7
    r = sp.relu_(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(r.view(np.uint32), O.relu(x).view(np.uint32))
    m = sp.relu_grad_mask(torch.from_numpy(x).cuda(), torch.from_numpy(up).cuda()).cpu().numpy()
    assert np.array_equal(m.view(np.uint32), O.relu_grad_mask(x, up).view(np.uint32))


def test_device_chwnn_transpose_matches_pack(sp):
    import torch
    rng = np.random.default_rng(3)
    for V, n in ((16, 19), (8, 8), (4, 3)):
        t = rng.standard_normal((n, 2 * V, 5, 6)).astype(np.float32)
        src = sp.pack_act_nchwc(t, V).to("cuda")
        got = sp.nchwc_to_chwnn(src)
        assert np.array_equal(got.data.cpu().numpy(), O.pack_act(t, V, chwnn=True))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("comp,check", ALL)
def test_config1_full_size_matches_reference_cpu(sp, comp, check):
    """BASELINE config 1 (N=16, C=K=64, 56x56, 3x3) at full size: GPU vs the
    reference's own CPU kernel on identical seeded inputs, values within TOL
    of max-abs and FMA counters exact; plus a 64-bit oracle check on an image slice."""
    from paper_1911_10175_b200 import workloads as wl
    V = 16
    sh = sp.ConvShape.make(16, 64, 64, 56, 56, 3, 3, 1, 1)
    D, G, dY = wl.config1_inputs_host(seed=0)
    a, b = {0: (D, G), 1: (dY, G), 2: (D, dY)}[comp]
    r = O.RefRun(comp, check, sh.astuple(), V, a, b)
    r.exec(0, os.cpu_count() or 1)
    ref_out, ref_cnt, _ = r.result()
    import torch
    ba, bb = torch.from_numpy(r.operand(0)).cuda(), torch.from_numpy(r.operand(1)).cuda()
    lay = {0: (sp.Layout.act_nchwc, sp.Layout.filter_kcrs_blk), 1: (sp.Layout.act_nchwc, sp.Layout.filter_kcrs_blk),
           2: ((sp.Layout.act_chwnn, sp.Layout.act_nchwc) if check == 0 else (sp.Layout.act_nchwc, sp.Layout.act_chwnn))}[comp]
    ta = sp.BlockedTensor(lay[0], V, sh.N, sh.C if comp != 1 else sh.K, sh.H if comp != 1 else sh.out_h(),
                          sh.W if comp != 1 else sh.out_w(), data=ba)
    if comp == 2:
        tb = sp.BlockedTensor(lay[1], V, sh.N, sh.K, sh.out_h(), sh.out_w(), data=bb)
    else:
        tb = sp.BlockedTensor(lay[1], V, k=sh.K if comp == 0 else sh.C, c=sh.C if comp == 0 else sh.K,
                              s=sh.S, r=sh.R, data=bb)
    _, res, got = run(sp, sh, comp, check, V, ta, tb, 0)
    assert O.max_abs_rel(got, ref_out) <= TOL
    assert res.counters.executed_vector_fmas == ref_cnt["executed_vector_fmas"]
    assert res.counters.checked_vectors == ref_cnt["checked_vectors"]
    # 64-bit oracle on a 2-image slice (FWD/BWI are per-image independent)
    if comp in (0, 1):
        sl = sh.with_batch(2).astuple()
        ref2 = O.dense(comp, sl, a[:2], b)
        assert O.max_abs_rel(got[:2], ref2) <= TOL


@pytest.mark.parametrize("R,stride", [(3, 1), (3, 2), (1, 1), (1, 2)])
def test_tuned_tile_kernels_match_oracle(sp, R, stride):
    """The V=16 tile kernels (C,K multiples of 64) on ragged image sizes that
    leave partial tiles, both KK variants, sparse and dense mode, exact counts."""
    V = 16
    rng = np.random.default_rng(1000 + 10 * R + stride)
    cases = [(2, 64, 64, 13, 11), (1, 128, 64, 9, 17), (2, 64, 128, 10, 10), (1, 128, 256, 7, 15),
             (3, 192, 64, 5, 6)]
    for n, C, K, H, W in cases:
        if H + 2 * ((R - 1) // 2) < R:
            continue
        sh = sp.ConvShape.make(n, C, K, H, W, R, R, stride, stride)
        for comp, check in ALL:
          for s in (0.0, 0.5, 0.8, 0.93):  # 0.8, 0.93: the jump-table kernels (density <= 28% / 21%)
            a, b, ba, bb = make_inputs(sp, sh, comp, check, s, V, int(rng.integers(1, 1000)))
            ref = O.dense(comp, sh.astuple(), a, b)
            want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), comp, V, 30, check),
                                     mask_of(comp, check, a, b))
            for mode in (0, 1):
                _, res, got = run(sp, sh, comp, check, V, ba, bb, mode)
                assert O.max_abs_rel(got, ref) <= TOL, (sh, comp, s, mode)
                if mode == 0:
                    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"], (sh, comp, s)
                else:
                    assert res.counters.executed_vector_fmas == want["dense_total"]


def test_jump_table_and_branch_kernels_agree_bitwise(sp):
    """The two sparse inner loops (per-pixel branches / jump table over the
    nonzeros) accumulate in the same order: identical bits, identical counts."""
    import ctypes as C
    import torch
    V = 16
    L = sp._lib.load()
    # 128 channels: the production branch kernel (42, KK=4 7x4), branches on a 4x8 tile (2), the
    # 2-warp (17) and the production one-warp (41) jump tables; 64 channels: the KK=2 8x16 CTA pair
    # that launch_tile_conv runs on 64-channel multiples (6 branches, 14 jump table)
    for C_, variants in ((128, (42, 2, 17, 41)), (64, (6, 14))):
      sh = sp.ConvShape.make(2, C_, C_, 20, 22, 3, 3, 1, 1)
      for comp in (0, 1):
        for s in (0.5, 0.95):
            a, b, ba, bb = make_inputs(sp, sh, comp, 0, s, V, 77)
            pl = sp.plan(sh, sp.Component(comp), V)
            outs = []
            for variant in variants:
                out = torch.empty(sh.N * (sh.K if comp == 0 else sh.C) * (sh.out_h() if comp == 0 else sh.H)
                                  * (sh.out_w() if comp == 0 else sh.W), device="cuda")
                cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
                ca, cb, cs, cp = ba.to_c(), bb.to_c(), sh.to_c(), pl.to_c()
                cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.data_ptr(), out.numel())
                st = L.spc_debug_conv_variant(variant, C.byref(ca), C.byref(cb), C.byref(cs), C.byref(cp), 0,
                                              C.byref(cd), C.c_void_p(cnt.data_ptr()),
                                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
                assert st == 0, sp._lib.last_error()
                torch.cuda.synchronize()
                outs.append((out.cpu().numpy(), cnt.cpu().numpy()))
            for o in outs[1:]:
                assert np.array_equal(outs[0][0].view(np.uint32), o[0].view(np.uint32))
                assert np.array_equal(outs[0][1], o[1])


def test_cxx_dropin_matches_reference_library():
    """The C++ drop-in (spconv::cuda::*) against the reference's own
    spconv::run_parallel on identical blocked tensors (tests/cxx/test_dropin.cpp)."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_1911_10175_b200", "cxx", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("C++ drop-in test binary not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]


def test_host_path_pipelined_chunks_match_device_path(sp):
    """Large host-buffer calls run in pipelined batch chunks: FWD/BWI stay
    bitwise equal to the device call; BWW (16-image-block chunks summed in
    fixed order) stays within rounding of it, counters exact."""
    V = 16
    sh = sp.ConvShape.make(40, 64, 128, 56, 56, 3, 3, 1, 1)  # > 64 MB of host I/O per call
    for comp, check in ALL:
        a, b, ba, bb = make_inputs(sp, sh, comp, check, 0.6, V, 11)
        pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
        rd = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
        ha, hb = ba.to(None), bb.to(None)  # pageable numpy: the pinned staging ring (host_stage.cu)
        import torch
        pa = sp.BlockedTensor(**{**ha.header(), "data": torch.from_numpy(ha.data).pin_memory().numpy()})
        pb = sp.BlockedTensor(**{**hb.header(), "data": torch.from_numpy(hb.data).pin_memory().numpy()})
        runs = [sp.run_parallel(ha, hb, sh, pl, sp.RunMode.sparse), sp.run_parallel(pa, pb, sh, pl, sp.RunMode.sparse)]
        ref = rd.out.data.cpu().numpy()
        for rh in runs:
            got = rh.out.data
            if comp == 2:
                # Two GPU summation orders (chunked vs whole-batch split reduction);
                # each is separately within 1e-5 of the oracle (test_bww_*).
                assert O.max_abs_rel(got, ref) <= 2e-6
            else:
                assert np.array_equal(got, ref)
            assert rh.counters == rd.counters
        assert np.array_equal(runs[0].out.data, runs[1].out.data)  # pageable == pinned, bitwise


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg,idx", [("resnet50_b64", 1), ("resnet50_b64", 2), ("resnet50_b64", 11),
                                     ("resnet34_b64", 7), ("resnet34_b64", 8), ("vgg16_b32", 8)])
@pytest.mark.parametrize("math", ["fp32", "tf32x3"])
def test_baseline_layers_match_reference_cpu(sp, cfg, idx, math):
    """BASELINE layer geometries (stride-2 3x3, 1x1 reduce/expand/projection,
    VGG 512-channel) at full spatial size and a 4-image batch: GPU vs the
    reference's own CPU kernels on identical inputs, all three passes, in both
    arithmetics (FP32 FFMA; the 3xTF32 tensor-core variant, same 1e-5 bar)."""
    import torch
    from paper_1911_10175_b200 import workloads as wl
    V = 16
    sh = wl.CONFIGS[cfg]()[idx].shape.with_batch(4)
    t = sh.astuple()
    rng = np.random.default_rng(idx)
    D = wl.host_activation((sh.N, sh.C, sh.H, sh.W), 0.6, rng)
    G = wl.host_weights(sh.K, sh.C, sh.S, sh.R, rng)
    dY = wl.host_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), 0.6, rng)
    for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY), (2, 1, D, dY)):
        r = O.RefRun(comp, check, t, V, a, b)
        r.exec(0, os.cpu_count() or 1)
        ref_out, ref_cnt, _ = r.result()
        ta, tb = torch.from_numpy(r.operand(0)).cuda(), torch.from_numpy(r.operand(1)).cuda()
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
        with sp.math_mode(sp.Math[math]):
            _, res, got = run(sp, sh, comp, check, V, ba, bb, 0)
        assert O.max_abs_rel(got, ref_out) <= TOL, (cfg, idx, comp, check, math)
        assert res.counters.executed_vector_fmas == ref_cnt["executed_vector_fmas"]
        assert res.counters.checked_vectors == ref_cnt["checked_vectors"]
        r.close()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("comp", [0, 1])
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("R", [1, 3])
def test_pointwise_nonfinite_filter_keeps_skip_semantics(sp, comp, stride, R):
    """The 1x1 kernels and the 3x3 stride-2 FWD kernel execute zero products
    (exact for finite filters); a filter with Inf/NaN must still follow the
    reference's skip semantics (0 inputs are skipped, so 0*Inf never happens):
    GPU == reference CPU incl. NaN/Inf positions."""
    V = 16
    sh = sp.ConvShape.make(3, 64, 128, 9, 10, R, R, stride, stride)
    rng = np.random.default_rng(11 + comp + stride + R)
    hp, wp = sh.out_h(), sh.out_w()
    G = rng.standard_normal((sh.K, sh.C, R, R)).astype(np.float32)
    if comp == 0:
        X = np.maximum(rng.standard_normal((sh.N, sh.C, sh.H, sh.W)), 0).astype(np.float32)
        X[:, 5] = 0.0       # channel 5 all zero: its Inf/NaN weights must be skipped
        X[:, 9, 0, 0] = 3.0  # channel 9 has one nonzero: Inf propagates there only
        G[7, 5, 0, 0], G[100, 5, 0, 0], G[3, 9, 0, 0] = np.inf, np.nan, np.inf
        a, b = X, G
    else:
        X = np.maximum(rng.standard_normal((sh.N, sh.K, hp, wp)), 0).astype(np.float32)
        X[:, 40] = 0.0
        G[40, 7, 0, 0], G[40, 60, 0, 0] = np.inf, -np.inf
        a, b = X, G
    r = O.RefRun(comp, 0, sh.astuple(), V, a, b)
    r.exec(0, 4)
    ref_out, ref_cnt, _ = r.result()
    pl = sp.plan(sh, sp.Component(comp), V)
    ta = sp.pack_act_nchwc(a, V)
    tb = sp.pack_filter(b, V, swap_kc=(comp == 1))
    res = sp.run_parallel(ta, tb, sh, pl, sp.RunMode.sparse)
    got = sp.unpack(res.out)
    assert np.array_equal(np.isnan(got), np.isnan(ref_out))
    assert np.array_equal(np.isinf(got), np.isinf(ref_out))
    fin = np.isfinite(ref_out)
    assert O.max_abs_rel(np.where(fin, got, 0), np.where(fin, ref_out, 0)) <= TOL
    assert res.counters.executed_vector_fmas == ref_cnt["executed_vector_fmas"]


def test_gated_host_path_equals_device_path(tmp_path):
    """SPC_HOST_GATE=1: FWD/BWI host-buffer calls as one launch whose CTAs wait
    for their input chunk (Gate, common.cuh) -- bitwise equal to the device call."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl
V = 16
for dims in [(12, 64, 128, 20, 22, 3, 1), (9, 128, 128, 15, 14, 3, 1), (7, 64, 256, 14, 14, 1, 1), (5, 64, 128, 14, 14, 1, 2)]:
    N, C, K, H, W, R, O = dims
    sh = sp.ConvShape.make(N, C, K, H, W, R, R, O, O)
    rng = np.random.default_rng(N)
    G = rng.standard_normal((K, C, R, R)).astype(np.float32)
    for comp in (sp.Component.fwd, sp.Component.bwi):
        shp = (N, C, H, W) if comp == sp.Component.fwd else (N, K, sh.out_h(), sh.out_w())
        x = np.maximum(rng.standard_normal(shp) - 0.3, 0).astype(np.float32)
        a, b = sp.pack_act_nchwc(x, V), sp.pack_filter(G, V, comp == sp.Component.bwi)
        pl = sp.plan(sh, comp, V)
        host = sp.run_parallel(a, b, sh, pl, sp.RunMode.sparse)
        dev = sp.run_parallel(a.to("cuda"), b.to("cuda"), sh, pl, sp.RunMode.sparse)
        assert np.array_equal(host.out.data, dev.out.data.cpu().numpy()), (dims, comp)
        assert host.counters == dev.counters
print("ok")
'''
    env = dict(os.environ, SPC_HOST_GATE="1", SPC_HOST_CHUNK_MB="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("stride", [1, 2])
def test_pointwise_bww_nonfinite_grad_keeps_skip_semantics(sp, stride):
    """1x1 BWW (check = input) executes zero products for finite dY; a dY with
    Inf/NaN must follow the reference's skip semantics (GPU == reference CPU)."""
    V = 16
    sh = sp.ConvShape.make(19, 64, 128, 9, 10, 1, 1, stride, stride)
    rng = np.random.default_rng(5 + stride)
    hp, wp = sh.out_h(), sh.out_w()
    D = np.maximum(rng.standard_normal((sh.N, sh.C, sh.H, sh.W)), 0).astype(np.float32)
    dY = rng.standard_normal((sh.N, sh.K, hp, wp)).astype(np.float32)
    D[:, 3] = 0.0                      # channel 3 all zero: dY's Inf/NaN must not reach dG[:, 3]
    dY[2, 7, 1, 1], dY[5, 90, 0, 2] = np.inf, np.nan
    for finite in (True, False):
        y = np.nan_to_num(dY, nan=0.0, posinf=0.0) if finite else dY
        r = O.RefRun(2, 0, sh.astuple(), V, D, y)
        r.exec(0, 4)
        ref_out, ref_cnt, _ = r.result()
        pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.input)
        res = sp.run_parallel(sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(y, V), sh, pl, sp.RunMode.sparse)
        got = sp.unpack(res.out)
        assert np.array_equal(np.isnan(got), np.isnan(ref_out)), finite
        assert np.array_equal(np.isinf(got), np.isinf(ref_out)), finite
        fin = np.isfinite(ref_out)
        assert O.max_abs_rel(np.where(fin, got, 0), np.where(fin, ref_out, 0)) <= TOL
        assert res.counters.executed_vector_fmas == ref_cnt["executed_vector_fmas"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("K,stride,check", [(64, 1, 0), (128, 1, 0), (128, 2, 0), (64, 1, 1), (128, 2, 1)])
def test_bww_3x3_nonfinite_checked_keeps_skip_semantics(sp, K, stride, check):
    """The 3x3 BWW tile kernels add d * 0 for partner pixels outside the image
    (tiles overhanging the right/bottom edge, virtual padding): exact only for
    a finite checked tensor.  A checked tensor holding Inf/NaN must switch to
    the exact-skip kernel: GPU == reference CPU incl. NaN/Inf positions, in
    both arithmetics; finite tensors keep the tile kernels (same values)."""
    V = 16
    sh = sp.ConvShape.make(5, 32, K, 9, 10, 3, 3, stride, stride)
    hp, wp = sh.out_h(), sh.out_w()
    rng = np.random.default_rng(K + 10 * stride + check)
    D = np.maximum(rng.standard_normal((sh.N, sh.C, sh.H, sh.W)) - 0.3, 0).astype(np.float32)
    dY = np.maximum(rng.standard_normal((sh.N, sh.K, hp, wp)) - 0.3, 0).astype(np.float32)
    for finite in (True, False):
        X, Y = D.copy(), dY.copy()
        if not finite:
            T = X if check == 0 else Y
            T[1, 3, 0, 0] = np.inf   # corner: its out-of-image partners must not produce NaN
            T[2, 7, T.shape[2] - 1, T.shape[3] - 1] = np.nan
        r = O.RefRun(2, check, sh.astuple(), V, X, Y)
        r.exec(0, 4)
        ref_out, ref_cnt, _ = r.result()
        pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck(check))
        a = sp.pack_act_chwnn(X, V) if check == 0 else sp.pack_act_nchwc(X, V)
        b = sp.pack_act_nchwc(Y, V) if check == 0 else sp.pack_act_chwnn(Y, V)
        for math in (sp.Math.fp32, sp.Math.tf32x3):
            with sp.math_mode(math):
                res = sp.run_parallel(a.to("cuda"), b.to("cuda"), sh, pl, sp.RunMode.sparse)
            got = sp.unpack(res.out).cpu().numpy()
            assert np.array_equal(np.isnan(got), np.isnan(ref_out)), (finite, math)
            assert np.array_equal(np.isinf(got), np.isinf(ref_out)), (finite, math)
            fin = np.isfinite(ref_out)
            assert O.max_abs_rel(np.where(fin, got, 0), np.where(fin, ref_out, 0)) <= TOL
            assert res.counters.executed_vector_fmas == ref_cnt["executed_vector_fmas"]


def test_row_bww_kernel_matches_oracle(tmp_path):
    """The opt-in row-window BWW kernel (SPC_ROW_BWW=1, csrc/row_bww.cu) on
    shapes with partial strips, both KK variants, sparse and dense mode,
    exact counters, and non-finite D (exact fallback)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, oracle as O, paper_1911_10175_b200 as sp
V = 16
for (n, C, K, H, W) in [(3, 16, 64, 9, 10), (2, 32, 128, 14, 13), (17, 16, 128, 7, 30), (1, 64, 64, 5, 5)]:
    sh = sp.ConvShape.make(n, C, K, H, W, 3, 3, 1, 1)
    for s in (0.0, 0.5, 0.9):
        D = O.gen_sparse(n, C, H, W, s, n + C)
        dY = O.gen_sparse(n, K, H, W, 0.0, K + W)
        ref = O.dense(2, sh.astuple(), D, dY)
        want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), 2, V), D)
        pl = sp.plan(sh, sp.Component.bww, V)
        for mode in (0, 1):
            res = sp.run_parallel(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh, pl,
                                  sp.RunMode(mode))
            got = sp.unpack(res.out).cpu().numpy()
            assert O.max_abs_rel(got, ref) <= 1e-5, (sh, s, mode)
            assert res.counters.executed_vector_fmas == (want["executed_vector_fmas"] if mode == 0
                                                         else want["dense_total"]), (sh, s, mode)
print("ok")
'''
    env = dict(os.environ, SPC_ROW_BWW="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_tma_bww_kernel_matches_oracle(sp):
    """The TMA-staged BWW tile kernel (csrc/tma_bww.cu; the default for
    check=input 3x3 s1 with K % 128 == 0): ragged image blocks (N % 16 != 0),
    widths that are not tile multiples (overhanging tiles, plane pitch > W + 1),
    one-tile images, sparse and dense mode, exact counters, run-to-run bitwise."""
    V = 16
    for (n, C, K, H, W) in [(3, 16, 128, 9, 10), (17, 32, 128, 14, 13), (2, 16, 256, 7, 30), (1, 48, 128, 5, 5),
                            (33, 16, 128, 3, 4), (2, 16, 128, 28, 28)]:
        sh = sp.ConvShape.make(n, C, K, H, W, 3, 3, 1, 1)
        for s in (0.0, 0.5, 0.9):
            D = O.gen_sparse(n, C, H, W, s, n + C)
            dY = O.gen_sparse(n, K, H, W, 0.0, K + W)
            ref = O.dense(2, sh.astuple(), D, dY)
            want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), 2, V), D)
            pl = sp.plan(sh, sp.Component.bww, V)
            a, b = sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda")
            for mode in (0, 1):
                res = sp.run_parallel(a, b, sh, pl, sp.RunMode(mode))
                got = sp.unpack(res.out).cpu().numpy()
                assert O.max_abs_rel(got, ref) <= TOL, (sh, s, mode)
                assert res.counters.executed_vector_fmas == (want["executed_vector_fmas"] if mode == 0
                                                             else want["dense_total"]), (sh, s, mode)
                again = sp.run_parallel(a, b, sh, pl, sp.RunMode(mode))
                assert np.array_equal(sp.unpack(again.out).cpu().numpy(), got)


def test_tma_bww_nonfinite_input_takes_the_exact_fallback(sp):
    """Inf/NaN in D at image corners and edges: the TMA kernel (which adds
    d * 0 for partner pixels outside the image) must not run; the exact
    shape-general kernel does, and the result equals the oracle's."""
    V = 16
    sh = sp.ConvShape.make(2, 16, 128, 9, 10, 3, 3, 1, 1)
    D = O.gen_sparse(2, 16, 9, 10, 0.5, 5)
    dY = O.gen_sparse(2, 128, 9, 10, 0.0, 6)
    D[0, 0, 0, 0] = np.inf
    D[1, 3, 8, 9] = np.nan
    D[1, 5, 4, 0] = -np.inf
    ref = O.dense(2, sh.astuple(), D, dY)
    pl = sp.plan(sh, sp.Component.bww, V)
    res = sp.run_parallel(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh, pl,
                          sp.RunMode.sparse)
    got = sp.unpack(res.out).cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(np.isinf(got), np.isinf(ref))
    fin = np.isfinite(ref)
    assert O.max_abs_rel(np.where(fin, got, 0), np.where(fin, ref, 0)) <= TOL


def test_tma_bww_equals_cp_async_tile_kernel(tmp_path):
    """A/B: SPC_TMA_BWW=0 (the cp.async tile kernel of tile_bww.cu) against the
    default TMA kernel on one shape -- same counters, values within the bar."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, oracle as O, paper_1911_10175_b200 as sp
V = 16
sh = sp.ConvShape.make(18, 32, 128, 14, 14, 3, 3, 1, 1)
D = O.gen_sparse(18, 32, 14, 14, 0.6, 1)
dY = O.gen_sparse(18, 128, 14, 14, 0.0, 2)
pl = sp.plan(sh, sp.Component.bww, V)
res = sp.run_parallel(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh, pl, sp.RunMode.sparse)
np.save(sys.argv[1], sp.unpack(res.out).cpu().numpy())
print("ok", res.counters.executed_vector_fmas)
'''
    outs = []
    for knob in ("1", "0"):
        env = dict(os.environ, SPC_TMA_BWW=knob)
        f = str(tmp_path / f"dg{knob}.npy")
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
        outs.append((np.load(f), r.stdout.split()[-1]))
    assert outs[0][1] == outs[1][1]
    assert O.max_abs_rel(outs[0][0], outs[1][0]) <= TOL


def test_host_batch_equals_per_call(sp):
    """spc_run_parallel_host_batch: pinned and pageable passes mixed, FWD / BWI /
    BWW (multi-chunk: N = 40 gives three 16-image blocks), more passes than
    pipeline slots -- outputs and counters bitwise those of one
    spc_run_parallel_host call per pass."""
    import torch
    V = 16
    rng = np.random.default_rng(3)
    hb = sp.HostBatch()
    want = []
    for i, (n, C, K, H, W) in enumerate([(40, 32, 128, 14, 14), (5, 16, 32, 9, 11), (40, 128, 128, 14, 14),
                                          (18, 64, 64, 12, 12)]):
        sh = sp.ConvShape.make(n, C, K, H, W, 3, 3, 1, 1)
        D = O.gen_sparse(n, C, H, W, 0.6, 10 + i)
        G = O.gen_sparse(K, C, 3, 3, 0.0, 20 + i)
        dY = O.gen_sparse(n, K, H, W, 0.5, 30 + i)
        ops = [(sp.Component.fwd, sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)),
               (sp.Component.bwi, sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)),
               (sp.Component.bww, sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V))]
        for j, (comp, a, b) in enumerate(ops):
            pl = sp.plan(sh, comp, V)
            ref = sp.run_parallel(a, b, sh, pl, sp.RunMode.sparse)  # per-call host path (pageable numpy)
            if (i + j) % 2 == 0:  # pinned operands and output: the pipelined path
                a = sp.BlockedTensor(**{**a.header(), "data": torch.from_numpy(a.data).pin_memory().numpy()})
                b = sp.BlockedTensor(**{**b.header(), "data": torch.from_numpy(b.data).pin_memory().numpy()})
                out = torch.empty(ref.out.data.size, dtype=torch.float32).pin_memory().numpy()
            else:
                out = None
            hb.add(a, b, sh, pl, sp.RunMode.sparse, out=out)
            want.append(ref)
    for rep in range(2):  # the second run reuses the arena and the slots
        got = hb.run()
        assert len(got) == len(want) == 12
        for g, w in zip(got, want):
            assert np.array_equal(g.out.data, w.out.data)
            assert g.counters == w.counters
            assert g.out.header() == w.out.header()


def test_host_batch_shared_and_chained_buffers(sp):
    """Batch passes that name the same host buffers: (1) BWI and BWW read one
    dY buffer (uploaded once, read in place by the second pass); (2) a pass
    reads the buffer an earlier pass of the batch writes (the batch must keep
    the order of a sequential loop); (3) a later pass overwrites a buffer an
    earlier pass read, and a still later pass reads the new contents.  All
    pinned; results bitwise those of sequential per-call runs."""
    import torch
    V = 16
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()

    def pinned(t):
        return sp.BlockedTensor(**{**t.header(), "data": pin(t.data)})

    n, C, K, H, W = 20, 32, 32, 12, 12
    sh = sp.ConvShape.make(n, C, K, H, W, 3, 3, 1, 1)
    D = O.gen_sparse(n, C, H, W, 0.6, 1)
    G = O.gen_sparse(K, C, 3, 3, 0.0, 2)
    pf, pb, pw = (sp.plan(sh, c, V) for c in (sp.Component.fwd, sp.Component.bwi, sp.Component.bww))
    bD, bG, bGt, bDc = (pinned(t) for t in (sp.pack_act_nchwc(D, V), sp.pack_filter(G, V), sp.pack_filter(G, V, True),
                                            sp.pack_act_chwnn(D, V)))
    # sequential reference through the per-call path
    r_fwd = sp.run_parallel(bD, bG, sh, pf, sp.RunMode.sparse)
    Y = sp.BlockedTensor(**{**r_fwd.out.header(), "data": pin(r_fwd.out.data)})
    r_bwi = sp.run_parallel(Y, bGt, sh, pb, sp.RunMode.sparse)
    r_bww = sp.run_parallel(bDc, Y, sh, pw, sp.RunMode.sparse)
    r_fwd2 = sp.run_parallel(sp.BlockedTensor(**{**bD.header(), "data": r_bwi.out.data}), bG, sh, pf, sp.RunMode.sparse)
    r_bww2 = sp.run_parallel(bDc, sp.BlockedTensor(**{**Y.header(), "data": r_fwd2.out.data}), sh, pw,
                             sp.RunMode.sparse)
    # the same five passes as one batch over shared buffers
    ybuf = pin(np.zeros_like(r_fwd.out.data))
    dbuf = pin(np.zeros_like(r_bwi.out.data))
    Yb = sp.BlockedTensor(**{**r_fwd.out.header(), "data": ybuf})
    hb = sp.HostBatch()
    hb.add(bD, bG, sh, pf, out=ybuf)                      # writes ybuf
    hb.add(Yb, bGt, sh, pb, out=dbuf)                     # reads ybuf (chained), writes dbuf
    hb.add(bDc, Yb, sh, pw)                               # reads ybuf again (shared upload)
    hb.add(sp.BlockedTensor(**{**bD.header(), "data": dbuf}), bG, sh, pf, out=ybuf)  # overwrites ybuf
    hb.add(bDc, Yb, sh, pw)                               # must see the NEW ybuf
    for rep in range(2):
        got = hb.run()
        for i, (g, w) in enumerate(zip(got, (r_fwd, r_bwi, r_bww, r_fwd2, r_bww2))):
            # pass 0's output buffer is overwritten by pass 3; its value is checked through passes 1 and 2
            assert i == 0 or np.array_equal(g.out.data, w.out.data), i
            assert g.counters == w.counters, i


def test_host_batch_at_size_with_shared_dy(sp):
    """VGG conv3_2 / conv4_2 at batch 32 (100 MB / 50 MB tensors), FWD / BWI /
    BWW per layer with BWI and BWW naming one pinned dY buffer, eight layers'
    worth of passes (24 > pipeline slots, so every slot is refilled while a
    borrower may still read it): every output and counter bitwise those of
    the per-call path."""
    import torch
    from paper_1911_10175_b200 import workloads as wl
    V = 16
    g = torch.Generator(device="cuda").manual_seed(5)
    pin = lambda t: sp.BlockedTensor(**{**t.header(), "data": t.data.cpu().pin_memory().numpy()})
    hb = sp.HostBatch()
    want = []
    layers = wl.CONFIGS["vgg16_b32"]()
    for rep in range(4):
        for li in (4, 7):
            sh = layers[li].shape
            G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
            D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), 0.7, g)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), 0.7, g)
            bD = sp.pack_act_nchwc(D, V)
            hD, hY = pin(bD), pin(sp.pack_act_nchwc(dY, V))
            ops = [(sp.Component.fwd, hD, pin(sp.pack_filter(G, V))), (sp.Component.bwi, hY, pin(sp.pack_filter(G, V, True))),
                   (sp.Component.bww, pin(sp.nchwc_to_chwnn(bD)), hY)]
            for comp, a, b in ops:
                pl = sp.plan(sh, comp, V)
                want.append(sp.run_parallel(a, b, sh, pl, sp.RunMode.sparse))
                out = torch.empty(want[-1].out.data.size, dtype=torch.float32).pin_memory().numpy()
                hb.add(a, b, sh, pl, out=out)
            del D, dY, bD
    got = hb.run()
    for i, (gr, w) in enumerate(zip(got, want)):
        assert np.array_equal(gr.out.data, w.out.data), i
        assert gr.counters == w.counters, i


def test_host_batch_packs_the_bww_checked_operand_on_device(sp):
    """SPC_PASS_CHECKED_NCHWC: a batch BWW whose checked operand is the ActNCHWc
    buffer (shared with the layer's FWD pass, so it is uploaded once) equals the
    per-call BWW on the host-packed ActCHWNn operand, bitwise, for both check
    sides, ragged batches (N % 16 != 0), pinned and pageable buffers."""
    import torch
    V = 16
    pin = lambda t: sp.BlockedTensor(**{**t.header(), "data": torch.from_numpy(t.data).pin_memory().numpy()})
    for (n, C, K, H, W), pinned in [((40, 32, 128, 14, 14), True), ((19, 64, 64, 9, 10), True),
                                     ((33, 128, 128, 7, 7), False)]:
        sh = sp.ConvShape.make(n, C, K, H, W, 3, 3, 1, 1)
        D = O.gen_sparse(n, C, H, W, 0.6, n)
        G = O.gen_sparse(K, C, 3, 3, 0.0, n + 1)
        dY = O.gen_sparse(n, K, H, W, 0.5, n + 2)
        nD, nY, bG = sp.pack_act_nchwc(D, V), sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V)
        if pinned:
            nD, nY, bG = pin(nD), pin(nY), pin(bG)
        pf = sp.plan(sh, sp.Component.fwd, V)
        pi = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.input)
        po = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.output_grad)
        want = [sp.run_parallel(nD, bG, sh, pf, sp.RunMode.sparse),
                sp.run_parallel(sp.pack_act_chwnn(D, V), nY, sh, pi, sp.RunMode.sparse),
                sp.run_parallel(nD, sp.pack_act_chwnn(dY, V), sh, po, sp.RunMode.sparse)]
        hb = sp.HostBatch()
        hb.add(nD, bG, sh, pf)      # FWD uploads D (ActNCHWc)
        hb.add(nD, nY, sh, pi)      # BWW check=input: D again, in ActNCHWc -> packed on the device
        hb.add(nD, nY, sh, po)      # BWW check=output_grad: dY in ActNCHWc -> packed on the device
        for rep in range(2):
            got = hb.run()
            for i, (g, w) in enumerate(zip(got, want)):
                assert np.array_equal(g.out.data, w.out.data), (sh, pinned, i)
                assert g.counters == w.counters, (sh, pinned, i)
    # the flag is BWW-only and wants ActNCHWc
    with pytest.raises(sp.SpconvError):
        bad = sp.HostBatch()
        bad.add(sp.pack_act_chwnn(D, V), nY, sh, pi)
        bad._items[0]["flags"] = 1
        bad.run()


def test_host_batch_validates_every_pass_before_device_work(sp):
    V = 16
    sh = sp.ConvShape.make(2, 16, 16, 5, 5, 3, 3, 1, 1)
    D = O.gen_sparse(2, 16, 5, 5, 0.5, 1)
    G = O.gen_sparse(16, 16, 3, 3, 0.0, 2)
    pl = sp.plan(sh, sp.Component.fwd, V)
    hb = sp.HostBatch()
    hb.add(sp.pack_act_nchwc(D, V), sp.pack_filter(G, V), sh, pl)
    hb.add(sp.pack_act_nchwc(D, V), sp.pack_filter(G, V), sh, pl, out=np.empty(7, np.float32))  # too small
    n0 = sp.launch_count()
    with pytest.raises(sp.SpconvError):
        hb.run()
    assert sp.launch_count() == n0


def test_s2_bww_counted_dense_keeps_the_skip_semantics_for_nonfinite_dy(sp):
    """3x3 stride-2 BWW (check=input) runs every FMA ("counted dense") only when
    both operands are finite: with Inf / NaN in dY at pixels whose D partners are
    zero, the reference skips those products (P/include/spconv/vec.hpp:120-128) and
    so must we (the exact kernel takes over); counters stay exact either way."""
    V = 16
    sh = sp.ConvShape.make(3, 64, 128, 13, 12, 3, 3, 2, 2)
    t = sh.astuple()
    D = O.gen_sparse(3, 64, 13, 12, 0.6, 11)
    dY = O.gen_sparse(3, 128, sh.out_h(), sh.out_w(), 0.0, 12)
    pl = sp.plan(sh, sp.Component.bww, V)
    for poison in (False, True):
        d = D.copy()
        g = dY.copy()
        if poison:
            d[1, :, 0:5, 0:5] = 0.0          # every D partner of dY[1, :, 0..1, 0..1] is zero
            g[1, 5, 0, 0] = np.inf
            g[1, 77, 1, 1] = np.nan
        # the skipped products contribute nothing: the expected dG is the dense oracle's on the
        # unpoisoned dY (the poisoned pixels only ever meet zero D values)
        ref = O.dense(2, t, d, dY)
        res = sp.run_parallel(sp.pack_act_chwnn(d, V).to("cuda"), sp.pack_act_nchwc(g, V).to("cuda"), sh, pl,
                              sp.RunMode.sparse)
        got = sp.unpack(res.out).cpu().numpy()
        assert np.isfinite(got).all(), poison
        assert O.max_abs_rel(got, ref) <= TOL
        assert res.counters.executed_vector_fmas == O.expected_counts(t, O.plan(t, 2, V), d)["executed_vector_fmas"]


def test_tma_pw_bww_stage_reuse_is_race_free(sp):
    """The TMA-staged 1x1 BWW GEMM on a shape whose CTAs reuse their pipeline
    stages (56x56 images, K = 64: short steps).  Before the proxy fence that
    orders the warps' reads of a stage against its TMA refill, this shape gave
    ~1e-4 relative errors that changed from run to run (csrc/tma_pw_bww.cu)."""
    V = 16
    n, C, K, H, W = 16, 256, 64, 56, 56
    sh = sp.ConvShape.make(n, C, K, H, W, 1, 1, 1, 1)
    D = O.gen_sparse(n, C, H, W, 0.5, 1)
    dY = O.gen_sparse(n, K, H, W, 0.0, 2)
    ref = O.dense(2, sh.astuple(), D, dY)
    pl = sp.plan(sh, sp.Component.bww, V)
    a, b = sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda")
    first = None
    for rep in range(4):
        got = sp.unpack(sp.run_parallel(a, b, sh, pl, sp.RunMode.sparse).out).cpu().numpy()
        assert O.max_abs_rel(got, ref) <= TOL, rep
        if first is None:
            first = got
        assert np.array_equal(got, first), rep


def test_vector_probes_match_reference_semantics(sp):  # test_vec.cpp:38-57, kernels.hpp:90-98
    rng = np.random.default_rng(8)
    for V in (4, 8, 16):
        (p,) = sp.vector_probes(V)
        assert p.width == V and p.native
        for _ in range(50):
            v = rng.standard_normal(V).astype(np.float32)
            v[rng.random(V) < 0.4] = 0.0
            if V >= 8:
                v[1], v[2], v[3] = -0.0, np.nan, np.inf
            assert p.cmp_neq_zero(v) == O.cmp_neq_zero(v)
            a, w = rng.standard_normal(V).astype(np.float32), rng.standard_normal(V).astype(np.float32)
            s = np.float32(rng.standard_normal())
            fused = (a.astype(np.float64) + np.float64(s) * w.astype(np.float64)).astype(np.float32)
            assert np.array_equal(p.broadcast_fma(a, s, w), fused)
            assert np.array_equal(p.add(a, w), (a + w).astype(np.float32))

