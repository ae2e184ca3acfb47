"""Pin the C oracle (oracle/spconv_oracle.c) before trusting it.

Three anchors:
  1. the reference's own known answers (P/tests/test_oracle.cpp, test_kernels.cpp,
     test_tensor.cpp, test_planner.cpp, test_vec.cpp, test_sparsity.cpp);
  2. golden fixtures generated from the UNMODIFIED reference library
     (tests/golden/make_golden.py);
  3. the live reference library in oracle/_ref when it was built.
"""
import glob
import math
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
TAGS = [(0, 0, "fwd"), (1, 0, "bwi"), (2, 0, "bww_in"), (2, 1, "bww_og")]


def rng_tiny_shape(rng, V):
    """random_tiny_shape (P/tests/testutil.hpp:16-29), with numpy's RNG."""
    C = V * int(rng.choice([1, 2, 4]))
    K = V * int(rng.choice([1, 2, 4]))
    R = int(rng.choice([1, 3, 3, 5]))
    Os = 1 if R == 1 else int(rng.choice([1, 1, 2]))
    H = int(rng.integers(0, 6)) + R
    W = int(rng.integers(0, 6)) + R
    N = int(rng.integers(1, 6))
    return O.shape_make(N, C, K, H, W, R, R, Os, Os)


# ---------------------------------------------------------------- known answers
def test_all_ones_3x3_same_padding():  # test_oracle.cpp:12-20
    sh = O.shape_make(1, 1, 1, 3, 3, 3, 3, 1, 1)
    Y = O.dense(0, sh, np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 3, 3), np.float32))
    assert Y.ravel().tolist() == [4, 6, 4, 6, 9, 6, 4, 6, 4]


def test_center_delta_identity():  # test_oracle.cpp:22-29
    sh = O.shape_make(2, 3, 3, 4, 5, 3, 3, 1, 1)
    D = O.gen_sparse(2, 3, 4, 5, 0.2, 42)
    G = np.zeros((3, 3, 3, 3), np.float32)
    for k in range(3):
        G[k, k, 1, 1] = 1
    assert np.array_equal(O.dense(0, sh, D, G), D)


def test_zero_in_zero_out():  # test_oracle.cpp:31-62
    sh = O.shape_make(1, 2, 2, 4, 4, 3, 3, 1, 1)
    G = O.gen_sparse(2, 2, 3, 3, 0.0, 1)
    D = O.gen_sparse(1, 2, 4, 4, 0.0, 2)
    z = np.zeros((1, 2, 4, 4), np.float32)
    assert not O.dense(0, sh, z, G).any()
    assert not O.dense(1, sh, z, G).any()
    assert not O.dense(2, sh, D, z).any()


def test_bwi_1x1_is_channel_matmul():  # test_oracle.cpp:39-53
    sh = O.shape_make(1, 3, 2, 2, 2, 1, 1, 1, 1)
    dY = O.gen_sparse(1, 2, 2, 2, 0.0, 3)
    G = O.gen_sparse(2, 3, 1, 1, 0.0, 4)
    dD = O.dense(1, sh, dY, G)
    want = np.einsum("kyx,kc->cyx", dY[0].astype(np.float64), G[:, :, 0, 0].astype(np.float64))
    np.testing.assert_allclose(dD[0], want, rtol=1e-6)


def test_bww_single_pixel_outer_product():  # test_oracle.cpp:64-75
    sh = O.shape_make(1, 3, 2, 1, 1, 1, 1, 1, 1)
    D = O.gen_sparse(1, 3, 1, 1, 0.0, 5)
    dY = O.gen_sparse(1, 2, 1, 1, 0.0, 6)
    dG = O.dense(2, sh, D, dY)
    np.testing.assert_allclose(dG[:, :, 0, 0], np.outer(dY[0, :, 0, 0], D[0, :, 0, 0]), rtol=1e-6)


def test_linearity():  # test_oracle.cpp:77-99
    sh = O.shape_make(2, 3, 2, 5, 5, 3, 3, 1, 1)
    rng = np.random.default_rng(9)
    sg = lambda *s: ((rng.integers(0, 2001, size=s) - 1000) / 500.0).astype(np.float32)
    D1, D2, G = sg(2, 3, 5, 5), sg(2, 3, 5, 5), sg(2, 3, 3, 3)
    a, b = np.float32(0.75), np.float32(-1.25)
    lhs = O.dense(0, sh, (a * D1 + b * D2).astype(np.float32), G)
    rhs = (a * O.dense(0, sh, D1, G) + b * O.dense(0, sh, D2, G)).astype(np.float32)
    # the reference checks elementwise max_rel_error < 1e-5 on its own RNG
    # draw; with a different draw near-cancelled outputs make the elementwise
    # metric ill-conditioned, so the max-abs-normalised form is used here.
    assert O.max_abs_rel(lhs, rhs) < 1e-6


def test_adjointness():  # test_oracle.cpp:101-119
    rng = np.random.default_rng(31)
    for trial in range(50):
        sh = rng_tiny_shape(rng, 4)
        N, C, K, H, W, R, S = sh[:7]
        hp, wp = O.out_hw(sh)
        D = O.gen_sparse(N, C, H, W, 0.3, trial * 3 + 1)
        G = O.gen_sparse(K, C, S, R, 0.0, trial * 3 + 2)
        dY = O.gen_sparse(N, K, hp, wp, 0.3, trial * 3 + 3)
        a = O.dot(O.dense(0, sh, D, G), dY)
        b = O.dot(D, O.dense(1, sh, dY, G))
        c = O.dot(G, O.dense(2, sh, D, dY))
        assert abs(a - b) <= 1e-5 * max(1.0, abs(a))
        assert abs(a - c) <= 1e-5 * max(1.0, abs(a))


def test_expected_counts_1x1_k128():  # test_oracle.cpp:141-153
    sh = O.shape_make(1, 16, 128, 4, 4, 1, 1, 1, 1)
    pl = O.plan(sh, 0, 16)
    assert pl["Q"] == 128
    D = np.zeros((1, 16, 4, 4), np.float32)
    D[0, 3, 1, 2], D[0, 5, 0, 0], D[0, 9, 3, 3] = 1, 2, 3
    rep = O.expected_counts(sh, pl, D)
    assert rep["executed_vector_fmas"] == 24 and rep["nonzero_elements"] == 3


def test_single_interior_nonzero_36_fmas():  # test_kernels.cpp:97-110
    sh = O.shape_make(1, 32, 32, 8, 8, 3, 3, 1, 1)
    D = np.zeros((1, 32, 8, 8), np.float32)
    D[0, 5, 4, 4] = 0.7
    assert O.expected_counts(sh, O.plan(sh, 0, 8), D)["executed_vector_fmas"] == 36


def test_expected_counts_all_zero_and_dense():  # test_oracle.cpp:155-182
    rng = np.random.default_rng(13)
    for trial in range(20):
        sh = rng_tiny_shape(rng, 4)
        N, C, K, H, W = sh[:5]
        hp, wp = O.out_hw(sh)
        for comp in (0, 1, 2):
            pl = O.plan(sh, comp, 4)
            mc, mh, mw = (K, hp, wp) if comp == 1 else (C, H, W)
            rz = O.expected_counts(sh, pl, np.zeros((N, mc, mh, mw), np.float32))
            assert rz["executed_vector_fmas"] == 0 and rz["skipped_vector_fmas"] == rz["dense_total"]
            rd = O.expected_counts(sh, pl, O.gen_sparse(N, mc, mh, mw, 0.0, trial))
            assert rd["executed_vector_fmas"] == rd["dense_total"]


def test_cmp_neq_zero_bits():  # test_vec.cpp:38-57
    assert O.cmp_neq_zero([0] * 8) == 0
    assert O.cmp_neq_zero([0, 2, 0, 0, 5, 0, 7, 0]) == 0b01010010
    assert O.cmp_neq_zero([-0.0, 1e-30, -3.5, 0.0]) == 0b0110
    assert O.cmp_neq_zero([math.nan, 0.0, math.inf, -0.0]) == 0b0101


def test_affected_outputs_examples():  # test_tensor.cpp:44-65
    assert O.affected_outputs(O.shape_make(1, 1, 1, 5, 5, 3, 3, 1, 1), 2) == [(2, 1), (1, 2), (0, 3)]
    assert O.affected_outputs(O.shape_make(1, 1, 1, 5, 5, 3, 3, 2, 2), 0) == [(1, 0)]
    sh = O.shape_make(1, 1, 1, 9, 9, 1, 1, 1, 1)
    for x in range(9):
        assert O.affected_outputs(sh, x) == [(0, x)]


def test_output_shape_goldens_and_rejection():  # test_tensor.cpp:14-42
    assert O.out_hw(O.shape_make(16, 128, 256, 56, 56, 3, 3, 1, 1)) == (56, 56)
    assert O.out_hw(O.shape_make(16, 128, 128, 56, 56, 3, 3, 2, 2)) == (28, 28)
    sh = O.shape_make(1, 4, 4, 5, 5, 1, 1, 1, 1)
    assert O.out_hw(sh) == (5, 5) and sh[9] == 0 and sh[10] == 0
    assert not O.shape_valid((1, 1, 1, 2, 2, 5, 5, 1, 1, 1, 1))
    with pytest.raises(ValueError):
        O.shape_make(0, 1, 1, 4, 4, 1, 1, 1, 1)
    assert not O.shape_valid((1, 1, 1, 4, 4, 3, 3, 1, 1, 3, 1))
    with pytest.raises(ValueError):
        O.shape_make(1, 1, 1, 4, 4, 3, 3, -1, 1)


def test_golden_plans_table2():  # test_planner.cpp:11-36
    for R, (Q, T, pipe, ring) in {1: (128, 8, 1, 16), 3: (128, 24, 0, 24), 5: (64, 20, 1, 24)}.items():
        p = O.plan(O.shape_make(16, 256, 256, 28, 28, R, R, 1, 1), 0, 16)
        assert (p["Q"], p["T"], p["pipelined"], p["ring_size"]) == (Q, T, pipe, ring)


def test_relu_semantics():  # sparsity.cpp:11-28, test_sparsity.cpp:12-57
    x = np.array([-1.0, -0.0, 0.0, 2.5, math.nan, math.inf, -math.inf, 1e-38], np.float32)
    r = O.relu(x)
    assert r.tolist()[:4] == [0.0, 0.0, 0.0, 2.5]
    assert not np.signbit(r[:3]).any() and r[4] == 0.0 and r[5] == math.inf and r[6] == 0.0
    up = np.arange(8, dtype=np.float32) + 1
    assert O.relu_grad_mask(x, up).tolist() == [0, 0, 0, 4, 0, 6, 0, 8]


def test_gen_sparse_statistics_and_determinism():  # test_sparsity.cpp:59-76
    a = O.gen_sparse(4, 16, 32, 32, 0.7, 123)
    assert np.array_equal(a, O.gen_sparse(4, 16, 32, 32, 0.7, 123))
    assert abs((a == 0).mean() - 0.7) < 0.01
    nz = a[a != 0]
    assert nz.min() >= 0.1 and nz.max() <= 1.0


def test_pack_roundtrip_and_ragged_lanes():  # test_tensor.cpp:142-210
    rng = np.random.default_rng(2)
    t = rng.standard_normal((5, 8, 3, 4)).astype(np.float32)
    for V in (4, 8):
        assert np.array_equal(O.unpack_act(O.pack_act(t, V), 5, 8, 3, 4, V), t)
        b = O.pack_act(t, V, chwnn=True)
        assert np.array_equal(O.unpack_act(b, 5, 8, 3, 4, V, chwnn=True), t)
        lanes = b.reshape(-1, 8, 3, 4, V)
        assert not lanes[-1, ..., 5 % V:].any() if V == 8 else True
    g = rng.standard_normal((8, 16, 3, 3)).astype(np.float32)
    assert np.array_equal(O.unpack_filter(O.pack_filter(g, 8), 8, 16, 3, 3, 8), g)
    gt = O.pack_filter(g, 8, swap_kc=True)
    assert np.array_equal(O.unpack_filter(gt, 16, 8, 3, 3, 8), g.transpose(1, 0, 2, 3))


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_reference_fixtures(path):
    z = np.load(path)
    sh = tuple(int(v) for v in z["shape"])
    V = int(z["V"])
    for comp, check, tag in TAGS:
        a, b = z[f"{tag}_a"], z[f"{tag}_b"]
        # 64-bit dense oracle: bitwise identical to the reference's dense_*
        assert np.array_equal(O.dense(comp, sh, a, b), z[f"{tag}_oracle64"]), tag
        # packing: bitwise identical blocked operands
        if comp == 0:
            pa, pb = O.pack_act(a, V), O.pack_filter(b, V)
        elif comp == 1:
            pa, pb = O.pack_act(a, V), O.pack_filter(b, V, True)
        elif check == 0:
            pa, pb = O.pack_act(a, V, chwnn=True), O.pack_act(b, V)
        else:
            pa, pb = O.pack_act(a, V), O.pack_act(b, V, chwnn=True)
        assert np.array_equal(pa, z[f"{tag}_a_blk"]) and np.array_equal(pb, z[f"{tag}_b_blk"]), tag
        # exact skip accounting: simulation == the reference kernel's counters
        pl = O.plan(sh, comp, V, 30, check)
        mask = b if (comp == 2 and check == 1) else a
        rep = O.expected_counts(sh, pl, mask)
        cs, cd = z[f"{tag}_counters_sparse"], z[f"{tag}_counters_dense"]
        assert rep["checked_vectors"] == cs[0] and rep["executed_vector_fmas"] == cs[1], tag
        assert rep["dense_total"] == cd[1] and cd[0] == 0, tag
        # the reference's own CPU kernel sits well inside the gate vs the oracle
        assert O.max_abs_rel(z[f"{tag}_ref_sparse"], z[f"{tag}_oracle64"]) <= 1e-5, tag


# ---------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_mt19937_64_stream_matches_std():
    for seed in (0, 1, 5489, 2**63 + 7):
        assert np.array_equal(O.mt64_stream(seed, 2000), O.ref_mt64_stream(seed, 2000))


@needs_ref
def test_generators_match_reference():
    for s in (0.0, 0.3, 0.9, 1.0):
        assert np.array_equal(O.gen_sparse(3, 5, 7, 11, s, 77), O.ref_gen_sparse(3, 5, 7, 11, s, 77))


@needs_ref
def test_random_shapes_dense_plans_counts_match_reference():
    rng = np.random.default_rng(101)
    for trial in range(40):
        V = [4, 8, 16][trial % 3]
        sh = rng_tiny_shape(rng, V)
        N, C, K, H, W, R, S = sh[:7]
        hp, wp = O.out_hw(sh)
        assert sh == O.ref_shape_make(N, C, K, H, W, R, S, sh[7], sh[8])
        D = O.gen_sparse(N, C, H, W, 0.5, trial)
        G = O.gen_sparse(K, C, S, R, 0.0, trial + 1)
        dY = O.gen_sparse(N, K, hp, wp, 0.4, trial + 2)
        for comp, a, b in ((0, D, G), (1, dY, G), (2, D, dY)):
            assert np.array_equal(O.dense(comp, sh, a, b), O.ref_dense(comp, sh, a, b))
        for comp, check, mask in ((0, 0, D), (1, 0, dY), (2, 0, D), (2, 1, dY)):
            p = O.plan(sh, comp, V, 30, check)
            rp = O.ref_plan(sh, comp, V, 30, check)
            assert all(p[k] == rp[k] for k in rp)
            mine = O.expected_counts(sh, p, mask)
            theirs = O.ref_expected_counts(comp, check, sh, V, mask)
            assert all(mine[k] == theirs[k] for k in theirs)
