"""Full-size parity on the BENCHED configuration (BASELINE cfg 2, VGG16 b32).

Every one of the 12 layers x FWD / BWI / BWW (check = input AND check =
output_grad) x sparsity {0.4, 0.6, 0.8, 0.9}, at the bench's batch of 32 and
224x224, through the production dispatch (the same ``spc_sparse_*`` entry
``bench.py`` launches: per-shape BWW split count, KK=2 / KK=4 branch +
jump-table pairs selected on the device by density, block order for large
sources).  Each pass is compared with the reference's own CPU
``run_parallel`` (P/src/kernels.cpp:304-313; backend automatic, all host
threads) on byte-identical packed operands:

* values: max|got - ref| / max|ref| <= 1e-5 (north_star);
* zero/nonzero indexing: all four ``kernel_counters`` integer-equal.

Plus the 64-bit oracle (``dense_*``, P/src/oracle.cpp:39-148, rounded once to
fp32): FWD/BWI on a 2-image slice of every layer (images are independent), and
SURVEY 8(c'): the deepest BWW reduction in the configs -- VGG conv1_2, N=32,
64->64 @224, 1.6 M terms per weight -- against ``dense_bww`` at full size.

Inputs: BASELINE cfg-2 distributions (workloads.vgg16_inputs_host, seeded).
"""
import os

import numpy as np
import pytest

import oracle as O
from parity_util import TOL, assert_counts_equal, ref_vs_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

GRID = (0.4, 0.6, 0.8, 0.9)


@pytest.mark.parametrize("s", GRID)
def test_vgg16_b32_every_layer_every_pass_matches_reference(sp, s):
    from paper_1911_10175_b200 import workloads as wl
    layers = wl.vgg16(32)
    worst = {}
    for li, layer in enumerate(layers):
        sh = layer.shape
        D, G, dY = wl.layer_inputs_host("vgg16_b32", li, sh, s)
        for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY), (2, 1, D, dY)):
            ctx = (layer.name, s, comp, check)
            res = ref_vs_gpu(sp, sh, comp, check, a, b, keep_gpu=comp < 2)
            assert res["finite"], ctx
            assert res["err"] <= TOL, (ctx, res["err"])
            assert_counts_equal(res, ctx)
            worst[(comp, check)] = max(worst.get((comp, check), 0.0), res["err"])
            if comp < 2:
                # 64-bit oracle on the first 2 images of the same batch
                sl = sh.with_batch(2).astuple()
                ref64 = O.dense(comp, sl, a[:2], b)
                e64 = O.max_abs_rel(res["out"][:2], ref64)
                assert e64 <= TOL, (ctx, "dense64", e64)
            del res
        del D, G, dY
    print(f"s={s}: worst max|d|/max|ref| vs reference CPU per (comp, check): "
          + ", ".join(f"{k}: {v:.2e}" for k, v in sorted(worst.items())))


@pytest.mark.parametrize("s", (0.4, 0.9))
@pytest.mark.parametrize("check", (0, 1))
def test_conv1_2_n32_deepest_bww_reduction_vs_64bit_oracle(sp, s, check):
    """SURVEY 8(c'): dG of VGG conv1_2 at N=32 sums 32*224*224 = 1.6 M products
    per weight; the production split reduction must stay within 1e-5 of the
    64-bit oracle (the reference's CPU kernels reach 1.03e-6 here)."""
    import torch
    from paper_1911_10175_b200 import workloads as wl
    sh = wl.vgg16(32)[0].shape
    D, _, dY = wl.layer_inputs_host("vgg16_b32", 0, sh, s)
    V = 16
    if check == 0:
        ba, bb = sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V)
    else:
        ba, bb = sp.pack_act_nchwc(D, V), sp.pack_act_chwnn(dY, V)
    ba, bb = ba.to("cuda"), bb.to("cuda")
    pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck(check))
    res = sp.run_parallel(ba, bb, sh, pl, sp.RunMode.sparse)
    got = sp.unpack(res.out).cpu().numpy()
    del ba, bb
    torch.cuda.empty_cache()
    ref64 = O.dense(2, sh.astuple(), D, dY)
    err = O.max_abs_rel(got, ref64)
    print(f"conv1_2 N=32 BWW check={check} s={s}: max|d|/max|ref| vs 64-bit oracle = {err:.2e}")
    assert err <= TOL
    want = O.expected_counts(sh.astuple(), O.plan(sh.astuple(), 2, V, 30, check), D if check == 0 else dY)
    assert res.counters.executed_vector_fmas == want["executed_vector_fmas"]
    assert res.counters.checked_vectors == want["checked_vectors"]


def test_vgg16_b32_dense_mode_matches_reference_dense_mode(sp):
    """run_mode::dense (the reference's speedup denominator, P/include/spconv/
    kernels.hpp:24): every layer x FWD / BWI / BWW (both checks) at the full
    batch, against the reference's own dense-mode run_parallel; counters
    equal its dense totals (checked_vectors = 0)."""
    from paper_1911_10175_b200 import workloads as wl
    worst = 0.0
    for li, layer in enumerate(wl.vgg16(32)):
        sh = layer.shape
        D, G, dY = wl.layer_inputs_host("vgg16_b32", li, sh, 0.4, seed=1)
        for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY), (2, 1, D, dY)):
            ctx = (layer.name, "dense", comp, check)
            res = ref_vs_gpu(sp, sh, comp, check, a, b, mode=1)
            assert res["finite"] and res["err"] <= TOL, (ctx, res["err"])
            assert_counts_equal(res, ctx)
            assert res["gpu"].checked_vectors == 0
            worst = max(worst, res["err"])
    print(f"dense mode: worst max|d|/max|ref| vs reference CPU {worst:.2e}")


def test_vgg16_b32_tf32x3_variant_matches_reference(sp):
    """The optional 3xTF32 tensor-core variant (DESIGN 4.7, stated tolerance
    1e-5) through its production dispatch at the benched size: every layer x
    FWD / BWI / BWW (both checks) at s = 0.6 vs the reference CPU, counters
    exact."""
    from paper_1911_10175_b200 import workloads as wl
    worst = 0.0
    with sp.math_mode(sp.Math.tf32x3):
        for li, layer in enumerate(wl.vgg16(32)):
            sh = layer.shape
            D, G, dY = wl.layer_inputs_host("vgg16_b32", li, sh, 0.6, seed=2)
            for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY), (2, 1, D, dY)):
                ctx = (layer.name, "tf32x3", comp, check)
                res = ref_vs_gpu(sp, sh, comp, check, a, b)
                assert res["finite"] and res["err"] <= TOL, (ctx, res["err"])
                assert_counts_equal(res, ctx)
                worst = max(worst, res["err"])
    print(f"tf32x3: worst max|d|/max|ref| vs reference CPU {worst:.2e}")
