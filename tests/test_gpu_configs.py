"""Parity per BASELINE config with its OWN input distributions
(workloads.layer_inputs_host; cfg 2 is tests/test_gpu_fullsize.py, cfg 1 is
test_gpu_parity.test_config1_full_size_matches_reference_cpu).

* cfg 3, ResNet-34: every one of the 35 convs (3x3 s1/s2, 1x1 s2
  projections) at its seeded per-layer sparsity U[0.4, 0.8], dense dY
  (BatchNorm before the ReLU), one full 16-image lane block of the batch;
* cfg 4, ResNet-50: every one of the 52 convs with spatially correlated
  ReLU(conv3x3_rand(N(0,1)) - tau) inputs (mean sparsity 0.6), dense dY;
* cfg 5, Fixup ResNet-50 at the full batch of 256: the calibrated chain
  reaches ~0.7 activation sparsity, and its passes agree with the 64-bit
  oracle fed the chain's own device tensors (FWD/BWI on an image slice of
  every conv; BWW of the stage-4 convs over the whole batch).

Each pass: the reference's CPU run_parallel on the byte-identical packed
operands, max|d|/max|ref| <= 1e-5, all four counters integer-equal.
"""
import numpy as np
import pytest
import torch

import oracle as O
from parity_util import TOL, assert_counts_equal, ref_vs_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("config", ["resnet34_b64", "resnet50_b64"])
def test_every_layer_of_the_config_matches_reference(sp, config):
    from paper_1911_10175_b200 import workloads as wl
    layers = wl.CONFIGS[config]()
    worst = 0.0
    sp_in = []
    for li, layer in enumerate(layers):
        sh = layer.shape.with_batch(16)
        D, G, dY = wl.layer_inputs_host(config, li, sh)
        sp_in.append(float((D == 0).mean()))
        assert (dY == 0).mean() < 1e-4  # BatchNorm nets: dense output gradients (no ReLU mask)
        for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY)):
            res = ref_vs_gpu(sp, sh, comp, check, a, b)
            ctx = (config, layer.name, comp)
            assert res["finite"] and res["err"] <= TOL, (ctx, res["err"])
            assert_counts_equal(res, ctx)
            worst = max(worst, res["err"])
    mean_s = float(np.mean(sp_in))
    if config == "resnet34_b64":
        assert 0.4 <= min(sp_in) and max(sp_in) <= 0.8 + 0.02 and 0.5 < mean_s < 0.7
    else:
        assert abs(mean_s - 0.6) < 0.03
    print(f"{config}: {len(layers)} layers x 3 passes, worst max|d|/max|ref| {worst:.2e}, "
          f"mean input sparsity {mean_s:.3f}")


def test_fixup_resnet50_b256_chain_full_size():
    import paper_1911_10175_b200 as sp
    from paper_1911_10175_b200 import chain as CH
    ch = CH.fixup_resnet50(256)
    ch.step()
    torch.cuda.synchronize()
    rep = ch.sparsity_report()
    assert 0.65 < rep["activation_sparsity_mean"] < 0.75, rep["activation_sparsity_mean"]
    assert 0.6 < rep["gradient_sparsity_mean"] < 0.8, rep["gradient_sparsity_mean"]
    relu = lambda v: np.where(v > 0, v, np.float32(0))
    npb = lambda bt: sp.unpack(bt).cpu().numpy()
    G = {n: w[2].cpu().numpy() for n, w in ch.weights.items()}
    n2 = 2  # images checked per FWD/BWI pass (images are independent)
    for bi, A in enumerate(ch.acts):
        x, a, b, out = npb(A["x"])[:n2], npb(A["a"])[:n2], npb(A["b"])[:n2], npb(A["out"])[:n2]
        s1, s2, s3 = (A[k].with_batch(n2).astuple() for k in ("s1", "s2", "s3"))
        b1, b2, b3 = (np.float32(ch.bias[f"b{bi}.{c}"]) for c in ("c1", "c2", "c3"))
        for got, ref, what in ((a, relu(O.dense(0, s1, x, G[f"b{bi}.c1"]) + b1), "a"),
                               (b, relu(O.dense(0, s2, a, G[f"b{bi}.c2"]) + b2), "b")):
            assert O.max_abs_rel(got, ref) <= TOL, (bi, what)
        sc = npb(A["sc"])[:n2] if A["sp"] is not None else x
        ref_out = relu((O.dense(0, s3, b, G[f"b{bi}.c3"]).astype(np.float64) * np.float32(ch.scale)
                        + sc).astype(np.float32) + b3)
        assert O.max_abs_rel(out, ref_out) <= TOL, (bi, "out")
    # backward: BWI on the image slice, BWW of the stage-4 convs (7x7) over the whole batch
    for (seq, names, T), bi in zip(ch._bwd_blocks, reversed(range(len(ch.blocks)))):
        A = ch.acts[bi]
        dz, db, da = npb(T["dz_in"]), npb(T["db"]), npb(T["da"])
        b, a = npb(A["b"]), npb(A["a"])
        s3, s2 = A["s3"], A["s2"]
        rdb = np.where(b[:n2] > 0, np.float32(ch.scale) * O.dense(1, s3.with_batch(n2).astuple(), dz[:n2],
                                                                   G[f"b{bi}.c3"]), np.float32(0))
        assert O.max_abs_rel(db[:n2], rdb) <= TOL, (bi, "db")
        rda = np.where(a[:n2] > 0, O.dense(1, s2.with_batch(n2).astuple(), db[:n2], G[f"b{bi}.c2"]), np.float32(0))
        assert O.max_abs_rel(da[:n2], rda) <= TOL, (bi, "da")
        if A["s3"].H == 7:
            q = s3
            g3 = sp.unpack(sp.BlockedTensor(sp.Layout.filter_kcrs_blk, 16, 0, q.C, 0, 0, q.K, q.R, q.S,
                                            ch.grad_slice[f"b{bi}.c3"])).cpu().numpy()
            assert O.max_abs_rel(g3, np.float32(ch.scale) * O.dense(2, q.astuple(), b, dz)) <= TOL, (bi, "dG3")
    print(f"fixup b256: activation sparsity {rep['activation_sparsity_mean']:.3f}, "
          f"gradient sparsity {rep['gradient_sparsity_mean']:.3f}")
