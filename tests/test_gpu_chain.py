"""Layer-chain driver (paper_1911_10175_b200/chain.py) on a small bottleneck
stack: every pass of one training step is checked against the 64-bit oracle
(P/src/oracle.cpp:39-148) fed the chain's own recorded device tensors, and
every ReLU / ReLU-grad mask against the reference semantics
(P/src/sparsity.cpp:11-28).  Tolerance: max|d|/max|ref| <= 1e-5 per pass (the
north-star bar); masks and zero patterns exact."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import chain as CH

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _np(bt):
    return sp.unpack(bt).cpu().numpy() if torch.is_tensor(bt.data) else sp.unpack(bt)


def _filt_np(t, K, Cc, S, R):
    return sp.unpack(sp.BlockedTensor(sp.Layout.filter_kcrs_blk, 16, 0, Cc, 0, 0, K, R, S, t)).cpu().numpy()


def _close(got, ref, what):
    err = O.max_abs_rel(got, ref)
    assert err <= TOL, f"{what}: {err:.3e}"


def _fma(a, alpha, add):  # fmaf(a, alpha, add) per element (exact in float64 here for these magnitudes)
    return (a.astype(np.float64) * np.float64(np.float32(alpha)) + add.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("mode", [sp.RunMode.sparse, sp.RunMode.dense])
def test_chain_step_matches_oracle_pass_by_pass(mode):
    blocks = CH.resnet50_blocks(H=10, W=10, cin=32, stages=((16, 1), (32, 2)))
    assert [b.proj for b in blocks] == [True, True, False]
    _check_chain(CH.FixupChain(3, blocks, scale=0.5, seed=7, mode=mode, x_sparsity=0.6), blocks)


def test_chain_step_tf32x3_matches_oracle_pass_by_pass():
    """The same step with the 3xTF32 tensor-core variant (64-channel multiples,
    so its 1x1 / 3x3 stride-1 passes run on tcgen05; stride-2 passes stay FP32)."""
    blocks = CH.resnet50_blocks(H=8, W=8, cin=64, stages=((64, 1), (128, 2)))
    launches = sp.launch_count()
    with sp.math_mode(sp.Math.tf32x3):
        _check_chain(CH.FixupChain(3, blocks, scale=0.5, seed=11, mode=sp.RunMode.sparse, x_sparsity=0.6),
                     blocks)
    assert sp.launch_count() > launches


def _check_chain(ch, blocks):
    ch.set_upstream()
    ch.step()
    torch.cuda.synchronize()
    scale = np.float32(0.5)
    G = {n: w[2].cpu().numpy() for n, w in ch.weights.items()}
    relu = lambda v: np.where(v > 0, v, np.float32(0))
    # ---- forward
    for bi, A in enumerate(ch.acts):
        x, a, b, out = _np(A["x"]), _np(A["a"]), _np(A["b"]), _np(A["out"])
        s1, s2, s3, spj = (A[k].astuple() if A[k] is not None else None for k in ("s1", "s2", "s3", "sp"))
        b1, b2, b3 = (np.float32(ch.bias[f"b{bi}.{c}"]) for c in ("c1", "c2", "c3"))
        ra = O.dense(0, s1, x, G[f"b{bi}.c1"]) + b1
        _close(a, relu(ra), f"b{bi} a")
        assert np.array_equal(a == 0, relu(ra) == 0) or O.max_abs_rel(a, relu(ra)) < TOL
        _close(b, relu(O.dense(0, s2, a, G[f"b{bi}.c2"]) + b2), f"b{bi} b")
        sc = _np(A["sc"]) if spj is not None else x
        if spj is not None:
            _close(sc, O.dense(0, spj, x, G[f"b{bi}.proj"]), f"b{bi} proj")
        c = O.dense(0, s3, b, G[f"b{bi}.c3"])
        _close(out, relu(_fma(c, scale, sc) + b3), f"b{bi} out")
        assert (out >= 0).all() and not np.signbit(out).any()  # ReLU maps -0 to +0
    # ---- backward
    last = ch.acts[-1]["out"]
    dout = sp.unpack(sp.BlockedTensor(sp.Layout.act_nchwc, 16, last.n, last.c, last.h, last.w, data=ch.dout))
    dz = _np(ch.dz_last)
    assert np.array_equal(dz, np.where(_np(last) > 0, dout.cpu().numpy(), np.float32(0)))  # bit-exact mask
    for (seq, names, T), bi in zip(ch._bwd_blocks, reversed(range(len(blocks)))):
        A = ch.acts[bi]
        x, a, b = _np(A["x"]), _np(A["a"]), _np(A["b"])
        s1, s2, s3 = A["s1"], A["s2"], A["s3"]
        dz, db, da = _np(T["dz_in"]), _np(T["db"]), _np(T["da"])
        shp = {"c1": s1, "c2": s2, "c3": s3, "proj": A["sp"]}
        gs = {}
        for n in names:
            q = shp[n.split(".")[1]]
            gs[n] = _filt_np(ch.grad_slice[n], q.K, q.C, q.S, q.R)
        _close(gs[f"b{bi}.c3"], scale * O.dense(2, s3.astuple(), b, dz), f"b{bi} dG3")
        rdb = np.where(b > 0, scale * O.dense(1, s3.astuple(), dz, G[f"b{bi}.c3"]), np.float32(0))
        _close(db, rdb, f"b{bi} db")
        assert not (db[b <= 0]).any()  # masked exactly where !(pre > 0)
        _close(gs[f"b{bi}.c2"], O.dense(2, s2.astuple(), a, db), f"b{bi} dG2")
        _close(da, np.where(a > 0, O.dense(1, s2.astuple(), db, G[f"b{bi}.c2"]), np.float32(0)), f"b{bi} da")
        _close(gs[f"b{bi}.c1"], O.dense(2, s1.astuple(), x, da), f"b{bi} dG1")
        skip = dz
        if A["sp"] is not None:
            spj = A["sp"].astuple()
            _close(gs[f"b{bi}.proj"], O.dense(2, spj, x, dz), f"b{bi} dGp")
            skip = O.dense(1, spj, dz, G[f"b{bi}.proj"])
        nxt = _np(ch.dx0) if bi == 0 else _np(ch._bwd_blocks[len(blocks) - bi][2]["dz_in"])
        ref = np.where(x > 0, O.dense(1, s1.astuple(), da, G[f"b{bi}.c1"]) + skip, np.float32(0))
        _close(nxt, ref, f"b{bi} dz_prev")
        assert not nxt[x <= 0].any()
    rep = ch.sparsity_report()
    assert 0.3 < rep["activation_sparsity_mean"] < 0.95
    assert ch.dense_flops() == sum(sh.dense_flops() for _, _, sh in ch.passes)
    # every conv has FWD, BWI and BWW passes
    for name in ch.weights:
        kinds = sorted(int(c) for n, c, _ in ch.passes if n == name)
        assert kinds == [0, 1, 2], (name, kinds)


def test_chain_sparse_equals_dense_mode_within_rounding():
    blocks = CH.resnet50_blocks(H=8, W=8, cin=64, stages=((16, 2),))
    outs = []
    for mode in (sp.RunMode.sparse, sp.RunMode.dense):
        ch = CH.FixupChain(2, blocks, scale=0.5, seed=3, mode=mode)
        ch.set_upstream()
        ch.step()
        torch.cuda.synchronize()
        outs.append((_np(ch.out), ch.grads.cpu().numpy().copy()))
    _close(outs[0][0], outs[1][0], "out")
    _close(outs[0][1], outs[1][1], "grads")


def test_resnet50_blocks_are_the_52_conv_shapes():
    from paper_1911_10175_b200 import workloads as wl
    blocks = CH.resnet50_blocks()
    shapes = []
    for b in blocks:
        Ho = (b.H - 1) // b.stride + 1
        shapes.append((b.cin, b.width, b.H, 1, 1))
        shapes.append((b.width, b.width, b.H, 3, b.stride))
        if b.proj:
            shapes.append((b.cin, 4 * b.width, b.H, 1, b.stride))
        shapes.append((b.width, 4 * b.width, Ho, 1, 1))
    ref = [(L.shape.C, L.shape.K, L.shape.H, L.shape.R, L.shape.O) for L in wl.resnet50(64)]
    assert sorted(shapes) == sorted(ref) and len(ref) == 52


def test_calibrated_biases_hit_the_target_sparsity():
    """BASELINE cfg 5: ReLU masks of the seeded forward pass at ~0.7 mean
    activation sparsity (Fixup biases calibrated on that pass)."""
    blocks = CH.resnet50_blocks(H=14, W=14, cin=64, stages=((32, 2), (64, 2)))
    ch = CH.FixupChain(8, blocks, scale=0.25, seed=5)
    ch.step()
    torch.cuda.synchronize()
    rep = ch.sparsity_report()
    assert 0.62 < rep["activation_sparsity_mean"] < 0.78, rep["activation_sparsity_mean"]
    assert any(v != 0.0 for v in ch.bias.values())


def test_two_rank_shards_equal_the_full_batch_step():
    """Data parallelism: the step of the global batch split over 2 ranks (each
    its slice, the same weights from one seed, the same biases) equals the
    single-rank full-batch step -- outputs per image, dG summed over ranks."""
    blocks = CH.resnet50_blocks(H=8, W=8, cin=64, stages=((16, 1), (32, 1)))
    full = CH.FixupChain(6, blocks, scale=0.5, seed=9)
    full.set_upstream()
    full.step()
    parts = []
    for r in range(2):
        ch = CH.FixupChain(6, blocks, scale=0.5, seed=9, world=2, rank=r, bias=full.bias)
        ch.set_upstream()
        ch.step()
        parts.append(ch)
    torch.cuda.synchronize()
    for name in full.weights:  # identical weights on every rank
        assert all(torch.equal(p.weights[name][2], full.weights[name][2]) for p in parts)
    out = np.concatenate([_np(p.out) for p in parts])
    _close(out, _np(full.out), "out")
    g = parts[0].grads.cpu().numpy() + parts[1].grads.cpu().numpy()
    _close(g, full.grads.cpu().numpy(), "dG summed over ranks")
