"""Fused FWD/BWI output epilogues (include/spconv_b200.h spc_epilogue): the
fused result equals the plain pass followed by the reference's relu /
relu_grad_mask semantics (P/src/sparsity.cpp:11-28), bit for bit, on the
tile kernels (branch and jump-table variants) and the shape-general path."""
import zlib

import pytest
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

pytestmark = pytest.mark.gpu
V = 16

SHAPES = [
    ("3x3 s1 KK4", (4, 32, 128, 14, 14, 3, 1)),
    ("3x3 s1 KK2", (3, 64, 64, 9, 11, 3, 1)),
    ("3x3 s2", (4, 64, 128, 15, 13, 3, 2)),
    ("1x1 s1", (4, 64, 256, 7, 9, 1, 1)),
    ("1x1 s2", (2, 128, 256, 14, 14, 1, 2)),
    ("5x5 generic", (2, 16, 32, 8, 8, 5, 1)),
]


def _inputs(comp, sh, s, g):
    G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
    if comp == sp.Component.fwd:
        x = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g)
        return sp.pack_act_nchwc(x, V), sp.pack_filter(G, V)
    dy = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g)
    return sp.pack_act_nchwc(dy, V), sp.pack_filter(G, V, True)


def _run(a, b, sh, pl, mode, epi=None):
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    pp = sp.PreparedPass(a, b, sh, pl, mode, counters=cnt, epilogue=epi)
    pp.launch(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return pp.out.clone(), pp.read_counters()


@pytest.mark.parametrize("name,dims", SHAPES)
@pytest.mark.parametrize("comp", [sp.Component.fwd, sp.Component.bwi])
@pytest.mark.parametrize("s", [0.5, 0.93])
def test_fused_epilogue_equals_separate_passes(name, dims, comp, s):
    N, Cc, K, H, W, R, O = dims
    sh = sp.ConvShape.make(N, Cc, K, H, W, R, R, O, O)
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(f"{name}/{int(comp)}/{s}".encode()))
    a, b = _inputs(comp, sh, s, g)
    pl = sp.plan(sh, comp, V)
    mode = sp.RunMode.sparse
    plain, c0 = _run(a, b, sh, pl, mode)
    n = plain.numel()
    add = torch.randn(n, device="cuda", generator=g)
    mask = torch.randn(n, device="cuda", generator=g)
    mask[::7] = -0.0
    for epi in [sp.Epilogue(relu=True), sp.Epilogue(mask=mask), sp.Epilogue(alpha=0.37, add=add, relu=True),
                sp.Epilogue(alpha=-1.5, add=add, relu=True, mask=mask)]:
        fused, c1 = _run(a, b, sh, pl, mode, epi)
        assert c1 == c0  # the epilogue never changes the counters
        ref = plain.clone()
        sp.epilogue_apply(epi, ref)  # the standalone pass (same per-element code)
        torch.cuda.synchronize()
        assert torch.equal(fused, ref), (name, epi)
        if epi.add is None and epi.alpha == 1.0:
            want = plain
            if epi.relu:
                want = torch.where(want > 0, want, torch.zeros_like(want))  # sparsity.cpp:13
            if epi.mask is not None:
                want = torch.where(epi.mask > 0, want, torch.zeros_like(want))  # sparsity.cpp:26
            assert torch.equal(fused, want)


def test_relu_epilogue_maps_negative_zero_and_nan_to_positive_zero():
    sh = sp.ConvShape.make(1, 16, 16, 4, 4, 1, 1, 1, 1)
    plain = torch.tensor([-0.0, float("nan"), -1.0, 2.0] * 64, device="cuda")
    out = plain.clone()
    sp.epilogue_apply(sp.Epilogue(relu=True), out)
    torch.cuda.synchronize()
    assert torch.equal(out, torch.tensor([0.0, 0.0, 0.0, 2.0] * 64, device="cuda"))
    assert not torch.signbit(out).any()
    del sh


def test_bww_rejects_epilogue():
    sh = sp.ConvShape.make(2, 16, 16, 4, 4, 3, 3, 1, 1)
    a = sp.pack_act_chwnn(torch.rand(2, 16, 4, 4, device="cuda"), V)
    b = sp.pack_act_nchwc(torch.rand(2, 16, 4, 4, device="cuda"), V)
    pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.input)
    with pytest.raises(sp.SpconvError):
        sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse, epilogue=sp.Epilogue(relu=True))
