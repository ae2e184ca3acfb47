"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/spconv_b200.h declares; shape/plan/counter/pack logic
and the contract checks match the reference (no device compute here)."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import HAS_GPU, ROOT

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
TAGS = [(0, 0, "fwd"), (1, 0, "bwi"), (2, 0, "bww_in"), (2, 1, "bww_og")]

# The reference's 27-layer registry geometries (P/src/bench.cpp:21-52) and the
# BASELINE.json conv shapes (VGG16 b32, ResNet-34/50 b64).
REGISTRY = [
    (64, 64, 224, 3, 1), (64, 128, 112, 3, 1), (128, 128, 112, 3, 1), (128, 256, 56, 3, 1),
    (256, 256, 56, 3, 1), (256, 512, 28, 3, 1), (512, 512, 28, 3, 1), (512, 512, 14, 3, 1),
    (64, 64, 56, 1, 1), (256, 64, 56, 1, 1), (64, 64, 56, 3, 1), (64, 256, 56, 1, 1), (256, 128, 56, 1, 1),
    (512, 128, 28, 1, 1), (128, 128, 28, 3, 1), (128, 128, 56, 3, 2), (128, 512, 28, 1, 1),
    (512, 256, 28, 1, 1), (1024, 256, 14, 1, 1), (256, 256, 14, 3, 1), (256, 256, 28, 3, 2),
    (256, 1024, 14, 1, 1), (1024, 512, 14, 1, 1), (2048, 512, 7, 1, 1), (512, 512, 7, 3, 1),
    (512, 512, 14, 3, 2), (512, 2048, 7, 1, 1), (64, 128, 56, 1, 2), (1024, 2048, 14, 1, 2),
]


def header_functions(name="spconv_b200.h"):
    src = open(os.path.join(ROOT, "include", name)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(sp):
    lib = ctypes.CDLL(sp._lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(sp._lib.EXPORTED)
    assert lib.spc_abi_version() == 3
    dev = header_functions("spconv_b200_dev.h")
    assert set(dev) == set(sp._lib.DEV_EXPORTED)
    for n in dev:
        assert hasattr(lib, n), n


def test_library_is_sm100a_only(sp):
    """The product .so carries sm_100a SASS only (no PTX/CPU fallback)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sp._lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_shape_make_parity(sp):
    rng = np.random.default_rng(4)
    for _ in range(300):
        dims = [int(rng.integers(-1, 9)) for _ in range(7)] + [int(rng.integers(0, 3)), int(rng.integers(0, 3))]
        try:
            want = O.shape_make(*dims)
        except ValueError:
            want = None
        try:
            got = sp.ConvShape.make(*dims).astuple()
        except sp.SpconvError as e:
            assert e.status == sp._lib.SPC_ERR_SHAPE
            got = None
        assert got == want, dims


def test_plan_parity_registry_and_baseline(sp):
    for C, K, HW, R, O_ in REGISTRY:
        for N in (16, 32, 64, 256):
            sh = sp.ConvShape.make(N, C, K, HW, HW, R, R, O_, O_)
            for V in (4, 8, 16):
                for comp in (0, 1, 2):
                    for check in ((0, 1) if comp == 2 else (0,)):
                        for budget in (30, 12, 64):
                            try:
                                want = O.plan(sh.astuple(), comp, V, budget, check)
                            except ValueError:
                                with pytest.raises(sp.SpconvError):
                                    sp.plan(sh, sp.Component(comp), V, budget, sp.BwwCheck(check))
                                continue
                            got = sp.plan(sh, sp.Component(comp), V, budget, sp.BwwCheck(check))
                            for k, v in want.items():
                                assert int(getattr(got, k)) == v, (k, sh, V, comp)


def test_plan_rejections(sp):
    # test_kernels.cpp:348-351: tiled channel dim not divisible by V
    with pytest.raises(sp.SpconvError):
        sp.plan(sp.ConvShape.make(2, 16, 12, 6, 6, 3, 3, 1, 1), sp.Component.fwd, 8)
    with pytest.raises(sp.SpconvError):
        sp.plan(sp.ConvShape.make(2, 16, 16, 6, 6, 3, 3, 1, 1), sp.Component.fwd, 5)
    with pytest.raises(sp.SpconvError):  # no Q fits a budget of 2 with R=3
        sp.plan(sp.ConvShape.make(2, 16, 16, 6, 6, 3, 3, 1, 1), sp.Component.fwd, 16, 2)


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_analytic_counters_match_reference_fixtures(sp, path):
    z = np.load(path)
    sh = sp.ConvShape(*[int(v) for v in z["shape"]])
    V = int(z["V"])
    for comp, check, tag in TAGS:
        pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
        cs, cd = z[f"{tag}_counters_sparse"], z[f"{tag}_counters_dense"]
        a = sp.analytic_counters(sh, pl, sp.RunMode.sparse)
        assert (a.checked_vectors, a.output_vector_loads, a.output_vector_stores) == (cs[0], cs[2], cs[3]), tag
        d = sp.analytic_counters(sh, pl, sp.RunMode.dense)
        assert (d.checked_vectors, d.executed_vector_fmas, d.output_vector_loads) == (cd[0], cd[1], cd[2]), tag


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_analytic_counters_match_reference_random(sp):
    from test_oracle import rng_tiny_shape
    rng = np.random.default_rng(77)
    for trial in range(30):
        V = [4, 8, 16][trial % 3]
        t = rng_tiny_shape(rng, V)
        sh = sp.ConvShape(*t)
        N, C, K, H, W, R, S = t[:7]
        hp, wp = O.out_hw(t)
        D = O.gen_sparse(N, C, H, W, 0.5, trial)
        G = O.gen_sparse(K, C, S, R, 0.0, trial + 1)
        dY = O.gen_sparse(N, K, hp, wp, 0.5, trial + 2)
        for comp, check, a, b in ((0, 0, D, G), (1, 0, dY, G), (2, 0, D, dY), (2, 1, D, dY)):
            r = O.RefRun(comp, check, t, V, a, b)
            pl = sp.plan(sh, sp.Component(comp), V, 30, sp.BwwCheck(check))
            for mode in (0, 1):
                r.exec(mode, 1)
                _, cnt, _ = r.result()
                mine = sp.analytic_counters(sh, pl, sp.RunMode(mode))
                assert mine.checked_vectors == cnt["checked_vectors"]
                assert mine.output_vector_loads == cnt["output_vector_loads"]
                assert mine.output_vector_stores == cnt["output_vector_stores"]
                if mode == 1:
                    assert mine.executed_vector_fmas == cnt["executed_vector_fmas"]
            r.close()


def test_pack_unpack_parity(sp):
    import torch
    rng = np.random.default_rng(8)
    for V in (4, 8, 16):
        t = rng.standard_normal((5, 2 * V, 3, 4)).astype(np.float32)
        t[0, 0, 0, 0] = -0.0
        b = sp.pack_act_nchwc(t, V)
        assert np.array_equal(b.data, O.pack_act(t, V))
        assert np.array_equal(sp.unpack(b), t)
        c = sp.pack_act_chwnn(t, V)
        assert np.array_equal(c.data, O.pack_act(t, V, chwnn=True))
        assert np.array_equal(sp.unpack(c), t)
        g = rng.standard_normal((V, 2 * V, 3, 3)).astype(np.float32)
        f = sp.pack_filter(g, V)
        assert np.array_equal(f.data, O.pack_filter(g, V))
        assert np.array_equal(sp.unpack(f), g)
        ft = sp.pack_filter(g, V, swap_kc=True)
        assert np.array_equal(ft.data, O.pack_filter(g, V, True))
        assert (ft.k, ft.c) == (2 * V, V)
        # torch (device-agnostic) packing gives the same bytes
        assert np.array_equal(sp.pack_act_nchwc(torch.from_numpy(t), V).data.numpy(), b.data)
        assert np.array_equal(sp.pack_act_chwnn(torch.from_numpy(t), V).data.numpy(), c.data)
        assert np.array_equal(sp.pack_filter(torch.from_numpy(g), V, True).data.numpy(), ft.data)
        # index helpers agree with the reference's address maps (tensor.hpp:98-119)
        assert b.data[b.act_index(3, V + 1, 2, 1)] == t[3, V + 1, 2, 1]
        assert c.data[c.chwnn_index(4, V + 1, 2, 3)] == t[4, V + 1, 2, 3]
        assert f.data[f.filter_index(V - 1, V + 2, 1, 2)] == g[V - 1, V + 2, 2, 1]


def _fwd_inputs(sp, V=8):
    sh = sp.ConvShape.make(2, 16, 16, 6, 6, 3, 3, 1, 1)
    D = O.gen_sparse(2, 16, 6, 6, 0.5, 1)
    G = O.gen_sparse(16, 16, 3, 3, 0.0, 2)
    return sh, sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)


def test_layout_and_plan_mismatches_rejected(sp):
    """test_kernels.cpp:328-352 -- rejected before any device work."""
    import dataclasses
    V = 8
    sh, a, b = _fwd_inputs(sp, V)
    pl = sp.plan(sh, sp.Component.fwd, V)
    E = sp.SpconvError
    with pytest.raises(E) as e:
        sp.sparse_fwd(a, dataclasses.replace(b, layout=sp.Layout.act_nchwc), sh, pl)
    assert e.value.status == sp._lib.SPC_ERR_LAYOUT
    with pytest.raises(E) as e:
        sp.sparse_fwd(dataclasses.replace(a, V=4), b, sh, pl)
    assert e.value.status == sp._lib.SPC_ERR_LAYOUT
    with pytest.raises(E) as e:
        sp.sparse_fwd(a, b, sh, sp.plan(sh, sp.Component.bwi, V))
    assert e.value.status == sp._lib.SPC_ERR_PLAN
    with pytest.raises(E) as e:
        sp.sparse_fwd(dataclasses.replace(a, data=a.data[:-1]), b, sh, pl)
    assert e.value.status == sp._lib.SPC_ERR_LAYOUT
    with pytest.raises(E) as e:
        sp.sparse_fwd(dataclasses.replace(a, h=5), b, sh, pl)
    assert e.value.status == sp._lib.SPC_ERR_LAYOUT
    with pytest.raises(E) as e:
        sp.sparse_fwd(a, b, sh, dataclasses.replace(pl, Q=24))
    assert e.value.status == sp._lib.SPC_ERR_PLAN
    with pytest.raises(E) as e:  # ring (R+pipe)*Q/V > 64
        sp.sparse_fwd(a, b, sp.ConvShape.make(2, 16, 256, 6, 6, 3, 3, 1, 1),
                      dataclasses.replace(pl, Q=256, pipelined=True))
    with pytest.raises(E):
        sp.sparse_fwd(a, b, sh, pl, workers=0)
    # bww: the checked tensor must be ActCHWNn
    D = O.gen_sparse(2, 16, 6, 6, 0.5, 1)
    dY = O.gen_sparse(2, 16, 6, 6, 0.0, 3)
    plw = sp.plan(sh, sp.Component.bww, V)
    with pytest.raises(E) as e:
        sp.sparse_bww(sp.pack_act_nchwc(D, V), sp.pack_act_nchwc(dY, V), sh, plw)
    assert e.value.status == sp._lib.SPC_ERR_LAYOUT
    # bwi wants the (C,K)-transposed filter dims
    with pytest.raises(E) as e:
        sp.sparse_bwi(a, sp.pack_filter(O.gen_sparse(16, 8, 3, 3, 0, 1), V),
                      sp.ConvShape.make(2, 8, 16, 6, 6, 3, 3, 1, 1),
                      sp.plan(sp.ConvShape.make(2, 8, 16, 6, 6, 3, 3, 1, 1), sp.Component.bwi, V))


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device path")
def test_no_device_fails_loudly(sp):
    sh, a, b = _fwd_inputs(sp)
    with pytest.raises(sp.SpconvError) as e:
        sp.sparse_fwd(a, b, sh, sp.plan(sh, sp.Component.fwd, 8))
    assert e.value.status == sp._lib.SPC_ERR_NO_DEVICE
    assert not sp.native_backend_available(16)


def test_math_mode_is_per_thread_and_validated(sp):
    """spc_set_math / spc_get_math (include/spconv_b200.h): FP32 by default,
    unknown modes rejected with the mode unchanged, per host thread."""
    import threading
    L = sp._lib.load()
    assert sp.get_math() == sp.Math.fp32
    assert L.spc_set_math(7) == -1 and sp.get_math() == sp.Math.fp32
    with sp.math_mode(sp.Math.tf32x3):
        assert sp.get_math() == sp.Math.tf32x3
        seen = []
        th = threading.Thread(target=lambda: seen.append(sp.get_math()))
        th.start()
        th.join()
        assert seen == [sp.Math.fp32]  # another host thread keeps its own mode
    assert sp.get_math() == sp.Math.fp32
    with pytest.raises(sp.SpconvError):
        sp.set_math(5)
