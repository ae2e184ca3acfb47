"""CPU tests of the BASELINE workload generators (workloads.py), the layer
tables, the batch-shard plan and the reference arm's isolation from the
product library (bench.py --impl reference must not load libspconv_b200)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1911_10175_b200 import workloads as wl
from paper_1911_10175_b200.dist import ShardPlan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_layer_tables_match_the_baseline_configs():
    counts = {k: len(f()) for k, f in wl.SPECS.items()}
    assert counts == {"cfg1_single3x3_b16": 1, "vgg16_b32": 12, "resnet34_b64": 35, "resnet50_b64": 52,
                      "fixup_resnet50_b256": 52}
    assert {t[1] for t in wl.SPECS["vgg16_b32"]()} == {32}
    assert {t[1] for t in wl.SPECS["fixup_resnet50_b256"]()} == {256}
    r34 = wl.SPECS["resnet34_b64"]()
    assert sum(1 for t in r34 if t[5] == 1) == 3 and all(t[6] == 2 for t in r34 if t[5] == 1)  # 1x1 s2 projections
    r50 = wl.SPECS["resnet50_b64"]()
    assert sum(1 for t in r50 if t[5] == 3 and t[6] == 2) == 3  # stride 2 on the first 3x3 of stages 2-4


def test_generators_are_seeded_and_follow_the_config_distributions():
    sh = wl.PlainShape((2, 32, 48, 14, 14, 3, 3, 1, 1, 1, 1))
    a = wl.layer_inputs_host("vgg16_b32", 3, sh, 0.8)
    b = wl.layer_inputs_host("vgg16_b32", 3, sh, 0.8)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    D, G, dY = a
    assert abs((D == 0).mean() - 0.8) < 0.02 and abs((dY == 0).mean() - 0.8) < 0.02
    assert (D >= 0).all() and G.shape == (48, 32, 3, 3)
    assert abs(G.std() - np.sqrt(2.0 / (32 * 9))) < 0.01
    # cfg 1: fixed 50 % (no grid); cfg 3: per-layer U[0.4, 0.8]; BatchNorm nets: dense dY
    assert wl.layer_sparsity("cfg1_single3x3_b16", 0, None) == 0.5
    s34 = [wl.layer_sparsity("resnet34_b64", i) for i in range(35)]
    assert 0.4 <= min(s34) and max(s34) <= 0.8 and len(set(s34)) == 35
    D3, _, dY3 = wl.layer_inputs_host("resnet34_b64", 5, sh)
    assert abs((D3 == 0).mean() - s34[5]) < 0.03 and (dY3 == 0).mean() < 1e-4


def test_resnet50_inputs_are_spatially_correlated_at_mean_06():
    sh = wl.PlainShape((2, 16, 16, 28, 28, 3, 3, 1, 1, 1, 1))
    D, _, dY = wl.layer_inputs_host("resnet50_b64", 1, sh)
    z = D == 0
    assert abs(z.mean() - 0.6) < 0.03
    # a zero's right neighbour is zero more often than chance (ReLU of a 3x3 conv of noise)
    p_joint = (z[..., :, 1:] & z[..., :, :-1]).mean()
    assert p_joint > z.mean() ** 2 + 0.05
    assert (dY == 0).mean() < 1e-4


def test_shard_plan_slices_the_global_nchwc_tensor_without_copies():
    import paper_1911_10175_b200 as sp
    x = np.random.default_rng(0).standard_normal((7, 32, 5, 6)).astype(np.float32)
    g = sp.pack_act_nchwc(x, 16)
    got = []
    for r in range(3):
        p = ShardPlan(7, 3, r)
        t = p.slice_nchwc(g)
        assert np.shares_memory(t.data, g.data) and t.n == p.count
        got.append(sp.unpack(t))
    assert np.array_equal(np.concatenate(got), x)
    with pytest.raises(Exception):
        ShardPlan(7, 3, 0).slice_nchwc(sp.pack_act_nchwc(x[:3], 16))


def test_reference_arm_never_loads_the_product_library():
    code = r"""
import sys, json
sys.argv = ["bench.py"]
sys.path.insert(0, %r)
import bench
layers = bench.ref_layers("vgg16_b32", 1)
maps = open("/proc/self/maps").read()
bench.emit({"n": len(layers), "loaded": "libspconv_b200" in maps, "N": layers[0][1].N})
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out == {"n": 12, "loaded": False, "N": 1}
