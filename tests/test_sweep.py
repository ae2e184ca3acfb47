"""The sweep harness (paper_1911_10175_b200/sweep.py) against the reference's
own harness (P/src/bench.cpp, P/src/projector.cpp) -- CPU parts: registry,
scaled shapes, the generator stream, CSV bytes and the projector's parser.
The timed GPU sweep is in test_gpu_sweep.py."""
import io

import numpy as np
import pytest

import oracle as O
from paper_1911_10175_b200 import sweep as S
from paper_1911_10175_b200.api import Component, RunMode, SpconvError

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built (oracle/_ref)")


@needs_ref
def test_registry_matches_reference():
    ref = O.ref_registry()
    mine = {lc.name: lc.shape.astuple() for lc in S.layer_registry()}
    assert set(ref) == set(mine) and len(mine) == 27
    for name, sh in ref.items():
        assert tuple(sh) == tuple(mine[name]), name
    assert S.find_layer("nope") is None


@needs_ref
@pytest.mark.parametrize("name", ["vgg1_2", "resnet2_2", "resnet2_1a", "resnet5_2/r", "resnet5_1b"])
@pytest.mark.parametrize("mb,scale", [(2, 8), (4, 2), (1, 64), (3, 1000), (16, 1)])
def test_scaled_shape_matches_reference(name, mb, scale):
    base = S.find_layer(name).shape
    assert S.scaled_shape(base, mb, scale).astuple() == O.ref_scaled_shape(base.astuple(), mb, scale)


def test_scaled_shape_rejects_bad_request():
    base = S.find_layer("resnet2_2").shape
    with pytest.raises(SpconvError):
        S.scaled_shape(base, 0, 2)
    with pytest.raises(SpconvError):
        S.scaled_shape(base, 2, 0)


@pytest.mark.parametrize("s,seed", [(0.0, 1), (0.5, 7), (0.9, 42), (1.0, 3)])
def test_gen_sparse_is_the_reference_stream(s, seed):
    mine = S.gen_sparse(2, 3, 5, 7, s, seed)
    assert np.array_equal(mine, O.gen_sparse(2, 3, 5, 7, s, seed))
    if O.ref_available():
        assert np.array_equal(mine, O.ref_gen_sparse(2, 3, 5, 7, s, seed))
    with pytest.raises(SpconvError):
        S.gen_sparse(1, 1, 1, 1, 1.5, 0)


def _records():
    R = S.BenchRecord
    return [
        R("resnet2_2", Component.fwd, 0.0, RunMode.dense, 1, 1234567.0, 9437184, 1.0),
        R("resnet2_2", Component.fwd, 0.5, RunMode.sparse, 1, 654321.5, 4718592, 1234567.0 / 654321.5),
        R("resnet2_2", Component.fwd, 0.9, RunMode.sparse, 1, 98765.4321, 943718, 1234567.0 / 98765.4321),
        R("resnet3_2/r", Component.bww, 0.0, RunMode.dense, 1, 1e6, 100, 1.0),
        R("resnet3_2/r", Component.bww, 0.3, RunMode.sparse, 1, 0.5e6, 70, 2.0),
        R("resnet3_2/r", Component.bww, 0.7, RunMode.sparse, 1, 0.25e6, 30, 4.0),
        R("geomean", Component.fwd, 0.5, RunMode.sparse, 1, 0.0, 0, 1.88679),
    ]


@needs_ref
def test_csv_bytes_match_reference_writers():
    recs = _records()
    a, b = io.StringIO(), io.StringIO()
    S.write_sweep_csv(recs, a)
    S.write_curves_csv(recs, b)
    ra, rb = O.ref_format_csv(recs)
    assert a.getvalue() == ra
    assert b.getvalue() == rb


@needs_ref
def test_reference_projector_parses_our_curves(tmp_path):
    p = tmp_path / "curves.csv"
    with open(p, "w") as f:
        S.write_curves_csv(_records(), f)
    assert O.ref_load_curves(p) == 2  # (resnet2_2, fwd) and (resnet3_2/r, bww)


def test_curves_need_a_dense_baseline():
    recs = [r for r in _records() if r.mode == RunMode.sparse]
    with pytest.raises(SpconvError):
        S.write_curves_csv(recs, io.StringIO())


def test_geo_mean_and_median():
    assert S.geo_mean([2.0, 8.0]) == pytest.approx(4.0)
    with pytest.raises(SpconvError):
        S.geo_mean([])
    with pytest.raises(SpconvError):
        S.geo_mean([1.0, 0.0])
    calls = []
    assert S.time_median_ns(lambda: calls.append(1), 5, 2) >= 0.0
    assert len(calls) == 7
    with pytest.raises(SpconvError):
        S.time_median_ns(lambda: None, 0, 0)
