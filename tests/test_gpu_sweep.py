"""GPU sweep harness vs the reference's (P/tests/test_bench.cpp:123-199,
P/src/bench.cpp:215-327): same record structure, same CSV columns, and the
non-timing columns (layer, component, sparsity, mode, workers, exec_fmas)
identical to the reference's own run_sweep on the same request."""
import csv
import io

import pytest

import oracle as O
from paper_1911_10175_b200 import sweep as S
from paper_1911_10175_b200.api import Component, RunMode

pytestmark = pytest.mark.gpu


def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def test_sweep_emits_records_baselines_and_geomean():
    req = S.SweepRequest(layers=["resnet2_2", "resnet3_2"], comps=[Component.fwd, Component.bww], grid=[0.0, 0.9],
                         minibatch=2, scale=8, repeats=1)
    recs = S.run_sweep(req)
    dense = [r for r in recs if r.layer != "geomean" and r.mode == RunMode.dense]
    sparse = [r for r in recs if r.layer != "geomean" and r.mode == RunMode.sparse]
    summary = [r for r in recs if r.layer == "geomean"]
    assert (len(dense), len(sparse), len(summary)) == (4, 8, 4)
    assert all(r.speedup_vs_dense == 1.0 for r in dense)
    assert all(r.median_ns > 0.0 for r in sparse)
    for s in summary:
        vals = [r.speedup_vs_dense for r in sparse if r.comp == s.comp and r.sparsity == s.sparsity]
        assert s.speedup_vs_dense == pytest.approx(S.geo_mean(vals))
    a, b = io.StringIO(), io.StringIO()
    S.write_sweep_csv(recs, a)
    S.write_curves_csv(recs, b)
    la, lb = a.getvalue().splitlines(), b.getvalue().splitlines()
    assert la[0] == "layer,component,sparsity,mode,workers,median_ns,exec_fmas,speedup_vs_dense"
    assert len(la) - 1 == len(recs)
    assert lb[0] == "layer,component,sparsity,median_ns,dense_ns"
    assert len(lb) - 1 == len(sparse)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built (oracle/_ref)")
@pytest.mark.parametrize("timing", ["device", "host"])
def test_sweep_non_timing_columns_equal_reference_sweep(timing, tmp_path):
    layers = ["resnet2_2", "resnet3_2/r", "resnet2_1a", "vgg5_1"]
    comps = [Component.fwd, Component.bwi, Component.bww]
    grid = [0.0, 0.3, 0.8]
    req = S.SweepRequest(layers=layers, comps=comps, grid=grid, minibatch=3, scale=4, repeats=1, seed=42,
                         timing=timing)
    recs = S.run_sweep(req)
    mine = io.StringIO()
    S.write_sweep_csv(recs, mine)
    ref_sweep, _ = O.ref_run_sweep(layers, comps, grid, 3, 4, 42, repeats=1)
    ra, rb = _rows(mine.getvalue()), _rows(ref_sweep)
    assert len(ra) == len(rb)
    for x, y in zip(ra, rb):
        for col in ("layer", "component", "sparsity", "mode", "workers", "exec_fmas"):
            assert x[col] == y[col], (col, x, y)
    # our curves load in the reference projector
    p = tmp_path / "curves.csv"
    with open(p, "w") as f:
        S.write_curves_csv(recs, f)
    assert O.ref_load_curves(p) == len(layers) * len(comps)


def test_sweep_non_timing_columns_deterministic_per_seed():
    req = S.SweepRequest(layers=["resnet2_2"], comps=[Component.fwd], grid=[0.3, 0.8], minibatch=2, scale=8,
                         repeats=1, seed=42)
    a, b = S.run_sweep(req), S.run_sweep(req)
    assert [(r.layer, r.comp, r.sparsity, r.mode, r.workers, r.exec_fmas) for r in a] == \
        [(r.layer, r.comp, r.sparsity, r.mode, r.workers, r.exec_fmas) for r in b]


def test_sweep_cli_writes_both_csvs(tmp_path):
    sw, cu = tmp_path / "sweep.csv", tmp_path / "curves.csv"
    assert S.main(["--layers", "resnet2_2", "--comps", "fwd", "bww", "--grid", "0.5", "0.9", "--minibatch", "2",
                   "--scale", "8", "--repeats", "1", "--csv", str(sw), "--curves", str(cu)]) == 0
    assert len(open(sw).read().splitlines()) == 1 + 2 * 3 + 2 * 2  # + geomean per (comp, s)
    assert len(open(cu).read().splitlines()) == 1 + 2 * 2
