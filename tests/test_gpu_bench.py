"""GPU: the bench front end -- bench_filter's protocol and
report (bench.cpp:71-126) and the read-only bandwidth probe (bench.cpp:44-67)
on HBM.  Model fields (flops, intensity, roofline) are bit-identical to the
compiled reference's on the same matrices (tests/golden/bench_filter.json);
timing fields obey the reference's definitions."""
import json
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bench_filter.json")


@pytest.mark.parametrize("name", ["graphene_32x32", "ti_4x4x4"])
def test_bench_filter_model_fields_match_reference(ctx, name):
    g = json.load(open(GOLDEN))[name]
    if name.startswith("graphene"):
        A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(32, 32, disorder=0.2, seed=3))
    else:
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(4, 4, 4, disorder=0.5,
                                                                      seed=2))
    rep = cf.bench_filter(A, g["sizes"], g["degree"], g["bandwidth"])
    assert rep.bandwidth_gbs == g["bandwidth"] and rep.degree == 16 and rep.dim == A.dim()
    assert [p.n_b for p in rep.points] == g["sizes"]
    assert [p.flops for p in rep.points] == g["flops"]
    assert [p.intensity for p in rep.points] == g["intensity"]
    assert [p.roofline for p in rep.points] == g["roofline"]
    for p in rep.points:
        assert p.seconds > 0
        assert p.gflops == p.flops / p.seconds / 1e9
        assert p.efficiency == p.gflops / p.roofline
        traffic = (A.nnz() / A.dim() / p.n_b * ((16 if A.kind else 8) + 4)
                   + 5.0 * (16 if A.kind else 8)) * A.dim() * p.n_b * 16
        assert abs(p.gbs_proxy - traffic / p.seconds / 1e9) <= 1e-12 * p.gbs_proxy
    j = rep.to_json()
    assert set(j) == {"bandwidth_gbs", "degree", "dim", "traffic_overhead", "points"}
    assert set(j["points"][0]) == {"n_b", "seconds", "flops", "gflops", "gbs_proxy", "intensity",
                                   "roofline_gflops", "efficiency"}
    assert "n_b" in rep.table()


def test_bench_filter_errors(ctx):
    """bench.cpp:74-75,89"""
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(8, 8))
    with pytest.raises(cf.InvalidArgument, match="degree"):
        cf.bench_filter(A, [1], 15, 100.0)
    with pytest.raises(cf.InvalidArgument, match="empty"):
        cf.bench_filter(A, [], 16, 100.0)
    with pytest.raises(cf.InvalidArgument, match="block size"):
        cf.bench_filter(A, [2, 0], 16, 100.0)


def test_bandwidth_probe_on_hbm(ctx):
    lo = cf.bandwidth_probe_min_bytes(ctx)
    assert lo >= 8 * 100 * 2**20  # 8 x the ~126 MB L2
    with pytest.raises(cf.InvalidArgument, match="8x"):
        cf.bandwidth_probe(ctx, lo - 1)
    b = cf.bandwidth_probe(ctx, lo, 5)
    # HBM3e read stream on B200: several TB/s, below the 8 TB/s spec
    assert 3000.0 < b < 8200.0, b


def test_bench_filter_probes_when_no_bandwidth_given(ctx):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1))
    rep = cf.bench_filter(A, [4], 16)
    assert 3000.0 < rep.bandwidth_gbs < 8200.0
    p = rep.points[0]
    assert np.isclose(p.roofline, p.intensity * rep.bandwidth_gbs, rtol=0, atol=0)
