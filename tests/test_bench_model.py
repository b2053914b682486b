"""bench.py's counting conventions (CPU): the flop model equals the compiled reference's
bench_filter numbers (tests/golden/bench_filter.json, bench.cpp:28-30,116), and the
minimal-schedule byte count (api.filter_schedule_bytes) follows the step kinds
apply_filter launches (capi.cu enqueue_filter)."""
import json
import os

import pytest

import bench
import paper_1510_04895_b200 as cf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bench_filter.json")


@pytest.mark.parametrize("name", ["graphene_32x32", "ti_4x4x4"])
def test_model_flops_match_reference_golden(name):
    g = json.load(open(GOLDEN))[name]
    if name.startswith("graphene"):
        o, c, v = cf.csr_graphene(cf.LatticeSpec(32, 32, disorder=0.2, seed=3))
        cplx = False
    else:
        o, c, v = cf.csr_topological_insulator(cf.LatticeSpec(4, 4, 4, disorder=0.5, seed=2))
        cplx = True
    dim, nnz = len(o) - 1, len(c)
    for nb, flops in zip(g["sizes"], g["flops"]):
        assert bench.model_flops(dim, nnz, nb, g["degree"], cplx) == pytest.approx(flops, rel=1e-15)


def test_schedule_bytes_follow_the_step_kinds():
    D, nnz, nb = 1000, 11000, 8
    mat, blk = nnz * 20, D * nb * 16
    # degree 2: spmmvm (2 streams) + start-up step 2 (4 streams)
    assert cf.filter_schedule_bytes(D, nnz, nb, True, 2) == 2 * mat + 6 * blk
    # degree 5: + one triple (two V_n-only steps of 3 streams, one X step of 5)
    assert cf.filter_schedule_bytes(D, nnz, nb, True, 5) == 5 * mat + 6 * blk + 11 * blk
    # degree 6: + a single fused step (5 streams) for the tail
    assert cf.filter_schedule_bytes(D, nnz, nb, True, 6) == 6 * mat + 6 * blk + 16 * blk
    # group 1 (X every step): every fused step moves the reference's 5 streams
    assert (cf.filter_schedule_bytes(D, nnz, nb, True, 100, group=1)
            == 2 * mat + 6 * blk + 98 * bench.model_step_bytes(D, nnz, nb))
    assert bench.recur_step_bytes(D, nnz, nb) == mat + 3 * blk
