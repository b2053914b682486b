"""CPU: the product library (libchebfd_b200.so) without a GPU.

* it loads and exports every function include/chebfd_b200.h declares;
* its host-side pieces (stencil-direct lattice generators, filter
  coefficients, DOS counts, lattice partition planning) agree with the
  oracle bit for bit;
* device entry points fail loudly (CudaError) instead of falling back.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1510_04895_b200 as cf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chebfd_b200.h")


def bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(chebfd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib_built):
    lib = C.CDLL(lib_built)
    names = declared_functions()
    assert len(names) >= 55
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    from paper_1510_04895_b200 import _lib
    assert sorted(set(names) - set(_lib.EXPORTED)) == []


def test_cpp_wrapper_header_compiles(lib_built, tmp_path):
    """include/chebfd_b200.hpp (the reference-signature C++ layer) builds and
    links against the library."""
    src = tmp_path / "use.cpp"
    src.write_text(open(os.path.join(ROOT, "tests", "cpp", "use_wrapper.cpp")).read())
    out = tmp_path / "use"
    import subprocess
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src),
                        "-o", str(out), f"-L{os.path.dirname(lib_built)}", "-lchebfd_b200",
                        f"-Wl,-rpath,{os.path.dirname(lib_built)}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    run = subprocess.run([str(out), "--host-only", str(tmp_path)], capture_output=True, text=True)
    assert run.returncode == 0, run.stdout + run.stderr


@pytest.mark.parametrize("boundary", ["periodic_xy_open_z", "periodic_all", "open_all"])
@pytest.mark.parametrize("l", [(3, 3, 3), (1, 2, 3), (2, 2, 2), (4, 3, 2), (1, 1, 1), (2, 1, 5)])
def test_ti_generator_bitexact(orc, boundary, l):
    spec = cf.LatticeSpec(*l, disorder=0.5, boundary=boundary, seed=5)
    offs, cols, vals = cf.csr_topological_insulator(spec)
    t = orc.topological_insulator(*l, disorder=0.5, boundary=boundary, seed=5)
    assert np.array_equal(offs, t.offs) and np.array_equal(cols, t.cols) and bits(vals, t.vals)
    d = t.dim
    r0, r1 = d // 3, 2 * d // 3 + 1
    o2, c2, v2 = cf.csr_topological_insulator(spec, r0, r1)
    assert np.array_equal(o2, t.offs[r0:r1 + 1] - t.offs[r0])
    assert np.array_equal(c2, t.cols[t.offs[r0]:t.offs[r1]])
    assert bits(v2, t.vals[t.offs[r0]:t.offs[r1]])


@pytest.mark.parametrize("boundary", ["periodic_xy_open_z", "open_all"])
@pytest.mark.parametrize("l", [(1, 1), (1, 2), (2, 2), (3, 5), (8, 8), (64, 64)])
def test_graphene_generator_bitexact(orc, boundary, l):
    spec = cf.LatticeSpec(l[0], l[1], disorder=0.1, boundary=boundary, seed=1)
    offs, cols, vals = cf.csr_graphene(spec)
    g = orc.graphene(*l, disorder=0.1, boundary=boundary, seed=1)
    assert np.array_equal(offs, g.offs) and np.array_equal(cols, g.cols) and bits(vals, g.vals)


def test_generator_at_bench_scale_matches_oracle(orc):
    """TI 64^3 slab, V = 0.5, seed 1 (BASELINE configs[1], C2): the library's
    stencil-direct generator against the oracle's Builder-equivalent restatement
    (models.cpp:80-140) on the whole 1,048,576-row operator, bit for bit, plus a
    rank-style row range from its middle."""
    spec = cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1)
    o, c, v = cf.csr_topological_insulator(spec)
    t = orc.topological_insulator(64, 64, 64, disorder=0.5, seed=1)
    assert t.dim == 1048576 and len(c) == 11517952
    assert np.array_equal(o, t.offs) and np.array_equal(c, t.cols) and bits(v, t.vals)
    r0, r1 = 499968, 500352
    o2, c2, v2 = cf.csr_topological_insulator(spec, r0, r1)
    assert np.array_equal(o2, t.offs[r0:r1 + 1] - t.offs[r0])
    assert np.array_equal(c2, t.cols[t.offs[r0]:t.offs[r1]])
    assert bits(v2, t.vals[t.offs[r0]:t.offs[r1]])


@pytest.mark.parametrize("k", ["none", "fejer", "jackson", "lanczos2", "lanczos3"])
def test_filter_coefficients_bitexact(orc, k):
    p = cf.make_filter((-0.1, 0.2), (-1.1, 1.3), 57, k)
    comb, a, b = orc.make_filter((-0.1, 0.2), (-1.1, 1.3), 57, k)
    assert bits(p.combined, comb) and p.alpha == a and p.beta == b
    assert bits(cf.window_coeffs((-0.1, 0.2), (-1.1, 1.3), 57),
                orc.window_coeffs((-0.1, 0.2), (-1.1, 1.3), 57))
    assert bits(cf.kernel_coeffs(k, 57), orc.kernel_coeffs(k, 57))
    for x in (-1.1, -0.3, 0.0, 0.15, 1.3):
        assert cf.eval_scalar(p, x) == orc.eval_scalar(comb, a, b, x)


def test_filter_errors_map_to_reference_exceptions():
    with pytest.raises(cf.InvalidArgument):  # filter.cpp:14-16
        cf.make_filter((0.5, 0.1), (-1, 1), 10)
    with pytest.raises(cf.InvalidArgument):
        cf.make_filter((-2.0, 0.1), (-1, 1), 10)
    with pytest.raises(cf.InvalidArgument):  # lanczos mu >= 1
        cf.Kernel.parse("lanczos0")
    with pytest.raises(cf.InvalidArgument):
        cf.Kernel.parse("boxcar")
    p = cf.make_filter((-0.5, 0.5), (-1.0, 1.0), 8)
    with pytest.raises(cf.DomainError):  # filter.cpp:102-103
        cf.eval_scalar(p, 1.0001)
    with pytest.raises(cf.InvalidArgument):  # LatticeSpec::validate
        cf.csr_topological_insulator(cf.LatticeSpec(0, 1, 1))
    with pytest.raises(cf.InvalidArgument):
        cf.csr_graphene(cf.LatticeSpec(2, 2, disorder=-1.0))
    for s in ("none", "fejer", "jackson", "lanczos2", "lanczos3"):  # test_filter.cpp:77-81
        assert cf.Kernel.parse(s).name() == s


def test_dos_count_matches_reference(ref):
    m = ref.diag_flat(1000, -1.0, 1.0)
    mu = ref.kpm_dos(m, (-1.05, 1.05), 500, 8, 3)
    dos = cf.DosEstimate(mu, cf.Interval(-1.05, 1.05))
    for lo, hi in ((-0.8, -0.6), (-0.2, 0.0), (0.1, 0.9), (-1.05, 1.05)):
        assert abs(dos.count(lo, hi) - ref.dos_count(mu, (-1.05, 1.05), lo, hi)) <= 1e-9


def test_intensity_model_matches_reference(ref):
    for args in ((13.0, 16, 4, 2, 6, 1), (10.98, 16, 4, 2, 6, 32), (4.0, 8, 4, 1, 1, 16)):
        assert abs(cf.intensity_model(*args) - ref.intensity_model(*args)) <= 1e-15


def test_device_calls_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(cf.CudaError):
        cf.Context(0)


@pytest.mark.parametrize("cplx", [False, True])
def test_parallel_randomize_is_the_reference_stream(orc, cplx):
    """chebfd_host_randomize (mt19937_64 jump-ahead + parallel polar method)
    must equal the serial libstdc++ stream bit for bit, across chunk
    boundaries and for row slices (distributed blocks)."""
    dim, w = (1 << 20, 9) if not cplx else (1 << 19, 9)   # >= 2^23 normals: parallel path
    full = orc.randomize(dim, w, 7, cplx)
    assert bits(cf.host_randomize(dim, w, 7, cplx), full)
    for r0, n in ((12345, 1000), (dim // 2 + 1, 777), (dim - 3, 3)):
        assert bits(cf.host_randomize(dim, w, 7, cplx, r0, n), full[r0:r0 + n])


def test_partition_plans_cover_rows_and_pair_up():
    spec = cf.LatticeSpec(4, 4, 8, disorder=0.5)
    for nranks in (1, 2, 3, 4):
        plans = [cf.plan_partition(spec, "ti", r, nranks) for r in range(nranks)]
        assert plans[0].row_begin == 0
        assert sum(p.local_rows for p in plans) == 4 * 4 * 4 * 8
        for r in range(1, nranks):
            assert plans[r].row_begin == plans[r - 1].row_begin + plans[r - 1].local_rows
            assert plans[r].row_begin % (4 * 4 * 4) == 0  # z-plane boundaries
        cf.plan_complete_sends(plans)
        for r, p in enumerate(plans):
            if p.hi_rank >= 0:
                q = plans[p.hi_rank]
                assert q.lo_rank == r and q.halo_lo == p.send_hi_n
            if p.lo_rank >= 0:
                q = plans[p.lo_rank]
                assert q.hi_rank == r and q.halo_hi == p.send_lo_n
        # open z: the end ranks have a single neighbour
        if nranks > 1:
            assert plans[0].lo_rank == -1 and plans[-1].hi_rank == -1


def test_python_option_codes_match_header():
    """Context.set_option's names map to the CHEBFD_OPT_* values of the C header."""
    text = open(HEADER).read()
    enum = {m.group(1).lower(): int(m.group(2))
            for m in re.finditer(r"CHEBFD_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", text)}
    import inspect
    from paper_1510_04895_b200 import api
    src = inspect.getsource(api.Context.set_option)
    codes = dict(re.findall(r'"([a-z_0-9]+)": (\d+)', src.split("}[name]")[0]))
    assert codes, "no option table found"
    for name, code in codes.items():
        assert enum.get(name) == int(code), (name, code, enum.get(name))
