"""CPU: on-disk formats around the hot path.

The product library's Matrix Market reader / writer and .cbfd block dumps
against (a) the compiled reference's own read_matrix_market /
write_matrix_market / BlockVector::save / load (oracle/_ref, this container),
(b) the numpy restatement oracle/formats.py and (c) committed golden files
the reference wrote (tests/golden/formats/, make_golden.py).  Integer / byte
work: everything bit-exact or byte-identical.
"""
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf
from oracle import formats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "formats")


def bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def same_csr(x, y):
    """(dim, offs, cols, vals, herm) tuples equal bit for bit"""
    return (x[0] == y[0] and np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2])
            and bits(x[3], y[3]) and x[4] == y[4])


def ref_csr(ref, path):
    m, herm = ref.read_matrix_market(path)
    c = m.csr()
    return m.dim, c.offs, c.cols, c.vals, herm


# hand-written files covering the reader's branches
CASES = {
    "general_real_dups.mtx": (
        "%%MatrixMarket matrix coordinate real general\n% a comment\n%\n"
        "4 4 7\n1 1 0.5\n2 1 -1.25\n1 2 3e-3\n4 4 1\n2 1 0.1\n4 4 1e-17\n3 2 -0.0\n"),
    "symmetric_integer.mtx": (
        "%%MatrixMarket matrix coordinate integer symmetric\n"
        "3 3 4\n1 1 2\n2 1 -1\n3 2 -1\n3 3 2\n"),
    "hermitian_complex.mtx": (
        "%%MatrixMarket matrix coordinate complex hermitian\n"
        "3 3 4\n1 1 1.5 0\n2 1 0.25 -0.75\n3 1 0 1\n3 3 -2 0\n"),
    "symmetric_complex_dup_diag.mtx": (  # complex symmetric: mirrored WITHOUT conjugation
        "%%MatrixMarket matrix coordinate complex symmetric\n"
        "2 2 3\n1 1 1 1\n2 1 0.5 0.5\n1 1 0.25 -1\n"),
    "uppercase_banner_blank_lines.mtx": (
        "%%MatrixMarket MATRIX Coordinate REAL General\n\n% c\n2 2 2\n\n1 2 7\n2 1 7\n"),
    "empty_rows.mtx": ("%%MatrixMarket matrix coordinate real general\n5 5 1\n3 3 1\n"),
    "zero_nnz.mtx": ("%%MatrixMarket matrix coordinate real symmetric\n3 3 0\n"),
}

BAD = {
    "no_banner.mtx": ("1 1 1\n1 1 1\n", ValueError, cf.NumericalError, "missing MatrixMarket banner"),
    "array.mtx": ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", ValueError,
                  cf.NumericalError, "only coordinate"),
    "skew.mtx": ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
                 ValueError, cf.NumericalError, "unsupported symmetry"),
    "pattern.mtx": ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n2 1\n", ValueError,
                    cf.NumericalError, "unsupported field"),
    "rect.mtx": ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", ValueError,
                 cf.NumericalError, "not square"),
    "short.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n",
                  ValueError, cf.NumericalError, "fewer entries"),
    "size_line.mtx": ("%%MatrixMarket matrix coordinate real general\nx y z\n", ValueError,
                      cf.NumericalError, "malformed size line"),
    "no_imag.mtx": ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1\n",
                    ValueError, cf.NumericalError, "missing imaginary part"),
    "no_value.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", ValueError,
                     cf.NumericalError, "missing value"),
    "range.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", IndexError,
                  cf.OutOfRange, "index out of range"),
    "zero_index.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n",
                       IndexError, cf.OutOfRange, "index out of range"),
}


@pytest.fixture
def case_files(tmp_path):
    paths = {}
    for name, text in CASES.items():
        p = tmp_path / name
        p.write_text(text)
        paths[name] = str(p)
    return paths


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_restatement(lib_built, case_files, name):
    got = cf.read_matrix_market(case_files[name])
    want = formats.read_matrix_market(case_files[name])
    assert same_csr(got, want)


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(lib_built, ref, case_files, name):
    got = cf.read_matrix_market(case_files[name])
    assert same_csr(got, ref_csr(ref, case_files[name]))


@pytest.mark.parametrize("name", sorted(BAD))
def test_reader_errors_match_reference(lib_built, tmp_path, name):
    text, orc_exc, our_exc, msg = BAD[name]
    p = tmp_path / name
    p.write_text(text)
    with pytest.raises(our_exc, match=msg):
        cf.read_matrix_market(str(p))
    with pytest.raises(orc_exc, match=msg):
        formats.read_matrix_market(str(p))


@pytest.mark.parametrize("name", sorted(BAD))
def test_reader_error_class_is_the_references(lib_built, ref, tmp_path, name):
    text, orc_exc, _, msg = BAD[name]
    p = tmp_path / name
    p.write_text(text)
    exc = IndexError if orc_exc is IndexError else RuntimeError  # oracle.Ref exception mapping
    with pytest.raises(exc, match=msg):
        ref.read_matrix_market(str(p))


def test_missing_file(lib_built, tmp_path):
    with pytest.raises(cf.NumericalError, match="cannot open"):
        cf.read_matrix_market(str(tmp_path / "nope.mtx"))


@pytest.mark.parametrize("model", ["graphene", "ti"])
@pytest.mark.parametrize("herm", [True, False])
def test_writer_is_byte_identical_to_reference(lib_built, ref, tmp_path, model, herm):
    m = (ref.graphene(5, 4, disorder=0.7, seed=3) if model == "graphene"
         else ref.topological_insulator(3, 2, 2, disorder=0.9, seed=8))
    c = m.csr()
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "theirs.mtx"
    cf.write_matrix_market(str(ours), m.dim, c.offs, c.cols, c.vals, hermitian=herm)
    ref.write_matrix_market(m, str(theirs), hermitian=herm)
    assert ours.read_bytes() == theirs.read_bytes()
    # write -> read is exact (17 digits), Hermitian storage expands back to full
    back = cf.read_matrix_market(str(ours))
    assert back[0] == m.dim and back[4] == herm
    assert np.array_equal(back[1], c.offs) and np.array_equal(back[2], c.cols)
    assert bits(back[3], c.vals)


def test_writer_round_trip_extreme_values(lib_built, tmp_path):
    vals = np.array([5e-324, -1.7976931348623157e308, 0.1, -0.0, 1 / 3, 2.0 ** -1074 * 3])
    offs = np.array([0, 2, 4, 6])
    cols = np.array([0, 2, 1, 2, 0, 2])
    p = tmp_path / "x.mtx"
    cf.write_matrix_market(str(p), 3, offs, cols, vals, hermitian=False)
    d, o, c, v, h = cf.read_matrix_market(str(p))
    assert d == 3 and not h and np.array_equal(o, offs) and np.array_equal(c, cols)
    # exact, except that -0.0 reads back as +0.0: the Builder sums from S{} = +0.0
    # (sparse_matrix.hpp:64), as the reference's own round trip does
    assert bits(v, vals + 0.0)


def test_writer_rejects_inconsistent_csr(lib_built, tmp_path):
    with pytest.raises(cf.InvalidArgument):
        cf.write_matrix_market(str(tmp_path / "x.mtx"), 3, [0, 1, 2], [0, 1], [1.0, 2.0])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("shape", [(7, 3), (1, 1), (0, 4), (33, 0)])
def test_cbfd_bytes_match_reference(lib_built, ref, tmp_path, cplx, shape):
    rng = np.random.default_rng(1)
    a = rng.standard_normal(shape)
    if cplx:
        a = a + 1j * rng.standard_normal(shape)
    ours, theirs = tmp_path / "ours.cbfd", tmp_path / "theirs.cbfd"
    cf.save_block(str(ours), a)
    ref.block_save(a, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes() == formats.cbfd_bytes(a)
    assert bits(cf.load_block(str(theirs)), a)
    assert bits(ref.block_load(str(ours), cplx), a)


def test_cbfd_errors(lib_built, ref, tmp_path):
    a = np.arange(12.0).reshape(4, 3)
    good = formats.cbfd_bytes(a)
    cases = {
        "bad_magic": (b"XXXX" + good[4:], "bad header"),
        "short_header": (good[:10], "bad header"),
        "truncated": (good[:-8], "truncated payload"),
        "bad_kind": (good[:16] + (7).to_bytes(4, "little") + good[20:], "kind mismatch"),
    }
    for name, (raw, msg) in cases.items():
        p = tmp_path / name
        p.write_bytes(raw)
        with pytest.raises(cf.NumericalError, match=msg):
            cf.load_block(str(p))
        with pytest.raises(RuntimeError, match=msg):
            ref.block_load(str(p), False)
    # the reference's typed load: a real file read as complex is a kind mismatch
    p = tmp_path / "real.cbfd"
    p.write_bytes(good)
    with pytest.raises(RuntimeError, match="kind mismatch"):
        ref.block_load(str(p), True)
    with pytest.raises(cf.NumericalError, match="cannot open"):
        cf.load_block(str(tmp_path / "missing.cbfd"))


def test_golden_files_written_by_reference(lib_built):
    """Files the compiled reference wrote (make_golden.py) read back through
    the product reader / loader, against the restatement."""
    names = sorted(os.listdir(GOLDEN))
    assert any(n.endswith(".mtx") for n in names) and any(n.endswith(".cbfd") for n in names)
    for n in names:
        p = os.path.join(GOLDEN, n)
        if n.endswith(".mtx"):
            assert same_csr(cf.read_matrix_market(p), formats.read_matrix_market(p)), n
        elif n.endswith(".cbfd"):
            assert bits(cf.load_block(p), formats.parse_cbfd(open(p, "rb").read())), n
