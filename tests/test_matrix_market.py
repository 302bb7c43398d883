"""Matrix Market input at the boundary (paper_0901_2665_b200/matrix_market.py) against the
reference's own reader (matrix_market.cpp run as oracle/_ref/ref_mm_dump): the same CSR arrays bit
for bit on accepted files, the same InputError message on rejected ones, and save -> load round
trips (the reference's tests round-trip the same way)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_0901_2665_b200 import feast as F
from paper_0901_2665_b200 import matrix_market as MM
from paper_0901_2665_b200.problems import Operator, banded_csr

needs_ref = pytest.mark.skipif(not O.available("mm"), reason="oracle/_ref/ref_mm_dump not built")

BANNER = "%%MatrixMarket matrix coordinate real symmetric\n"

GOOD = {
    "plain": BANNER + "3 3 4\n1 1 2.0\n2 1 -1\n2 2 2\n3 3 1.5e-3\n",
    "comments_blanks": BANNER + "% a comment\n\n3 3 3\n% inside\n1 1 1\n\n3 1 0.25\n2 2 -7\n",
    "duplicates": BANNER + "2 2 4\n1 1 0.1\n1 1 0.2\n2 1 0.3\n2 1 0.4\n",
    "both_triangles": BANNER + "2 2 3\n1 2 5\n2 1 5\n2 2 1\n",   # mirrored twice: summed to 10
    "negative_zero": BANNER + "2 2 2\n1 1 -0\n2 2 1\n",
    "case_banner": "%%MatrixMarket MATRIX Coordinate REAL Symmetric\n1 1 1\n1 1 3\n",
    "no_trailing_newline": BANNER + "1 1 1\n1 1 3",
    # istream extraction takes the longest numeric prefix: '1.5d0' reads as 1.5
    "fortran_exponent_prefix": BANNER + "2 2 2\n1 1 1.5d0\n2 2 2\n",
    "signs_and_dots": BANNER + "2 2 3\n+1 +1 +.5\n2 1 -3.\n2 2 1e+2\n",
    "underscore_digits": BANNER + "2 2 1\n1 1 1_0\n",   # reads 1 (Python's float() says 10)
    "crlf": BANNER.replace("\n", "\r\n") + "2 2 2\r\n1 1 1\r\n2 2 4\r\n",
}

BAD = {
    "empty": "",
    "banner": "%MatrixMarket matrix coordinate real symmetric\n1 1 0\n",
    "object": "%%MatrixMarket vector coordinate real symmetric\n1 1 0\n",
    "format": "%%MatrixMarket matrix array real symmetric\n1 1 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "complex": "%%MatrixMarket matrix coordinate complex hermitian\n1 1 1\n1 1 1 0\n",
    "complex_missing_im": "%%MatrixMarket matrix coordinate complex hermitian\n1 1 1\n1 1 1\n",
    "no_size": BANNER + "% only comments\n",
    "bad_size": BANNER + "3 x 3\n",
    "not_square": BANNER + "3 4 0\n",
    "zero_dim": BANNER + "0 0 0\n",
    "negative_count": BANNER + "2 2 -1\n",
    "eof": BANNER + "2 2 3\n1 1 1\n",
    "malformed_entry": BANNER + "2 2 1\n1 one 1\n",
    "index_range": BANNER + "2 2 1\n3 1 1\n",
    "index_zero": BANNER + "2 2 1\n0 1 1\n",
    # what Python's int()/float() accept but C++ stream extraction rejects
    "nan_value": BANNER + "2 2 1\n1 1 nan\n",
    "inf_value": BANNER + "2 2 1\n1 1 inf\n",
    "incomplete_exponent": BANNER + "2 2 1\n1 1 1e\n",
    "overflow_value": BANNER + "2 2 1\n1 1 1e999\n",
    "float_size_line": BANNER + "2.0 2 1\n1 1 1\n",
    # a CRLF blank line is "\r": not empty for std::getline, so a malformed entry
    "crlf_blank_line": BANNER.replace("\n", "\r\n") + "2 2 1\r\n\r\n1 1 1\r\n",
}


def write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_text(text)
    return str(p)


@needs_ref
@pytest.mark.parametrize("name", sorted(GOOD))
def test_accepted_files_match_reference(tmp_path, name):
    p = write(tmp_path, name, GOOD[name])
    n, rp, ci, v = O.mm_load_reference(p)
    op = MM.load_matrix_market_real(p)
    assert op.n == n
    assert np.array_equal(op.row_ptr, rp) and np.array_equal(op.col_idx, ci)
    assert np.array_equal(op.values.view(np.int64), v.view(np.int64))  # bit for bit (signed zeros too)


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_rejected_files_match_reference(tmp_path, name):
    p = write(tmp_path, name, BAD[name])
    with pytest.raises(O.ReferenceInputError) as ref:
        O.mm_load_reference(p)
    with pytest.raises(F.InputError) as mine:
        MM.load_matrix_market_real(p)
    assert str(mine.value) == str(ref.value)


@needs_ref
def test_missing_file_and_both_triangles_disagreeing(tmp_path):
    p = str(tmp_path / "absent.mtx")
    with pytest.raises(O.ReferenceInputError) as ref:
        O.mm_load_reference(p)
    with pytest.raises(F.InputError) as mine:
        MM.load_matrix_market_real(p)
    assert str(mine.value) == str(ref.value)
    # (1,2) = 5 and (2,1) = 4 are each mirrored and summed: 9 on both sides, no error
    p = write(tmp_path, "both", BANNER + "2 2 2\n1 2 5\n2 1 4\n")
    n, rp, ci, v = O.mm_load_reference(p)
    op = MM.load_matrix_market_real(p)
    assert np.array_equal(op.values, v) and np.array_equal(v, [9.0, 9.0])


@needs_ref
def test_generated_banded_pencil_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    n = 700
    a = banded_csr(n, rng.uniform(-2, 2, n), {d: rng.standard_normal(n - d) for d in (1, 2, 5, 9)})
    p = str(tmp_path / "a.mtx")
    MM.save_matrix_market(p, a)
    back = MM.load_matrix_market_real(p)
    assert np.array_equal(back.row_ptr, a.row_ptr) and np.array_equal(back.col_idx, a.col_idx)
    assert np.array_equal(back.values, a.values)
    n2, rp, ci, v = O.mm_load_reference(p)
    assert n2 == n and np.array_equal(rp, a.row_ptr) and np.array_equal(ci, a.col_idx)
    assert np.array_equal(v, a.values)


def test_dense_and_blocktri_writers(tmp_path):
    rng = np.random.default_rng(1)
    m = rng.standard_normal((32, 32))
    m = m + m.T
    m[np.abs(m) < 0.5] = 0.0
    p = str(tmp_path / "d.mtx")
    MM.save_matrix_market(p, Operator.from_dense(m))
    back = MM.load_matrix_market_real(p)
    dense = np.zeros((32, 32))
    for i in range(32):
        for k in range(back.row_ptr[i], back.row_ptr[i + 1]):
            dense[i, back.col_idx[k]] = back.values[k]
    assert np.array_equal(dense, m)
    diag = np.stack([m[l * 8:(l + 1) * 8, l * 8:(l + 1) * 8] for l in range(4)])
    low = np.stack([m[(l + 1) * 8:(l + 2) * 8, l * 8:(l + 1) * 8] for l in range(3)])
    bt = Operator.from_blocktri(diag, low)
    MM.save_matrix_market(p, bt)
    back = MM.load_matrix_market_real(p)
    want = np.zeros_like(m)
    for l in range(4):
        want[l * 8:(l + 1) * 8, l * 8:(l + 1) * 8] = diag[l]
    for l in range(3):
        want[(l + 1) * 8:(l + 2) * 8, l * 8:(l + 1) * 8] = low[l]
        want[l * 8:(l + 1) * 8, (l + 1) * 8:(l + 2) * 8] = low[l].T
    got = np.zeros_like(m)
    for i in range(32):
        for k in range(back.row_ptr[i], back.row_ptr[i + 1]):
            got[i, back.col_idx[k]] = back.values[k]
    assert np.array_equal(got, want)


def test_triplet_assembly_errors():
    with pytest.raises(F.InputError, match="dimension must be positive"):
        MM.operator_from_triplets(0, [], [], [])
    with pytest.raises(F.InputError, match="triplet index out of range"):
        MM.operator_from_triplets(2, [0], [2], [1.0])
    with pytest.raises(F.InputError, match="missing mirror entry"):
        MM.operator_from_triplets(2, [0], [1], [1.0], mirror_off_diagonal=False)
