"""Matrix Market I/O (csrc/cvk_mmio.cu, mmio.py) against the reference's
reader (restated in the oracle) and its golden system.mtx, on CPU."""
import os

import numpy as np
import pytest

from conftest import GOLDEN


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_read_golden_equals_reference_reader(oracle, threads):
    from paper_2112_00087_b200.mmio import read_matrix_market
    path = os.path.join(GOLDEN, "system.mtx")
    A = read_matrix_market(path, threads)
    rp, ci, v = oracle.read_matrix_market(path)
    assert np.array_equal(np.asarray(A.row_offsets, np.int64), rp)
    assert np.array_equal(np.asarray(A.col_indices, np.int64), ci)
    assert np.array_equal(bits(A.values), bits(v))


def test_write_is_byte_identical_to_reference(tmp_path):
    from paper_2112_00087_b200.mmio import read_matrix_market, write_matrix_market
    path = os.path.join(GOLDEN, "system.mtx")
    A = read_matrix_market(path)
    out = tmp_path / "w.mtx"
    for t in (1, 7):
        write_matrix_market(str(out), A, t)
        assert out.read_bytes() == open(path, "rb").read()


def test_duplicates_order_comments_and_errors(oracle, tmp_path):
    from paper_2112_00087_b200.mmio import read_matrix_market
    rng = np.random.default_rng(7)
    n, m = 40, 400
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    re = rng.standard_normal(m) * 10.0 ** rng.integers(-5, 5, m)
    im = rng.standard_normal(m)
    lines = ["%%MatrixMarket matrix coordinate complex general", "% comment", "", f"{n} {n} {m}"]
    lines += [f"{a + 1}\t{b + 1}  {float(x)!r} {float(y)!r}" for a, b, x, y in zip(r, c, re, im)]
    p = tmp_path / "d.mtx"
    p.write_text("\n".join(lines))  # no trailing newline
    A = read_matrix_market(str(p), 4)
    rp, ci, v = oracle.csr_from_triplets(r, c, re + 1j * im, n, n)
    assert np.array_equal(np.asarray(A.row_offsets, np.int64), rp)
    assert np.array_equal(np.asarray(A.col_indices, np.int64), ci)
    assert np.array_equal(bits(A.values), bits(v))
    bad = {
        "x.mtx": ("hello\n1 1 1\n1 1 1 0\n", "missing header"),
        "y.mtx": ("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n", "unsupported header"),
        "z.mtx": ("%%MatrixMarket matrix coordinate complex general\n2 2 3\n1 1 1 0\n", "truncated"),
        "w.mtx": ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n0 1 1 0\n", "1-based"),
        "v.mtx": ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n3 1 1 0\n", r"out of range at \(2, 0\)"),
    }
    for name, (text, msg) in bad.items():
        q = tmp_path / name
        q.write_text(text)
        with pytest.raises(ValueError, match=msg):
            read_matrix_market(str(q))
