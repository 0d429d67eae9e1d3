"""QC expansion and alist round trips of the input plumbing (CPU)."""
import numpy as np

from gen import codes


def test_expand_qc_examples():
    assert np.array_equal(codes.expand_qc(1, 1, 3, [[[0]]]).dense(), np.eye(3, dtype=np.uint8))
    assert codes.expand_qc(1, 1, 3, [[[1]]]).dense().tolist() == [[0, 1, 0], [0, 0, 1], [1, 0, 0]]
    c = codes.expand_qc(1, 2, 3, [[[0, 2], []]])
    assert c.nnz == 6 and c.dense()[:, 3:].sum() == 0


def test_ccsds_shaped_qc():
    c = codes.qc_random()
    assert (c.m, c.n) == (1022, 8176)
    H = c.dense()
    assert np.all(H.sum(axis=1) == 32) and np.all(H.sum(axis=0) == 4)
    assert c.nnz == 2 * 16 * 511 * 2  # sum over blocks of Z x shifts (SPEC invariant)


def test_alist_round_trip():
    for c in (codes.paper_5x10(), codes.random_small(9, 17, 4, 2, 5), codes.regular(12, 24, 3, 6, 2)):
        text = codes.to_alist(c)
        d = codes.parse_alist(text)
        assert all(np.array_equal(a, b) for a, b in zip(c.rows, d.rows)) and (d.m, d.n) == (c.m, c.n)
        assert codes.to_alist(d) == text
    lines = codes.to_alist(codes.paper_5x10()).splitlines()
    assert lines[0] == "10 5" and lines[1].endswith("6")


def test_alist_rejects_inconsistent():
    import pytest

    bad = "2 1\n1 2\n1 1\n2\n1\n1\n1 1\n"
    with pytest.raises(ValueError):
        codes.parse_alist(bad)
