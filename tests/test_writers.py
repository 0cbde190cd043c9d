"""Writers: the reference io tests' known answers (test_io.cpp:140-252), CPU only."""
import io

import numpy as np

from paper_0909_2000_b200.alignplot import PlotGrid
from paper_0909_2000_b200 import writers as wr


def grid(rows, cols, w, h, vals):
    return PlotGrid(rows, cols, w, h, values=np.array(vals, dtype=np.int32))


def test_half_to_decimal():
    assert wr.half_to_decimal(3) == "1.5" and wr.half_to_decimal(0) == "0.0"
    assert wr.half_to_decimal(-1) == "-0.5" and wr.half_to_decimal(-4) == "-2.0"


def test_tsv():
    g = grid(2, 2, 4, 5, [4, 1, 3, 8])
    s = io.StringIO(); wr.write_tsv(s, g)
    assert s.getvalue() == "# x_offset y_offset score\n0\t0\t2.0\n0\t1\t0.5\n5\t0\t1.5\n5\t1\t4.0\n"
    s = io.StringIO(); wr.write_tsv(s, g, 3)
    assert s.getvalue() == "# x_offset y_offset score\n0\t0\t2.0\n5\t0\t1.5\n5\t1\t4.0\n"
    s2 = io.StringIO(); wr.write_tsv(s2, g, 3, dense=True)
    s3 = io.StringIO(); wr.write_tsv(s3, g)
    assert s2.getvalue() == s3.getvalue()
    s = io.StringIO(); wr.write_tsv(s, g, 100)
    assert s.getvalue() == "# x_offset y_offset score\n"


def test_dots():
    g = grid(2, 2, 4, 1, [4, 1, 3, 4])
    s = io.StringIO(); wr.write_dots(s, g, 3)
    assert s.getvalue() == "0 0\n1 0\n1 1\n"
    s = io.StringIO(); wr.write_dots(s, g)
    assert s.getvalue() == "0 0\n0 1\n1 0\n1 1\n"


def test_pgm():
    for v, px in ((8, b"\xff"), (0, b"\x00"), (4, b"\x80")):
        b = io.BytesIO(); wr.write_pgm(b, grid(1, 1, 4, 1, [v]))
        assert b.getvalue() == b"P5\n1 1\n255\n" + px
    b = io.BytesIO(); wr.write_pgm(b, grid(1, 1, 4, 1, [4]), 6)
    assert b.getvalue() == b"P5\n1 1\n255\n\x00"
    rng = np.random.default_rng(22)
    vals = rng.integers(0, 15, 28)
    g = grid(4, 7, 7, 3, vals)
    assert np.array_equal(wr.pgm_pixels(g).reshape(-1), (255 * vals + 7) // 14)


def test_fasta_reader_matches_reference_cases():
    # test_io.cpp:107-150
    import pytest
    from paper_0909_2000_b200.fasta import ParseError, read_fasta_bytes, select_record
    one = read_fasta_bytes(b">s\nACGT\n")
    assert [(r.header, bytes(r.sequence)) for r in one] == [("s", b"ACGT")]
    two = read_fasta_bytes(b">a\nAC\nGT\n>b\nTT\n")
    assert [(r.header, bytes(r.sequence)) for r in two] == [("a", b"ACGT"), ("b", b"TT")]
    recs = read_fasta_bytes(b">s desc here\nacgt acgt\r\n  ttaa\n")
    assert recs[0].header == "s desc here" and bytes(recs[0].sequence) == b"ACGTACGTTTAA"
    for bad in (b"ACGT\n", b"", b"\n\n", b">a\n>b\nAC\n", b">a\nAC\n>b\n", b">a\nAC>GT\n", b">a\nAC\x01GT\n"):
        with pytest.raises(ParseError):
            read_fasta_bytes(bad, "test")
    with pytest.raises(ParseError, match="test:2"):
        read_fasta_bytes(b"\nACGT\n", "test")
    recs = read_fasta_bytes(b">alpha one\nAA\n>beta two\nCC\n")
    assert select_record(recs, "", "f").header == "alpha one"
    assert select_record(recs, "beta", "f").header == "beta two"
    assert select_record(recs, "beta two", "f").header == "beta two"
    with pytest.raises(ParseError):
        select_record(recs, "gamma", "f")
