"""proj/tests/test_matrix_market.cpp re-expressed against the B200 build's
host layer (csrc/host/matrix_market.cpp through fl_mm_read / fl_mm_write):
same parse results, error types, line numbers and lossless round trips; plus
the remaining reference error paths (matrix_market.cpp:31-117) and the
parsed matrix going through the filter path unchanged (no GPU needed for
the parse; the filter leg is marked gpu)."""
import numpy as np
import pytest

import oracle as O


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_coordinate_symmetric_file_parses_with_mirrored_lower_triangle(tmp_path):
    import paper_1605_08771_b200 as P
    f = _write(tmp_path, "coord.mtx",
               "%%MatrixMarket matrix coordinate real symmetric\n"
               "% comment line\n"
               "2 2 3\n"
               "1 1 1.0\n"
               "2 1 0.5\n"
               "2 2 2.0\n")
    M = P.read_matrix_market(f).mat()
    assert M[0, 0] == 1.0 and M[0, 1] == 0.5 and M[1, 0] == 0.5 and M[1, 1] == 2.0


def test_general_header_is_rejected_with_a_distinct_error(tmp_path):
    import paper_1605_08771_b200 as P
    f = _write(tmp_path, "general.mtx",
               "%%MatrixMarket matrix coordinate real general\n"
               "2 2 4\n1 1 1\n1 2 2\n2 1 2\n2 2 3\n")
    with pytest.raises(P.NotSymmetricError) as e:
        P.read_matrix_market(f)
    assert "general" in str(e.value)
    assert isinstance(e.value, P.MatrixMarketError) and e.value.line == 1


def test_parse_failures_carry_line_numbers(tmp_path):
    import paper_1605_08771_b200 as P
    f = _write(tmp_path, "bad.mtx",
               "%%MatrixMarket matrix coordinate real symmetric\n"
               "2 2 2\n"
               "1 1 1.0\n"
               "2 oops 0.5\n")
    with pytest.raises(P.MatrixMarketError) as e:
        P.read_matrix_market(f)
    assert e.value.line == 4
    assert "(line 4)" in str(e.value)


@pytest.mark.parametrize("fmt", ["coordinate", "array"])
def test_round_trip_is_lossless_in_both_formats(tmp_path, fmt):
    import paper_1605_08771_b200 as P
    M = P.SymmetricMatrix(O.random_symmetric(17, 31))
    f = str(tmp_path / "roundtrip.mtx")
    P.write_matrix_market(M, f, fmt)
    R = P.read_matrix_market(f)
    assert R.dim() == 17
    assert np.abs(R.mat() - M.mat()).max() == 0.0


def test_missing_file_and_truncated_file_are_reported(tmp_path):
    import paper_1605_08771_b200 as P
    with pytest.raises(P.FeastRuntimeError) as e:
        P.read_matrix_market("/nonexistent/feastlab.mtx")
    assert not isinstance(e.value, P.MatrixMarketError)
    f = _write(tmp_path, "trunc.mtx",
               "%%MatrixMarket matrix coordinate real symmetric\n"
               "3 3 6\n"
               "1 1 1.0\n")
    with pytest.raises(P.MatrixMarketError):
        P.read_matrix_market(f)


@pytest.mark.parametrize("text,line,frag", [
    ("", 1, "empty file"),
    ("%MatrixMarket matrix coordinate real symmetric\n1 1 1\n1 1 1\n", 1, "banner"),
    ("%%MatrixMarket vector coordinate real symmetric\n", 1, "unsupported object"),
    ("%%MatrixMarket matrix packed real symmetric\n", 1, "unsupported format"),
    ("%%MatrixMarket matrix coordinate complex symmetric\n", 1, "unsupported field"),
    ("%%MatrixMarket matrix coordinate real symmetric\n% only comments\n\n", 3, "missing size line"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 x 1\n", 2, "malformed size line"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n", 2, "must be square"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1.0\n", 3, "out of range"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n", 3, "upper-triangle"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n\n% c\nnan\n", 6, "malformed value"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n2.0\n", 4, "unexpected end"),
])
def test_reference_error_paths(tmp_path, text, line, frag):
    import paper_1605_08771_b200 as P
    f = _write(tmp_path, "err.mtx", text)
    with pytest.raises(P.MatrixMarketError) as e:
        P.read_matrix_market(f)
    assert e.value.line == line, (e.value.line, str(e.value))
    assert frag in str(e.value)


def test_header_is_case_insensitive_and_entries_tolerate_blanks_and_trailing_text(tmp_path):
    import paper_1605_08771_b200 as P
    f = _write(tmp_path, "case.mtx",
               "%%MatrixMarket MATRIX Array REAL Symmetric\n"
               "   \n"
               "2 2\n"
               "  1.5e0   extra\n"
               "\t-2\r\n"
               "+.25\n")
    M = P.read_matrix_market(f).mat()
    assert np.array_equal(M, np.array([[1.5, -2.0], [-2.0, 0.25]]))


@pytest.mark.gpu
def test_parsed_matrix_drives_the_filter(tmp_path):
    """A matrix read from disk goes through the B200 filter like the in-memory
    one (bitwise: the file holds %.17g round-trip digits)."""
    import paper_1605_08771_b200 as P
    n = 300
    A = O.random_symmetric(n, 9) / np.sqrt(n)
    f = str(tmp_path / "a.mtx")
    P.write_matrix_market(A, f)
    S = P.read_matrix_market(f)
    X = O.random_block(n, 16, 3)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.3), 8)
    assert np.array_equal(P.apply_filter(S, rule, X), P.apply_filter(A, rule, X))
