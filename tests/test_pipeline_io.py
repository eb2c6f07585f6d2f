"""Point-cloud files, host-side: the B200 library's
xyz / legacy-VTK reader and writer against the reference's own pipeline_io
(oracle/_ref): bit-exact round trips, identical parses of the same files, and
the same error class (and parse line) on malformed input."""
import os

import numpy as np
import pytest

from paper_1907_04834_b200 import (VTK, XYZ, ParseError, UnsupportedFormat, format_for_path,
                                   read_points, write_points)


@pytest.fixture
def pts():
    rng = np.random.default_rng(3)
    p = rng.normal(0, 1, (257, 3)) * np.array([1e-300, 1.0, 1e300])
    p[0] = [0.1, -0.0, 5e-324]  # awkward values: 0.1, -0, smallest denormal
    return p


def test_format_for_path():
    assert format_for_path("a/b.vtk") == VTK and format_for_path("x.xyz") == XYZ
    assert format_for_path("noext") == XYZ


@pytest.mark.parametrize("fmt,ext", [(XYZ, "xyz"), (VTK, "vtk")])
def test_round_trip_bit_exact(tmp_path, pts, fmt, ext):
    f = str(tmp_path / f"p.{ext}")
    write_points(pts, f, fmt, header=["moving shape", "second line"])
    back = read_points(f, fmt)
    assert back.tobytes() == np.ascontiguousarray(pts).tobytes()


GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("fmt,name", [(XYZ, "io_ref.xyz"), (VTK, "io_ref.vtk")])
def test_byte_identical_to_reference_writer(tmp_path, fmt, name):
    """Files written by the reference's write_points (tests/golden/make_golden_io.py)."""
    pts = np.fromfile(os.path.join(GOLD, "io_points.bin"), dtype="<f8").reshape(-1, 3)
    a = str(tmp_path / "ours")
    write_points(pts, a, fmt, header=["title"])
    assert open(a, "rb").read() == open(os.path.join(GOLD, name), "rb").read()
    assert read_points(os.path.join(GOLD, name), fmt).tobytes() == pts.tobytes()


CASES = {
    "ok_comments": (XYZ, "# c\n\n  1 2 3\n4.5e1 -6 +7\n# tail\n"),
    "missing_coord": (XYZ, "1 2 3\n4 5\n"),
    "trailing": (XYZ, "1 2 3\n4 5 6 7\n"),
    "bad_token": (XYZ, "1 2 x\n"),
    "empty": (XYZ, "# only comments\n\n"),
    "inf_text": (XYZ, "inf 0 0\n"),
    "vtk_ok": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 2 float\n"
                    "1 2 3 4\n5 6\nVERTICES 2 4\n1 0\n1 1\n"),
    "vtk_binary": (VTK, "# vtk DataFile Version 3.0\nt\nBINARY\nDATASET POLYDATA\n"),
    "vtk_grid": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET STRUCTURED_GRID\n"),
    "vtk_notvtk": (VTK, "hello\n"),
    "vtk_short": (VTK, "# vtk DataFile Version 3.0\nt\n"),
    "vtk_nopoints": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nLINES 1\n"),
    "vtk_badcount": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 1.5 float\n"),
    "vtk_badtype": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 1 int\n1 2 3\n"),
    "vtk_truncated": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 2 double\n1 2 3\n4\n"),
    "vtk_badnum": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 1 double\n1 2 z\n"),
    "vtk_nan": (VTK, "# vtk DataFile Version 3.0\nt\nASCII\nDATASET POLYDATA\nPOINTS 1 double\n1 nan 3\n"),
}


@pytest.mark.parametrize("case", list(CASES))
def test_parse_matches_reference(tmp_path, ref, case):
    fmt, text = CASES[case]
    f = str(tmp_path / "in.txt")
    open(f, "w").write(text)
    want_st, want, want_line = ref.read_points(f, fmt)
    try:
        got = read_points(f, fmt)
        got_st, got_line = 0, 0
    except ParseError as e:
        got_st, got_line, got = 10, e.line, None
    except UnsupportedFormat:
        got_st, got_line, got = 11, 0, None
    except ValueError:
        got_st, got_line, got = 7, 0, None
    assert got_st == want_st
    if want_st == 10:
        assert got_line == want_line
    if want_st == 0:
        assert np.array_equal(got, want)


def test_missing_file(tmp_path):
    with pytest.raises(OSError):
        read_points(str(tmp_path / "nope.xyz"))


# ---- property: every finite double survives a write/read round trip ----------
from hypothesis import given, settings, strategies as st  # noqa: E402

_finite = st.floats(allow_nan=False, allow_infinity=False, width=64)


@settings(max_examples=60, deadline=None)
@given(st.lists(st.tuples(_finite, _finite, _finite), min_size=1, max_size=40),
       st.sampled_from([(XYZ, "xyz"), (VTK, "vtk")]))
def test_round_trip_property(tmp_path_factory, rows, fmt_ext):
    fmt, ext = fmt_ext
    pts = np.array(rows, dtype=np.float64).reshape(-1, 3)
    f = str(tmp_path_factory.mktemp("rt") / f"p.{ext}")
    write_points(pts, f, fmt)
    back = read_points(f, fmt)
    assert back.shape == pts.shape
    # bit-exact, -0.0 included (%.17g keeps the sign)
    assert back.tobytes() == pts.tobytes()
