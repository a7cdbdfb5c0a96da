"""Native read_column (csrc/rqa_ingest.cpp) against the line-by-line reader.

The Python reader (_read_column_py) is the reference's algorithm
(ingest.py:95-129, also checked against tiledrqa itself below when the
reference is importable); the native reader must return the same values,
skipped-row counts and errors on every ASCII input.  CPU only.
"""

import os
import sys

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2402_16853_b200 import errors
from paper_2402_16853_b200.ingest import _read_column_native, _read_column_py, read_column

TOKENS = ["1", "-2.5", "+.5", "5.", "1e3", "1E-3", "1_000", "1__0", "_1", "1_", "1e1_0",
          "inf", "-Infinity", "nan", "NaN", "1e400", "1e-400", "0x10", "", " ", "abc", ".",
          "1.2.3", "  7  ", "\t8\x0b", "1 2", "+-1", "00012", "9" * 40, "1.5e+3", "e5",
          "\x1c3\x1f", "3\x00", "-0", "1e", "1._5", "2_.5", "infinit", "iNf"]
NEWLINES = ["\n", "\r\n", "\r"]


def _outcome(fn, *args):
    try:
        ts = fn(*args)
    except errors.RQAError as exc:
        return type(exc).__name__, str(exc)
    return "ok", ts.values.tolist(), ts.skipped_rows


@settings(max_examples=300, deadline=None)
@given(rows=st.lists(st.lists(st.sampled_from(TOKENS), min_size=0, max_size=4), max_size=25),
       nls=st.lists(st.sampled_from(NEWLINES), min_size=25, max_size=25),
       delim=st.sampled_from([",", ";", " ", "\t", "|"]),
       column=st.integers(0, 3), offset=st.integers(0, 4), skip=st.booleans(),
       trailing=st.booleans())
def test_native_matches_python_reader(tmp_path_factory, rows, nls, delim, column, offset, skip,
                                      trailing):
    text = "".join(delim.join(r) + nls[i] for i, r in enumerate(rows))
    if not trailing and text:
        text = text[:-len(nls[len(rows) - 1])]
    path = tmp_path_factory.mktemp("ing") / "x.txt"
    path.write_bytes(text.encode("ascii"))
    want = _outcome(_read_column_py, str(path), delim, column, offset, skip)
    got = _outcome(lambda *a: _read_column_native(*a, 0) or (_ for _ in ()).throw(
        AssertionError("native reader declined an ASCII file")), str(path), delim, column,
        offset, skip)
    assert got == want, (text, delim, column, offset, skip)


def test_large_file_multithreaded(tmp_path):
    rng = np.random.default_rng(0)
    n = 400_000
    vals = rng.normal(size=n) * 10.0 ** rng.integers(-5, 6, n)
    lines = [f"{i},{float(v)!r},x" for i, v in enumerate(vals)]
    lines[1000] = ""                    # blank rows do not count
    lines[123457] = "  "                # one field only: ColumnOutOfRange unless skipped
    path = tmp_path / "big.csv"
    path.write_text("hdr\n" + "\r\n".join(lines) + "\n")
    ts = read_column(path, column=1, offset=1, skip_invalid=True, threads=8)
    want = _read_column_py(path, ",", 1, 1, True)
    assert ts.skipped_rows == want.skipped_rows == 1
    assert np.array_equal(ts.values, want.values)
    with pytest.raises(errors.ColumnOutOfRange) as exc:
        read_column(path, column=1, offset=1, threads=8)
    assert exc.value.row == 123459     # physical line (1-based, header + blank counted)
    with pytest.raises(errors.ParseError) as exc:
        read_column(path, column=2, offset=1, threads=8)
    assert exc.value.row == 2 and exc.value.token == "x"


def test_fallbacks_and_errors(tmp_path):
    p = tmp_path / "u.csv"
    p.write_text("1\n٢\n3\n", encoding="utf-8")   # Arabic-Indic two: float() accepts it
    assert read_column(p).values.tolist() == [1.0, 2.0, 3.0]
    with pytest.raises(errors.FileNotReadable):
        read_column(tmp_path / "missing.csv")
    with pytest.raises(errors.FileNotReadable):
        read_column(tmp_path)
    q = tmp_path / "c.csv"
    q.write_text("1,2\n3\n")
    with pytest.raises(errors.ColumnOutOfRange) as exc:
        read_column(q, column=1)
    assert (exc.value.row, exc.value.n_fields, exc.value.column) == (2, 1, 1)
    e = tmp_path / "e.csv"
    e.write_text("\n\n")
    with pytest.raises(errors.EmptySeries):
        read_column(e)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_against_reference_reader(tmp_path):
    sys.path.insert(0, REF)
    try:
        import tiledrqa
    finally:
        sys.path.remove(REF)
    text = "t,v\n1,2\n\n3_0, 4e1 \r\n5,nan\r7,8\n9,1e400\n"
    p = tmp_path / "r.csv"
    p.write_text(text)
    for kw in ({"column": 1, "offset": 1, "skip_invalid": True}, {"column": 0, "offset": 1}):
        a = tiledrqa.read_column(str(p), **kw)
        b = read_column(str(p), **kw)
        assert a.values.tolist() == b.values.tolist() and a.skipped_rows == b.skipped_rows
    with pytest.raises(tiledrqa.ParseError) as ea:
        tiledrqa.read_column(str(p), column=1, offset=1)
    with pytest.raises(errors.ParseError) as eb:
        read_column(str(p), column=1, offset=1)
    assert str(ea.value) == str(eb.value)
