"""Edge-list text I/O (reference graph.py:177-225): the library's multi-threaded reader and
writer against the oracle restatement, which is pinned to the reference's own outputs
(tests/golden/edgelists.npz, written by the real read_edge_list / write_edge_list)."""

from __future__ import annotations

import ctypes as C
import json
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from conftest import golden
from oracle import cpu_ref as O
from paper_1602_02018_b200 import _lib, graph as G
from paper_1602_02018_b200._errors import GraphError


@pytest.fixture(scope="module")
def edge_golden():
    return golden("edgelists")


def _text(a) -> str:
    return bytes(np.asarray(a, dtype=np.uint8)).decode("utf-8")


def test_oracle_pinned_to_reference(edge_golden):
    rows, hdr = O.parse_edge_text(_text(edge_golden["messy_text"]))
    g = O.build_csr(rows[:, 0].astype(np.int64), rows[:, 1].astype(np.int64), rows[:, 2], int(hdr))
    assert hdr == int(edge_golden["messy_n"])
    assert np.array_equal(g.indptr, edge_golden["messy_indptr"])
    assert np.array_equal(g.indices, edge_golden["messy_indices"])
    assert np.array_equal(g.weights, edge_golden["messy_weights"])
    fmt = O.format_edge_list(int(edge_golden["write_n"]), edge_golden["write_indptr"], edge_golden["write_indices"],
                             edge_golden["write_weights"])
    assert fmt == bytes(edge_golden["write_bytes"])
    msgs = json.loads(_text(edge_golden["error_msgs"]))
    for name, text in json.loads(_text(edge_golden["error_texts"])).items():
        if name == "self_loop":  # raised by build_graph, not by the parse
            continue
        with pytest.raises(O.EdgeListError) as exc:
            O.parse_edge_text(text)
        assert str(exc.value) == msgs[name][1]


def test_native_parse_messy_file(edge_golden, tmp_path):
    p = tmp_path / "messy.edges"
    p.write_bytes(bytes(edge_golden["messy_text"]))
    rows, hdr = G.parse_edge_list(p)
    want, whdr = O.parse_edge_text(_text(edge_golden["messy_text"]))
    assert hdr == whdr and rows.shape == want.shape and np.array_equal(rows, want)


def test_native_parse_errors_match_reference(edge_golden, tmp_path):
    msgs = json.loads(_text(edge_golden["error_msgs"]))
    for name, text in json.loads(_text(edge_golden["error_texts"])).items():
        p = tmp_path / f"{name}.edges"
        p.write_text(text)
        if name == "self_loop":
            rows, _ = G.parse_edge_list(p)
            assert rows.tolist() == [[0.0, 0.0, 1.0]]
            continue
        with pytest.raises(GraphError) as exc:
            G.parse_edge_list(p)
        assert str(exc.value).replace(str(p), "<path>") == msgs[name][1]


def test_native_writer_bytes_match_reference(edge_golden, tmp_path):
    p = tmp_path / "w.edges"
    ip = np.ascontiguousarray(edge_golden["write_indptr"], dtype=np.int32)
    ix = np.ascontiguousarray(edge_golden["write_indices"], dtype=np.int32)
    w = np.ascontiguousarray(edge_golden["write_weights"], dtype=np.float64)
    _lib.call("csc_edgelist_write", str(p).encode(), int(edge_golden["write_n"]), _lib.ptr(ip), _lib.ptr(ix),
              _lib.ptr(w), 0)
    assert p.read_bytes() == bytes(edge_golden["write_bytes"])


def test_empty_and_comment_only_files(tmp_path):
    for text, hdr in (("", None), ("# nodes 5\n", 5), ("\n\n  \n# x\n", None), ("# nodes 3\n# nodes 1_0\n", 10)):
        p = tmp_path / "e.edges"
        p.write_text(text)
        rows, h = G.parse_edge_list(p)
        assert rows.shape == (0, 3) and h == hdr


def _repr(v: float) -> str:
    buf, n = C.create_string_buffer(64), C.c_int()
    _lib.call("csc_float_repr", float(v), buf, 64, C.byref(n))
    return buf.value.decode()


@settings(max_examples=3000, deadline=None)
@given(st.floats(allow_nan=True, allow_infinity=True))
def test_float_repr_is_pythons(v):
    assert _repr(v) == repr(v)


def test_float_repr_boundaries():
    for v in (0.0, -0.0, 1.0, 0.1, 1e15, 1e16, 9999999999999998.0, 1e-4, 1e-5, 0.00012, 5e-324, 2.2250738585072014e-308,
              1.7976931348623157e308, 123456789012345678.0, 1e22, 1e100, 1.5e-100, math.pi, float("nan"), float("inf")):
        assert _repr(v) == repr(v), v


TOKENS = ["0", "1", "2", "7", "12", "-3", "+4", "007", "1_0", "x", "٣", "1.5", ".5", "5.", "1e-3", "2.25E+1",
          "inf", "nan", "1__0", "1e400", "1e-400", "-0.0", "0x10", "", "#", "# nodes 9", "#nodes 4", "nodes"]
SEPS = [" ", "\t", "  ", "\x0b", "\x0c", " ", "\x1c"]
ENDS = ["\n", "\r\n", "\r"]


@st.composite
def messy_files(draw):
    lines = []
    for _ in range(draw(st.integers(0, 25))):
        toks = draw(st.lists(st.sampled_from(TOKENS), min_size=0, max_size=4))
        sep = draw(st.sampled_from(SEPS))
        lead = draw(st.sampled_from(["", " ", "\t"]))
        lines.append(lead + sep.join(toks) + draw(st.sampled_from(ENDS)))
    text = "".join(lines)
    if text and draw(st.booleans()):
        text = text.rstrip("\r\n")  # no terminator on the last line
    return text


@settings(max_examples=400, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(messy_files())
def test_native_parse_matches_oracle_on_messy_text(tmp_path, text):
    p = tmp_path / "f.edges"
    p.write_bytes(text.encode("utf-8"))
    try:
        want = O.parse_edge_text(text, name=str(p))
    except O.EdgeListError as exc:
        with pytest.raises(GraphError) as got:
            G.parse_edge_list(p)
        assert str(got.value) == str(exc)
        return
    rows, hdr = G.parse_edge_list(p)
    assert hdr == want[1]
    assert rows.shape == want[0].shape and np.array_equal(rows, want[0], equal_nan=True)


def test_parallel_chunks_match_oracle(tmp_path):
    """A file large enough to be split over several threads (>= 4 MB per thread), line
    terminators of all three kinds, a few complex lines spread through it."""
    rng = np.random.default_rng(3)
    n = 400_000
    src, dst = rng.integers(0, 10_000, n), rng.integers(0, 10_000, n)
    w = rng.uniform(0.01, 5.0, n)
    ends = np.array(["\n", "\r\n", "\r"])[rng.integers(0, 3, n)]
    parts = [f"{a} {b} {c!r}{e}" for a, b, c, e in zip(src.tolist(), dst.tolist(), w.tolist(), ends.tolist())]
    for k in rng.choice(n, 30, replace=False):
        parts[k] = f"{src[k]} {dst[k]} 1_0.5\n"
    parts.insert(1000, "# nodes 10001\n")
    text = "".join(parts)
    p = tmp_path / "big.edges"
    p.write_bytes(text.encode("utf-8"))
    rows, hdr = G.parse_edge_list(p)
    want, whdr = O.parse_edge_text(text)
    assert hdr == whdr == 10001 and np.array_equal(rows, want)


def test_writer_empty_graph_and_null_arrays(tmp_path):
    p = tmp_path / "e.edges"
    _lib.call("csc_edgelist_write", str(p).encode(), 0, None, None, None, 0)
    assert p.read_bytes() == O.format_edge_list(0, [0], [], [])
    with pytest.raises(ValueError):
        _lib.call("csc_edgelist_write", str(p).encode(), 3, None, None, None, 0)
    with pytest.raises(ValueError):
        _lib.call("csc_edgelist_read", str(tmp_path / "missing.edges").encode(), 0, C.byref(C.c_void_p()))
