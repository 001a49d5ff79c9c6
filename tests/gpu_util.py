"""Helpers for the GPU parity tests."""

from __future__ import annotations

import contextlib

from conftest import c1_config


@contextlib.contextmanager
def options(**kv):
    from paper_1602_02018_b200 import _lib

    old = {k: _lib.get_option(k) for k in kv}
    try:
        for k, v in kv.items():
            _lib.set_option(k, v)
        yield
    finally:
        for k, v in old.items():
            _lib.set_option(k, v)


_cache: dict = {}


def c1_graph():
    import paper_1602_02018_b200 as P

    if "c1" not in _cache:
        _cache["c1"] = P.sbm_generate(c1_config())
    return _cache["c1"]


def c1_op(dtype="float64"):
    import paper_1602_02018_b200 as P

    key = ("op", dtype)
    if key not in _cache:
        _cache[key] = P.laplacian_op(c1_graph()[0], dtype=dtype)
    return _cache[key]


def oracle_csr(graph):
    from oracle import cpu_ref as O

    return O.Csr(graph.num_nodes, graph.indptr, graph.indices, graph.weights, graph.degrees)
