"""CPU oracle for the compressive-spectral-clustering hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
directory; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` use it, and only as the checker or
as the timed CPU baseline.

``cpu_ref`` restates, with numpy and scipy, the reference algorithm of every
function on the hot path (each function cites the reference file:line it
follows, relative to ``/root/reference/pkg/src/cscluster/``).  It performs the
same floating-point operations in the same order as the reference, so on the
same numpy/scipy build its results are bit-identical to the reference's.

Pinning: ``tests/golden/make_golden.py`` imports the real reference (present
only in the build container) and records its outputs on seeded inputs as
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this oracle
against those fixtures (bit-exact), so the oracle is pinned to the reference.
"""
