"""Checker helpers for the BASELINE-config parity tests (test infrastructure).

The oracle (oracle/, a pinned C restatement of the reference engine) runs
on a row prefix of a workload: rows are independent (engine.py:237-251),
so the prefix of the GPU's full-batch result must equal the oracle's
result for those rows.  Layers are generated a chunk at a time; once no
prefix row holds an entry the remaining layers are the identity (zero rows
stay zero, the reference's own KAT test_engine.py:138-146), so the oracle
stops there while the GPU still runs every layer.
"""

from __future__ import annotations

import os

import numpy as np

from oracle import oracle as O
from paper_1909_05631_b200 import workloads as W

THREADS = os.cpu_count() or 8
F32_RTOL = 1e-5  # north_star: final Y within fp32 relative tolerance 1e-5 of the reference


def prefix_csr(n, off, cols, vals, rows):
    """The first `rows` rows of a CSR batch with n columns."""
    return O.CSR(rows, n, off[:rows + 1].copy(), cols[:off[rows]], vals[:off[rows]])


def oracle_stream(w: W.Workload, y0: O.CSR, precision: int, chunk: int = 8):
    """(final Y, live rows entering each layer + survivors) of the oracle
    over y0 through all w.layers layers."""
    y = O.CSR(y0.n_rows, w.n, y0.off, y0.cols, y0.vals)
    live = np.zeros(w.layers + 1, np.int64)
    l = 0
    while l < w.layers:
        rows_live = int(np.count_nonzero(np.diff(y.off)))
        if rows_live == 0:
            break
        m = min(chunk, w.layers - l)
        for c in W.layers_csr(w, l, m, THREADS):
            live[l] = int(np.count_nonzero(np.diff(y.off)))
            if live[l] == 0:
                break
            y = O.infer([O.CSR(w.n, w.n, *c)], [w.bias], y, w.ymax, precision=precision, threads=THREADS)
            l += 1
    live[w.layers] = int(np.count_nonzero(np.diff(y.off)))
    y.n_cols = w.n
    return y, live


def assert_f32_within(y32: O.CSR, y64: O.CSR, rtol: float = F32_RTOL) -> float:
    """float32 result vs the float64 reference: same stored pattern (so the
    same categories) and every value within `rtol` relative; returns the
    largest relative error seen."""
    assert y32.n_rows == y64.n_rows
    assert np.array_equal(y32.off, y64.off), "stored pattern differs (row counts)"
    assert np.array_equal(y32.cols, y64.cols), "stored pattern differs (columns)"
    if y64.vals.size == 0:
        return 0.0
    rel = np.abs(y32.vals - y64.vals) / np.abs(y64.vals)
    worst = float(rel.max())
    assert worst <= rtol, f"max relative error {worst:.3g} > {rtol}"
    return worst
