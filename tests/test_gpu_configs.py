"""GPU parity on the BASELINE configs as specified (C1-C5, all twelve C5
cells) and the live K2 companion, both precisions.

For every config: the full batch runs on the GPU; the oracle runs a row
prefix (rows are independent).  Checked: live rows entering every layer,
the prefix's final Y bit-identical to the oracle's same-precision instance,
categories equal to the float64 oracle's in BOTH precisions, the float32
final Y within relative 1e-5 of the float64 reference (north_star), and
the full batch's categories restricted to the prefix equal the prefix's.
Reference contract: challenge.py:123-128 (verify) and
tests/test_acceptance.py:231-250.
"""

import numpy as np
import pytest

from oracle import oracle as O
from parity import F32_RTOL, assert_f32_within, oracle_stream, prefix_csr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1909_05631_b200 import engine as E  # noqa: E402
from paper_1909_05631_b200 import workloads as W  # noqa: E402

PREFIX = {"C1": 60000, "C2": 3000, "C3": 1500, "C4": 600}


def _check(w, net, full_off, full_cols, full_vals, rows, want, live, want64, dtype):
    """Full batch + prefix on the GPU against the oracle's same-precision
    instance (`want`, its live rows per layer `live`) and the float64
    reference (`want64`).  The live sets of intermediate layers may differ
    between precisions (a row whose sum lands within rounding of -bias),
    so they are compared within a precision only."""
    full = net.run(net.upload_csr(w.batch, full_off, full_cols, full_vals), w.ymax)
    assert full.live_rows[0] == np.count_nonzero(np.diff(full_off))
    y0 = prefix_csr(w.n, full_off, full_cols, full_vals, rows)
    head = net.run(net.upload_csr(rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    got = O.CSR(rows, w.n, *head.y)
    assert np.array_equal(head.live_rows, live), f"{dtype}: live rows per layer"
    assert got.identical(want), f"{dtype}: prefix Y differs from the oracle's {dtype} instance"
    assert np.array_equal(head.categories, O.categorize(want64)), f"{dtype}: categories vs float64"
    if dtype == "f32":
        assert_f32_within(got, want64)
    assert np.array_equal(full.categories[full.categories <= rows], head.categories)
    return full


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_as_specified(name):
    """C1-C4 exactly as BASELINE.json specifies them (C4 = the benched
    flagship: N=65536, L=1920, 60,000 rows, w=0.0625, b=-0.45)."""
    w = W.CONFIGS[name]
    off, cols, vals = W.images(w)
    rows = PREFIX[name]
    y0 = prefix_csr(w.n, off, cols, vals, rows)
    want64, live64 = oracle_stream(w, y0, 64)
    want32, live32 = oracle_stream(w, y0, 32)
    for dtype, want, live in (("f32", want32, live32), ("f64", want64, live64)):
        net = E.DeviceNetwork(w.n, 0, dtype)
        net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
        _check(w, net, off, cols, vals, rows, want, live, want64, dtype)
        net.close()


@pytest.fixture(scope="module", params=["f32", "f64"])
def c5_net(request):
    """One C5 network per precision, reused by the twelve cells (pytest
    groups the cells by this module-scoped parameter, so only one network
    and its run scratch -- up to ~120 GB at 240,000 rows -- is resident)."""
    w = W.CONFIGS["C5"]
    net = E.DeviceNetwork(w.n, 0, request.param)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    yield request.param, net
    net.close()


@pytest.mark.parametrize("batch,p", W.C5_SWEEP)
def test_c5_sweep_cell(c5_net, batch, p):
    """All twelve cells of BASELINE config 5 (N=65536, L=120, B in
    {1000, 15000, 60000, 240000} x p in {0.1, 0.35, 0.7}), both precisions,
    against a 400-row oracle prefix."""
    dtype, net = c5_net
    w = W.CONFIGS["C5"].with_(batch=batch, p=p)
    off, cols, vals = W.images(w)
    rows = min(400, batch)
    y0 = prefix_csr(w.n, off, cols, vals, rows)
    want64, live64 = oracle_stream(w, y0, 64)
    if dtype == "f64":
        want, live = want64, live64
    else:
        want, live = oracle_stream(w, y0, 32)
    _check(w, net, off, cols, vals, rows, want, live, want64, dtype)


def test_k2_live_companion_f32_within_tolerance_of_f64():
    """K2 (the C4/C5 generator with w=0.125, 120 layers): rows stay alive
    and saturate, so every layer carries the full batch.  Full batch in both
    precisions: identical category lists; a 2,000-row block's final Y from
    the float32 path within 1e-5 of the (reference-exact) float64 path; a
    32-row prefix against the oracle in both precisions."""
    w = W.CONFIGS["K2"].with_(layers=120)
    off, cols, vals = W.images(w)
    rows = 32
    y0 = prefix_csr(w.n, off, cols, vals, rows)
    want64, live64 = oracle_stream(w, y0, 64)
    want32, live32 = oracle_stream(w, y0, 32)
    assert live64[-1] > 0  # a live workload
    block = prefix_csr(w.n, off, cols, vals, 2000)
    fulls, ys = {}, {}
    for dtype, want, live in (("f32", want32, live32), ("f64", want64, live64)):
        net = E.DeviceNetwork(w.n, 0, dtype)
        net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
        fulls[dtype] = _check(w, net, off, cols, vals, rows, want, live, want64, dtype)
        r = net.run(net.upload_csr(2000, block.off, block.cols, block.vals), w.ymax, want_y=True)
        ys[dtype] = O.CSR(2000, w.n, *r.y)
        net.close()
    assert fulls["f32"].categories.size > 50000
    assert np.array_equal(fulls["f32"].categories, fulls["f64"].categories)
    assert ys["f64"].nnz > 0
    assert_f32_within(ys["f32"], ys["f64"], F32_RTOL)
