"""Output pruning by line bounds (include/sdnn.h: sdnn_net_set_pruning).

A (tile, output) column whose input lines cannot lift any row above -bias
gathers nothing.  The bound is an upper bound of the chain the reference
computes (engine.py:64-137), so the result must be bit-identical with
pruning on and off and equal to the oracle's, on the BASELINE dynamics
(rows die at layer 2-3: on the flagship almost every column of the dying
layer is pruned),
on live rows (nothing may be pruned away), on mixed-sign general instances
and at the rounding boundary of `sum == -bias`.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1909_05631_b200 import engine as E  # noqa: E402
from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.model import SparseMatrix  # noqa: E402


def sm(c: O.CSR) -> SparseMatrix:
    return SparseMatrix(c.n_rows, c.n_cols, c.off, c.cols, c.vals, check=False)


def both(net, batch, ymax):
    """(pruning on, pruning off) runs of one staged batch, asserted identical."""
    net.set_pruning(True)
    on = net.run(batch, ymax, want_y=True)
    net.set_pruning(False)
    off = net.run(batch, ymax, want_y=True)
    net.set_pruning(True)
    assert off.pruned == 0
    assert all(np.array_equal(a, b) for a, b in zip(on.y, off.y))
    assert np.array_equal(on.categories, off.categories)
    assert np.array_equal(on.live_rows, off.live_rows)
    return on, off


@pytest.mark.parametrize("dtype,prec", [("f32", 32), ("f64", 64)])
@pytest.mark.parametrize("prune_pass", ["1", "0"])
@pytest.mark.parametrize("name,rows,layers", [("C1", 3000, 12), ("C2", 1500, 8), ("C3", 1200, 6), ("C4", 700, 6)])
def test_dying_configs_are_pruned_and_bit_identical(monkeypatch, name, rows, layers, prune_pass, dtype, prec):
    """BASELINE dynamics (w = 0.0625): layer 2's inputs are few and small,
    its columns are pruned, and the result is the oracle's -- through the
    prune pass (bound codes in shared memory, one bit per column; C3 leaves
    some columns of every warp to the exact-bound test and the gather) and
    with the per-column test alone."""
    monkeypatch.setenv("SDNN_PRUNE_PASS", prune_pass)
    w = W.CONFIGS[name].with_(batch=rows, layers=layers)
    off, cols, vals = W.images(w)
    y0 = O.CSR(rows, w.n, off, cols, vals)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    on, _ = both(net, net.upload_csr(rows, off, cols, vals), w.ymax)
    lw = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    want = O.infer(lw, [w.bias] * w.layers, y0, w.ymax, precision=prec, threads=8)
    assert O.CSR(rows, w.n, *on.y).identical(want)
    assert np.array_equal(on.categories, O.categorize(want))
    # layer 2 runs in the persistent kernel over every (tile, output).  C4's
    # layer-1 outputs are 5 % dense and at most ~0.3, so 32 * 0.0625 * (line
    # bound) stays below 0.45 for nearly every column; C1 / C2 (47 % / 26 %
    # dense, bias -0.30 / -0.35) are beyond a line-granular bound and simply
    # gather as before
    tiles = -(-int(on.live_rows[1]) // (256 if dtype == "f32" else 128))
    if name == "C4":
        assert on.pruned >= tiles * w.n * 8 // 10, (on.pruned, tiles * w.n)
    if name == "C3":
        assert tiles * w.n // 2 <= on.pruned < tiles * w.n, (on.pruned, tiles * w.n)
    net.close()


@pytest.mark.parametrize("dtype,prec", [("f32", 32), ("f64", 64)])
@pytest.mark.parametrize("bits", ["1", "0"])
def test_live_rows_survive_pruning(monkeypatch, dtype, prec, bits):
    """Rows that stay alive (w = 0.125) and rows that die gradually share
    tiles: pruning may only drop columns that end at zero for every row."""
    monkeypatch.setenv("SDNN_BIN", bits)
    side = 32
    w = W.Workload("t", 1024, 10, 2000, side, 20, 0.35, -0.45, value=0.125)
    off, cols, vals = W.images(w)
    y0 = O.CSR(w.batch, w.n, off, cols, vals)
    lw = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    want = O.infer(lw, [w.bias] * w.layers, y0, w.ymax, precision=prec, threads=8)
    assert 0 < O.categorize(want).size < w.batch
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    on, _ = both(net, net.upload_csr(w.batch, off, cols, vals), w.ymax)
    assert O.CSR(w.batch, w.n, *on.y).identical(want)
    net.close()


def test_mixed_sign_general_instances():
    """Mixed-sign weights, variable degree (ELL padded to 32 slots), biases of
    either sign, real-valued inputs: on == off == oracle, float64."""
    rng = np.random.default_rng(5631)
    pruned = 0
    for i in range(60):
        n = int(rng.integers(8, 97))
        layers, bias = [], []
        for _ in range(int(rng.integers(1, 7))):
            dens = rng.uniform(0.02, 0.3)
            m = np.where(rng.random((n, n)) < dens, rng.uniform(-1, 1, (n, n)), 0.0)
            layers.append(O.CSR.from_dense(m))
            bias.append(float(rng.uniform(-0.8, 0.2)))
        rows = int(rng.integers(1, 300))
        y = (rng.random((rows, n)) < rng.uniform(0.05, 0.6)).astype(np.float64)
        y *= rng.uniform(0.05, 2.0, y.shape)
        y0 = O.CSR.from_dense(y)
        net = E.DeviceNetwork(n, 0, "f64")
        for m, b in zip(layers, bias):
            net.add_layer_csr(sm(m), b)
        on, _ = both(net, net.upload_csr(rows, y0.off, y0.cols, y0.vals), 32.0)
        want = O.infer(layers, bias, y0, precision=64)
        assert O.CSR(rows, n, *on.y).identical(want), i
        pruned += on.pruned
        net.close()
    assert pruned > 0  # the bound fires on some of them


@pytest.mark.parametrize("dtype,prec", [("f32", 32), ("f64", 64)])
def test_rounding_boundary(dtype, prec):
    """Every output sums 32 inputs of value y with weight 1/16: z = 2y.  With
    bias = -(2y) the result is exactly zero (dropped); one ulp less negative
    and every entry survives with a tiny value.  The bound must not prune
    the second case (its margin only ever errs towards gathering)."""
    n, rows = 64, 300
    dense = np.zeros((n, n))
    for j in range(n):
        for s in range(32):
            dense[(j + s) % n, j] = 0.0625
    wm = O.CSR.from_dense(dense)
    yv = 1.7
    y = np.full((rows, n), yv)
    y0 = O.CSR.from_dense(y)
    ft = np.float32 if prec == 32 else np.float64
    z = ft(0)
    for _ in range(32):  # the chain's own rounding
        z = ft(z + ft(yv) * ft(0.0625))  # the product is exact (power-of-two weight)
    exact = -float(z)
    for bias, survive in ((exact, False), (float(np.nextafter(ft(exact), ft(0))), True),
                          (exact * 1.0005, False), (exact * 0.9995, True)):
        net = E.DeviceNetwork(n, 0, dtype)
        net.add_layer_csr(sm(wm), bias)
        on, _ = both(net, net.upload_csr(rows, y0.off, y0.cols, y0.vals), 32.0)
        want = O.infer([wm], [bias], y0, precision=prec)
        assert O.CSR(rows, n, *on.y).identical(want), bias
        assert (on.categories.size == rows) == survive, bias
        net.close()


@pytest.mark.parametrize("dtype,prec", [("f32", 32), ("f64", 64)])
@pytest.mark.parametrize("scale,bias", [(0.06, -0.45), (0.11, -0.45), (0.2, -0.1)])
def test_layer1_prefilter_with_uneven_weights(monkeypatch, dtype, prec, scale, bias):
    """Layer 1 over bit-lines with the row prefilter (bin_quad_item1): the
    count bound uses the column's largest |weight|, so uneven and mixed-sign
    weights only make it looser, never wrong.  scale 0.06: few rows pass the
    count test (listed rows, exact chains); 0.11: some columns list rows and
    some take the dense walk; 0.2 with a small bias: every row passes.
    Prefilter forced == probe's choice == prefilter off == oracle, bit for bit."""
    n, rows, layers = 1024, 3000, 3
    w = W.Workload("t", n, layers, rows, 32, 20, 0.35, bias, value=scale)
    off, cols, vals = W.images(w)
    y0 = O.CSR(rows, n, off, cols, vals)
    rng = np.random.default_rng(int(scale * 1000))
    lw = []
    for l in range(layers):
        o, c, v = W.layer_csr(w, l)
        v = rng.uniform(0.3 * scale, scale, v.shape) * np.where(rng.random(v.shape) < 0.15, -1.0, 1.0)
        lw.append(O.CSR(n, n, o, c, v))
    want = O.infer(lw, [bias] * layers, y0, w.ymax, precision=prec, threads=8)
    net = E.DeviceNetwork(n, 0, dtype)
    for m in lw:
        net.add_layer_csr(sm(m), bias)
    batch = net.upload_csr(rows, off, cols, vals)
    outs = []
    for pre in ("2", "1", "0"):  # 2: the prefilter walk whatever the probe says; 1: the probe picks; 0: dense
        monkeypatch.setenv("SDNN_PREFILTER", pre)
        r = net.run(batch, w.ymax, want_y=True)
        assert O.CSR(rows, n, *r.y).identical(want), (pre, dtype)
        outs.append(r)
    assert np.array_equal(outs[0].live_rows, outs[2].live_rows)
    net.close()


def test_forced_prune_pass_on_odd_sizes(monkeypatch):
    """SDNN_PRUNE_PASS=2 runs the prune pass (bound codes by bulk copy into
    shared memory, one bit per column) on every layer it applies to, whatever
    the samples say: odd neuron counts (the bulk copy moves the codes rounded
    up to 16 bytes), mixed-sign weights, live and dying rows, several tiles;
    forced == default == oracle, float64 and float32."""
    rng = np.random.default_rng(97)
    forced_pruned = 0
    for i in range(40):
        n = int(rng.integers(17, 200))
        layers, bias = [], []
        for _ in range(int(rng.integers(2, 6))):
            dens = rng.uniform(0.02, min(0.3, 30.0 / n))  # at most 32 per column (one batch of slots)
            m = np.where(rng.random((n, n)) < dens, rng.uniform(-0.3, 1.0, (n, n)), 0.0)
            while (m != 0).sum(axis=0).max() > 32:
                m[:, (m != 0).sum(axis=0).argmax()] *= rng.random(n) < 0.5
            layers.append(O.CSR.from_dense(m))
            bias.append(float(rng.uniform(-0.9, -0.05)))
        rows = int(rng.integers(1, 700))
        y = (rng.random((rows, n)) < rng.uniform(0.05, 0.5)).astype(np.float64)
        if i % 2:
            y *= rng.uniform(0.05, 1.5, y.shape)
        y0 = O.CSR.from_dense(y)
        for dtype, prec in (("f64", 64), ("f32", 32)):
            want = O.infer(layers, bias, y0, precision=prec)
            net = E.DeviceNetwork(n, 0, dtype)
            for m, b in zip(layers, bias):
                net.add_layer_csr(sm(m), b)
            batch = net.upload_csr(rows, y0.off, y0.cols, y0.vals)
            for mode in ("2", "1"):
                monkeypatch.setenv("SDNN_PRUNE_PASS", mode)
                r = net.run(batch, 32.0, want_y=True)
                assert O.CSR(rows, n, *r.y).identical(want), (i, dtype, mode)
                if mode == "2":
                    forced_pruned += r.pruned
            net.close()
    assert forced_pruned > 0
