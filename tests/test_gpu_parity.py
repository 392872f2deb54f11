"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

float64 must equal the reference bit for bit (golden vectors produced by
the reference itself, tests/golden) and the oracle's float64 instance.
float32 must equal the oracle's float32 instance bit for bit (same
algorithm, same order), and the category list must match the float64
reference wherever float32 keeps categories (the BASELINE configs); on the
fp32-hostile RadiX-Net workload the float32 tolerance is reported, not
asserted bitwise.
"""

import os

import numpy as np
import pytest

import goldens
from parity import assert_f32_within
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1909_05631_b200 import engine as E  # noqa: E402
from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.errors import ParameterError, ShapeError  # noqa: E402
from paper_1909_05631_b200.model import (  # noqa: E402
    FeatureBatch,
    LayerWeights,
    NetworkModel,
    SparseMatrix,
)


def sm(c: O.CSR) -> SparseMatrix:
    return SparseMatrix(c.n_rows, c.n_cols, c.off, c.cols, c.vals, check=False)


def model_of(layers, bias, n):
    return NetworkModel(n, tuple(LayerWeights(sm(w), float(b)) for w, b in zip(layers, bias)))


def as_csr(fb) -> O.CSR:
    d = fb.data
    return O.CSR(d.n_rows, d.n_cols, np.asarray(d.row_offsets), np.asarray(d.col_indices),
                 np.asarray(d.values))


@pytest.fixture
def env():
    saved = dict(os.environ)
    yield os.environ
    os.environ.clear()
    os.environ.update(saved)


# ------------------------------------------------------------ golden vectors

def test_general_goldens_f64_bit_exact():
    for i, t in enumerate(goldens.general()):
        model = model_of(t["layers"], t["bias"], t["n"])
        out = E.infer(model, FeatureBatch(sm(t["y0"])))
        assert as_csr(out).identical(t["y"]), f"instance {i}"
        assert np.array_equal(np.asarray(E.categorize(out).image_rows), t["cats"])


@pytest.mark.parametrize("cfg", [
    dict(mode="data_parallel", workers=2, devices=(0, 0)),
    dict(mode="data_parallel", workers=3, devices=(0, 0, 0)),
    dict(mode="pipeline", pipeline_stages=2),
    dict(mode="pipeline", workers=8),
])
def test_modes_bit_identical(cfg):
    for t in goldens.general()[:12]:
        model = model_of(t["layers"], t["bias"], t["n"])
        layers = len(t["layers"])
        c = dict(cfg)
        if c.get("pipeline_stages", 0) > layers:
            c["pipeline_stages"] = layers
        out = E.infer(model, FeatureBatch(sm(t["y0"])), E.InferenceConfig(**c))
        assert as_csr(out).identical(t["y"])


def test_general_goldens_f32_is_the_oracle_float_instance():
    for t in goldens.general():
        model = model_of(t["layers"], t["bias"], t["n"])
        out = E.infer(model, FeatureBatch(sm(t["y0"])), E.InferenceConfig(dtype="f32"))
        want = O.infer(t["layers"], t["bias"], t["y0"], precision=32)
        assert as_csr(out).identical(want)


def test_radixnet_digits_f64_bit_exact_and_f32_tolerance():
    """The reference's own acceptance workload (RadiX-Net 1024 + synthetic
    digits, golden from the reference).  float64: bit-exact.  float32: the
    oracle's float instance bit for bit, the same stored pattern and
    categories as the reference at 24 and 120 layers, and the final Y within
    the stated tolerance.  At 120 layers every survivor has saturated, so
    float32 meets north_star's 1e-5.  At 24 layers the values are in their
    unsaturated transient, where a bias of -0.3 against sums near 0.3
    cancels most significant bits: float32 then carries up to 0.59 relative
    error on 0.4 % of the entries (measured with the oracle's float
    instance, which our float32 path equals bit for bit), so this depth is
    outside the 1e-5 contract and the float64 path is the one to use."""
    r = goldens.radixnet()
    for L, y, cats, rtol in ((24, r["y24"], r["cats24"], 0.6), (120, r["y120"], r["cats120"], 1e-5)):
        model = model_of(r["layers"][:L], r["bias"][:L], r["n"])
        out = E.infer(model, FeatureBatch(sm(r["y0"])))
        assert as_csr(out).identical(y)
        out32 = E.infer(model, FeatureBatch(sm(r["y0"])), E.InferenceConfig(dtype="f32"))
        want32 = O.infer(r["layers"][:L], r["bias"][:L], r["y0"], precision=32)
        assert as_csr(out32).identical(want32)
        assert np.array_equal(O.categorize(as_csr(out32)), cats)
        worst = assert_f32_within(as_csr(out32), y, rtol)
        if L == 24:
            rel = np.abs(as_csr(out32).vals - y.vals) / np.abs(y.vals)
            assert (rel > 1e-5).mean() < 0.01 and worst > 1e-5


# -------------------------------------------------------------- KATs on GPU

def csr(dense):
    return sm(O.CSR.from_dense(np.asarray(dense, np.float64)))


class TestKAT:
    def test_spmm_identity_and_hand_sum(self):
        z = E.spmm(FeatureBatch(csr([[1.0, 0.0]])), csr(np.eye(2)))
        assert np.array_equal(z.to_dense(), [[1.0, 0.0]])
        z = E.spmm(FeatureBatch(csr([[1.0, 1.0]])), csr([[.5, .5], [.5, .5]]))
        assert np.array_equal(z.to_dense(), [[1.0, 1.0]])

    def test_spmm_empty_and_rectangular(self):
        y = SparseMatrix.empty(3, 4)
        w = csr(np.pad([[2.0]], ((0, 3), (0, 4))))  # 4 x 5
        z = E.spmm(FeatureBatch(y), w)
        assert z.shape == (3, 5) and z.nnz == 0

    def test_spmm_shape_mismatch(self):
        with pytest.raises(ShapeError):
            E.spmm(FeatureBatch(csr([[1.0, 0.0]])), csr(np.eye(3)))

    def test_exact_zero_dropped(self):
        z = E.spmm(FeatureBatch(csr([[1.0, 1.0]])), csr([[.5, 0], [-.5, 0]]))
        assert z.nnz == 0

    def test_ascending_inner_order(self, rng):
        yd = (rng.random((4, 40)) < 0.8).astype(float)
        wd = rng.uniform(-1, 1, size=(40, 7))
        z = E.spmm(FeatureBatch(csr(yd)), csr(wd))
        want = O.spmm(O.CSR.from_dense(yd), O.CSR.from_dense(wd))
        assert np.array_equal(z.to_dense(), want.to_dense())

    def test_bias_relu_clamp(self):
        assert E.apply_bias_relu_clamp(csr([[0.5]]), -0.3).values.tolist() == [0.5 + -0.3]
        assert E.apply_bias_relu_clamp(csr([[0.2]]), -0.3).nnz == 0
        assert E.apply_bias_relu_clamp(csr([[0.25]]), -0.25).nnz == 0
        assert E.apply_bias_relu_clamp(csr([[40.0]]), 0.0, 32.0).values.tolist() == [32.0]
        out = E.apply_bias_relu_clamp(csr([[0.5, 0.0]]), 0.4)
        assert out.col_indices.tolist() == [0] and out.values.tolist() == [0.5 + 0.4]

    def test_cancelled_entry_gets_no_bias(self):
        z = E.spmm(FeatureBatch(csr([[1.0, 1.0]])), csr([[.75, .5], [.25, -.5]]))
        assert z.col_indices.tolist() == [0]
        b = E.apply_bias_relu_clamp(z, 0.4)
        assert b.col_indices.tolist() == [0] and b.values.tolist() == [1.0 + 0.4]

    def test_worked_example_and_clamp(self):
        model = NetworkModel(2, (LayerWeights(csr([[.5, .5], [0, 1.0]]), -0.3),))
        out = E.infer(model, FeatureBatch(csr([[1.0, 0.0]])))
        assert np.array_equal(out.data.to_dense(), [[0.5 + -0.3, 0.5 + -0.3]])
        model = NetworkModel(1, (LayerWeights(csr([[5.0]]), 0.0),))
        assert E.infer(model, FeatureBatch(csr([[8.0]]))).data.values.tolist() == [32.0]

    def test_validation(self):
        model = NetworkModel(2, (LayerWeights(csr(np.eye(2)), 0.0),))
        with pytest.raises(ShapeError):
            E.infer(model, FeatureBatch(csr([[1.0, 0.0, 1.0]])))
        with pytest.raises(ParameterError):
            E.infer(model, FeatureBatch(csr([[1.0, 0.0]])),
                    E.InferenceConfig(mode="pipeline", pipeline_stages=5))

    def test_empty_and_single_row_batches(self):
        t = goldens.general()[0]
        model = model_of(t["layers"], t["bias"], t["n"])
        out = E.infer(model, FeatureBatch(SparseMatrix.empty(0, t["n"])))
        assert out.data.shape == (0, t["n"])
        out = E.infer(model, FeatureBatch(SparseMatrix.empty(5, t["n"])))
        assert out.data.nnz == 0 and out.data.n_rows == 5
        one = O.CSR(1, t["n"], t["y0"].off[:2], t["y0"].cols[:t["y0"].off[1]],
                    t["y0"].vals[:t["y0"].off[1]])
        got = as_csr(E.infer(model, FeatureBatch(sm(one))))
        assert got.identical(O.infer(t["layers"], t["bias"], one))

    def test_infer_timed(self):
        t = goldens.general()[3]
        model = model_of(t["layers"], t["bias"], t["n"])
        out, cats, sec = E.infer_timed(model, FeatureBatch(sm(t["y0"])))
        assert sec > 0 and as_csr(out).identical(t["y"])
        assert np.array_equal(np.asarray(cats.image_rows), t["cats"])


# ------------------------------------------------- kernel geometry variants

def permunion_case(n, layers, rows, value, p=0.35):
    side = int(round(n ** 0.5))
    w = W.Workload("t", n, layers, rows, side, int(side * 0.625), p, -0.45, value=value)
    off, cols, vals = W.images(w)
    return w, O.CSR(rows, n, off, cols, vals), [O.CSR(n, n, *W.layer_csr(w, l)) for l in range(layers)]


@pytest.mark.parametrize("jb,occ", [("1", "1"), ("7", "2"), ("100", "1"), ("4096", "3")])
@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_work_item_geometry(env, jb, occ, dtype, prec):
    """Output-block size and grid size change only the schedule, never bits."""
    env["SDNN_JB"] = jb
    env["SDNN_OCC"] = occ
    w, y0, layers = permunion_case(1024, 5, 97, 0.125)
    net = E.DeviceNetwork(w.n, 0, dtype)
    for l in range(w.layers):
        net.add_layer_csr(sm(layers[l]), w.bias)
    res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=4)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)
    assert res.live_rows[0] == np.count_nonzero(np.diff(y0.off))


@pytest.mark.parametrize("n", [4096, 16384, 65536])
def test_large_n_live_rows_f32_and_f64(n):
    rows = {4096: 48, 16384: 24, 65536: 8}[n]
    w, y0, layers = permunion_case(n, 6, rows, 0.125)
    for dtype, prec in (("f32", 32), ("f64", 64)):
        net = E.DeviceNetwork(w.n, 0, dtype)
        net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
        res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
        want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=8)
        assert O.CSR(y0.n_rows, w.n, *res.y).identical(want), dtype
        net.close()


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
@pytest.mark.parametrize("bits", ["1", "0"])
def test_live_row_compaction_is_bit_identical(env, dtype, prec, bits):
    """Rows die gradually here (2000 -> 1074 over 10 layers, every tile
    keeps some): repacking the live rows densely between layers (SURVEY.md
    7 step 3) only moves values, so every threshold -- never, whenever a
    tile is freed, the default, rarely -- gives the oracle's bits, through
    the device-side Y, the host assembly and multi-wave runs; bit-line
    (binary) and float first layers."""
    env["SDNN_BIN"] = bits
    env["SDNN_COMPACT_MIN"] = "1"  # this batch spans 8-16 tiles
    w, y0, layers = permunion_case(1024, 10, 2000, 0.125)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=8)
    cats = O.categorize(want)
    assert 0 < cats.size < 1500
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    batch = net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals)
    runs = {}
    for pct in (0, 1, 10, 60):
        net.set_compaction(pct)
        r = net.run(batch, w.ymax, want_y=True)
        assert O.CSR(y0.n_rows, w.n, *r.y).identical(want), pct
        assert np.array_equal(r.categories, cats), pct
        runs[pct] = r
    assert runs[0].compactions == 0
    assert runs[1].compactions >= 2 and runs[10].compactions >= 1
    for r in runs.values():
        assert np.array_equal(r.live_rows, runs[0].live_rows)
    net.set_compaction(1)
    env["SDNN_HOST_Y"] = "1"
    host = net.run(batch, w.ymax, want_y=True)
    assert host.compactions >= 2
    assert all(np.array_equal(a, b) for a, b in zip(host.y, runs[0].y))
    env["SDNN_HOST_Y"] = "0"
    env["SDNN_WAVE_ROWS"] = "700"
    waves = net.run(batch, w.ymax, want_y=True)
    assert waves.compactions >= 1
    assert all(np.array_equal(a, b) for a, b in zip(waves.y, runs[0].y))
    net.close()


def _random_instance(rng):
    """A general instance in the spirit of the reference's helpers.random_model /
    random_batch (tests/helpers.py:31-50): mixed-sign weights avoiding 0,
    variable degree, biases that may be positive, binary or real inputs."""
    n = int(rng.integers(8, 97))
    layers, bias = [], []
    for _ in range(int(rng.integers(1, 9))):
        dens = rng.uniform(0.02, 0.3)
        w = np.where(rng.random((n, n)) < dens, rng.uniform(-1, 1, (n, n)), 0.0)
        layers.append(O.CSR.from_dense(w))
        bias.append(float(rng.uniform(-0.5, 0.2)))
    rows = int(rng.integers(0, 300))
    y = (rng.random((rows, n)) < rng.uniform(0.05, 0.6)).astype(np.float64)
    if rng.random() < 0.5:
        y *= rng.uniform(0.1, 2.0, y.shape)  # real-valued inputs: float densify path
    return n, layers, bias, O.CSR.from_dense(y)


@pytest.mark.parametrize("compact", ["0", "1"])
def test_random_general_instances_f64_bit_exact(env, compact):
    """200 random general instances (acceptance criterion 4's shape,
    test_acceptance.py:231-250) through the C ABI in float64 against the
    oracle bit for bit (the oracle is pinned to the reference by the
    goldens), and in float32 against its float instance; with live-row
    compaction off, and forced whenever it frees a tile."""
    env["SDNN_COMPACT"] = compact
    env["SDNN_COMPACT_MIN"] = "1"
    rng = np.random.default_rng(20261020)
    for i in range(200):
        n, layers, bias, y0 = _random_instance(rng)
        for dtype, prec in (("f64", 64), ("f32", 32)):
            if prec == 32 and i % 4:
                continue
            net = E.DeviceNetwork(n, 0, dtype)
            for w, b in zip(layers, bias):
                net.add_layer_csr(sm(w), b)
            res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), 32.0, want_y=True)
            want = O.infer(layers, bias, y0, precision=prec)
            assert O.CSR(y0.n_rows, n, *res.y).identical(want), (i, dtype)
            assert np.array_equal(res.categories, O.categorize(want)), (i, dtype)
            net.close()


def test_wave_splitting_does_not_change_bits(env):
    env["SDNN_WAVE_ROWS"] = "37"
    w, y0, layers = permunion_case(1024, 4, 200, 0.125)
    net = E.DeviceNetwork(w.n, 0, "f64")
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    want = O.infer(layers, [w.bias] * w.layers, y0, threads=4)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_device_y_matches_host_assembly_and_oracle(env, dtype, prec):
    """Final Y materialised on the device (row-ordered int64/float64 CSR,
    SURVEY 8f rank 2) == the host assembly path == multi-wave runs == the
    oracle, on a workload where some rows and whole tiles die."""
    w, y0, layers = permunion_case(4096, 5, 700, 0.12)  # 20 of 700 rows survive
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=8)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    batch = net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals)
    dev = net.run(batch, w.ymax, want_y=True)
    assert O.CSR(y0.n_rows, w.n, *dev.y).identical(want)
    assert 0 < dev.categories.size < y0.n_rows
    env["SDNN_HOST_Y"] = "1"
    host = net.run(batch, w.ymax, want_y=True)
    env["SDNN_HOST_Y"] = "0"
    env["SDNN_WAVE_ROWS"] = "300"
    waves = net.run(batch, w.ymax, want_y=True)
    for r in (host, waves):
        assert all(np.array_equal(a, b) for a, b in zip(r.y, dev.y))
    net.close()


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
@pytest.mark.parametrize("waves", ["0", "150"])
def test_pipeline_handoff_on_device(env, dtype, prec, waves):
    """Layer ranges chained through sdnn_batch_from_result (device Y of one
    range -> staged batch of the next, no host round trip) == one run over
    all layers == the oracle; with waves the result is host-assembled and
    the hand-off uploads it instead."""
    if waves != "0":
        env["SDNN_WAVE_ROWS"] = waves
    w, y0, layers = permunion_case(4096, 7, 700, 0.12)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=8)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    other = E.DeviceNetwork(w.n, 0, dtype)  # a second stage network (same GPU here)
    other.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    b = net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals)
    b = net.run_to_batch(b, w.ymax, 0, 2)
    b = net.run_to_batch(b, w.ymax, 2, 3, target=other)
    res = other.run(b, w.ymax, 5, 2, want_y=True)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)
    with pytest.raises(ShapeError):
        small = E.DeviceNetwork(1024, 0, dtype)
        try:
            net.run_to_batch(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, 0, 1, target=small)
        finally:
            small.close()
    other.close()
    net.close()


def test_e2e_host_call_matches_device_resident_run():
    w, y0, layers = permunion_case(1024, 8, 300, 0.125)
    net = E.DeviceNetwork(w.n, 0, "f32")
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    a = net.infer_host(sm(y0))
    b = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    assert np.array_equal(a.categories, b.categories)
    assert all(np.array_equal(x, y) for x, y in zip(a.y, b.y))


@pytest.mark.parametrize("segments", [1, 2, 3, 7, 1000])
@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_streamed_e2e_segments_are_bit_identical(segments, dtype, prec):
    """sdnn_infer_streamed: Y0 uploaded in row segments by a second host
    thread while earlier segments run; every segment count gives the
    oracle's result bit for bit.  One segment holds real values (float
    tiles), the others are binary (bit-line tiles), and a block of empty
    rows sits in the middle."""
    w, y0, layers = permunion_case(1024, 6, 300, 0.125)
    vals = y0.vals.copy()
    lo, hi = int(y0.off[200]), int(y0.off[260])
    vals[lo:hi] = 0.75
    off = y0.off.copy()
    cols = y0.cols.copy()
    # rows 100..139 empty
    keep = np.ones(cols.size, bool)
    keep[int(off[100]):int(off[140])] = False
    counts = np.diff(off)
    counts[100:140] = 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    cols, vals = cols[keep], vals[keep]
    yy = O.CSR(y0.n_rows, w.n, off, cols, vals)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    got = net.infer_csr(yy.n_rows, off, cols, vals, w.ymax, want_y=True, segments=segments)
    assert got.segments == min(segments, yy.n_rows)
    want = O.infer(layers, [w.bias] * w.layers, yy, precision=prec, threads=8)
    assert O.CSR(yy.n_rows, w.n, *got.y).identical(want)
    assert np.array_equal(got.categories, O.categorize(want))
    ref = net.run(net.upload_csr(yy.n_rows, off, cols, vals), w.ymax)
    assert np.array_equal(got.live_rows, ref.live_rows)
    cats_only = net.infer_csr(yy.n_rows, off, cols, vals, w.ymax, want_y=False, segments=segments)
    assert cats_only.y is None and np.array_equal(cats_only.categories, got.categories)
    assert cats_only.h2d_bytes > 0
    net.close()


def test_streamed_e2e_empty_batch_and_bad_input():
    w, y0, layers = permunion_case(1024, 2, 10, 0.125)
    net = E.DeviceNetwork(w.n, 0, "f32")
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    r = net.infer_csr(0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0), w.ymax)
    assert r.categories.size == 0 and r.y[0].tolist() == [0]
    bad = y0.cols.copy()
    bad[-1] = w.n  # column outside the row: ParameterError from the producer thread
    with pytest.raises(ParameterError):
        net.infer_csr(y0.n_rows, y0.off, bad, y0.vals, w.ymax, segments=3)
    # the handle stays usable after the failed call
    ok = net.infer_csr(y0.n_rows, y0.off, y0.cols, y0.vals, w.ymax, segments=3)
    assert np.array_equal(ok.categories, O.categorize(O.infer(layers, [w.bias] * 2, y0, precision=32)))
    net.close()


# ------------------------------------------------ flagship width, full batch
# (the BASELINE configs as specified: tests/test_gpu_configs.py)

def test_c4_shape_full_batch_row_sample_consistency():
    """Flagship width at full batch: rows are independent, so a 64-row
    sample run alone (and by the oracle) must agree with the full run."""
    w = W.CONFIGS["K2"].with_(layers=8)
    off, cols, vals = W.images(w)
    net = E.DeviceNetwork(w.n, 0, "f32")
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    full = net.run(net.upload_csr(w.batch, off, cols, vals), w.ymax)
    assert full.live_rows[0] == w.batch
    rng = np.random.default_rng(3)
    sample = np.sort(rng.choice(w.batch, 64, replace=False))
    s_off = np.zeros(65, np.int64)
    np.cumsum(np.diff(off)[sample], out=s_off[1:])
    s_cols = np.concatenate([cols[off[r]:off[r + 1]] for r in sample])
    s_vals = np.concatenate([vals[off[r]:off[r + 1]] for r in sample])
    part = net.run(net.upload_csr(64, s_off, s_cols, s_vals), w.ymax, want_y=True)
    in_full = np.isin(sample + 1, full.categories)
    assert np.array_equal(np.nonzero(in_full)[0] + 1, part.categories)
    layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    want = O.infer(layers, [w.bias] * w.layers, O.CSR(64, w.n, s_off, s_cols, s_vals),
                   precision=32, threads=os.cpu_count() or 8)
    assert O.CSR(64, w.n, *part.y).identical(want)


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_real_valued_inputs_use_the_float_tiles(dtype, prec):
    """Y0 with arbitrary values (not the binary images): values are uploaded
    and expanded into float tiles; results must match the oracle bit for bit."""
    w, y0, layers = permunion_case(1024, 6, 300, 0.125)
    rng = np.random.default_rng(11)
    vals = rng.uniform(0.05, 2.0, size=y0.vals.size)
    y0 = O.CSR(y0.n_rows, y0.n_cols, y0.off, y0.cols, vals)
    net = E.DeviceNetwork(w.n, 0, dtype)
    for l in range(w.layers):
        net.add_layer_csr(sm(layers[l]), w.bias)
    batch = net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals)
    assert batch.h2d_bytes >= y0.vals.size * (8 if dtype == "f64" else 4)
    res = net.run(batch, w.ymax, want_y=True)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=4)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)


def test_binary_inputs_bit_tiles_and_float_tiles_agree(env):
    """The binary-image fast path (bit-line tiles for layer 1) and the
    general float tiles give identical bits."""
    t_cases = goldens.general()[:16]
    outs = []
    for flag in ("1", "0"):
        env["SDNN_BIN"] = flag
        res = []
        for t in t_cases:
            model = model_of(t["layers"], t["bias"], t["n"])
            res.append(as_csr(E.infer(model, FeatureBatch(sm(t["y0"])))))
        outs.append(res)
    for a, b, t in zip(outs[0], outs[1], t_cases):
        assert a.identical(b) and a.identical(t["y"])


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_non_finite_inputs_take_the_zero_fill_gather(dtype, prec):
    """Y0 holding inf (and, in float32, values that overflow to inf) must not
    leak into rows whose sector is dead: the host switches the gather to the
    zero-filling variant and the result equals the oracle bit for bit."""
    w, y0, layers = permunion_case(1024, 4, 300, 0.125)
    rng = np.random.default_rng(12)
    vals = rng.uniform(0.05, 2.0, size=y0.vals.size)
    hit = rng.choice(vals.size, size=40, replace=False)
    vals[hit[:20]] = np.inf
    vals[hit[20:]] = 1e300  # finite in float64, inf once rounded to float32
    y0 = O.CSR(y0.n_rows, y0.n_cols, y0.off, y0.cols, vals)
    net = E.DeviceNetwork(w.n, 0, dtype)
    for l in range(w.layers):
        net.add_layer_csr(sm(layers[l]), w.bias)
    res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=4)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)


def test_zero_fill_and_keep_gathers_agree(env):
    """Both dead-lane treatments of the gather (zero-filled registers, or kept
    registers with weight 0) give the reference's bits."""
    for flag in ("1", "0"):
        env["SDNN_ZFILL"] = flag
        for t in goldens.general()[:16]:
            model = model_of(t["layers"], t["bias"], t["n"])
            assert as_csr(E.infer(model, FeatureBatch(sm(t["y0"])))).identical(t["y"])


def test_device_weight_ingest_general_csr():
    """CSR -> ELL on the device (sort by column, ascending rows kept): column
    degrees 0..~70 (padded ELL of 96 slots, several batches per column),
    empty rows and columns, mixed signs; bit-exact against the oracle."""
    rng = np.random.default_rng(21)
    n = 300
    dense = np.zeros((n, n))
    for j in range(n):
        deg = int(rng.integers(0, 71)) if j % 7 else 0
        rows = rng.choice(n, size=deg, replace=False)
        dense[rows, j] = rng.uniform(-0.4, 0.6, size=deg)
    dense[5, :] = 0.0  # an empty input row
    layers = [O.CSR.from_dense(dense), O.CSR.from_dense(dense.T.copy())]
    y = np.where(rng.random((400, n)) < 0.2, rng.uniform(0.1, 2.0, (400, n)), 0.0)
    y0 = O.CSR.from_dense(y)
    bias = [-0.05, 0.1]
    for dtype, prec in (("f64", 64), ("f32", 32)):
        net = E.DeviceNetwork(n, 0, dtype)
        for lw, b in zip(layers, bias):
            net.add_layer_csr(sm(lw), b)
        res = net.run(net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), 32.0, want_y=True)
        want = O.infer(layers, bias, y0, precision=prec, threads=4)
        assert O.CSR(y0.n_rows, n, *res.y).identical(want)
        net.close()


def test_device_weight_ingest_rejects_bad_csr():
    net = E.DeviceNetwork(4, 0, "f64")
    bad_col = SparseMatrix(4, 4, np.array([0, 1, 1, 1, 1]), np.array([4]), np.array([1.0]), check=False)
    with pytest.raises(ParameterError):
        net.add_layer_csr(bad_col, 0.0)
    bad_off = SparseMatrix(4, 4, np.array([0, 2, 1, 2, 2]), np.array([0, 1]), np.array([1.0, 1.0]), check=False)
    with pytest.raises(ParameterError):
        net.add_layer_csr(bad_off, 0.0)
    net.close()


def test_layer_buffers_replicate_a_network():
    """The weight-replication path of the multi-GPU bench (rank 0 generates,
    the others receive the device ELL): a network whose layers were filled
    through the exposed device buffers runs bit-identically to the source."""
    w, y0, _ = permunion_case(1024, 5, 300, 0.125)
    for dtype in ("f32", "f64"):
        src = E.DeviceNetwork(w.n, 0, dtype)
        src.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
        dst = E.DeviceNetwork(w.n, 0, dtype)
        dst.add_layers_uninit(w.layers, w.width, w.bias)
        for l in range(w.layers):
            si, sv = src.layer_tensors(l)
            di, dv = dst.layer_tensors(l)
            assert si.shape == di.shape and sv.dtype == dv.dtype
            di.copy_(si)
            dv.copy_(sv)
        torch.cuda.synchronize()
        a = src.run(src.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
        b = dst.run(dst.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
        assert all(np.array_equal(x, y) for x, y in zip(a.y, b.y))
        assert np.array_equal(a.categories, b.categories)
        src.close()
        dst.close()


# ------------------------------------------- image preprocessing (8f rank 4)

def test_device_resize_matches_reference_golden():
    """sdnn_batch_from_images == the reference's resize_threshold_flatten on
    images holding values within 1e-9 of the threshold, at every side."""
    from paper_1909_05631_b200 import ingest as I

    z = np.load(goldens.GOLDEN / "images.npz")
    for t in (int(v) for v in z["sides"]):
        fb = I.resize_threshold_flatten(z["pixels"], t)
        d = fb.data
        assert np.array_equal(np.asarray(d.row_offsets), z[f"off{t}"]), t
        want = np.unpackbits(z[f"mask{t}"], axis=1)[:, :t * t].astype(bool)
        rows = np.repeat(np.arange(want.shape[0]), np.diff(z[f"off{t}"]))
        got = np.zeros_like(want)
        got[rows, np.asarray(d.col_indices)] = True
        assert np.array_equal(got, want), t
        assert np.all(np.asarray(d.values) == 1.0)


@pytest.mark.parametrize("side,t", [(28, 32), (28, 256), (64, 32), (17, 128), (40, 64)])
def test_device_resize_matches_oracle_other_sides(side, t):
    from paper_1909_05631_b200 import ingest as I

    rng = np.random.default_rng(side * 1000 + t)
    pix = rng.integers(0, 256, size=(37, side, side), dtype=np.uint8)
    pix[::3] = (pix[::3] > 128) * 255  # hard edges: exact 0.5 crossings
    want = O.resize_threshold_flatten(pix, t)
    d = I.resize_threshold_flatten(pix, t).data
    assert np.array_equal(np.asarray(d.row_offsets), want.off)
    assert np.array_equal(np.asarray(d.col_indices), want.cols)


def test_device_resize_errors_and_empty():
    from paper_1909_05631_b200 import ingest as I

    with pytest.raises(ParameterError):
        I.resize_threshold_flatten(np.zeros((2, 28, 28), np.uint8), 100)
    net = E.DeviceNetwork(1024, 0, "f32")
    with pytest.raises(ShapeError):
        net.upload_images(np.zeros((2, 28, 28), np.uint8), 64)
    b = net.upload_images(np.zeros((0, 28, 28), np.uint8), 32)
    off, cols, _ = b.to_csr()
    assert off.tolist() == [0] and cols.size == 0
    b.close()
    net.close()


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_images_to_categories_on_device(dtype, prec):
    """Raw images -> device resize -> all layers: the same result as the
    reference-format host batch (oracle resize + oracle engine)."""
    z = np.load(goldens.GOLDEN / "images.npz")
    w = W.CONFIGS["C1"].with_(layers=6, batch=int(z["pixels"].shape[0]), value=0.1)
    layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    y0 = O.resize_threshold_flatten(z["pixels"], 32)
    want = O.infer(layers, [w.bias] * w.layers, y0, w.ymax, precision=prec, threads=4)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    res = net.run(net.upload_images(z["pixels"], 32), w.ymax, want_y=True)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)
    assert np.array_equal(res.categories, O.categorize(want))
    net.close()


# ------------------------------------------- multi-GPU handle (C ABI group)

@pytest.mark.parametrize("devices", [(0,), (0, 0), (0, 0, 0)])
@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_group_handle_matches_one_gpu(devices, dtype, prec):
    """sdnn_open_devices / sdnn_group_*: weights converted on the first
    member and copied device to device, the batch split into ceil(B/G)-row
    blocks run concurrently from one host thread per member, merged in row
    order: bit-identical to the oracle (and so to one GPU), with the
    categories shifted by each block's first row."""
    w, y0, layers = permunion_case(1024, 6, 517, 0.125)
    g = E.DeviceGroup(w.n, devices, dtype)
    for l in range(w.layers):
        g.add_layer_csr(sm(layers[l]), w.bias)
    res = g.infer_csr(y0.n_rows, y0.off, y0.cols, y0.vals, w.ymax, want_y=True)
    want = O.infer(layers, [w.bias] * w.layers, y0, precision=prec, threads=4)
    assert O.CSR(y0.n_rows, w.n, *res.y).identical(want)
    assert np.array_equal(res.categories, O.categorize(want))
    assert res.live_rows[0] == np.count_nonzero(np.diff(y0.off))
    r2 = g.infer_csr(y0.n_rows, y0.off, y0.cols, y0.vals, w.ymax, want_y=False)
    assert np.array_equal(r2.categories, res.categories)
    g.close()
    g = E.DeviceGroup(w.n, devices, dtype)  # perm-union layers generated once, replicated
    g.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    r3 = g.infer_csr(y0.n_rows, y0.off, y0.cols, y0.vals, w.ymax, want_y=True)
    assert O.CSR(y0.n_rows, w.n, *r3.y).identical(want)
    empty = g.infer_csr(0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0), w.ymax)
    assert empty.categories.size == 0
    g.close()


# ------------------------------------ K1: RadiX-Net at flagship width (65536)

@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
def test_k1_radixnet_flagship_width(dtype, prec):
    """The reference's own network family at N=65536 (RadiX-Net preset,
    seed 42, weights pinned to the reference generator by
    tests/test_workloads.py) fed digit-like images resized to 256x256 on
    the device: 24 rows through 24 layers against the oracle's same
    precision instance (float64 = the reference's arithmetic), via both
    the device ingest and the host CSR."""
    n, L, rows = 65536, 24, 24
    w = W.CONFIGS["K1"].with_(layers=L, batch=rows)
    pix = W.stroke_images(rows)
    y0 = O.resize_threshold_flatten(pix, 256)
    layers = [O.CSR(n, n, *c) for c in
              (_ell_csr(W.radixnet_ell(n, l), n, w.value) for l in range(L))]
    want = O.infer(layers, [w.bias] * L, y0, precision=prec, threads=os.cpu_count() or 8)
    assert want.nnz > 0
    net = E.DeviceNetwork(n, 0, dtype)
    net.add_radixnet_layers(w.weight_seed, 0, L, w.value, w.bias)
    b = net.upload_images(pix, 256)
    off, cols, vals = b.to_csr()
    assert np.array_equal(off, y0.off) and np.array_equal(cols, y0.cols)
    res = net.run(b, w.ymax, want_y=True)
    assert O.CSR(rows, n, *res.y).identical(want)
    res2 = net.run(net.upload_csr(rows, y0.off, y0.cols, y0.vals), w.ymax, want_y=True)
    assert O.CSR(rows, n, *res2.y).identical(want)
    net.close()


def _ell_csr(idx, n, value):
    from paper_1909_05631_b200 import _lib
    off = np.zeros(n + 1, np.int64)
    cols = np.zeros(idx.size, np.int64)
    vals = np.zeros(idx.size)
    _lib.check_gen(_lib.gen().sdnn_gen_ell_to_csr(n, n, idx.shape[1], _lib.ptr(idx),
                                                  _lib.ptr(np.full(idx.size, value)), _lib.ptr(off),
                                                  _lib.ptr(cols), _lib.ptr(vals)))
    return off, cols, vals


@pytest.mark.parametrize("dtype,prec", [("f64", 64), ("f32", 32)])
@pytest.mark.parametrize("n,rows,p", [(1024, 700, 0.35), (4096, 300, 0.05), (1000, 513, 0.7)])
def test_both_bit_line_builders_agree(env, n, rows, p, dtype, prec):
    """Binary Y0 -> quad / oct bit-lines by densify_quad_kernel (a span of
    lines in shared memory, one row stream per warp: SDNN_DENSIFY_QUAD=2) and
    by densify_bin_kernel (0); the default picks by row density.  Same bits,
    equal to the oracle, for dense, sparse and ragged batches (empty rows,
    a neuron count that is no multiple of 32, a last tile with few rows)."""
    rng = np.random.default_rng(n + rows)
    layers, bias = [], []
    for _ in range(3):
        m = np.zeros((n, n))
        for j in range(n):
            m[rng.choice(n, 24, replace=False), j] = rng.uniform(0.05, 0.2, 24)
        layers.append(O.CSR.from_dense(m))
        bias.append(-0.3)
    y = (rng.random((rows, n)) < p).astype(np.float64)
    y[rng.choice(rows, rows // 7, replace=False)] = 0.0  # empty rows never enter a tile
    y0 = O.CSR.from_dense(y)
    want = O.infer(layers, bias, y0, precision=prec, threads=8)
    net = E.DeviceNetwork(n, 0, dtype)
    for m, b in zip(layers, bias):
        net.add_layer_csr(sm(m), b)
    batch = net.upload_csr(rows, y0.off, y0.cols, y0.vals)
    for mode in ("2", "0", "1"):
        env["SDNN_DENSIFY_QUAD"] = mode
        r = net.run(batch, 32.0, want_y=True)
        assert O.CSR(rows, n, *r.y).identical(want), (mode, dtype)
        assert np.array_equal(r.categories, O.categorize(want)), (mode, dtype)
    net.close()
