"""CPU-side checks of the C ABI boundary and the host generators (no GPU)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_1909_05631_b200 import _lib
from paper_1909_05631_b200 import workloads as W

ROOT = Path(__file__).resolve().parent.parent


def declared(header: str):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sdnn_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared("sdnn.h") + declared("sdnn_gen.h")
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES + _lib.GEN_SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_generator_library_exports():
    g = _lib.gen()
    for name in declared("sdnn_gen.h"):
        assert hasattr(g, name)


def test_library_loads_without_gpu_and_reports_no_device():
    assert _lib.lib().sdnn_version() == 1
    assert _lib.device_count() >= 0


@pytest.mark.parametrize("n,width", [(64, 32), (1024, 32), (37, 5), (4096, 32)])
def test_permunion_is_exactly_regular(n, width):
    w = W.Workload("t", n, 2, 1, 8, 4, 0.5, -0.3, width=width)
    for layer in range(2):
        idx = W.layer_ell(w, layer)
        assert idx.shape == (n, width)
        assert (np.diff(idx, axis=1) > 0).all()          # ascending, no collision
        assert (np.bincount(idx.ravel(), minlength=n) == width).all()  # row degree
        off, cols, vals = W.layer_csr(w, layer)
        assert (np.diff(off) == width).all()
        for i in range(0, n, max(1, n // 16)):            # transpose consistency
            js = cols[off[i]:off[i + 1]]
            assert (np.diff(js) > 0).all()
            assert all(i in idx[j] for j in js)


def test_permunion_is_seeded_and_layer_independent():
    w = W.CONFIGS["C1"]
    a = W.layer_ell(w, 5)
    b = W.layer_ell(w, 5)
    c = W.layer_ell(w, 6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    g = _lib.gen()
    many = np.zeros((3, w.n, w.width), np.int32)
    _lib.check_gen(g.sdnn_gen_permunion_ell_layers(w.weight_seed, 4, 3, w.n, w.width, 3, _lib.ptr(many)))
    assert np.array_equal(many[1], a)


def test_images_follow_the_config():
    w = W.CONFIGS["C2"].with_(batch=300)
    off, cols, vals = W.images(w)
    side, s = w.side, w.square
    o = (side - s) // 2
    r, c = cols // side, cols % side
    assert ((r >= o) & (r < o + s) & (c >= o) & (c < o + s)).all()
    assert (vals == 1.0).all()
    mean = off[-1] / w.batch
    assert abs(mean - w.p * s * s) < 0.05 * w.p * s * s
    for i in range(w.batch):
        assert (np.diff(cols[off[i]:off[i + 1]]) > 0).all()
    o2, c2, _ = W.images(w, n_rows=100, row0=200)
    assert np.array_equal(c2, cols[off[200]:off[300]])


def test_nominal_edges_match_challenge_rate_arithmetic():
    # challenge.rate: inputs x connections / seconds (challenge.py:131-135)
    w = W.CONFIGS["C1"]
    assert w.edges == 60000 * 1024 * 32 * 120
    assert W.CONFIGS["C4"].edges == 60000 * 65536 * 32 * 1920


@pytest.mark.parametrize("m", [0, 5, 16, 17, 1000, 4099])
def test_host_narrowing_of_y0_columns(m):
    """The upload's host pass (csrc/sdnn_host.c: AVX2, non-temporal staging
    stores): int64 columns -> uint16, range check, binary-value check; equal
    to the plain conversion for every length (16-entry blocks + tail)."""
    import ctypes

    lib = _lib.lib()
    f = lib.sdnn_host_narrow16
    f.restype = None
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int64] + [ctypes.POINTER(ctypes.c_int)] * 2
    rng = np.random.default_rng(m)
    n = 65536
    cols = rng.integers(0, n, m).astype(np.int64)
    vals = np.ones(m)
    raw = np.zeros(m + 32, np.uint16)
    off = (-raw.ctypes.data % 32) // 2  # 32-byte aligned destination
    dst = raw[off:off + m]

    def run(c, v):
        bad, binary = ctypes.c_int(0), ctypes.c_int(1)
        f(c.ctypes.data, v.ctypes.data, dst.ctypes.data, m, n, ctypes.byref(bad), ctypes.byref(binary))
        return bad.value, binary.value

    assert run(cols, vals) == (0, 1)
    assert np.array_equal(dst, cols.astype(np.uint16))
    if m:
        for at in (0, m - 1, m // 2):
            v2 = vals.copy()
            v2[at] = 0.5
            assert run(cols, v2) == (0, 0)
            v2[at] = np.nan
            assert run(cols, v2) == (0, 0)
            for badc in (-1, n, 1 << 40):
                c2 = cols.copy()
                c2[at] = badc
                assert run(c2, vals)[0] == 1


def test_null_handles_are_parameter_errors_without_a_gpu():
    """Entry points that take a handle reject NULL with the parameter code
    (2 -> ParameterError) before touching a device."""
    import ctypes

    lib = _lib.lib()
    n = ctypes.c_int64()
    assert lib.sdnn_net_set_compaction(None, 10) == 2
    assert lib.sdnn_net_set_layer_timing(None, 1) == 2
    assert lib.sdnn_result_compactions(None, ctypes.byref(n)) == 2
    assert lib.sdnn_result_launches(None, ctypes.byref(n)) == 2
    assert lib.sdnn_result_n_categories(None, ctypes.byref(n)) == 2
