"""Workload generators against the reference (CPU): the RadiX-Net
restatement (workloads.radixnet_ell, the K1 companion's weights) equals the
reference's own generator bit for bit."""

import sys

import numpy as np
import pytest

import goldens
from paper_1909_05631_b200 import _lib
from paper_1909_05631_b200 import workloads as W
from refpath import reference_path


def ell_to_csr(idx, n, value=0.0625):
    off = np.zeros(n + 1, np.int64)
    cols = np.zeros(idx.size, np.int64)
    vals = np.zeros(idx.size)
    ones = np.full(idx.size, value)
    _lib.check_gen(_lib.gen().sdnn_gen_ell_to_csr(n, n, idx.shape[1], _lib.ptr(np.ascontiguousarray(idx)),
                                                  _lib.ptr(ones), _lib.ptr(off), _lib.ptr(cols), _lib.ptr(vals)))
    return off, cols, vals


def test_radixnet_equals_the_reference_golden_network():
    """All 120 layers of the RadiX-Net (1024, 120) seed-42 network in
    tests/golden/radixnet.npz (written by the reference's generate_layers)."""
    r = goldens.radixnet()
    for l, want in enumerate(r["layers"]):
        off, cols, vals = ell_to_csr(W.radixnet_ell(1024, l), 1024)
        assert np.array_equal(off, want.off) and np.array_equal(cols, want.cols), l
        assert np.array_equal(vals, want.vals), l


@pytest.mark.skipif(reference_path() is None, reason="reference package not available")
@pytest.mark.parametrize("n,layers", [(4096, 10), (65536, 3)])
def test_radixnet_equals_the_reference_generator(n, layers):
    sys.path.insert(0, str(reference_path()))
    from sdnnbench.radixnet import GeneratorConfig, generate_layers
    it = generate_layers(GeneratorConfig.preset(n, 1920, rng_seed=W.RADIX_SEED))
    for l in range(layers):
        ref = next(it)
        off, cols, vals = ell_to_csr(W.radixnet_ell(n, l), n)
        assert np.array_equal(off, ref.row_offsets) and np.array_equal(cols, ref.col_indices), l
        assert np.array_equal(vals, ref.values), l


def test_radixnet_structure():
    for n in (1024, 65536):
        for l in (0, 5, 13):
            idx = W.radixnet_ell(n, l)
            assert idx.shape == (n, 32) and (np.diff(idx, axis=1) > 0).all()
            assert (np.bincount(idx.ravel(), minlength=n) == 32).all()
