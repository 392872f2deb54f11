"""Pin the CPU oracle before trusting it (CPU only, no GPU).

* Known-answer tests restated from the reference's own suite
  (test_engine.py:30-160, test_acceptance.py:253-299).
* Golden vectors produced by running the reference engine
  (tests/golden/make_golden.py): 49 general instances and the
  RadiX-Net + digits acceptance workload, bit for bit.
* The C Gustavson restatement agrees with the numpy dense-oracle
  restatement (challenge.py:70-112).
"""

import numpy as np
import pytest

import goldens
from oracle import oracle as O
from oracle.oracle import CSR


def csr(dense):
    return CSR.from_dense(np.asarray(dense, np.float64))


def wcsr(triples, n_rows, n_cols):
    d = np.zeros((n_rows, n_cols))
    for r, c, v in triples:  # 1-based like model.Triple
        d[r - 1, c - 1] = v
    return CSR.from_dense(d)


class TestSpmmKAT:
    def test_identity(self):  # test_engine.py:31-35
        z = O.spmm(csr([[1.0, 0.0]]), wcsr([(1, 1, 1.0), (2, 2, 1.0)], 2, 2))
        assert np.array_equal(z.to_dense(), [[1.0, 0.0]])

    def test_hand_sum(self):  # :37-44
        w = wcsr([(1, 1, .5), (1, 2, .5), (2, 1, .5), (2, 2, .5)], 2, 2)
        assert np.array_equal(O.spmm(csr([[1.0, 1.0]]), w).to_dense(), [[1.0, 1.0]])

    def test_empty_input(self):  # :46-51
        y = CSR(3, 4, np.zeros(4, np.int64), np.empty(0, np.int64), np.empty(0))
        z = O.spmm(y, wcsr([(1, 1, 2.0)], 4, 5))
        assert (z.n_rows, z.n_cols, z.nnz) == (3, 5, 0)

    def test_exact_zero_dropped(self):  # :59-63
        z = O.spmm(csr([[1.0, 1.0]]), wcsr([(1, 1, .5), (2, 1, -.5)], 2, 2))
        assert z.nnz == 0

    def test_ascending_inner_order(self, rng):  # :65-80
        yd = (rng.random((4, 40)) < 0.8).astype(float)
        wd = rng.uniform(-1, 1, size=(40, 7))
        z = O.spmm(csr(yd), CSR.from_dense(wd))
        want = np.zeros((4, 7))
        for i in range(4):
            for j in range(7):
                acc = 0.0
                for k in range(40):
                    acc += yd[i, k] * wd[k, j]
                want[i, j] = acc
        got = z.to_dense()
        assert np.array_equal(got[got != 0], want[got != 0])


class TestBiasReluClampKAT:  # test_engine.py:83-109
    def test_bias_applied(self):
        assert O.bias_relu_clamp(csr([[0.5]]), -0.3).vals.tolist() == [0.5 + -0.3]

    def test_negative_removed(self):
        assert O.bias_relu_clamp(csr([[0.2]]), -0.3).nnz == 0

    def test_exact_zero_removed(self):
        assert O.bias_relu_clamp(csr([[0.25]]), -0.25).nnz == 0

    def test_clamp(self):
        assert O.bias_relu_clamp(csr([[40.0]]), 0.0, 32.0).vals.tolist() == [32.0]

    def test_unstored_positions_get_no_bias(self):
        out = O.bias_relu_clamp(csr([[0.5, 0.0]]), 0.4)
        assert out.cols.tolist() == [0] and out.vals.tolist() == [0.5 + 0.4]


class TestInferKAT:
    def test_worked_example(self):  # test_engine.py:112-131
        w = wcsr([(1, 1, .5), (1, 2, .5), (2, 2, 1.0)], 2, 2)
        out = O.infer([w], [-0.3], csr([[1.0, 0.0]]))
        want = 0.5 + -0.3
        assert np.array_equal(out.to_dense(), [[want, want]])

    def test_clamp_40_to_32(self):  # test_acceptance.py:278-283
        z = O.spmm(csr([[8.0]]), wcsr([(1, 1, 5.0)], 1, 1))
        assert O.bias_relu_clamp(z, 0.0, 32.0).vals.tolist() == [32.0]

    def test_cancelled_entry_gets_no_bias(self):  # test_acceptance.py:285-296
        w = wcsr([(1, 1, .75), (1, 2, .5), (2, 1, .25), (2, 2, -.5)], 2, 2)
        z = O.spmm(csr([[1.0, 1.0]]), w)
        assert z.cols.tolist() == [0]
        b = O.bias_relu_clamp(z, 0.4)
        assert b.cols.tolist() == [0] and b.vals.tolist() == [1.0 + 0.4]

    def test_zero_input_stays_zero(self):
        w = CSR.from_dense(np.eye(8) * 0.5)
        y = CSR(5, 8, np.zeros(6, np.int64), np.empty(0, np.int64), np.empty(0))
        assert O.infer([w] * 4, [0.1] * 4, y).nnz == 0


class TestGoldens:
    def test_general_instances_bit_exact(self):
        cases = goldens.general()
        assert len(cases) >= 40
        for i, t in enumerate(cases):
            out = O.infer(t["layers"], t["bias"], t["y0"])
            assert out.identical(t["y"]), f"instance {i}"
            assert np.array_equal(O.categorize(out), t["cats"])

    @pytest.mark.parametrize("threads,tile", [(2, 0), (8, 0), (3, 7), (4, 1)])
    def test_tiling_and_threads_do_not_change_bits(self, threads, tile):
        for t in goldens.general()[:12]:
            out = O.infer(t["layers"], t["bias"], t["y0"], threads=threads, tile=tile)
            assert out.identical(t["y"])

    def test_dense_oracle_restatement_agrees(self):
        for t in goldens.general()[:16]:
            dense = O.dense_infer([w.to_dense() for w in t["layers"]], t["bias"],
                                  t["y0"].to_dense())
            assert np.array_equal(dense, t["y"].to_dense())

    def test_radixnet_digits(self):
        r = goldens.radixnet()
        out = O.infer(r["layers"][:24], r["bias"][:24], r["y0"], threads=4)
        assert out.identical(r["y24"])
        assert np.array_equal(O.categorize(out), r["cats24"])
        out = O.infer(r["layers"], r["bias"], r["y0"], threads=4)
        assert out.identical(r["y120"])
        assert np.array_equal(O.categorize(out), r["cats120"])

    def test_float32_instance_is_the_same_algorithm(self):
        # exact-in-float inputs (binary Y, power-of-two weights) give identical bits
        rng = np.random.default_rng(5)
        w = CSR.from_dense((rng.random((24, 24)) < 0.3) * 0.125)
        y = CSR.from_dense((rng.random((30, 24)) < 0.5).astype(float))
        a = O.infer([w] * 5, [-0.25] * 5, y, precision=64)
        b = O.infer([w] * 5, [-0.25] * 5, y, precision=32)
        assert a.identical(b)


# ------------------------------------------- image preprocessing (8f rank 4)

def test_oracle_resize_matches_reference_golden():
    """The C restatement of ingest.resize_threshold_flatten reproduces the
    reference's output on images chosen because they hold values within
    1e-9 of the threshold (where a reordered or unfused sum flips pixels)."""
    z = np.load(goldens.GOLDEN / "images.npz")
    for t in z["sides"]:
        t = int(t)
        m = O.resize_threshold_masks(z["pixels"], t)
        want = np.unpackbits(z[f"mask{t}"], axis=1)[:, :t * t].astype(bool)
        assert np.array_equal(m, want), t
        csr = O.resize_threshold_flatten(z["pixels"], t)
        assert np.array_equal(csr.off, z[f"off{t}"]), t
