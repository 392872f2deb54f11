"""The drop-in with the reference package importable.

Both adoption routes of INTEGRATION.md run here against the UNMODIFIED
reference (``sdnnbench``): section 1 (our engine fed the reference's own
objects, errors caught as the reference's classes) and section 2 (the
``mode="b200"`` branch at the reference's dispatch point,
engine.py:317-323, installed by ``paper_1909_05631_b200.integration``).
Each case runs in a fresh interpreter so the reference is importable
before our package is (the error classes pick their bases at import).
"""

import os
import subprocess
import sys
import textwrap

import pytest

from refpath import ROOT, reference_path

REF = reference_path()
pytestmark = pytest.mark.skipif(REF is None, reason="reference package not available")


def run_py(code: str, timeout: int = 600) -> str:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT)])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/sdnn_numba_cache")
    out = subprocess.run([sys.executable, "-c", textwrap.dedent(code)], capture_output=True, text=True,
                         timeout=timeout, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    return out.stdout


def test_package_imports_beside_the_reference_and_subclasses_its_errors():
    out = run_py("""
        import sdnnbench.errors as R
        import paper_1909_05631_b200 as P
        from paper_1909_05631_b200 import errors as E
        for name in ("SdnnError", "ParameterError", "CapacityError", "ShapeError", "BoundsError"):
            assert issubclass(getattr(E, name), getattr(R, name)), name
        assert issubclass(E.ShapeError, E.SdnnError)
        assert isinstance(E.from_code(4, "x"), R.ShapeError)
        assert isinstance(E.from_code(2, "x"), R.ParameterError)
        assert isinstance(E.from_code(3, "x"), R.CapacityError)
        print("ok")
    """)
    assert out.strip().endswith("ok")


def test_reference_objects_in_reference_errors_out():
    """Section 1: real sdnnbench.model objects through our engine.  Shape
    and parameter errors are raised before any device work and caught as
    the reference's classes; without a GPU the call itself fails loudly
    with the reference's CapacityError (no CPU fallback)."""
    out = run_py("""
        import numpy as np, torch
        import sdnnbench.errors as R
        from sdnnbench.model import FeatureBatch, LayerWeights, NetworkModel, SparseMatrix
        from paper_1909_05631_b200 import engine as b200
        w = SparseMatrix(4, 4, np.arange(5), np.arange(4), np.full(4, 0.5))
        model = NetworkModel(4, (LayerWeights(w, -0.1), LayerWeights(w, -0.1)))
        y_bad = FeatureBatch(SparseMatrix(2, 5, [0, 1, 2], [0, 4], [1.0, 1.0]))
        y = FeatureBatch(SparseMatrix(2, 4, [0, 1, 2], [0, 3], [1.0, 1.0]))
        try:
            b200.infer(model, y_bad)
        except R.ShapeError:
            pass
        else:
            raise AssertionError("no ShapeError")
        try:
            b200.infer(model, y, b200.InferenceConfig(mode="pipeline", pipeline_stages=3))
        except R.ParameterError:
            pass
        else:
            raise AssertionError("no ParameterError")
        if not torch.cuda.is_available():
            try:
                b200.infer(model, y)
            except R.CapacityError:
                pass
            else:
                raise AssertionError("ran without a device")
        print("ok")
    """)
    assert out.strip().endswith("ok")


def test_b200_mode_branch_at_the_reference_dispatch():
    """Section 2: install the mode="b200" branch; the reference's own
    InferenceConfig accepts the mode, every other mode still runs the
    reference, and the branch reaches our engine (CapacityError without a
    GPU)."""
    out = run_py("""
        import numpy as np, torch
        import sdnnbench.errors as R
        from sdnnbench import engine
        from sdnnbench.model import FeatureBatch, LayerWeights, NetworkModel, SparseMatrix
        from paper_1909_05631_b200 import integration
        integration.install(engine)
        integration.install(engine)  # idempotent
        assert engine.MODES.count("b200") == 1
        cfg = engine.InferenceConfig(mode="b200")
        w = SparseMatrix(2, 2, [0, 2, 3], [0, 1, 1], [0.5, 0.5, 1.0])
        model = NetworkModel(2, (LayerWeights(w, -0.3),))
        y0 = FeatureBatch(SparseMatrix(1, 2, [0, 1], [0], [1.0]))
        ref = engine.infer(model, y0)   # serial: the reference's own kernels
        assert np.array_equal(ref.data.to_dense(), [[0.2, 0.2]])  # test_engine.py:112-131
        if not torch.cuda.is_available():
            try:
                engine.infer(model, y0, cfg)
            except R.CapacityError:
                pass
            else:
                raise AssertionError("b200 mode ran without a device")
        integration.uninstall(engine)
        assert "b200" not in engine.MODES
        print("ok")
    """)
    assert out.strip().endswith("ok")


@pytest.mark.gpu
def test_b200_mode_bit_exact_with_the_reference_engine_on_gpu():
    """On the B200: reference objects in, the reference's serial engine and
    the b200 branch (and infer_timed through it) agree bit for bit on the
    reference's own random-instance generator shape (mixed-sign weights,
    variable degree, positive bias) and on a perm-union network; result
    types are the reference's classes."""
    out = run_py("""
        import numpy as np, torch
        assert torch.cuda.is_available()
        from sdnnbench import engine
        from sdnnbench.model import FeatureBatch, LayerWeights, NetworkModel, SparseMatrix, CategorySet
        from paper_1909_05631_b200 import integration, workloads as W
        integration.install(engine)
        rng = np.random.default_rng(7)
        def rand_sm(r, c, dens, lo, hi):
            d = np.where(rng.random((r, c)) < dens, rng.uniform(lo, hi, (r, c)), 0.0)
            m = d != 0
            off = np.concatenate([[0], np.cumsum(m.sum(1))])
            return SparseMatrix(r, c, off, np.nonzero(m)[1], d[m])
        for trial in range(6):
            n = int(rng.integers(8, 300)); L = int(rng.integers(1, 7)); B = int(rng.integers(1, 400))
            model = NetworkModel(n, tuple(LayerWeights(rand_sm(n, n, 0.1, -1, 1), float(rng.uniform(-0.4, 0.2)))
                                          for _ in range(L)))
            y0 = FeatureBatch(rand_sm(B, n, 0.3, 0, 2))
            want = engine.infer(model, y0)
            got = engine.infer(model, y0, engine.InferenceConfig(mode="b200"))
            assert type(got) is FeatureBatch and type(got.data) is SparseMatrix
            assert got.data == want.data, trial  # bitwise (model.py:110-119)
        w = W.CONFIGS["C1"].with_(layers=12, batch=500, value=0.125)
        model = NetworkModel(w.n, tuple(LayerWeights(SparseMatrix(w.n, w.n, *c, check=False), w.bias)
                                        for c in W.layers_csr(w)))
        y0 = FeatureBatch(SparseMatrix(w.batch, w.n, *W.images(w), check=False))
        want, wcats, _ = engine.infer_timed(model, y0, engine.InferenceConfig(mode="data_parallel", workers=4))
        got, gcats, _ = engine.infer_timed(model, y0, engine.InferenceConfig(mode="b200"))
        assert got.data == want.data and isinstance(gcats, CategorySet)
        assert list(gcats.image_rows) == list(wcats.image_rows) and len(wcats.image_rows) > 0
        print("ok", len(wcats.image_rows))
    """, timeout=900)
    assert "ok" in out
