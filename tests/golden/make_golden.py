"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every expected output below comes from ``sdnnbench.engine.infer`` (the
reference's own numba engine) on inputs built by the reference's own test
helpers and generators; nothing here is hand-written.  The fixtures are
small ``.npz`` files so they travel to the GPU box, where the reference does
not exist.

Files:
  general.npz   criterion-4-style random instances (helpers.random_model /
                random_batch: mixed-sign weights, variable degree, positive
                and negative biases), as in test_acceptance.py:231-250.
  radixnet.npz  the reference's own acceptance workload shape: RadiX-Net
                preset (1024 neurons) + synthetic digits resized to 32x32
                (radixnet.py:293-310, helpers.py:59-84, ingest.py:128-156),
                24 layers (fp32-hostile, unsaturated transients) and the
                full 120 layers on fewer rows.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

from helpers import random_batch, random_model, synthetic_digits  # noqa: E402
from sdnnbench.engine import infer  # noqa: E402
from sdnnbench.ingest import ImageSet, resize_threshold_flatten  # noqa: E402
from sdnnbench.model import FeatureBatch, SparseMatrix  # noqa: E402
from sdnnbench.radixnet import GeneratorConfig, generate_layers  # noqa: E402
from sdnnbench.challenge import categorize  # noqa: E402

OUT = Path(__file__).resolve().parent


def pack_csr(d: dict, prefix: str, m: SparseMatrix) -> None:
    d[prefix + "_shape"] = np.array([m.n_rows, m.n_cols], np.int64)
    d[prefix + "_off"] = np.asarray(m.row_offsets, np.int64)
    d[prefix + "_cols"] = np.asarray(m.col_indices, np.int64)
    d[prefix + "_vals"] = np.asarray(m.values, np.float64)


def make_general() -> None:
    gen = np.random.default_rng(20240601)
    d = {}
    count = 0
    for trial in range(48):
        n = int(gen.integers(4, 65))
        layers = int(gen.integers(1, 9))
        rows = int(gen.integers(1, 101))
        density = float(gen.uniform(0.05, 0.6))
        model = random_model(gen, n, layers, density=density)
        y0 = random_batch(gen, rows, n, float(gen.uniform(0.1, 0.6)))
        out = infer(model, y0)
        p = f"t{count}"
        d[p + "_meta"] = np.array([n, layers, rows], np.int64)
        d[p + "_bias"] = np.array([lw.bias for lw in model.layers], np.float64)
        for li, lw in enumerate(model.layers):
            pack_csr(d, f"{p}_w{li}", lw.weights)
        pack_csr(d, p + "_y0", y0.data)
        pack_csr(d, p + "_y", out.data)
        d[p + "_cats"] = np.asarray(categorize(out).image_rows, np.int64)
        count += 1
    # deep net with forced zero rows (test_engine.py:138-146 shape)
    gen = np.random.default_rng(1234)
    model = random_model(gen, 16, 120, density=0.4)
    mask = gen.random((10, 16)) < 0.5
    mask[3] = False
    mask[7] = False
    from helpers import csr_from_mask
    y0 = FeatureBatch(csr_from_mask(mask))
    out = infer(model, y0)
    p = f"t{count}"
    d[p + "_meta"] = np.array([16, 120, 10], np.int64)
    d[p + "_bias"] = np.array([lw.bias for lw in model.layers], np.float64)
    for li, lw in enumerate(model.layers):
        pack_csr(d, f"{p}_w{li}", lw.weights)
    pack_csr(d, p + "_y0", y0.data)
    pack_csr(d, p + "_y", out.data)
    d[p + "_cats"] = np.asarray(categorize(out).image_rows, np.int64)
    count += 1
    d["count"] = np.array([count], np.int64)
    np.savez_compressed(OUT / "general.npz", **d)
    print("general.npz", count, "instances")


def make_radixnet() -> None:
    n, depth = 1024, 120
    cfg = GeneratorConfig.preset(n, depth, rng_seed=42)
    ws = list(generate_layers(cfg))
    # weights: every layer is degree-32 by row with one constant value; store
    # the exact arrays (cols as uint16, offsets, values) so nothing is implied
    d = {"n": np.array([n], np.int64), "layers": np.array([depth], np.int64)}
    d["w_off"] = np.stack([np.asarray(w.row_offsets, np.int64) for w in ws])
    d["w_cols"] = np.stack([np.asarray(w.col_indices, np.uint16) for w in ws])
    vals = np.stack([np.asarray(w.values, np.float64) for w in ws])
    d["w_vals"] = vals.astype(np.float32)
    assert np.array_equal(d["w_vals"].astype(np.float64), vals), "values not float32-exact"
    d["bias"] = np.full(depth, -0.30)
    corpus = ImageSet(600, 28, synthetic_digits(600, seed=7))
    y0 = resize_threshold_flatten(corpus, 32)
    pack_csr(d, "y0", y0.data)
    # 24-layer prefix over all 600 rows (precision stress, unsaturated)
    from sdnnbench.model import LayerWeights, NetworkModel
    for L in (24, 120):
        model = NetworkModel(n, tuple(LayerWeights(w, -0.30) for w in ws[:L]))
        out = infer(model, y0)
        pack_csr(d, f"y{L}", out.data)
        d[f"cats{L}"] = np.asarray(categorize(out).image_rows, np.int64)
        print(f"radixnet L={L}: {len(d[f'cats{L}'])} categories, nnz {out.data.nnz}")
    np.savez_compressed(OUT / "radixnet.npz", **d)


if __name__ == "__main__":
    make_general()
    make_radixnet()
