"""Golden fixture for the device image preprocessing,
produced by running the REFERENCE's own ``ingest.resize_threshold_flatten``
(ingest.py:128-156) on the reference's own synthetic digits
(tests/helpers.py ``synthetic_digits``).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_images_golden.py

The images kept are the ones that discriminate summation orders: every
image of the first 2,000 digits holding a resampled value within 1e-9 of
the 0.5 threshold at some target side (there a non-fused or reordered sum
flips the pixel), plus 32 ordinary ones.  Stored per target side: the
reference's row offsets and its dense masks, bit-packed.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

from helpers import synthetic_digits  # noqa: E402
from sdnnbench.ingest import TARGET_SIDES, ImageSet, _interp_matrix, resize_threshold_flatten  # noqa: E402

OUT = Path(__file__).resolve().parent


def main() -> None:
    pix = np.ascontiguousarray(synthetic_digits(2000, seed=7))
    near = np.zeros(pix.shape[0], bool)
    p = pix.astype(np.float64) / 255.0
    for t in TARGET_SIDES:
        h = _interp_matrix(pix.shape[1], t)
        x = h @ p @ h.T
        near |= (np.abs(x - 0.5) < 1e-9).reshape(pix.shape[0], -1).any(axis=1)
    pick = np.nonzero(near)[0][:96].tolist() + [i for i in range(pix.shape[0]) if not near[i]][:32]
    pick = np.array(sorted(pick), np.int64)
    sel = np.ascontiguousarray(pix[pick])
    out = {"pixels": sel, "index": pick, "sides": np.array(TARGET_SIDES, np.int64)}
    imgs = ImageSet(sel.shape[0], sel.shape[1], sel)
    for t in TARGET_SIDES:
        fb = resize_threshold_flatten(imgs, t).data
        mask = np.zeros((sel.shape[0], t * t), bool)
        off = np.asarray(fb.row_offsets, np.int64)
        for r in range(sel.shape[0]):
            mask[r, np.asarray(fb.col_indices[off[r]:off[r + 1]])] = True
        out[f"off{t}"] = off
        out[f"mask{t}"] = np.packbits(mask, axis=1)
    np.savez_compressed(OUT / "images.npz", **out)
    print(f"{sel.shape[0]} images ({int(near.sum())} near-threshold of 2000)")


if __name__ == "__main__":
    main()
