"""Loaders for the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by running the reference engine itself
(tests/golden/make_golden.py); these helpers only unpack them.
"""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

from oracle.oracle import CSR

GOLDEN = Path(__file__).resolve().parent / "golden"


def _csr(z, prefix) -> CSR:
    shape = z[prefix + "_shape"]
    return CSR(int(shape[0]), int(shape[1]), z[prefix + "_off"], z[prefix + "_cols"],
               z[prefix + "_vals"])


@lru_cache(maxsize=None)
def general():
    """List of dicts: layers (CSR list), bias, y0, y (reference output), cats."""
    z = np.load(GOLDEN / "general.npz")
    out = []
    for t in range(int(z["count"][0])):
        p = f"t{t}"
        n, layers, rows = (int(v) for v in z[p + "_meta"])
        out.append({
            "n": n,
            "layers": [_csr(z, f"{p}_w{i}") for i in range(layers)],
            "bias": z[p + "_bias"],
            "y0": _csr(z, p + "_y0"),
            "y": _csr(z, p + "_y"),
            "cats": z[p + "_cats"],
        })
    return out


@lru_cache(maxsize=None)
def radixnet():
    """RadiX-Net (1024 neurons, 120 layers) + synthetic digits, reference output."""
    z = np.load(GOLDEN / "radixnet.npz")
    n = int(z["n"][0])
    layers = []
    for i in range(int(z["layers"][0])):
        layers.append(CSR(n, n, z["w_off"][i], z["w_cols"][i].astype(np.int64),
                          z["w_vals"][i].astype(np.float64)))
    return {
        "n": n,
        "layers": layers,
        "bias": z["bias"],
        "y0": _csr(z, "y0"),
        "y24": _csr(z, "y24"),
        "cats24": z["cats24"],
        "y120": _csr(z, "y120"),
        "cats120": z["cats120"],
    }
