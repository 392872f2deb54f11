"""Calibrate the reference arm: time the UNMODIFIED reference engine
(sdnnbench from baseline/_ref, numba) on a row sample of a workload's
first layers and on the full batch of empty rows through dead layers.

    python tools/ref_probe.py C4 600 4 16
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sdnn_numba_cache")

import numpy as np  # noqa: E402

from paper_1909_05631_b200 import workloads as W  # noqa: E402


def main():
    name, S, Lp, D = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    from sdnnbench import engine as RE
    from sdnnbench.model import FeatureBatch, LayerWeights, NetworkModel, SparseMatrix
    w = W.CONFIGS[name]
    t0 = time.time()
    lay = W.layers_csr(w, 0, Lp + D)
    print("gen", time.time() - t0, flush=True)
    lw = [LayerWeights(SparseMatrix(w.n, w.n, *c, check=False), w.bias) for c in lay]
    off, cols, vals = W.images(w, n_rows=S)
    y0 = FeatureBatch(SparseMatrix(S, w.n, off, cols, vals, check=False))
    cfg = RE.InferenceConfig(mode="data_parallel", workers=os.cpu_count())
    RE.warmup()
    for i in range(2):
        _, cats, sec = RE.infer_timed(NetworkModel(w.n, tuple(lw[:Lp])), y0, cfg)
        print(f"live {S} rows x {Lp} layers: {sec:.3f} s, cats {len(cats.image_rows) if hasattr(cats,'image_rows') else cats}", flush=True)
    empty = FeatureBatch(SparseMatrix.empty(w.batch, w.n))
    for i in range(2):
        _, cats, sec = RE.infer_timed(NetworkModel(w.n, tuple(lw[Lp:])), empty, cfg)
        print(f"dead {w.batch} rows x {D} layers: {sec:.3f} s ({sec / D * 1e3:.2f} ms/layer)", flush=True)


if __name__ == "__main__":
    main()
