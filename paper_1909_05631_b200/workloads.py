"""BASELINE.json workloads (configs[0..4]) and the live companions.

Synthetic stand-ins, generated from seeds: the paper's inputs are MNIST-
derived images on RadiX-Net networks, neither of which is
available here.  W_l is the union of 32 seeded permutation matrices (exactly
32 nonzeros per row and column, each `value`), Y0 rows are side x side
binary images with Bernoulli(p) pixels in the centred square.

C1..C5 as specified die by layer 2-3, so K2 (the C4/C5
generator with weight 0.125 = 2^-3) is carried beside them as the live-row
throughput companion: survivors saturate at YMAX and stay dense.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

from . import _lib

WEIGHT_SEED = 20190912
IMAGE_SEED = 1909


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    layers: int
    batch: int
    side: int
    square: int
    p: float
    bias: float
    width: int = 32
    value: float = 0.0625
    ymax: float = 32.0
    weight_seed: int = WEIGHT_SEED
    image_seed: int = IMAGE_SEED
    kind: str = "permunion"  # weights: "permunion" (BASELINE generator) or "radixnet" (K1)

    @property
    def edges(self) -> int:
        """Nominal edges (inputs x connections), the challenge rate numerator."""
        return self.batch * self.n * self.width * self.layers

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


CONFIGS = {
    "C1": Workload("C1", 1024, 120, 60000, 32, 20, 0.35, -0.30),
    "C2": Workload("C2", 4096, 480, 60000, 64, 40, 0.35, -0.35),
    "C3": Workload("C3", 16384, 1920, 60000, 128, 80, 0.35, -0.40),
    "C4": Workload("C4", 65536, 1920, 60000, 256, 160, 0.35, -0.45),
    "C5": Workload("C5", 65536, 120, 60000, 256, 160, 0.35, -0.45),
    "K2": Workload("K2", 65536, 1920, 60000, 256, 160, 0.35, -0.45, value=0.125),
    # K1: the reference's own workload shape at flagship width -- RadiX-Net
    # preset (65536, 1920) seed 42 and digit-like 28x28 images resized to
    # 256x256 on the device (stroke_images; rows stay alive and saturate).
    # A 6,000-row sample of the 60,000-image batch.
    "K1": Workload("K1", 65536, 1920, 6000, 256, 0, 0.0, -0.45, weight_seed=42, kind="radixnet"),
}
C5_SWEEP = [(b, p) for b in (1000, 15000, 60000, 240000) for p in (0.1, 0.35, 0.7)]


# ------------------------------------------------------------- RadiX-Net (K1)
# The reference's own network family (sdnnbench.radixnet): a radix-2
# butterfly base of S stages over n/16 neurons (stage s links i with
# i XOR 2^s, radixnet.py:148-175), each stage Kronecker-expanded by the
# 16 x 16 all-ones block (radixnet.py:178-208: 32 inputs per neuron), and
# layer t the base stage (t-1) mod S conjugated by seeded neuron
# relabelings on both sides (perm_{t-1} on inputs, perm_t on outputs,
# perm_0 = identity; radixnet.py:246-268,293-310).  perm_t is a uniform
# permutation from numpy's counter-based Philox stream keyed (seed, t)
# (radixnet.py:192-196), so any layer is produced alone, in any order.
RADIX_PRESETS = {1024: (6, 16), 4096: (8, 16), 16384: (10, 16), 65536: (12, 16)}  # radixnet.py:46-51
RADIX_BIAS = {1024: -0.30, 4096: -0.35, 16384: -0.40, 65536: -0.45}  # radixnet.py:39
RADIX_SEED = 42  # the reference's acceptance workload seed


def radix_perm(seed: int, t: int, n: int) -> np.ndarray:
    key = np.array([seed & 0xFFFFFFFFFFFFFFFF, t], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).permutation(n).astype(np.int64)


def radixnet_ell(n: int, layer: int, seed: int = RADIX_SEED) -> np.ndarray:
    """Layer `layer` (0-based; depth slot t = layer + 1) of the RadiX-Net
    preset network over n neurons as ELL by output column: [n][32] int32,
    the 32 inputs of each output ascending."""
    stages, k = RADIX_PRESETS[n]
    t = layer + 1
    place = 1 << ((t - 1) % stages)
    cur = radix_perm(seed, t, n)
    inv = np.empty(n, np.int64)
    inv[cur] = np.arange(n, dtype=np.int64)    # output j' is expanded-stage neuron inv[j']
    i = inv // k                               # its base-butterfly neuron
    base = np.stack([i & ~place, i | place], axis=1)  # the stage's two partners (symmetric)
    inputs = (base[:, :, None] * k + np.arange(k, dtype=np.int64)[None, None, :]).reshape(n, 2 * k)
    if t > 1:
        inputs = radix_perm(seed, t - 1, n)[inputs]
    inputs.sort(axis=1)
    return inputs.astype(np.int32)


def radixnet_ell_layers(n: int, first: int, count: int, seed: int = RADIX_SEED,
                        threads: int | None = None) -> list:
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=threads or _threads()) as pool:
        return list(pool.map(lambda l: radixnet_ell(n, l, seed), range(first, first + count)))


def _threads() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


def images(w: Workload, n_rows: int | None = None, threads: int | None = None, row0: int = 0):
    """Rows [row0, row0 + n_rows) of Y0 as CSR arrays (off int64, cols
    int64, vals float64); n_rows defaults to the whole batch."""
    g = _lib.gen()
    B = w.batch - row0 if n_rows is None else int(n_rows)
    t = threads or _threads()
    cnt = np.zeros(max(B, 1), np.int64)
    _lib.check_gen(g.sdnn_gen_images_count(w.image_seed, row0, B, w.side, w.square, w.p, t,
                                           _lib.ptr(cnt)))
    off = np.zeros(B + 1, np.int64)
    np.cumsum(cnt[:B], out=off[1:])
    nnz = int(off[-1])
    cols = np.zeros(max(nnz, 1), np.int64)
    vals = np.zeros(max(nnz, 1), np.float64)
    _lib.check_gen(g.sdnn_gen_images_fill(w.image_seed, row0, B, w.side, w.square, w.p, t,
                                          _lib.ptr(off), _lib.ptr(cols), None, _lib.ptr(vals)))
    return off, cols[:nnz], vals[:nnz]


def layer_ell(w: Workload, layer: int) -> np.ndarray:
    """Layer `layer` as ELL by output column, [n][width] int32 ascending."""
    idx = np.zeros((w.n, w.width), np.int32)
    _lib.check_gen(_lib.gen().sdnn_gen_permunion_ell(w.weight_seed, layer, w.n, w.width, _lib.ptr(idx)))
    return idx


def layer_csr(w: Workload, layer: int):
    """Layer `layer` in the reference's CSR-by-input layout (off, cols, vals)."""
    idx = layer_ell(w, layer)
    vals = np.full(idx.size, w.value, np.float64)
    off = np.zeros(w.n + 1, np.int64)
    cols = np.zeros(idx.size, np.int64)
    out = np.zeros(idx.size, np.float64)
    _lib.check_gen(_lib.gen().sdnn_gen_ell_to_csr(w.n, w.n, w.width, _lib.ptr(idx), _lib.ptr(vals),
                                                  _lib.ptr(off), _lib.ptr(cols), _lib.ptr(out)))
    return off, cols, out


def layers_csr(w: Workload, first: int = 0, count: int | None = None, threads: int | None = None):
    """Layers [first, first + count) in CSR-by-input form, generated and
    transposed by `threads` host threads (for the CPU oracle and tests)."""
    from concurrent.futures import ThreadPoolExecutor

    count = w.layers - first if count is None else count
    t = threads or _threads()
    idx = np.zeros((max(count, 1), w.n, w.width), np.int32)
    if count:
        _lib.check_gen(_lib.gen().sdnn_gen_permunion_ell_layers(
            w.weight_seed, first, count, w.n, w.width, t, _lib.ptr(idx)))
    vals = np.full(w.n * w.width, w.value, np.float64)

    def one(i):
        off = np.zeros(w.n + 1, np.int64)
        cols = np.zeros(w.n * w.width, np.int64)
        out = np.zeros(w.n * w.width, np.float64)
        _lib.check_gen(_lib.gen().sdnn_gen_ell_to_csr(w.n, w.n, w.width, _lib.ptr(idx[i]), _lib.ptr(vals),
                                                      _lib.ptr(off), _lib.ptr(cols), _lib.ptr(out)))
        return off, cols, out

    with ThreadPoolExecutor(max_workers=t) as pool:
        return list(pool.map(one, range(count)))


def stroke_images(n: int, seed: int = IMAGE_SEED, side: int = 28) -> np.ndarray:
    """Seeded MNIST-shaped stand-in corpus for the device ingest path: each
    image holds 2-4 thick strokes with soft (anti-aliased) edges, so the
    resampled values cross the 0.5 threshold at fractional positions.
    uint8, shape (n, side, side)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:side, 0:side].astype(np.float32)
    img = np.zeros((n, side, side), np.float32)
    for s in range(4):
        a = rng.uniform(4, side - 4, size=(n, 2)).astype(np.float32)
        b = rng.uniform(4, side - 4, size=(n, 2)).astype(np.float32)
        width = rng.uniform(1.0, 2.2, size=n).astype(np.float32)
        on = rng.random(n) < (1.0 if s < 2 else 0.5)
        d = b - a
        L2 = np.maximum((d ** 2).sum(axis=1), 1e-3)
        px = xx[None] - a[:, 0, None, None]
        py = yy[None] - a[:, 1, None, None]
        t = np.clip((px * d[:, 0, None, None] + py * d[:, 1, None, None]) / L2[:, None, None], 0, 1)
        dist = np.hypot(px - t * d[:, 0, None, None], py - t * d[:, 1, None, None])
        ink = np.clip(width[:, None, None] + 0.5 - dist, 0.0, 1.0) * on[:, None, None]
        img = np.maximum(img, ink)
    return np.rint(img * 255.0).astype(np.uint8)
