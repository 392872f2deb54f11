"""Device image preprocessing: drop-in for ``sdnnbench.ingest.
resize_threshold_flatten`` (reference ingest.py:128-156), SURVEY.md 8f rank 4.

Raw uint8 images go to the GPU (784 bytes per MNIST image instead of a
~9,000-entry int64/float64 CSR row at 256x256), where
``sdnn_batch_from_images`` (libsdnn.so) resamples, thresholds and flattens
them into the engine's staged batch layout.  The result is bit-identical to
the reference: both bilinear products are evaluated as the reference's BLAS
dgemm evaluates them (one fused multiply-add chain per entry), pinned on the
reference's own digits at every target side (tests/golden/images.npz).
"""

from __future__ import annotations

from .errors import ParameterError

TARGET_SIDES = (32, 64, 128, 256)  # ingest.py TARGET_SIDES


def resize_threshold_flatten(images, target_side: int, device: int = 0):
    """Resize, binarize at 0.5 and flatten images into sparse feature rows
    (reference ingest.py:128-156); returns the caller's FeatureBatch class
    when the images come from ``sdnnbench``."""
    from .engine import DeviceNetwork, _make_matrix

    if target_side not in TARGET_SIDES:
        raise ParameterError(f"target side {target_side} is not one of {TARGET_SIDES}")
    net = DeviceNetwork(target_side * target_side, device, "f32")
    try:
        batch = net.upload_images(images, target_side)
        off, cols, vals = batch.to_csr()
        batch.close()
    finally:
        net.close()
    sm_cls, fb_cls, _ = _image_family(images)
    n = int(off.size - 1)
    return fb_cls(_make_matrix(sm_cls, n, target_side * target_side, off, cols, vals))


def _image_family(images):
    """(SparseMatrix, FeatureBatch, CategorySet) of the module the ImageSet
    came from (the reference's own classes for a reference ImageSet)."""
    import sys

    from . import model

    mod = sys.modules.get(type(images).__module__)
    pkg = sys.modules.get(mod.__name__.rsplit(".", 1)[0] + ".model") if mod and "." in mod.__name__ else None
    fb = getattr(pkg, "FeatureBatch", model.FeatureBatch)
    sm = getattr(pkg, "SparseMatrix", model.SparseMatrix)
    cs = getattr(pkg, "CategorySet", model.CategorySet)
    return sm, fb, cs
