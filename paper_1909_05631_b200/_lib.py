"""ctypes binding of libsdnn.so (include/sdnn.h).

The CUDA extension is the product: there is no CPU fallback.  If the shared
object is missing or no CUDA device is visible, calls raise loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CapacityError, from_code

PKG = Path(__file__).resolve().parent
# SDNN_LIB selects another build of the same sources (tuning variants)
LIB_PATH = Path(os.environ["SDNN_LIB"]) if os.environ.get("SDNN_LIB") else PKG / "libsdnn.so"
GEN_PATH = PKG / "libsdnn_gen.so"

i64, i32, u64, dbl, cint = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
vp = ctypes.c_void_p
P = ctypes.POINTER

# (name, restype, argtypes) for every symbol declared in include/sdnn.h
SIGNATURES = [
    ("sdnn_version", cint, []),
    ("sdnn_last_error", ctypes.c_char_p, []),
    ("sdnn_device_count", cint, [P(cint)]),
    ("sdnn_net_create", cint, [cint, cint, i64, P(vp)]),
    ("sdnn_net_destroy", None, [vp]),
    ("sdnn_net_add_layer_csr", cint, [vp, vp, vp, vp, i64, dbl]),
    ("sdnn_net_add_layer_ell", cint, [vp, i32, vp, vp, dbl]),
    ("sdnn_net_add_layers_permunion", cint, [vp, u64, i64, i64, i32, dbl, dbl, cint]),
    ("sdnn_net_add_layers_uninit", cint, [vp, i64, i32, dbl]),
    ("sdnn_net_layer_buffers", cint, [vp, i64, P(vp), P(vp), P(i32), P(i64)]),
    ("sdnn_net_n_layers", cint, [vp, P(i64)]),
    ("sdnn_net_weight_bytes", cint, [vp, P(i64)]),
    ("sdnn_batch_upload", cint, [vp, i64, vp, vp, vp, P(vp)]),
    ("sdnn_batch_free", None, [vp]),
    ("sdnn_batch_from_images", cint, [vp, i64, i32, vp, i32, P(vp)]),
    ("sdnn_batch_nnz", cint, [vp, P(i64)]),
    ("sdnn_batch_from_result", cint, [vp, vp, P(vp)]),
    ("sdnn_batch_csr", cint, [vp, vp, vp, vp]),
    ("sdnn_batch_h2d_bytes", cint, [vp, P(i64)]),
    ("sdnn_run", cint, [vp, vp, dbl, i64, i64, P(vp)]),
    ("sdnn_run_y", cint, [vp, vp, dbl, i64, i64, P(vp)]),
    ("sdnn_infer", cint, [vp, i64, vp, vp, vp, dbl, P(vp)]),
    ("sdnn_infer_streamed", cint, [vp, i64, vp, vp, vp, dbl, cint, cint, P(vp)]),
    ("sdnn_result_h2d_bytes", cint, [vp, P(i64)]),
    ("sdnn_result_segments", cint, [vp, P(i64)]),
    ("sdnn_result_n_categories", cint, [vp, P(i64)]),
    ("sdnn_result_categories", cint, [vp, vp]),
    ("sdnn_result_device_ms", dbl, [vp]),
    ("sdnn_result_wall_ms", dbl, [vp]),
    ("sdnn_result_n_layers", cint, [vp, P(i64)]),
    ("sdnn_result_live_rows", cint, [vp, vp]),
    ("sdnn_net_set_layer_timing", cint, [vp, cint]),
    ("sdnn_result_layer_ms", cint, [vp, vp]),
    ("sdnn_result_stage_ms", cint, [vp, vp]),
    ("sdnn_result_launches", cint, [vp, P(i64)]),
    ("sdnn_net_set_compaction", cint, [vp, cint]),
    ("sdnn_result_compactions", cint, [vp, P(i64)]),
    ("sdnn_net_set_pruning", cint, [vp, cint]),
    ("sdnn_result_pruned", cint, [vp, P(i64)]),
    ("sdnn_result_y_nnz", cint, [vp, P(i64)]),
    ("sdnn_result_y_csr", cint, [vp, vp, vp, vp]),
    ("sdnn_result_free", None, [vp]),
    ("sdnn_spmm", cint, [cint, cint, i64, i64, i64, vp, vp, vp, vp, vp, vp, P(vp)]),
    ("sdnn_bias_relu_clamp", cint, [cint, cint, i64, i64, vp, vp, vp, dbl, dbl, P(vp)]),
    ("sdnn_open", cint, [cint, cint, i64, P(vp)]),
    ("sdnn_open_devices", cint, [vp, cint, cint, i64, P(vp)]),
    ("sdnn_close", None, [vp]),
    ("sdnn_group_size", cint, [vp, P(cint)]),
    ("sdnn_group_net", vp, [vp, cint]),
    ("sdnn_group_add_layer_csr", cint, [vp, vp, vp, vp, i64, dbl]),
    ("sdnn_group_add_layers_permunion", cint, [vp, u64, i64, i64, i32, dbl, dbl, cint]),
    ("sdnn_group_infer", cint, [vp, i64, vp, vp, vp, dbl, cint, P(vp)]),
]

GEN_SIGNATURES = [
    ("sdnn_gen_permunion_ell", cint, [u64, i64, i32, i32, vp]),
    ("sdnn_gen_permunion_ell_layers", cint, [u64, i64, i64, i32, i32, cint, vp]),
    ("sdnn_gen_ell_to_csr", cint, [i32, i32, i32, vp, vp, vp, vp, vp]),
    ("sdnn_gen_images_count", cint, [u64, i64, i64, i32, i32, dbl, cint, vp]),
    ("sdnn_gen_images_fill", cint, [u64, i64, i64, i32, i32, dbl, cint, vp, vp, vp, vp]),
]

_lib = None
_gen = None


def _bind(lib, sigs):
    for name, res, args in sigs:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise CapacityError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        _lib = _bind(ctypes.CDLL(str(LIB_PATH)), SIGNATURES + GEN_SIGNATURES)
    return _lib


def gen():
    """Host-only generator library (usable without CUDA)."""
    global _gen
    if _gen is None:
        if not GEN_PATH.exists():
            raise CapacityError(f"{GEN_PATH} is missing: build the package first")
        _gen = _bind(ctypes.CDLL(str(GEN_PATH)), GEN_SIGNATURES)
    return _gen


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().sdnn_last_error()
        raise from_code(rc, msg.decode() if msg else f"libsdnn error {rc}")


def ptr(a) -> int:
    return a.ctypes.data if a is not None else None


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().sdnn_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0


def check_gen(rc: int) -> None:
    if rc != 0:
        raise from_code(rc, f"generator failed with code {rc}")
