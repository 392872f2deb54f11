"""The reference-side binding, applied at run time.

INTEGRATION.md section 2 shows the one branch a maintainer adds to the
reference's dispatch point (``sdnnbench.engine.infer``, engine.py:317-323,
plus the mode name in ``MODES``, engine.py:38).  ``install`` makes exactly
that change to an imported ``sdnnbench.engine`` module without editing its
source, for callers who cannot patch the reference:

    from sdnnbench import engine
    from paper_1909_05631_b200 import integration
    integration.install(engine)
    out = engine.infer(model, y0, engine.InferenceConfig(mode="b200"))

Every other mode still runs the reference's own code.  ``infer_timed``
(engine.py:327-340) looks ``infer`` up in its module at call time, so it
times the B200 path for ``mode="b200"`` as well.
"""

from __future__ import annotations

MODE = "b200"


def install(ref_engine=None, dtype: str = "f64"):
    """Add ``mode="b200"`` to a reference engine module; idempotent.
    ``dtype="f64"`` (default) is bit-exact with the reference."""
    if ref_engine is None:
        from sdnnbench import engine as ref_engine
    if getattr(ref_engine.infer, "_b200_branch", False):
        return ref_engine
    original = ref_engine.infer
    if MODE not in ref_engine.MODES:
        ref_engine.MODES = tuple(ref_engine.MODES) + (MODE,)

    def infer(model, y0, cfg=None):
        cfg = cfg or ref_engine.InferenceConfig()
        if cfg.mode != MODE:
            return original(model, y0, cfg)
        from . import engine as b200

        return b200.infer(model, y0, b200.InferenceConfig(
            ymax=cfg.ymax, mode="data_parallel", workers=cfg.workers,
            pipeline_stages=cfg.pipeline_stages, batch_tile=cfg.batch_tile, dtype=dtype))

    infer.__doc__ = original.__doc__
    infer._b200_branch = True
    infer._original = original
    ref_engine.infer = infer
    return ref_engine


def uninstall(ref_engine) -> None:
    """Undo ``install`` (tests)."""
    fn = ref_engine.infer
    if getattr(fn, "_b200_branch", False):
        ref_engine.infer = fn._original
        ref_engine.MODES = tuple(m for m in ref_engine.MODES if m != MODE)
