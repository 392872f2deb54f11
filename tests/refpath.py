"""Where the reference package (sdnnbench) can be imported from, if anywhere.

``baseline/_ref`` is the offline pip install of the unmodified reference
(git-ignored, travels to the GPU box with the repo snapshot); the build
container also has the read-only source tree.  Tests that need the
reference skip when neither exists.
"""

from __future__ import annotations

from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def reference_path() -> Path | None:
    for p in CANDIDATES:
        if (p / "sdnnbench" / "engine.py").exists():
            return p
    return None
