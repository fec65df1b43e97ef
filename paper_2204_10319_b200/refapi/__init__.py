"""Drop-in numpy boundary: the reference package's import name and types
on top of the B200 engine.

Put this directory on ``sys.path`` (or call :func:`install`) and
``import sparseconv`` resolves to :mod:`paper_2204_10319_b200.refapi.sparseconv`:
the reference's public API (``sparseconv.core``, ``.mapping``,
``.execution``, ``.network``, ``.autotune``) with its numpy signatures —
int64 coordinates, f32/f16 feature matrices, read-only arrays, the same
errors — where every operation runs on the device engine
(``libsparseconv_b200.so``) and results come back as host numpy arrays.
Model code written against the reference runs unmodified; the reference's
own test suite runs against it (tests/test_reference_suite.py).

The reference's out-of-scope modules (oracle, synth, traffic, bench, cli,
pointio) are not mirrored (not on the hot path).
"""

from __future__ import annotations

import sys
from pathlib import Path

PATH = str(Path(__file__).resolve().parent)


def install() -> None:
    """Make ``import sparseconv`` resolve to the B200-backed mirror."""
    if PATH not in sys.path:
        sys.path.insert(0, PATH)
