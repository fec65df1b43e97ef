"""pytest plugin for running the reference's own test files UNMODIFIED
against the B200 engine (tests/test_reference_suite.py launches it).

``import sparseconv`` resolves to the engine's numpy mirror
(paper_2204_10319_b200/refapi).  The reference modules that are not on the
hot path and not mirrored (oracle, synth, traffic, bench, pointio, cli,
kernels) are the UNMODIFIED reference's own, imported from baseline/_ref
under a private package name and registered as ``sparseconv.<name>``:
the dense oracle the tests check against is therefore the reference's, not
ours.  Test infrastructure only."""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_PKG = Path(os.environ.get("SCB_REFERENCE_PKG", ROOT / "baseline" / "_ref" / "sparseconv"))
PASSTHROUGH = ("oracle", "synth", "traffic", "bench", "pointio", "cli", "kernels")


def _load_reference_as(alias: str):
    spec = importlib.util.spec_from_file_location(alias, REF_PKG / "__init__.py",
                                                  submodule_search_locations=[str(REF_PKG)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[alias] = mod
    spec.loader.exec_module(mod)
    return mod


def _install() -> None:
    sys.path.insert(0, str(ROOT))
    from paper_2204_10319_b200 import refapi
    refapi.install()
    import sparseconv  # the mirror
    assert Path(sparseconv.__file__).resolve().is_relative_to(ROOT / "paper_2204_10319_b200"), \
        sparseconv.__file__
    _load_reference_as("_sparseconv_reference")
    for name in PASSTHROUGH:
        m = importlib.import_module(f"_sparseconv_reference.{name}")
        sys.modules[f"sparseconv.{name}"] = m
        setattr(sparseconv, name, m)


_install()
