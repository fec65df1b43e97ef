"""Stage the UNMODIFIED reference for the GPU box (run in the build
container, where /root/reference exists; __graft_entry__.build() calls it):

  baseline/_ref        pip install --no-deps --target of a /tmp copy of
                       /root/reference/pkg (the CPU arm of bench.py and the
                       whole-network oracle, oracle/reference_runner.py)
  baseline/_ref_tests  the reference's own test files, run unmodified
                       against the B200 engine by tests/test_reference_suite.py

Both are git-ignored (reference sources stay out of this repo's history)
but not gpurun-ignored, so they travel with the snapshot."""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")


def main() -> int:
    if not REF.exists():
        print("stage_reference: /root/reference absent (GPU box): using the staged copies")
        return 0
    ref_pkg = ROOT / "baseline" / "_ref" / "sparseconv"
    if not ref_pkg.exists():
        with tempfile.TemporaryDirectory() as tmp:
            src = Path(tmp) / "pkg"
            shutil.copytree(REF, src)
            subprocess.run([sys.executable, "-m", "pip", "install", "-q", "--no-index",
                            "--no-build-isolation", "--no-deps", "--find-links", "/opt/wheelhouse",
                            "--target", str(ROOT / "baseline" / "_ref"), str(src)], check=True)
    tests = ROOT / "baseline" / "_ref_tests"
    if tests.exists():
        shutil.rmtree(tests)
    shutil.copytree(REF / "tests", tests, ignore=shutil.ignore_patterns("__pycache__"))
    print(f"stage_reference: {ref_pkg.parent} and {tests} ready")
    return 0


if __name__ == "__main__":
    sys.exit(main())
