"""Stage the unmodified reference package and its own test modules as
TEST-ONLY fixtures for the GPU box (VERDICT r01 "prove the drop-in").

    python tools/stage_reference.py [--force]

* ``baseline/_ref/sparse_sampler`` -- the reference installed with the offline
  recipe the task prescribes (``pip install --no-index --no-build-isolation
  --no-deps --target baseline/_ref``; pip needs a writable copy of the tree,
  so the install runs from a copy under /tmp -- /root/reference is read-only
  and has its pyproject under pkg/);
* ``baseline/_ref/ref_tests/*.py`` -- the reference's own test modules
  (pkg/tests), byte-for-byte.

Both are git-ignored (``baseline/_ref/``), so no reference source enters the
repo history, and NOT gpurun-ignored, so they travel to the GPU box with the
snapshot, where ``tests/test_gpu_reference_suite.py`` runs them under
``compat.install()``.  Nothing in the product package imports them
(``tests/test_hygiene.py``).  Runs only where /root/reference exists (this
container); a no-op elsewhere.
"""

from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(DEST, "ref_tests")


def staged() -> bool:
    return os.path.isfile(os.path.join(DEST, "sparse_sampler", "pyramid.py")) and bool(
        glob.glob(os.path.join(TESTS, "test_*.py")))


def stage(force: bool = False) -> bool:
    """Returns True when the fixtures are present after the call."""
    if staged() and not force:
        return True
    if not os.path.isdir(REF_PKG):
        return staged()
    if os.path.isdir(DEST):
        shutil.rmtree(DEST)
    os.makedirs(DEST)
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", DEST, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{res.stdout}\n{res.stderr}")
    os.makedirs(TESTS)
    for f in sorted(glob.glob(os.path.join(REF_PKG, "tests", "*.py"))):
        shutil.copy2(f, TESTS)
    return staged()


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args(argv)
    ok = stage(args.force)
    print(f"reference staged in {DEST}: {ok}")


if __name__ == "__main__":
    main()
