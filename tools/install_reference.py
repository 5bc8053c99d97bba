"""Install the unmodified reference into baseline/_ref (git-ignored; it travels
to the GPU box with the gpurun snapshot).

    python tools/install_reference.py [--force]

* ``baseline/_ref/fastgabor``: ``pip install --no-index --no-build-isolation
  --no-deps --target baseline/_ref`` of a /tmp copy of /root/reference/pkg
  (the build writes into its source tree; /root/reference is read-only).
  Its dependencies (numpy, scipy, numba) are already in the image.
  ``bench.py --impl reference`` imports it from there.
* ``baseline/_ref/tests``: a copy of the reference's own test suite, run
  against the drop-in by ``tools/run_reference_suite.py``.

Only runs where /root/reference exists (this container); the GPU box uses
the copy that travelled.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")


def install(force: bool = False, quiet: bool = True) -> bool:
    if not os.path.isdir(REF):
        return os.path.isdir(os.path.join(DEST, "fastgabor"))
    if force or not os.path.isdir(os.path.join(DEST, "fastgabor")):
        with tempfile.TemporaryDirectory() as tmp:
            src = os.path.join(tmp, "pkg")
            shutil.copytree(REF, src)
            cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                   "--find-links", "/opt/wheelhouse", "--target", DEST, "--upgrade", src]
            r = subprocess.run(cmd, capture_output=quiet, text=True)
            if r.returncode != 0:
                print(f"reference install failed:\n{r.stdout}\n{r.stderr}", file=sys.stderr)
                return False
    tests = os.path.join(DEST, "tests")
    if force or not os.path.isdir(tests):
        shutil.rmtree(tests, ignore_errors=True)
        shutil.copytree(os.path.join(REF, "tests"), tests, ignore=shutil.ignore_patterns("__pycache__"))
    return True


if __name__ == "__main__":
    ok = install(force="--force" in sys.argv, quiet=False)
    print("baseline/_ref:", "ok" if ok else "unavailable")
    sys.exit(0 if ok else 1)
