"""The reference's own test suite (/root/reference/pkg/tests, copied to
baseline/_ref/tests) run against the drop-in through tools/run_reference_suite.py,
which aliases ``fastgabor`` to ``paper_1704_05231_b200``.

CPU: collection of every module (all drop-in names resolve) and the host-only
modules (image_io, metrics).  GPU: the whole suite except acceptance criteria
7 (CPU wall-clock timing of the reference's scheduler) and 8 (red in the
reference itself, pkg/test_output.txt:204).
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
RUNNER = os.path.join(ROOT, "tools", "run_reference_suite.py")

needs_ref = pytest.mark.skipif(not os.path.isdir(TESTS), reason="baseline/_ref/tests absent (tools/install_reference.py)")


def _run(args, timeout):
    r = subprocess.run([sys.executable, RUNNER, *args], capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    return r.returncode, (r.stdout + r.stderr)[-6000:]


@needs_ref
def test_reference_suite_collects_against_dropin():
    rc, out = _run(["--co"], 300)
    assert rc == 0, out
    assert "139 tests collected" in out or "tests collected" in out, out


@needs_ref
def test_reference_host_modules_pass():
    rc, out = _run(["-k", "image_io or metrics"], 300)
    assert rc == 0, out


@needs_ref
@pytest.mark.gpu
def test_reference_suite_passes_on_gpu():
    rc, out = _run(["-rfE"], 1800)
    print(out)
    assert rc == 0, out
