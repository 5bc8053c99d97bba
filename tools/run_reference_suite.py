"""Run the reference's own test suite against the B200 drop-in.

    python tools/run_reference_suite.py [pytest args...]

The reference's tests (a copy of /root/reference/pkg/tests under
baseline/_ref/tests, git-ignored, made by ``__graft_entry__.build()`` or
``tools/install_reference.py``) import ``fastgabor`` and its submodules.  This
runner aliases ``fastgabor`` and every submodule the tests import to
``paper_1704_05231_b200`` (same module names: gaussian, gabor, bank, sdft,
image_io, metrics, cli; ``fastgabor.oracle`` -> ``bruteforce``) BEFORE pytest
collects, so every call in those tests runs through libfgb200 on the GPU --
the real reference package next to them is never imported.

Deselected: acceptance criterion 7 (wall-clock speedup of the reference's
own reuse scheduler on the CPU, timing-only) and criterion 8 (the
reference's recursive-smoother accuracy criterion, red in the reference
itself: pkg/test_output.txt).
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
DESELECT = ("test_acceptance.py::test_criterion_7_wall_clock_speedup",
            "test_acceptance.py::test_criterion_8_recursive_smoother_accuracy")


def install_alias() -> None:
    sys.path.insert(0, ROOT)
    import importlib

    pkg = importlib.import_module("paper_1704_05231_b200")
    sys.modules["fastgabor"] = pkg
    for sub in ("gaussian", "gabor", "bank", "sdft", "image_io", "metrics", "cli"):
        sys.modules[f"fastgabor.{sub}"] = importlib.import_module(f"paper_1704_05231_b200.{sub}")
    sys.modules["fastgabor.oracle"] = importlib.import_module("paper_1704_05231_b200.bruteforce")


def main(argv: list[str]) -> int:
    if not os.path.isdir(TESTS):
        print(f"reference tests not found at {TESTS} (run tools/install_reference.py)", file=sys.stderr)
        return 4
    install_alias()
    import pytest

    args = [TESTS, "-q", "-p", "no:cacheprovider", "--rootdir", os.path.dirname(TESTS)]
    for d in DESELECT:
        args += ["--deselect", "tests/" + d]
    return int(pytest.main(args + argv))


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
