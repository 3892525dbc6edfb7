"""pytest plugin: make ``import repeatscan`` resolve to paper_1501_06663_b200.

Used by run_reference_suite.py to run the REFERENCE package's own test suite
(/root/reference/pkg/tests, staged into the git-ignored baseline/_ref/tests
by tools/stage_reference_tests.sh so it travels to the GPU box) against the
B200 package through the drop-in boundary (SURVEY 8(b) "Interop for parity").
Every reference module the tests import maps to the module of the same name
here; ``repeatscan.oracle`` (the substring-search ground truth) maps to
bruteforce.py.  ``repeatscan._backend`` (the numba/numpy backend selector) is
out of scope: its tests are deselected by the runner.
"""

from __future__ import annotations

import importlib
import sys

_MODULES = {
    "repeatscan": "paper_1501_06663_b200",
    "repeatscan.engine": "paper_1501_06663_b200.engine",
    "repeatscan.llr": "paper_1501_06663_b200.llr",
    "repeatscan.query": "paper_1501_06663_b200.query",
    "repeatscan.suffixes": "paper_1501_06663_b200.suffixes",
    "repeatscan.text": "paper_1501_06663_b200.text",
    "repeatscan.stats": "paper_1501_06663_b200.stats",
    "repeatscan.oracle": "paper_1501_06663_b200.bruteforce",
    "repeatscan.cli": "paper_1501_06663_b200.cli",
}


def install() -> None:
    for alias, real in _MODULES.items():
        sys.modules[alias] = importlib.import_module(real)


install()
