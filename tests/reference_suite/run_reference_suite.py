"""Run the reference package's own pytest suite against paper_1501_06663_b200.

    python tests/reference_suite/run_reference_suite.py [pytest args...]

The suite is the reference's (not copied into this repository's history):
it is read from /root/reference/pkg/tests when present, else from the
git-ignored copy baseline/_ref/tests that tools/stage_reference_tests.sh
makes in the build container (it travels to the GPU box with the snapshot).
``import repeatscan`` resolves to this package through repeatscan_alias.py.
Deselected, with the reason: test_backends.py -- the numba/numpy backend
SELECTOR (_backend.py:10-34 env handling), out of scope (the
north star forbids multi-backend dispatch).  ``python -m repeatscan`` in the
suite's subprocesses runs this package's CLI through shim/repeatscan.
Exit status is pytest's.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
CANDIDATES = [Path("/root/reference/pkg/tests"), REPO / "baseline" / "_ref" / "tests"]


def suite_dir() -> Path | None:
    for p in CANDIDATES:
        if (p / "conftest.py").exists():
            return p
    return None


def main(argv: list[str]) -> int:
    d = suite_dir()
    if d is None:
        print("reference test suite not found (run tools/stage_reference_tests.sh)", file=sys.stderr)
        return 5
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(HERE), str(HERE / "shim"), str(REPO), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "repeatscan_alias", "-p", "no:cacheprovider",
           "--rootdir", str(d), str(d), "--ignore", str(d / "test_backends.py"), *argv]
    return subprocess.call(cmd, env=env, cwd=str(d.parent) if os.access(d.parent, os.W_OK) else "/tmp")


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
