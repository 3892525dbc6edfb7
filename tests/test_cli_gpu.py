"""The CLI (paper_1501_06663_b200.cli) against the reference CLI's behaviour
(test_cli.py) and the reference's serialised TSV digests (cli.py:72-93)."""

from __future__ import annotations

import hashlib
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO, golden_digests
from paper_1501_06663_b200 import workloads
from paper_1501_06663_b200.cli import main

pytestmark = pytest.mark.gpu


@pytest.fixture
def miss_file(tmp_path):
    p = tmp_path / "miss.txt"
    p.write_bytes(b"mississippi")
    return p


def run_cli(capsys, *argv):
    code = main([str(a) for a in argv])
    out = capsys.readouterr()
    return code, out.out, out.err


def test_query_formats(capsys, miss_file, tmp_path):
    code, out, _ = run_cli(capsys, "query", "--mode", "leftmost", "--path", "raw", miss_file)
    lines = out.splitlines()
    assert code == 0 and len(lines) == 11 and lines[0] == "1\t-1\t0" and lines[4] == "5\t2\t4"
    code, out, _ = run_cli(capsys, "query", "--mode", "all", miss_file)
    lines = out.splitlines()
    assert code == 0 and lines[0] == "1\t-1,0" and lines[4] == "5\t2,4;5,4"
    for path in ("raw", "compact"):
        code, out, _ = run_cli(capsys, "query", "--path", path, "--pos", "5", miss_file)
        assert code == 0 and out == "5\t2\t4\n"
    code, out, _ = run_cli(capsys, "query", "--range", "9:11", miss_file)
    assert code == 0 and out.splitlines() == ["9\t9\t1", "10\t10\t1", "11\t11\t1"]
    empty = tmp_path / "empty.txt"
    empty.write_bytes(b"")
    code, out, _ = run_cli(capsys, "query", empty)
    assert code == 0 and out == ""
    code, out, _ = run_cli(capsys, "query", "--verify", miss_file)
    assert code == 0 and len(out.splitlines()) == 11
    dest = tmp_path / "out.tsv"
    code, out, _ = run_cli(capsys, "query", "--output", dest, miss_file)
    assert code == 0 and out == "" and dest.read_bytes().count(b"\n") == 11


def test_query_errors(capsys, miss_file, tmp_path):
    code, _, err = run_cli(capsys, "query", "--pos", "99", miss_file)
    assert code != 0 and "out of range" in err
    code, _, err = run_cli(capsys, "query", tmp_path / "nope.txt")
    assert code != 0 and "missing file" in err
    code, _, err = run_cli(capsys, "query", "--range", "5:2", miss_file)
    assert code != 0


def test_stats_selftest_bench(capsys, miss_file):
    code, out, _ = run_cli(capsys, "stats", miss_file)
    assert code == 0 and out.splitlines()[0] == "path\tmin\tmax\tavg" and len(out.splitlines()) == 3
    code, out, _ = run_cli(capsys, "selftest", miss_file)
    assert code == 0 and "selftest OK" in out
    code, out, _ = run_cli(capsys, "bench", "--exec", "par", "--threads", "2", miss_file)
    report = dict(line.split("=", 1) for line in out.splitlines())
    for key in ("dataset", "n", "sigma", "mode", "path", "exec", "workers", "backend",
                "build_seconds", "raw_llr_seconds", "compaction_seconds", "query_seconds",
                "total_seconds"):  # test_acceptance.py:215-220
        assert key in report


def test_module_entry_point(miss_file):
    r = subprocess.run([sys.executable, "-m", "paper_1501_06663_b200", "query", str(miss_file)],
                       capture_output=True, text=True, cwd=REPO)
    assert r.returncode == 0 and r.stdout.splitlines()[4] == "5\t2\t4"


@pytest.mark.parametrize("mode", ["leftmost", "all"])
def test_tsv_digest_matches_reference_1mb(tmp_path, capsys, mode):
    # byte identity with the reference serializers on its 1 MB acceptance
    # fixture (test_acceptance.py:129-146), digest produced by the reference
    rec = golden_digests()["acgt_1e6_seed99"]
    data = eval(rec["expr"])
    p = tmp_path / "acgt.txt"
    p.write_bytes(data.tobytes())
    dest = tmp_path / "out.tsv"
    for path in ("raw", "compact"):
        code, _, _ = run_cli(capsys, "query", "--mode", mode, "--path", path, "--output", dest, p)
        assert code == 0
        assert hashlib.sha256(dest.read_bytes()).hexdigest()[:16] == rec[f"{mode}_tsv"]


def test_reference_test_suite_runs_against_this_package():
    """The reference's own pytest suite (pkg/tests: suffixes, llr, query,
    engine, stats, oracle, text, cli, acceptance) through ``import repeatscan``
    -> this package (tests/reference_suite).  The suite is read from the
    git-ignored baseline/_ref/tests staged in the build container (it is not
    part of this repository's history); skipped where it was not staged."""
    import subprocess
    import sys
    from pathlib import Path
    runner = Path(__file__).resolve().parent / "reference_suite" / "run_reference_suite.py"
    sys.path.insert(0, str(runner.parent))
    try:
        import run_reference_suite as rrs
    finally:
        sys.path.pop(0)
    if rrs.suite_dir() is None:
        pytest.skip("reference test suite not staged (tools/stage_reference_tests.sh)")
    proc = subprocess.run([sys.executable, str(runner), "-q", "-p", "no:randomly"],
                          capture_output=True, text=True, timeout=1800)
    assert proc.returncode == 0, proc.stdout[-4000:] + proc.stderr[-2000:]
