"""Shared test setup: the `gpu` marker, repo on sys.path, golden fixtures."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


class GoldenCase:
    """One reference-computed case from golden_small.npz (int64 arrays)."""

    def __init__(self, z, i):
        for f in ("text", "sa", "rank", "lcp", "raw", "flags", "ps", "c_starts",
                  "c_lengths", "l_starts", "l_lengths", "a_lengths", "a_offsets", "a_flat",
                  "w_raw", "w_comp"):
            off = z[f + "_off"]
            setattr(self, f, z[f][off[i]:off[i + 1]])
        self.data = self.text.astype(np.uint8)
        self.n = int(self.data.size)

    def __repr__(self):
        return f"GoldenCase(n={self.n}, {self.data[:24].tobytes()!r})"


_cases = None


def golden_cases() -> list[GoldenCase]:
    global _cases
    if _cases is None:
        z = np.load(GOLDEN / "golden_small.npz")
        z = {k: z[k] for k in z.files}
        count = z["sa_off"].size - 1
        _cases = [GoldenCase(z, i) for i in range(count)]
    return _cases


def golden_digests() -> dict:
    return json.loads((GOLDEN / "digests.json").read_text())


def digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()[:16]


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(0xC0FFEE)
