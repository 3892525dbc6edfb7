"""Synthetic input generators for the five BASELINE.json configurations.

Shapes and seeds follow SURVEY.md section 8(d) (binary sizes as the paper uses,
``PAPER.md:1185-1187``).  Every generator is deterministic (numpy PCG64) so the
parity tests can regenerate an input on the GPU box and compare digests that
were computed from the reference package in this container.

  C1  n=2^20      i.i.d. uniform over b"ACGT", default_rng(1)
  C2  n=64*2^20   i.i.d. ACGT + 20 Alu-like 300 bp families planted at 30%
                  coverage with 10% substitutions, default_rng(2)
  C3  n=256*2^20  i.i.d. ACGT, default_rng(3)            (headline metric)
  C4  n=100*2^20  English-like bytes, sigma=96, Zipf(1) over 50k words, rng(4)
  C5  n=2^30      Fibonacci word over {A,C} with 1e-4 point mutations, rng(5)

``reference_dna`` reproduces the reference's own acceptance fixture
(``tests/test_acceptance.py:50-51``: lowercase ``acgt``, rng.choice).
"""

from __future__ import annotations

import numpy as np

MiB = 1 << 20

ACGT = np.frombuffer(b"ACGT", np.uint8)


def iid_dna(n: int, seed: int, alphabet: bytes = b"ACGT") -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.choice(np.frombuffer(alphabet, np.uint8), size=n)


def reference_dna(n: int, seed: int) -> np.ndarray:
    """test_acceptance.py:50-51 -- ``dna(default_rng(seed), n)``."""
    rng = np.random.default_rng(seed)
    return rng.choice(np.frombuffer(b"acgt", np.uint8), size=n)


def planted_dna(n: int, seed: int = 2, families: int = 20, family_len: int = 300,
                coverage: float = 0.3, divergence: float = 0.10) -> np.ndarray:
    """C2 shape: i.i.d. background + mutated copies of random consensus families."""
    rng = np.random.default_rng(seed)
    data = ACGT[rng.integers(0, 4, size=n, dtype=np.uint8)]
    cons = ACGT[rng.integers(0, 4, size=(families, family_len), dtype=np.uint8)]
    copies = int(coverage * n) // family_len
    if n < family_len or copies == 0:
        return data
    fam = rng.integers(0, families, size=copies)
    offs = rng.integers(0, n - family_len + 1, size=copies)
    for c in range(copies):
        seq = cons[fam[c]].copy()
        mut = rng.random(family_len) < divergence
        k = int(mut.sum())
        if k:
            seq[mut] = ACGT[rng.integers(0, 4, size=k, dtype=np.uint8)]
        data[offs[c]: offs[c] + family_len] = seq
    return data


def english_like(n: int, seed: int = 4, vocab: int = 50_000) -> np.ndarray:
    """C4 shape: Zipf(1) words of 1-12 symbols over printable ASCII, sigma=96."""
    rng = np.random.default_rng(seed)
    symbols = np.frombuffer(bytes(range(0x21, 0x7F)), np.uint8)  # 94 non-space printables
    wlen = rng.integers(1, 13, size=vocab)
    woff = np.zeros(vocab + 1, np.int64)
    np.cumsum(wlen, out=woff[1:])
    wbytes = symbols[rng.integers(0, symbols.size, size=int(woff[-1]))]
    weights = 1.0 / np.arange(1, vocab + 1)
    weights /= weights.sum()
    out = np.empty(n, np.uint8)
    pos = 0
    while pos < n:
        batch = max(1024, (n - pos) // 6 + 1024)
        ids = rng.choice(vocab, size=batch, p=weights)
        lens = wlen[ids] + 1  # word + separator
        ends = np.cumsum(lens)
        keep = int(np.searchsorted(ends, n - pos, side="left")) + 1
        keep = min(keep, batch)
        ids, lens, ends = ids[:keep], lens[:keep], ends[:keep]
        total = int(ends[-1])
        starts_out = ends - lens
        # gather word bytes: for output byte j in word w at offset o -> wbytes[woff[w] + o]
        word_of = np.repeat(np.arange(keep), lens)
        within = np.arange(total) - np.repeat(starts_out, lens)
        chunk = np.empty(total, np.uint8)
        is_sep = within == (lens[word_of] - 1)
        src = woff[ids[word_of]] + within
        chunk[~is_sep] = wbytes[src[~is_sep]]
        seps = np.where(rng.random(int(is_sep.sum())) < 0.08, ord("\n"), ord(" "))
        chunk[is_sep] = seps.astype(np.uint8)
        take = min(total, n - pos)
        out[pos: pos + take] = chunk[:take]
        pos += take
    return out


def fibonacci_mutated(n: int, seed: int = 5, rate: float = 1e-4,
                      alphabet: bytes = b"AC") -> np.ndarray:
    """C5 shape: Fibonacci word prefix over {A,C} + i.i.d. point substitutions."""
    a, b = alphabet[0:1], alphabet[0:1] + alphabet[1:2]  # f1 = "A", f2 = "AC"
    prev, cur = a, b
    while len(cur) < n:
        prev, cur = cur, cur + prev
    data = np.frombuffer(cur[:n], np.uint8).copy()
    del prev, cur
    rng = np.random.default_rng(seed)
    k = int(rng.binomial(n, rate)) if n else 0
    if k:
        pos = rng.choice(n, size=k, replace=False)
        data[pos] = ACGT[rng.integers(0, 4, size=k, dtype=np.uint8)]
    return data


def periodic_mutated(n: int, seed: int = 5, period: int = 1000, rate: float = 1e-4) -> np.ndarray:
    """Alternative C5 shape: a random period-p ACGT block tiled, with substitutions."""
    rng = np.random.default_rng(seed)
    block = ACGT[rng.integers(0, 4, size=period, dtype=np.uint8)]
    data = np.resize(block, n).copy()
    k = int(rng.binomial(n, rate)) if n else 0
    if k:
        pos = rng.choice(n, size=k, replace=False)
        data[pos] = ACGT[rng.integers(0, 4, size=k, dtype=np.uint8)]
    return data


CONFIGS = {
    "C1": dict(n=1 * MiB, make=lambda n: iid_dna(n, 1),
               desc="1 MiB i.i.d. ACGT, leftmost (CPU oracle config)"),
    "C2": dict(n=64 * MiB, make=lambda n: planted_dna(n, 2),
               desc="64 MiB DNA with planted Alu-like families, all ties"),
    "C3": dict(n=256 * MiB, make=lambda n: iid_dna(n, 3),
               desc="256 MiB i.i.d. ACGT, end-to-end SA+LCP+all-ties query"),
    "C4": dict(n=100 * MiB, make=lambda n: english_like(n, 4),
               desc="100 MiB English-like bytes (sigma~96, Zipf words)"),
    "C5": dict(n=1024 * MiB, make=lambda n: fibonacci_mutated(n, 5),
               desc="1 GiB Fibonacci word + 1e-4 mutations (compact path)"),
}


def make(config: str, n: int | None = None) -> np.ndarray:
    """Input bytes for a config, optionally truncated/resized to n."""
    c = CONFIGS[config]
    return c["make"](c["n"] if n is None else int(n))
