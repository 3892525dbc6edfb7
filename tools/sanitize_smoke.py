"""Small end-to-end run for compute-sanitizer (memcheck): every kernel family once."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1501_06663_b200 as rb
from paper_1501_06663_b200 import workloads

for data in (workloads.iid_dna(20000, 1), workloads.planted_dna(30000, 2, family_len=100),
             workloads.english_like(20000, 4), workloads.fibonacci_mutated(30000, 5, rate=1e-3),
             np.frombuffer(b"mississippi", np.uint8), np.frombuffer(b"a", np.uint8)):
    t = rb.Text(data)
    s = rb.build_suffix_structures(t)
    assert rb.verify_suffix_structures(t, s)
    raw = rb.build_raw_llr(s)
    c = rb.build_compact_llr(raw)
    f = rb.compute_flags(raw)
    rb.scatter_compact(raw, f, rb.prefix_sum(f))
    for path in ("raw", "compact"):
        for mode in ("leftmost", "all"):
            rb.all_positions(t, mode=mode, path=path)
            rb.all_positions(t, mode=mode, path=path, structures=s)
print("sanitize smoke done")
