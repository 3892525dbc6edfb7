"""Suffix-sort time with text-order round keys vs the list gather (RS_SA_LIST_KEYS).

Each config: build the SA twice per mode (the second timed), compare the sa /
rank / lcp digests with tests/golden/fullsize_digests.json.
"""
import hashlib, json, os, subprocess, sys, time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]

CHILD = r'''
import hashlib, json, sys, time
import numpy as np
sys.path.insert(0, %r)
import paper_1501_06663_b200 as rb
from paper_1501_06663_b200 import workloads, _native
cfg = sys.argv[1]
rec = json.load(open(%r))[cfg]
t = rb.Text(workloads.make(cfg))
ctx = _native.context(0)
def dg(a):
    a = np.ascontiguousarray(a, dtype=np.int64); return hashlib.sha256(memoryview(a).cast("B")).hexdigest()[:16]
for rep in range(2):
    t0 = time.perf_counter()
    with ctx.lock:
        ctx.call("rs_set_text", _native.u8(t.data), t.n)
        ctx.call("rs_build_structures")
        ctx.call("rs_synchronize")
    dt = time.perf_counter() - t0
s = rb.build_suffix_structures(t)
ok = dg(s.sa) == rec["sa"] and dg(s.rank) == rec["rank"] and dg(s.lcp) == rec["lcp"]
print(json.dumps({"config": cfg, "sa_s": dt, "rounds": ctx.sa_rounds(), "digests_ok": ok}))
'''
for cfg in sys.argv[1:] or ["C3", "C4", "C5"]:
    for mode in ("text", "list"):
        env = dict(os.environ)
        if mode == "list":
            env["RS_SA_LIST_KEYS"] = "1"
        code = CHILD % (str(REPO), str(REPO / "tests/golden/fullsize_digests.json"))
        r = subprocess.run([sys.executable, "-c", code, cfg], env=env, capture_output=True, text=True)
        print(mode, r.stdout.strip() or r.stderr[-2000:], flush=True)
