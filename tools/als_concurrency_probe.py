"""Per-call cost of the device CP-ALS as the reference pipeline uses it
(pipeline.cpp:410-434: one cp_als per replica from parallel_for workers) vs one
batched call: 40^3 rank-20 replicas (the factors1000 drop-in case)."""
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_13693_b200 as xt  # noqa: E402

n, R, Q = int(sys.argv[1]) if len(sys.argv) > 1 else 40, 20, 16
rng = np.random.default_rng(0)
ts = []
for q in range(Q):
    a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
    ts.append(np.einsum("ir,jr,kr->ijk", a, b, c))
xt.cp_als(ts[0], R, seed=1)  # warm-up
out = {"n": n, "rank": R, "tensors": Q}
t0 = time.perf_counter()
r = xt.cp_als(ts[0], R, seed=1)
out["single_call_s"] = time.perf_counter() - t0
out["single_iters"] = r.iters
t0 = time.perf_counter()
rs = xt.cp_als_batched(ts, R, seeds=list(range(Q)))
out["batched_s"] = time.perf_counter() - t0
out["batched_iters"] = [x.iters for x in rs]
res = [None] * Q
def work(q):
    res[q] = xt.cp_als(ts[q], R, seed=q)
th = [threading.Thread(target=work, args=(q,)) for q in range(Q)]
t0 = time.perf_counter()
for t in th:
    t.start()
for t in th:
    t.join()
out["threads_s"] = time.perf_counter() - t0
out["thread_iters"] = [x.iters for x in res]
print(json.dumps(out))
