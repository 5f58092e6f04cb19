"""Probe: device CP-ALS on config-1 replicas (30^3, rank 10), batched and per call."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2311_13693_b200 as xt
from bench import derive
from oracle.oracle import Reference

dims, red, P, S, R = (200, 200, 200), (30, 30, 30), 12, 10, 10
a = xt.gen_gaussian(200, R, derive(1, 1)); b = xt.gen_gaussian(200, R, derive(1, 2)); c = xt.gen_gaussian(200, R, derive(1, 3))
ens = xt.make_ensemble(dims, red, P, S, derive(2, 11))
reps = [xt.comp_from_factors((a, b, c), ens.u[p], ens.v[p], ens.w[p]) for p in range(P)]
seeds = [derive(derive(2, 500 + p), 0) for p in range(P)]
xt.cp_als_batched(reps[:1], R, seeds=seeds[:1])
t = time.perf_counter(); res = xt.cp_als_batched(reps, R, seeds=seeds); dt = time.perf_counter() - t
print("batched 12:", round(dt, 4), "s iters", [r.iters for r in res], "conv", [r.converged for r in res],
      "err", ["%.1e" % r.final_error() for r in res])
t = time.perf_counter(); r1 = xt.cp_als(reps[0], R, seed=seeds[0]); dt = time.perf_counter() - t
print("single:", round(dt, 4), "s iters", r1.iters)
try:
    ref = Reference(); ref.L.xref_set_blas_threads(1)
    t = time.perf_counter(); out = [ref.cp_als(x, R, seed=s) for x, s in zip(reps, seeds)]; dt = time.perf_counter() - t
    print("reference serial 12:", round(dt, 4), "s iters", [o[1] for o in out], "err", ["%.1e" % o[2][-1] for o in out])
except Exception as e:
    print("no reference", e)
