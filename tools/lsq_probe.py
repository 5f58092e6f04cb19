"""Probe: stacked least squares at config-3 size (124 replicas x 128 rows
stacked = 15,872 x 10,000 per mode, rank-20 right-hand sides) through the
public solve_stacked_ls (host fp64 in and out, as the pipeline's recovery
stage calls it per mode)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import paper_2311_13693_b200 as xt

P, L, I, R = 124, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 10000, 20
rng = np.random.default_rng(0)
x = rng.standard_normal((I, R))
us = [np.asfortranarray(rng.standard_normal((L, I))) for _ in range(P)]
fs = [np.asfortranarray(u @ x) for u in us]
xt.solve_stacked_ls(fs[:2], [u[:, :200] for u in us[:2]])  # warm-up (context, kernels)
for rep in range(2):
    t0 = time.perf_counter()
    sol = xt.solve_stacked_ls(fs, us)
    dt = time.perf_counter() - t0
    print(f"{P * L} x {I}, {R} rhs: {dt:.3f} s, rel err {np.linalg.norm(sol - x) / np.linalg.norm(x):.2e}")
