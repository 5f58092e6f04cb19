"""Probe: per-sweep time of the batched device CP-ALS at C3 replica size
(128^3, rank 20), noisy replicas like the bf16 compression produces."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2311_13693_b200 as xt

n, R = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 20
count = int(sys.argv[2]) if len(sys.argv) > 2 else 124
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(0)
a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
t = np.einsum("ir,jr,kr->ijk", a, b, c)
t = t + 3e-3 * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(t.shape)
t = np.asfortranarray(t)
ts = [t] * count
xt.cp_als_batched(ts[:1], R, max_iters=2, tol=1e-300, seeds=[1])
for cnt in (1, count):
    t0 = time.perf_counter()
    res = xt.cp_als_batched(ts[:cnt], R, max_iters=iters, tol=1e-300, seeds=list(range(cnt)))
    dt = time.perf_counter() - t0
    print(f"n={n} R={R} batch={cnt}: {dt / iters * 1e3:.2f} ms/sweep, err {res[0].final_error():.3e}")
