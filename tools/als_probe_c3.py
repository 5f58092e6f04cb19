"""Probe: per-sweep time of the batched device CP-ALS at config-3 replica size
(128^3, rank 20) on noisy replicas like the bf16 compression produces. The
replicas are device-resident (no host staging inside the timed call)."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2311_13693_b200 as xt
from paper_2311_13693_b200._lib import AlsConfig, check, lib, ptr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
count = int(sys.argv[2]) if len(sys.argv) > 2 else 124
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
R = int(sys.argv[4]) if len(sys.argv) > 4 else 20
rng = np.random.default_rng(0)
a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
t = np.einsum("ir,jr,kr->ijk", a, b, c)
t = t + 3e-3 * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(t.shape)
td = torch.from_numpy(np.asfortranarray(t).ravel(order="F")).cuda().repeat(count)


def run(cnt, its):
    cfgs = (AlsConfig * cnt)()
    for q in range(cnt):
        cfgs[q] = AlsConfig(R, its, 1e-300, q + 1, 0, 0)
    fa = torch.zeros(cnt * n * R, dtype=torch.float64, device="cuda")
    fb, fc = torch.zeros_like(fa), torch.zeros_like(fa)
    it = torch.zeros(cnt, dtype=torch.int64, device="cuda")
    cv = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    h = torch.zeros(cnt * its, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(lib.xtsg_cp_als_batched(cnt, ptr(td), n, n, n, cfgs, ptr(fa), ptr(fb), ptr(fc), ptr(it), ptr(cv), ptr(h)))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if "--abs" in sys.argv:
        print(f"  batch={cnt} its={its}: {dt * 1e3:.2f} ms total, iters {sorted(set(it.cpu().tolist()))}")
    return dt, h[its - 1].item()


run(1, 2)
for cnt in (1, count):
    d1, _ = run(cnt, iters)
    d2, err = run(cnt, 2 * iters)
    print(f"n={n} R={R} batch={cnt}: {(d2 - d1) / iters * 1e3:.3f} ms/sweep (marginal), err {err:.3e}")
