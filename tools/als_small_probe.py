"""Probe: one batched launch of the small-replica CP-ALS kernel at config-1
size (12 noisy 30^3 replicas, rank 10, a fixed number of sweeps) for ncu."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2311_13693_b200._lib import AlsConfig, check, lib, ptr

n, R, cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 30, 10, 12
its = int(sys.argv[2]) if len(sys.argv) > 2 else 200
rng = np.random.default_rng(0)
a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
t = np.einsum("ir,jr,kr->ijk", a, b, c)
t = t + 1e-2 * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(t.shape)
td = torch.from_numpy(np.asfortranarray(t).ravel(order="F")).cuda().repeat(cnt)
cfgs = (AlsConfig * cnt)()
for q in range(cnt):
    cfgs[q] = AlsConfig(R, its, 1e-300, q + 1, 0, 0)
fa = torch.zeros(cnt * n * R, dtype=torch.float64, device="cuda")
fb, fc = torch.zeros_like(fa), torch.zeros_like(fa)
it = torch.zeros(cnt, dtype=torch.int64, device="cuda")
cv = torch.zeros(cnt, dtype=torch.int32, device="cuda")
h = torch.zeros(cnt * its, dtype=torch.float64, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record()
check(lib.xtsg_cp_als_batched(cnt, ptr(td), n, n, n, cfgs, ptr(fa), ptr(fb), ptr(fc), ptr(it), ptr(cv), ptr(h)))
ev1.record()
torch.cuda.synchronize()
print(f"{cnt} x {n}^3 R={R}: iters {it.cpu().tolist()}, {ev0.elapsed_time(ev1) / max(1, int(it.max())) * 1e3:.1f} us/sweep")
if __import__("os").environ.get("XTSG_ALS_CL_DBG"):
    hh = h.view(cnt, its)[:, :8].cpu().numpy()
    names = ["mttkrp_A", "reduce+solve+gram_A", "P=A'T", "M_B reduce+solve+gram_B", "C rows+solve+allgather",
             "norms+grams", "residual+sync"]
    sw = hh[:, 7]
    print("cycles per sweep (mean over instances):", {n_: round(float(np.mean(hh[:, q] / sw))) for q, n_ in enumerate(names)},
          "total", round(float(np.mean(hh[:, :7].sum(1) / sw))))
    hs = h.view(cnt, its)[:, 8:12].cpu().numpy()
    print("A update split:", {n_: round(float(np.mean(hs[:, q] / sw))) for q, n_ in
                              enumerate(["H + cluster sync", "DSMEM reduce", "solve_gram", "gram"])})
