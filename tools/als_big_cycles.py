"""Probe: per-phase SM cycles of the large-replica CP-ALS kernel (pass 1,
pass 2, mode-3 MTTKRP from P, whole loop) at config-3 replica size, from the
kernel's XTSG_ALS_BIG_DBG=8 instrumentation (timing experiments only)."""
import os
import sys
sys.path.insert(0, ".")
os.environ["XTSG_ALS_BIG_DBG"] = "8"
import numpy as np
import torch
from paper_2311_13693_b200._lib import AlsConfig, check, lib, ptr

n, cnt, its, R = 128, int(sys.argv[1]) if len(sys.argv) > 1 else 124, int(sys.argv[2]) if len(sys.argv) > 2 else 10, 20
rng = np.random.default_rng(0)
a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
t = np.einsum("ir,jr,kr->ijk", a, b, c)
t = t + 3e-3 * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(t.shape)
td = torch.from_numpy(np.asfortranarray(t).ravel(order="F")).cuda().repeat(cnt)
cfgs = (AlsConfig * cnt)()
for q in range(cnt):
    cfgs[q] = AlsConfig(R, its, 1e-300, q + 1, 0, 0)
fa = torch.zeros(cnt * n * R, dtype=torch.float64, device="cuda")
fb, fc = torch.zeros_like(fa), torch.zeros_like(fa)
it = torch.zeros(cnt, dtype=torch.int64, device="cuda")
cv = torch.zeros(cnt, dtype=torch.int32, device="cuda")
h = torch.zeros(cnt * its, dtype=torch.float64, device="cuda")
for rep in range(2):
    check(lib.xtsg_cp_als_batched(cnt, ptr(td), n, n, n, cfgs, ptr(fa), ptr(fb), ptr(fc), ptr(it), ptr(cv), ptr(h)))
    torch.cuda.synchronize()
hh = h.view(cnt, its)[:, :5].cpu().numpy()
sw = hh[:, 4]
print(f"batch {cnt}, sweeps {sorted(set(sw.tolist()))}; cycles per sweep (mean over CTAs): "
      f"pass1 {np.mean(hh[:, 0] / sw):.0f}, pass2 {np.mean(hh[:, 1] / sw):.0f}, mttkrp_c {np.mean(hh[:, 2] / sw):.0f}, "
      f"loop {np.mean(hh[:, 3] / sw):.0f}")
