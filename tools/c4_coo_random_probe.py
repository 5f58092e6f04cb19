"""Probe: C4 (10^6^3 rank 10, 464 nonzeros per factor column, 9.99e8
nonzeros) as device COO in random order, the bench's sparse_c4 input, timed
per call; run with XTSG_TRACE=1 for the phase split of the COO path."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2311_13693_b200 as xt

dev = torch.device("cuda", 0)
dims, R, npc, red, P, S = (10 ** 6,) * 3, 10, 464, (32, 32, 32), 16, 8
f = xt.generate_factors(dims, R, law="sparse", nnz_per_col=npc, seed=1)
ci, cj, ck, cv = [], [], [], []
for r in range(R):
    sup = [np.nonzero(f[m][:, r])[0] for m in range(3)]
    val = [torch.tensor(f[m][sup[m], r], dtype=torch.float32, device=dev) for m in range(3)]
    idx = [torch.tensor(x, dtype=torch.int32, device=dev) for x in sup]
    na, nb, nc = (len(x) for x in sup)
    ck.append(idx[2].repeat_interleave(nb * na))
    cj.append(idx[1].repeat_interleave(na).repeat(nc))
    ci.append(idx[0].repeat(nc * nb))
    cv.append((val[2].view(nc, 1, 1) * val[1].view(1, nb, 1) * val[0].view(1, 1, na)).reshape(-1))
ci, cj, ck, cv = (torch.cat(x) for x in (ci, cj, ck, cv))
order = sys.argv[1] if len(sys.argv) > 1 else "random"
if order == "random":
    perm = torch.randperm(cv.numel(), device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    ci, cj, ck, cv = ci[perm], cj[perm], ck[perm], cv[perm]
    del perm
plan = xt.Plan(dims, red, P, S, 7, precision=xt.PREC_BF16)
y = torch.zeros(P * 32 ** 3, dtype=torch.float32, device=dev)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.compress_coo(ci, cj, ck, cv, y=y)
    torch.cuda.synchronize()
    print(f"{order} COO, {cv.numel():.3e} nonzeros: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
