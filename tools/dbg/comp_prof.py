import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13693_b200 as xt
from oracle.oracle import Restated
o = Restated()
dims, red, P, S = (2000, 2000, 2000), (64, 64, 64), 32, 40
f = o.generate_dense(dims, 20, 1)
dev = torch.device("cuda", 0)
for prec in (xt.PREC_BF16, xt.PREC_FP16X3):
    plan = xt.Plan(dims, red, P, S, o.derive(2, 11), precision=prec)
    y = plan.compress_factors(f, device=dev)
    torch.cuda.synchronize()
    plan.set_profiling(True)
    plan.profile(reset=True)
    for _ in range(3):
        t0 = time.perf_counter()
        plan.compress_factors(f, y=y, device=dev)
        torch.cuda.synchronize()
        print("  wall %.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
    print(prec, "%.1f ms" % ((time.perf_counter() - t0) * 1e3), plan.profile(reset=True), flush=True)
    plan.close()
