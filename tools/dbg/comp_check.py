"""Compensated (fp16x3) tensor-core mode: replica errors vs the oracle at
several sizes, and timing vs bf16 (debug tool)."""
import os, sys, time
sys.path.insert(0, '.')
from concurrent.futures import ThreadPoolExecutor
import numpy as np, torch
import paper_2311_13693_b200 as xt
from oracle.oracle import Restated, rel_diff
o = Restated()
dev = torch.device("cuda", 0)
which = sys.argv[1:] or ["small", "mid", "c2", "c3"]


def oracle_fac(f, dims, red, P, S, seed, cols=None):
    cols = cols or [np.arange(n) for n in dims]
    a, b, c = (np.asfortranarray(x[i]) for x, i in zip(f, cols))
    ens = o.ensemble_cols(dims, red, P, S, seed, cols=cols)
    with ThreadPoolExecutor(16) as ex:
        return list(ex.map(lambda p: o.comp_from_factors(a, b, c, ens[0][p], ens[1][p], ens[2][p]), range(P)))


def errs(want, y, P, red):
    y = y.cpu().numpy() if isinstance(y, torch.Tensor) else y
    n = int(np.prod(red))
    return [rel_diff(w, y[p * n:(p + 1) * n].reshape(red, order="F")) for p, w in enumerate(want)]


kpc = os.environ.get("XTSG_COMP_KPC", "32")
if "small" in which:
    dims, red, P, S = (256, 300, 72), (64, 64, 64), 4, 8
    seed = 77
    t = np.asfortranarray(np.random.default_rng(0).standard_normal(dims))
    ens = o.make_ensemble(dims, red, P, S, seed)
    want = [o.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    for prec in (xt.PREC_BF16, xt.PREC_FP16X3):
        plan = xt.Plan(dims, red, P, S, seed, precision=prec)
        y = plan.compress(t)
        print("small dense", prec, "max err %.3e" % max(errs(want, y, P, red)), flush=True)
    # L=30 (padded), P=12 odd row blocks
    dims, red, P, S = (200, 200, 200), (30, 30, 30), 12, 10
    ens = o.make_ensemble(dims, red, P, S, seed)
    t = np.asfortranarray(np.random.default_rng(1).standard_normal(dims))
    want = [o.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = xt.Plan(dims, red, P, S, seed, precision=xt.PREC_FP16X3)
    print("C1 shape dense fp16x3 max err %.3e" % max(errs(want, plan.compress(t), P, red)), flush=True)
for name, dims, red, P, S, k in [("mid", (600, 500, 300), (64, 64, 64), 32, 40, None),
                                ("c2", (2000, 2000, 2000), (64, 64, 64), 32, 40, None),
                                ("c3", (10000, 10000, 10000), (128, 128, 128), 124, 40, (0, 40))]:
    if name not in which:
        continue
    seed = o.derive(2, 11)
    f = o.generate_dense(dims, 20, 1)
    cols = None if k is None else [np.arange(dims[0]), np.arange(dims[1]), np.arange(*k)]
    want = oracle_fac(f, dims, red, P, S, seed, cols)
    for prec in (xt.PREC_BF16, xt.PREC_FP16X3):
        plan = xt.Plan(dims, red, P, S, seed, precision=prec)
        kk = k or (0, dims[2])
        y = plan.compress_factors(f, kk[0], kk[1], device=dev)
        torch.cuda.synchronize()
        e = errs(want, y, P, red)
        t0 = time.perf_counter()
        for _ in range(2):
            plan.compress_factors(f, kk[0], kk[1], y=y, device=dev)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 2
        print(f"{name} prec {prec} kpc {kpc}: max err {max(e):.3e} mean {np.mean(e):.3e}  {dt*1e3:.1f} ms", flush=True)
        plan.close()
