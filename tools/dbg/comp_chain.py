"""Error of the compensated mode vs the contraction lengths (debug)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2311_13693_b200 as xt
from oracle.oracle import Restated, rel_diff
o = Restated()
for dims in [(64, 64, 40), (64, 256, 40), (64, 1024, 40), (256, 64, 40), (1024, 64, 40), (4096, 64, 40)]:
    red, P, S, seed = (64, 64, 32), 4, 8, 5
    t = np.asfortranarray(np.random.default_rng(0).standard_normal(dims))
    ens = o.make_ensemble(dims, red, P, S, seed)
    want = [o.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = xt.Plan(dims, red, P, S, seed, precision=xt.PREC_FP16X3)
    y = plan.compress(t)
    n = int(np.prod(red))
    e = [rel_diff(w, y[p * n:(p + 1) * n].reshape(red, order="F")) for p, w in enumerate(want)]
    # the same in fp64 emulation of the split arithmetic (no accumulation error)
    print(dims, "kpc", os.environ.get("XTSG_COMP_KPC", "32"), "max err %.3e" % max(e), flush=True)
