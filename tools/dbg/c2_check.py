import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13693_b200 as xt
from oracle.oracle import Restated, rel_diff
o = Restated()
for dims, red, P, S in [((2000, 2000, 2000), (64, 64, 64), 32, 40), ((600, 500, 300), (64, 64, 64), 32, 40),
                        ((600, 500, 300), (64, 64, 64), 4, 40), ((600, 500, 300), (64, 64, 64), 32, 8)]:
    seed = o.derive(2, 11)
    f = o.generate_dense(dims, 20, 1)
    ens_o = o.ensemble_cols(dims, red, P, S, seed)
    ens_x = xt.make_ensemble(dims, red, P, S, seed)
    same = all(np.array_equal(ens_o[m][p], [ens_x.u, ens_x.v, ens_x.w][m][p]) for m in range(3) for p in range(P))
    plan = xt.Plan(dims, red, P, S, seed)
    y = xt.Plan.replicas(plan.compress_factors(f), P, red)
    e_o = [rel_diff(o.comp_from_factors(*f, ens_o[0][p], ens_o[1][p], ens_o[2][p]), y[p]) for p in range(P)]
    e_x = [rel_diff(xt.comp_from_factors(f, ens_x.u[p], ens_x.v[p], ens_x.w[p]), y[p]) for p in range(min(P, 4))]
    print(dims, P, S, "ens same", same, "err vs oracle", max(e_o), "vs xt", max(e_x), flush=True)
