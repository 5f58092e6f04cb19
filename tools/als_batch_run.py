import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2311_13693_b200 as xt
n, R, Q = int(sys.argv[1]), int(sys.argv[2]), 16
rng = np.random.default_rng(0)
ts = []
for q in range(Q):
    a, b, c = (rng.standard_normal((n, R)) for _ in range(3))
    ts.append(np.einsum("ir,jr,kr->ijk", a, b, c))
rs = xt.cp_als_batched(ts, R, seeds=list(range(Q)), max_iters=60)
print([x.iters for x in rs])
