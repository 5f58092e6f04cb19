"""Tensor-core tile path vs SIMT fiber kernel (XTSG_SPARSE_TC=0) on
hypersparse random COO (one nonzero per fiber, ~nnz/dims per slice)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_13693_b200 as xt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10 ** 6
nnz = int(sys.argv[2]) if len(sys.argv) > 2 else 10 ** 7
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
i, j, k = (torch.randint(0, n, (nnz,), device=dev, dtype=torch.int32, generator=g) for _ in range(3))
v = torch.randn(nnz, device=dev, generator=g)
order = torch.argsort(k.long() * n + j.long())
i, j, k, v = i[order], j[order], k[order], v[order]
plan = xt.Plan((n, n, n), (32, 32, 32), 16, 8, 3, precision=xt.PREC_BF16)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
y = torch.zeros(16 * 32 ** 3, device=dev)
out = {"dims": n, "nnz": nnz}
for mode in ("1", "0"):
    os.environ["XTSG_SPARSE_TC"] = mode
    plan.compress_coo(i, j, k, v, y=y, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3):
        plan.compress_coo(i, j, k, v, y=y, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    out["tc_ms" if mode == "1" else "fiber_ms"] = e0.elapsed_time(e1) / 3
    out["y_" + mode] = y.clone()
out["rel_diff"] = float((out["y_1"] - out["y_0"]).norm() / out["y_0"].norm())
del out["y_1"], out["y_0"]
print(json.dumps(out))
