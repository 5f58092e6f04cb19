"""Throughput of the fp64 plan path (XTSG_PREC_FP64: the reference's own
precision, what comp / comp_blocked promise) on a resident f64 n^3 block,
P = 32 replicas of 64^3, vs the bf16 tensor-core path on the same block."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_13693_b200 as xt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dev = torch.device("cuda", 0)
torch.manual_seed(0)
X64 = torch.randn((n, n, n), dtype=torch.float64, device=dev).permute(2, 1, 0)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
out = {"n": n, "replicas": 32, "reduced": 64}
for name, prec, X in (("fp64", xt.PREC_FP64, X64), ("bf16", xt.PREC_BF16, X64.to(torch.bfloat16))):
    plan = xt.Plan((n, n, n), (64, 64, 64), 32, 40, 2, precision=prec)
    y = torch.zeros(32 * 64 ** 3, dtype=torch.float64 if prec == xt.PREC_FP64 else torch.float32, device=dev)
    plan.compress(X, y=y, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3):
        plan.compress(X, y=y, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    flops = 2.0 * 32 * 64 * (n ** 3 + 64 * n * n + 64 * 64 * n)
    out[name] = {"ms": ms, "elements_per_s": n ** 3 / (ms / 1e3), "tflops": flops / (ms / 1e3) / 1e12}
    plan.close()
print(json.dumps(out))
