"""Probe: C3 compression (10^4^3 rank 20, P = 124 x 128^3) on a k-range of
device-generated slabs, with the plan's live profile (fused TTM / mode-3
time) so the generator's share is the remainder."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2311_13693_b200 as xt

k1 = int(sys.argv[1]) if len(sys.argv) > 1 else 400
prec = {"bf16": xt.PREC_BF16, "fp16": xt.PREC_FP16, "fp16x3": xt.PREC_FP16X3}[sys.argv[2] if len(sys.argv) > 2 else "bf16"]
dims, red, P, S, R = (10000, 10000, 10000), (128, 128, 128), 124, 40, 20
f = xt.generate_factors(dims, R, seed=1)
plan = xt.Plan(dims, red, P, S, 7, precision=prec)
y = torch.zeros(P * 128 ** 3, dtype=torch.float32, device="cuda")
plan.compress_factors(f, 0, 40, y=y, device="cuda")
torch.cuda.synchronize()
plan.set_profiling(True)
plan.profile(reset=True)
t0 = time.perf_counter()
plan.compress_factors(f, 0, k1, y=y, device="cuda")
torch.cuda.synchronize()
dt = time.perf_counter() - t0
pr = plan.profile()
el = dims[0] * dims[1] * k1
print(f"k-range {k1}: {dt:.3f} s wall, {el / dt:.3e} elem/s; fused {pr['fused_ms']:.1f} ms "
      f"({pr['fused_flops'] / pr['fused_ms'] / 1e9:.1f} TF/s, {pr['fused_launches']} launches), "
      f"mode3 {pr['mode3_ms']:.1f} ms, rest (generator + glue) {dt * 1e3 - pr['fused_ms'] - pr['mode3_ms']:.1f} ms")
