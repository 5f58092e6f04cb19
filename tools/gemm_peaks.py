"""Library GEMM peaks on this B200 for the roofline denominators the survey
lists as unmeasured (tf32 tensor cores, fp64 DMMA) next to bf16: cuBLAS via
torch.matmul on square n^3 problems, CUDA events, best of 5 after warm-up.
These are reference points for the precision modes, not a kernel of ours."""
import json
import sys

import torch


def rate(dtype, n, tf32=False, reps=5):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 4)
    return 2.0 * n ** 3 / (best / 1e3) / 1e12, best


out = {}
for name, dt, n, tf32 in (("bf16", torch.bfloat16, 8192, False), ("tf32", torch.float32, 8192, True),
                          ("fp32_simt", torch.float32, 8192, False), ("fp64", torch.float64, 8192, False)):
    tf, ms = rate(dt, n, tf32)
    out[name] = {"tflops": round(tf, 1), "ms": round(ms, 3), "n": n}
out["how"] = "cuBLAS through torch.matmul, square n^3, best of 5 x 4 back-to-back calls, 2 flop per FMA"
out["device"] = torch.cuda.get_device_name(0)
print(json.dumps(out))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        f.write(json.dumps(out) + "\n")
