"""Where the compensated (fp16x3) C2 step goes: one plan.compress of a
resident f32 2000^3 block timed with CUDA events, the fused-TTM / mode-3
share from xtsg_plan_profile, and the rest (X hi/lo staging, gaps)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_13693_b200 as xt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
dev = torch.device("cuda", 0)
torch.manual_seed(0)
X = torch.randn((n, n, n), dtype=torch.float32, device=dev).permute(2, 1, 0)  # (i, j, k) column-major view
plan = xt.Plan((n, n, n), (64, 64, 64), 32, 40, 2, precision=xt.PREC_FP16X3)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
y = torch.zeros(32 * 64 ** 3, dtype=torch.float32, device=dev)
plan.compress(X, y=y, stream=s)
torch.cuda.synchronize()
plan.set_profiling(True)
plan.profile(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record(s)
for _ in range(reps):
    plan.compress(X, y=y, stream=s)
e1.record(s)
torch.cuda.synchronize()
prof = plan.profile(reset=True)
step = e0.elapsed_time(e1) / reps
print(json.dumps({"n": n, "ms_per_step": step, "profile": {k: (v / reps if "ms" in k else v) for k, v in prof.items()}}))
