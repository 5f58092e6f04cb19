import sys, time
sys.path.insert(0, ".")
import paper_2311_13693_b200 as xt
dims, R, red, P, S = (200, 200, 200), 10, (30, 30, 30), 12, 10
f = xt.generate_factors(dims, R, seed=1)
cfg = xt.PipelineConfig(reduced=red, rank=R, replicas=P, shared=S, precision=xt.PREC_FP64, seed=2)
xt.decompose(cfg, factors=f)
t0 = time.perf_counter(); rec, met = xt.decompose(cfg, factors=f); print(time.perf_counter() - t0, met.stage_seconds)
