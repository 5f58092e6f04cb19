"""Device pipeline with the compensated compression at the reference's
default replica_fit_tol (1e-6): survivors, factor errors (debug)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2311_13693_b200 as xt
for dims, R, L, S in [((1000,) * 3, 10, 64, 20), ((2000,) * 3, 20, 64, 40)]:
    f = xt.generate_factors(dims, R, seed=1)
    for prec in (xt.PREC_FP16X3, xt.PREC_BF16):
        cfg = xt.PipelineConfig(reduced=(L, L, L), rank=R, shared=S, precision=prec, seed=2)
        t0 = time.perf_counter()
        try:
            rec, met = xt.decompose(cfg, factors=f)
            ev = xt.evaluate(f, rec)
            print(dims[0], "prec", prec, "dropped", met.replicas_dropped, "of", met.replicas_total,
                  "factor err", ["%.2e" % e for e in ev.mode_rel_err], "stages", {k: round(v, 2) for k, v in met.stage_seconds.items()},
                  "%.1f s" % (time.perf_counter() - t0), flush=True)
        except Exception as e:
            print(dims[0], "prec", prec, "FAILED:", str(e)[:200], flush=True)
