"""Measurements of BASELINE.json's non-headline configs (SURVEY §8 d), one JSON
line each, for profiles/:

  c1  dense 200^3 rank 10, P = 12 x 30^3, S = 10: the device pipeline
      (decompose, fp64 compression) end to end vs the reference's own
      decompose (oracle/_ref) on the host cores, factor errors of both.
  c4  sparse COO 10^6^3, rank 10, 464 nonzeros per factor column (R rank-1
      blocks of 464^3 = 9.99e8 nonzeros, int32 coordinates + fp32 values,
      resident in HBM), P = 16 x 32^3: nonzeros/s, HBM roofline on the
      16 B/nonzero algorithmic traffic, plus a check against the exact
      comp_from_factors of the generating factors.
  c5  4000^3 dense bf16 (resident, 128 GB), L = M = N in {32, 64, 128},
      P in {16, 32, 64, 128}: fused-kernel TFLOP/s and fraction of the
      sustained bf16 peak per (L, P) point.

Timing: CUDA events on the launching stream after warm-up; inputs larger
than L2.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import derive, peaks  # noqa: E402


def emit(d, out):
    line = json.dumps(d)
    print(line, flush=True)
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


def c1(args):
    import paper_2311_13693_b200 as xt
    from oracle.oracle import Reference
    dims, R, red, P, S = (200, 200, 200), 10, (30, 30, 30), 12, 10
    xt.lib.xtsg_warmup()
    f = xt.generate_factors(dims, R, seed=1)
    cfg = xt.PipelineConfig(reduced=red, rank=R, replicas=P, shared=S, precision=xt.PREC_FP64, seed=2)
    xt.decompose(cfg, factors=f)  # warm-up (module load, pools)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        rec, met = xt.decompose(cfg, factors=f)
        walls.append(time.perf_counter() - t0)
    rep = xt.evaluate(f, rec)
    ref = Reference()
    ref.L.xref_set_blas_threads(1)
    threads = os.cpu_count() or 1
    rwalls = []
    for _ in range(2):
        t0 = time.perf_counter()
        rc, rrec, st = ref.decompose(f, dims, red, R, P, S, 2, workers=threads)
        rwalls.append(time.perf_counter() - t0)
    rerr, rmse = ref.evaluate(f, rrec)
    emit({"config": "C1: dense 200^3 rank-10, P=12 replicas of 30^3, S=10 (decompose end to end)",
          "xtsg": {"decompose_s": float(np.median(walls)), "stage_seconds": met.stage_seconds,
                   "mode_rel_err": rep.mode_rel_err, "sample_mse": rep.sample_mse,
                   "precision": "fp64 compression + fp64 ALS/LS on the device"},
          "reference": {"decompose_s": float(np.median(rwalls)), "rc": rc, "mode_rel_err": rerr,
                        "sample_mse": rmse, "threads": threads, "kind": "oracle/_ref (reference compiled in place)"},
          "speedup": float(np.median(rwalls) / np.median(walls))}, args.out)


def c4(args):
    import torch
    import paper_2311_13693_b200 as xt
    from oracle.oracle import rel_diff
    dims, R, npc, red, P, S = (10 ** 6,) * 3, 10, args.nnz_per_col, (32, 32, 32), 16, 8
    dev = torch.device("cuda", 0)
    f = xt.generate_factors(dims, R, law="sparse", nnz_per_col=npc, seed=1)
    # COO stream: the R rank-1 blocks a_r (x) b_r (x) c_r over their supports,
    # built on the device (k fastest within a block, blocks back to back)
    parts = []
    for r in range(R):
        sup = [np.nonzero(f[m][:, r])[0] for m in range(3)]
        val = [torch.tensor(f[m][sup[m], r], dtype=torch.float32, device=dev) for m in range(3)]
        idx = [torch.tensor(sup[m], dtype=torch.int32, device=dev) for m in range(3)]
        na, nb, nc = (len(s) for s in sup)
        ii = idx[0].view(na, 1, 1).expand(na, nb, nc).reshape(-1)
        jj = idx[1].view(1, nb, 1).expand(na, nb, nc).reshape(-1)
        kk = idx[2].view(1, 1, nc).expand(na, nb, nc).reshape(-1)
        vv = (val[0].view(na, 1, 1) * val[1].view(1, nb, 1) * val[2].view(1, 1, nc)).reshape(-1)
        parts.append((ii, jj, kk, vv))
    ci, cj, ck, cv = (torch.cat([p[q] for p in parts]) for q in range(4))
    del parts
    nnz = int(cv.numel())
    csf = None
    if args.csf:
        # the same nonzeros in CSF form (each rank-1 block is a dense 464^3
        # sub-cube: slices = its k support, fibers = its j support)
        sk, fj, ni, nv = [], [], [], []
        for r in range(R):
            sup = [torch.tensor(np.nonzero(f[m][:, r])[0], dtype=torch.int32, device=dev) for m in range(3)]
            val = [torch.tensor(f[m][np.nonzero(f[m][:, r])[0], r], dtype=torch.float32, device=dev)
                   for m in range(3)]
            na, nb, nc = (len(x) for x in sup)
            sk.append(sup[2])
            fj.append(sup[1].repeat(nc))
            ni.append(sup[0].repeat(nc * nb))
            nv.append((val[2].view(nc, 1, 1) * val[1].view(1, nb, 1) * val[0].view(1, 1, na)).reshape(-1))
        sk, fj, ni, nv = (torch.cat(x) for x in (sk, fj, ni, nv))
        per_slice = int(fj.numel() // sk.numel())
        per_fiber = int(ni.numel() // fj.numel())
        sp = torch.arange(0, sk.numel() + 1, dtype=torch.int64, device=dev) * per_slice
        fp = torch.arange(0, fj.numel() + 1, dtype=torch.int64, device=dev) * per_fiber
        csf = (sk, sp, fj, fp, ni, nv)
        del ci, cj, ck, cv
        nnz = int(nv.numel())
    if args.presorted:
        order = torch.argsort(ck.long() * dims[1] + cj.long())
        ci, cj, ck, cv = ci[order], cj[order], ck[order], cv[order]
        del order
    torch.cuda.synchronize()
    plan = xt.Plan(dims, red, P, S, derive(2, 11), precision=xt.PREC_BF16)
    y = torch.zeros(P * int(np.prod(red)), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    def step():
        if csf is not None:
            plan.compress_csf(*csf, y=y, stream=stream)
        else:
            plan.compress_coo(ci, cj, ck, cv, y=y, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = xt.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    mem_free, mem_total = torch.cuda.mem_get_info()
    launches = (xt.launch_count() - l0) / args.steps
    # exact check: comp_from_factors of the generating factors (linear in X;
    # duplicates sum), fp64 on the device, for a few replicas
    ens = xt.make_ensemble(dims, red, P, S, derive(2, 11))
    got = xt.Plan.replicas(y.cpu().numpy(), P, red)
    errs = []
    for p in range(0, P, max(1, P // 4)):
        want = xt.comp_from_factors(f, ens.u[p], ens.v[p], ens.w[p])
        errs.append(rel_diff(want, got[p]))
    _, _, hbm, src = peaks()
    rate = nnz / (ms / 1e3)
    achieved = 16.0 * rate / 1e9
    host_multi = None
    if args.host_multi:
        # the same nonzeros from HOST memory through xtsg_multi_compress_* on
        # this GPU (the C++ caller's route): H2D, validation, chunked device
        # calls, NCCL reduce and the replica read-back all inside the wall time
        host = [t.cpu().numpy() for t in (csf if csf is not None else (ci, cj, ck, cv))]
        del y, plan
        if csf is not None:
            del csf, sk, sp, fj, fp, ni, nv
        else:
            del ci, cj, ck, cv
        torch.cuda.empty_cache()
        mp = xt.MultiPlan(dims, red, P, S, derive(2, 11), gpus=[0], precision=xt.PREC_BF16)
        host_multi = []
        for chunk in args.chunks:
            os.environ["XTSG_SPARSE_CHUNK"] = str(chunk)
            run = (lambda: mp.compress_csf(*host)) if args.csf else (lambda: mp.compress_coo(*host))
            yh = run()
            walls, dev_ms = [], []
            for _ in range(args.steps):
                t0 = time.perf_counter()
                yh = run()
                walls.append(time.perf_counter() - t0)
                dev_ms.append(mp.last_ms())
            got = xt.Plan.replicas(yh, P, red)
            herr = max(rel_diff(xt.comp_from_factors(f, ens.u[p], ens.v[p], ens.w[p]), got[p])
                       for p in range(0, P, max(1, P // 4)))
            w = float(np.median(walls))
            host_multi.append({"chunk_nnz": chunk, "calls_per_step": -(-nnz // chunk), "wall_s": w,
                               "e2e_nnz_per_s": nnz / w, "device_ms_max_over_gpus": float(np.median(dev_ms)),
                               "h2d_bytes_per_step": int(sum(a.nbytes for a in host)),
                               "max_rel_err_vs_comp_from_factors": float(herr)})
        os.environ.pop("XTSG_SPARSE_CHUNK", None)
        mp.close()
    emit({"config": f"C4: sparse COO 10^6^3 rank-{R}, {npc} nnz/col -> {nnz:.4g} nonzeros "
                    f"({'CSF input, no sort' if args.csf else 'pre-sorted by (k, j)' if args.presorted else 'unsorted: sort inside the step'}), "
                    f"P={P} replicas of 32^3",
          "metric": "nonzeros compressed/sec", "value": rate, "unit": "nnz/s", "ms_per_step": ms,
          "steps": args.steps, "warmup": args.warmup, "kernel_launches_per_step": launches,
          "roofline": {"bound": "hbm (algorithmic 16 B/nnz) vs SIMT fp32 FMA (2*P*L = 1024 flop/nnz)",
                       "achieved_gbs": achieved, "peak_gbs": hbm, "frac": achieved / hbm,
                       "fma_tflops": 2.0 * P * red[0] * rate / 1e12, "peak_source": src},
          "max_rel_err_vs_comp_from_factors": float(max(errs)), "tolerance": 1e-2,
          "device_mem_free_gb": mem_free / 2**30, "torch_reserved_gb": torch.cuda.memory_reserved() / 2**30,
          "host_input_multi_api": host_multi}, args.out)


def c5(args):
    import torch
    import paper_2311_13693_b200 as xt
    from oracle.oracle import rel_diff
    n = args.n
    dims = (n, n, n)
    dev = torch.device("cuda", 0)
    R = 20
    A, B, Cf = (torch.from_numpy(xt.gen_gaussian(n, R, derive(1, m + 1))).to(dev, torch.float32) for m in range(3))
    X = torch.empty((n, n, n), dtype=torch.bfloat16, device=dev)
    for k in range(0, n, 50):
        X[k:k + 50] = torch.einsum("kr,jr,ir->kji", Cf[k:k + 50], B, A).to(torch.bfloat16)
    Xv = X.permute(2, 1, 0)
    torch.cuda.synchronize()
    _, sustained, _, src = peaks()
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    fac = tuple(t.double().cpu().numpy() for t in (A, B, Cf))
    for L in args.L:
        for P in args.P:
            red = (L, L, L)
            S = min(L // 2, 40)
            try:
                plan = xt.Plan(dims, red, P, S, derive(2, 11), precision=xt.PREC_BF16)
            except xt.XtsError as e:
                emit({"config": f"C5 point L={L} P={P}", "unsupported": str(e)}, args.out)
                continue
            y = torch.zeros(P * L ** 3, dtype=torch.float32, device=dev)
            plan.compress(Xv, y=y, stream=stream)
            torch.cuda.synchronize()
            plan.set_profiling(True)
            plan.profile(reset=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                plan.compress(Xv, y=y, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            pr = plan.profile(reset=True)
            tf = pr["fused_flops"] / (pr["fused_ms"] / 1e3) / 1e12
            fe = 2.0 * P * L * (1 + L / n + L * L / (n * n))
            # spot check replica 0 against the exact fp64 comp_from_factors of
            # the (bf16-rounded X's) generating factors
            ens = xt.make_ensemble(dims, red, P, S, derive(2, 11))
            got = xt.Plan.replicas(y.cpu().numpy(), P, red)
            err = max(rel_diff(xt.comp_from_factors(fac, ens.u[p], ens.v[p], ens.w[p]), got[p]) for p in (0, P - 1))
            emit({"config": f"C5: {n}^3 dense bf16 resident, L=M=N={L}, P={P}",
                  "elements_per_s": n ** 3 / (ms / 1e3), "ms_per_step": ms,
                  "flop_per_element": fe, "step_tflops": fe * n ** 3 / (ms / 1e3) / 1e12,
                  "fused_kernel_tflops": tf, "frac_of_sustained_bf16": tf / sustained,
                  "fused_share_of_step": pr["fused_ms"] / (ms * args.steps), "peak_source": src,
                  "max_rel_err_vs_fp64": err}, args.out)
            plan.close()
            del y


def twostage(args):
    """Two-stage compression as a true two-pass on the C2 tensor:
    2000^3 bf16 resident, P = 32 replicas of 64^3, inner 1.6x (102^3, sparse
    inner law): stage 1 on the tensor cores is one 102-row replica, so the
    pass is HBM-bound (2 B per element, 2*102*(1+...) flop per element)."""
    import torch
    import paper_2311_13693_b200 as xt
    from oracle.oracle import rel_diff
    n, R = args.n if args.n != 4000 else 2000, 20
    dims, red, P, S = (n, n, n), (64, 64, 64), 32, 40
    dev = torch.device("cuda", 0)
    A, B, Cf = (torch.from_numpy(xt.gen_gaussian(n, R, derive(1, m + 1))).to(dev, torch.float32) for m in range(3))
    X = torch.empty((n, n, n), dtype=torch.bfloat16, device=dev)
    for k in range(0, n, 50):
        X[k:k + 50] = torch.einsum("kr,jr,ir->kji", Cf[k:k + 50], B, A).to(torch.bfloat16)
    Xv = X.permute(2, 1, 0)
    spec = dict(kind="two_stage", alpha=1.6, beta=1.6, gamma=1.6, inner_kind="sparse", inner_s=2.0)
    plan = xt.Plan(dims, red, P, S, derive(2, 11), **spec)
    y = torch.zeros(P * 64 ** 3, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    plan.compress(Xv, y=y, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.compress(Xv, y=y, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    _, _, hbm, src = peaks()
    rate = n ** 3 / (ms / 1e3)
    ens = xt.make_ensemble(dims, red, P, S, derive(2, 11), **spec)
    fac = tuple(t.double().cpu().numpy() for t in (A, B, Cf))
    got = xt.Plan.replicas(y.cpu().numpy(), P, red)
    err = max(rel_diff(xt.comp_from_factors(fac, ens.u[p], ens.v[p], ens.w[p]), got[p]) for p in (0, P - 1))
    emit({"config": f"two-stage (true two-pass) on {n}^3 bf16 resident, P={P} x 64^3, inner 1.6x (sparse law, s=2)",
          "elements_per_s": rate, "ms_per_step": ms, "steps": args.steps,
          "vs_one_stage_c2": "bench.py (same tensor, one-stage): ~2.8e11 elements/s",
          "roofline": {"bound": "hbm (2 B per element of X)", "achieved_gbs": 2.0 * rate / 1e9, "peak_gbs": hbm,
                       "frac": 2.0 * rate / 1e9 / hbm, "peak_source": src},
          "max_rel_err_vs_fp64_materialized_ensemble": err, "tolerance": 1e-2}, args.out)


def omp(args):
    """OMP recovery on the device at large dictionaries (sparse
    factors at 10^6 atoms): rows = stacked compressed rows, R columns with s
    nonzeros each, Gaussian dictionary (unit columns); time and support recovery."""
    import torch
    from paper_2311_13693_b200._lib import check, lib
    dev = torch.device("cuda", 0)
    rows, R, s = 512, 10, args.sparsity
    for atoms in (10 ** 4, 10 ** 5, 10 ** 6):
        g = torch.Generator(device=dev)
        g.manual_seed(atoms)
        D = torch.randn(atoms, rows, dtype=torch.float64, device=dev, generator=g).t().contiguous()  # column-major rows x atoms
        D = D / D.norm(dim=0, keepdim=True)
        Dcm = D.t().contiguous()          # (atoms, rows) row-major == rows x atoms column-major
        X = torch.zeros(R, atoms, dtype=torch.float64, device=dev)
        rng = np.random.default_rng(atoms)
        supp = [np.sort(rng.choice(atoms, s, replace=False)) for _ in range(R)]
        for c in range(R):
            X[c, supp[c]] = torch.tensor(rng.choice([-1.0, 1.0], s) * (1 + rng.random(s)), dtype=torch.float64,
                                         device=dev)
        Y = (D @ X.t()).t().contiguous()  # (R, rows) row-major == rows x R column-major
        out = torch.zeros(R, atoms, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        check(lib.xtsg_omp_recover(Y.data_ptr(), rows, R, Dcm.data_ptr(), atoms, s, 1e-9, out.data_ptr()))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        check(lib.xtsg_omp_recover(Y.data_ptr(), rows, R, Dcm.data_ptr(), atoms, s, 1e-9, out.data_ptr()))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        got = out.cpu().numpy()
        ok = sum(set(np.nonzero(np.abs(got[c]) > 1e-6)[0]) == set(supp[c]) for c in range(R))
        err = float((out - X).norm() / X.norm())
        emit({"config": f"OMP: {rows} measured rows x {atoms:.0e} atoms, {R} columns, sparsity {s}",
              "seconds": dt, "supports_recovered": f"{ok}/{R}", "rel_err": err}, args.out)
        del D, Dcm, X, Y, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c1", "c4", "c5", "twostage", "omp"])
    ap.add_argument("--sparsity", type=int, default=16)
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--nnz-per-col", type=int, default=464)
    ap.add_argument("--presorted", action="store_true")
    ap.add_argument("--csf", action="store_true")
    ap.add_argument("--host-multi", action="store_true",
                    help="c4: also time host input through xtsg_multi_compress_* (1 GPU)")
    ap.add_argument("--chunks", type=int, nargs="+", default=[2 ** 31, 250_000_000])
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--L", type=int, nargs="+", default=[32, 64, 128])
    ap.add_argument("--P", type=int, nargs="+", default=[16, 32, 64, 128])
    a = ap.parse_args()
    {"c1": c1, "c4": c4, "c5": c5, "twostage": twostage, "omp": omp}[a.which](a)


if __name__ == "__main__":
    main()
