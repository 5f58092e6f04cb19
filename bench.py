#!/usr/bin/env python
"""Headline benchmark: input tensor elements compressed per second (BASELINE.json).

Workload (BASELINE.json configs[1], "C2"): dense 2000^3 rank-20 tensor,
P = 32 replicas of 64^3, S = 40 shared anchor rows, Gaussian ensemble from the
bit-exact device RNG. One step = one pass of the hot path (fused tcgen05
mode-1/2 TTM + mode-3 GEMM) over the rank's 2000^3 block resident in HBM as
bf16 (16 GB > L2, so no flush is needed between steps); for N > 1 every rank
owns one mode-3 slab of a (2000, 2000, 2000*N) tensor (weak scaling, per-GPU
work fixed) and the partial replicas are summed with one NCCL reduce.

`e2e` is the same metric through the public C ABI with HOST buffers: the
rank's block sits in pinned host memory and every step streams it H2D inside
xtsg_plan_compress (double-buffered copy/convert/compute) and reads the
replicas back D2H.

`--impl reference` times the reference's own CPU implementation (compiled in
place into oracle/_ref) on the box's host cores: comp_blocked fast mode on a
bounded mode-3 slab sample of the same workload.

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU); NCCL_DEBUG=INFO is set so
the communicator's rank count is in the log. `--cpu-smoke` runs the same rank
plumbing (spawn, slab split, reduce, max-over-ranks timing, JSON line) on CPU
with gloo and a torch einsum per rank, for the CPU test suite; it is never a
bench number. After the timed region rank 0 checks two replicas of the timed
output against the CPU oracle (comp_from_factors of the generating factors)
and reports `parity.max_rel_err`.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GOLD = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1

C2 = dict(I=2000, J=2000, K=2000, L=64, M=64, N=64, P=32, S=40, R=20, seed=2, factor_seed=1)


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def derive(seed, tag):
    """rng.hpp:46-50"""
    s = (seed ^ ((GOLD * (tag + 0x632BE59BD9B4E019)) & M64)) & M64
    return _mix((s + 2 * GOLD) & M64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--cpu-smoke", action="store_true",
                    help="rank plumbing on CPU (gloo, torch einsum per rank): for the CPU test suite, not a bench")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="xtsg", choices=["xtsg", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-dtype", default="f32", choices=["bf16", "f32", "f64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cp-time", action="store_true")
    ap.add_argument("--no-c3", action="store_true",
                    help="skip the north-star C3 decompose (10^4^3 rank 20, P = 124 x 128^3) after the C2 timing")
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the sparse C4 line (10^6^3, 1e9 nonzeros as CSF; one GPU runs only)")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp16", "fp16x3"],
                    help="tensor-core operand type (fp16: 3 more mantissa bits, same speed; fp16x3: the "
                         "compensated hi/lo mode, ~1e-6 replicas at ~3x the tensor-core work)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--K", type=int, default=C2["K"], help="mode-3 extent per rank (testing)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampler for the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_block(torch, xt, cfg, k0, K, device, dtype=None):
    """Rank's block X[:, :, k0:k0+K] of reconstruct(A, B, C) as bf16, (I, J, K) column-major.

    Factors follow generate({dims, R, dense, seed}) (pipeline.cpp:182-193): one
    polar stream per matrix from derive(seed, 1|2|3), drawn on the device."""
    I, J, R = cfg["I"], cfg["J"], cfg["R"]
    Ktot = cfg["Ktot"]
    A = torch.from_numpy(xt.gen_gaussian(I, R, derive(cfg["factor_seed"], 1))).to(device, torch.float32)
    B = torch.from_numpy(xt.gen_gaussian(J, R, derive(cfg["factor_seed"], 2))).to(device, torch.float32)
    Cf = torch.from_numpy(xt.gen_gaussian(Ktot, R, derive(cfg["factor_seed"], 3))).to(device, torch.float32)
    dtype = dtype or torch.bfloat16
    X = torch.empty((K, J, I), dtype=dtype, device=device)
    step = 50
    for k in range(0, K, step):
        kk = min(step, K - k)
        ck = Cf[k0 + k:k0 + k + kk]                       # (kk, R)
        # X[k, j, i] = sum_r A[i, r] B[j, r] C[k, r]
        X[k:k + kk] = torch.einsum("kr,jr,ir->kji", ck, B, A).to(dtype)
    return X.permute(2, 1, 0), (A, B, Cf)


def cpu_reference_rate(cfg, seconds, threads):
    """Reference comp_blocked (fast mode, compression.cpp:381-403) on a
    (I, J, ks) mode-3 slab of the workload; returns (elements/s, sample)."""
    from oracle.oracle import Reference
    ref = Reference()
    ref.L.xref_set_blas_threads(1)      # one BLAS thread per parallel_for worker
    I, J, P = cfg["I"], cfg["J"], cfg["P"]
    red = (cfg["L"], cfg["M"], cfg["N"])
    rng = np.random.default_rng(0)

    def run(ks):
        ks = max(ks, cfg["N"])  # make_ensemble needs reduced <= dims on every mode
        t = np.asfortranarray(rng.standard_normal((I, J, ks)))
        # the slab's ensemble == leading columns of the full one (per-row streams)
        ens = ref.make_ensemble((I, J, ks), red, P, cfg["S"], seed=derive(cfg["seed"], 11))
        t0 = time.perf_counter()
        ref.comp_blocked(t, (500, 500, ks), ens, deterministic=False, workers=threads)
        return time.perf_counter() - t0

    ks = cfg["N"]
    dt = run(ks)
    if dt < 0.5 * seconds:
        ks = int(min(400, ks * seconds / max(dt, 1e-3)))
        dt = run(ks)
    n = I * J * ks
    return n / dt, f"comp_blocked fast mode, {I}x{J}x{ks} slab ({n:.3g} elements, 500x500x{ks} blocks), " \
                   f"P={P} replicas of {red[0]}^3, {dt:.1f} s, OPENBLAS 1 thread x {threads} workers"


def cp_time_c1():
    """The metric's second half, end-to-end CP time, on the reference's own
    CPU-runnable config (BASELINE configs[0], C1): decompose from the rank-10
    factors on the device (fp64 compression, the reference's precision) next
    to the reference's decompose on the host cores (oracle/_ref), with the
    recovered-factor errors of both (evaluate, pipeline.cpp:577-609)."""
    import paper_2311_13693_b200 as xt
    dims, R, red, P, S = (200, 200, 200), 10, (30, 30, 30), 12, 10
    f = xt.generate_factors(dims, R, seed=1)
    cfg = xt.PipelineConfig(reduced=red, rank=R, replicas=P, shared=S, precision=xt.PREC_FP64, seed=2)
    xt.decompose(cfg, factors=f)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        rec, met = xt.decompose(cfg, factors=f)
        walls.append(time.perf_counter() - t0)
    out = {"config": "C1: dense 200^3 rank-10, P=12 x 30^3, S=10, decompose end to end (fp64)",
           "seconds": float(np.median(walls)), "stage_seconds": met.stage_seconds,
           "mode_rel_err": xt.evaluate(f, rec).mode_rel_err}
    try:
        from oracle.oracle import Reference
        ref = Reference()
        ref.L.xref_set_blas_threads(1)
        threads = os.cpu_count() or 1
        rw = []
        for _ in range(2):
            t0 = time.perf_counter()
            rc, rrec, _ = ref.decompose(f, dims, red, R, P, S, 2, workers=threads)
            rw.append(time.perf_counter() - t0)
        out["reference_seconds"] = float(np.median(rw))
        out["reference_cores"] = threads
        out["reference_mode_rel_err"] = ref.evaluate(f, rrec)[0]
    except Exception as e:  # reference build absent on this box
        out["reference_seconds"] = None
        out["reference_note"] = f"unavailable: {e}"
    return out


def cp_time_c3(xt, torch, world, rank, dev):
    """north_star: the dense 10,000^3 rank-20 tensor compressed and decomposed
    end to end (C3: P = 124 replicas of 128^3, S = 40, blocks generated on the
    device from the factors). One GPU: decompose on the device. N ranks:
    mode-3 slabs per rank, one reduce-scatter of the replicas, stage 1
    (CP-ALS) on every rank for its share, stages 2-3 on rank 0
    (dist.decompose_distributed). bf16 compression at the relaxed replica fit
    tolerance 1e-2 (the compensated mode meets the default 1e-6 at ~5x the
    compression time, profiles/r2_pipeline_c3_fp16x3.json); recovered-factor
    errors from evaluate (pipeline.cpp:577-609)."""
    import torch.distributed as dist
    dims, R, red, P, S = (10000, 10000, 10000), 20, (128, 128, 128), 124, 40
    f = xt.generate_factors(dims, R, seed=1)
    cfg = xt.PipelineConfig(reduced=red, rank=R, replicas=P, shared=S, precision=xt.PREC_BF16,
                            replica_fit_tol=1e-2, seed=2)
    if world == 1:
        t0 = time.perf_counter()
        rec, met = xt.decompose(cfg, factors=f)
        wall = time.perf_counter() - t0
    else:
        from paper_2311_13693_b200.dist import decompose_distributed
        lmn = int(np.prod(red))
        per = -(-P // world)
        plan = xt.Plan(dims, red, P, S, derive(2, 11), precision=xt.PREC_BF16)
        yy = torch.zeros(per * world * lmn, dtype=torch.float32, device=dev)

        def slab(k0, k1, ybuf):
            plan.compress_factors(f, k0, k1, y=ybuf[:P * lmn], device=dev)
            torch.cuda.synchronize()

        dist.barrier()
        t0 = time.perf_counter()
        rec, met, t_s1 = decompose_distributed(
            slab, dims[2], P, lmn, yy, lambda reps, ids: xt.decompose_stage1(cfg, dims, reps, ids),
            lambda merged: xt.decompose_finish(cfg, merged, factors=f))
        wall = time.perf_counter() - t0
        tw = torch.tensor([wall, t_s1], device=dev, dtype=torch.float64)
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw[0].item())
        plan.close()
        if rank != 0:
            return None
        met.stage_seconds["decomposition"] = float(tw[1].item())
        met.stage_seconds["compression"] = wall - sum(v for k, v in met.stage_seconds.items() if k != "compression")
    rep = xt.evaluate(f, rec)
    return {"config": "C3 (north_star): dense 10000^3 rank-20, P=124 x 128^3, S=40, factored source, "
                      "bf16 compression, replica fit tol 1e-2, decompose end to end",
            "n_gpus": world, "seconds": wall, "stage_seconds": met.stage_seconds,
            "replicas_dropped": met.replicas_dropped, "mode_rel_err": rep.mode_rel_err,
            "compression_elements_per_s": float(np.prod(dims)) / met.stage_seconds["compression"]}


def sparse_c4(xt, torch, dev):
    """north_star config 4 (one GPU): the sparse 10^6 x 10^6 x 10^6 rank-10
    tensor (464 nonzeros per factor column -> 10 dense 464^3 sub-cubes,
    9.99e8 nonzeros), P = 16 replicas of 32^3, as CSF resident on the device
    (tile planner + dense-tile tensor kernel, CUDA events on the call's
    stream), then the same CSF from host memory through the multi-GPU C ABI
    (xtsg_multi_compress_csf: pinned-staged H2D + NCCL reduce in the wall
    time). Checked against comp_from_factors of the generating factors."""
    dims, R, npc, red, P, S = (10 ** 6,) * 3, 10, 464, (32, 32, 32), 16, 8
    f = xt.generate_factors(dims, R, law="sparse", nnz_per_col=npc, seed=1)
    sk, fj, ni, nv = [], [], [], []
    for r in range(R):
        sup = [np.nonzero(f[m][:, r])[0] for m in range(3)]
        val = [torch.tensor(f[m][sup[m], r], dtype=torch.float32, device=dev) for m in range(3)]
        idx = [torch.tensor(x, dtype=torch.int32, device=dev) for x in sup]
        na, nb, nc = (len(x) for x in sup)
        sk.append(idx[2])
        fj.append(idx[1].repeat(nc))
        ni.append(idx[0].repeat(nc * nb))
        nv.append((val[2].view(nc, 1, 1) * val[1].view(1, nb, 1) * val[0].view(1, 1, na)).reshape(-1))
    sk, fj, ni, nv = (torch.cat(x) for x in (sk, fj, ni, nv))
    sp = torch.arange(0, sk.numel() + 1, dtype=torch.int64, device=dev) * (fj.numel() // sk.numel())
    fp = torch.arange(0, fj.numel() + 1, dtype=torch.int64, device=dev) * (ni.numel() // fj.numel())
    csf = (sk, sp, fj, fp, ni, nv)
    nnz = int(nv.numel())
    seed = derive(2, 11)
    plan = xt.Plan(dims, red, P, S, seed, precision=xt.PREC_BF16)
    y = torch.zeros(P * int(np.prod(red)), dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        for _ in range(2):
            plan.compress_csf(*csf, y=y, stream=st)
        steps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            plan.compress_csf(*csf, y=y, stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ens = xt.make_ensemble(dims, red, P, S, seed)
    from oracle.oracle import rel_diff
    got = xt.Plan.replicas(y.cpu().numpy(), P, red)
    err = max(rel_diff(xt.comp_from_factors(f, ens.u[p], ens.v[p], ens.w[p]), got[p]) for p in (0, P - 1))
    # the same nonzeros as unsorted COO (north_star config 4's input format):
    # a random permutation, so every call groups them into fibers itself
    nf_per_slice = fj.numel() // sk.numel()
    npf = ni.numel() // fj.numel()
    perm = torch.randperm(nnz, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    ck = sk.repeat_interleave(nf_per_slice * npf)[perm]
    cj = fj.repeat_interleave(npf)[perm]
    ci, cv = ni[perm], nv[perm]
    del perm
    yc = torch.zeros_like(y)
    with torch.cuda.stream(st):
        plan.compress_coo(ci, cj, ck, cv, y=yc, stream=st)
        csteps = 3
        e0.record(st)
        for _ in range(csteps):
            plan.compress_coo(ci, cj, ck, cv, y=yc, stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    coo_ms = e0.elapsed_time(e1) / csteps
    got = xt.Plan.replicas(yc.cpu().numpy(), P, red)
    coo_err = max(rel_diff(xt.comp_from_factors(f, ens.u[p], ens.v[p], ens.w[p]), got[p]) for p in (0, P - 1))
    del ci, cj, ck, cv, yc
    plan.close()
    host = [t.cpu().numpy() for t in csf]
    del csf, sk, sp, fj, fp, ni, nv, y
    torch.cuda.empty_cache()
    mp = xt.MultiPlan(dims, red, P, S, seed, gpus=[dev.index or 0], precision=xt.PREC_BF16)
    mp.compress_csf(*host)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        yh = mp.compress_csf(*host)
        walls.append(time.perf_counter() - t0)
    mp.close()
    got = xt.Plan.replicas(yh, P, red)
    herr = max(rel_diff(xt.comp_from_factors(f, ens.u[p], ens.v[p], ens.w[p]), got[p]) for p in (0, P - 1))
    hbm = peaks()[2]
    rate = nnz / (ms / 1e3)
    wall = float(np.median(walls))
    return {"config": "C4: sparse 10^6^3 rank-10, 464 nnz/col -> %.4g nonzeros as CSF, P=16 replicas of 32^3, "
                      "bf16 tile path" % nnz,
            "metric": "nonzeros compressed/sec", "value": rate, "unit": "nnz/s", "ms_per_step": ms,
            "steps": steps, "roofline": {"bound": "hbm", "algorithmic_bytes_per_nnz": 16,
                                         "achieved": 16.0 * rate / 1e9, "peak": hbm, "unit": "GB/s",
                                         "frac": 16.0 * rate / 1e9 / hbm},
            "max_rel_err_vs_comp_from_factors": float(err),
            "coo_unsorted": {"value": nnz / (coo_ms / 1e3), "unit": "nnz/s", "ms_per_step": coo_ms, "steps": 3,
                             "input": "the same nonzeros as device COO in random order (grouped into fibers "
                                      "inside every call: 25-bit radix sort of compact (rank k, rank j) keys)",
                             "max_rel_err_vs_comp_from_factors": float(coo_err)},
            "e2e_host_csf_multi_api": {"value": nnz / wall, "unit": "nnz/s", "wall_s": wall,
                                       "h2d_bytes_per_step": int(sum(a.nbytes for a in host)),
                                       "d2h_bytes_per_step": int(yh.nbytes),
                                       "max_rel_err_vs_comp_from_factors": float(herr)}}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args):
    """--gpus N outside torchrun: re-launch under torch.distributed.run, one rank per GPU."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd, env=env))


def run_cpu_smoke(args):
    """The multi-rank plumbing on CPU: gloo, mode-3 slabs, one reduce, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2311_13693_b200.dist import slab_range
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    I, J, K, P, L = 64, 48, 16 * world, 4, 8
    g = torch.Generator().manual_seed(0)
    X = torch.randn(I, J, K, generator=g, dtype=torch.float64)
    U, V, W = (torch.randn(P, L, n, generator=g, dtype=torch.float64) for n in (I, J, K))
    k0, k1 = slab_range(K, rank, world)
    y = torch.zeros(P, L, L, L, dtype=torch.float64)

    def step():
        y.copy_(torch.einsum("ijk,pai,pbj,pck->pabc", X[:, :, k0:k1], U, V, W[:, :, k0:k1]))
        if world > 1:
            dist.reduce(y, dst=0)

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    if world > 1:
        dist.barrier()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = torch.einsum("ijk,pai,pbj,pck->pabc", X, U, V, W)
        err = float((y - full).abs().max() / full.abs().max())
        print(json.dumps({"impl": "cpu-smoke", "metric": "input tensor elements compressed/sec",
                          "value": I * J * K * args.steps / float(dt.item()), "unit": "elements/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "config": {"workload": f"cpu smoke {I}x{J}x{K}", "parallelism": f"mode-3 slabs x{world}"},
                          "check_max_rel_err": err}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def parity_check(y, cfg, dims, red, P, reps):
    """Outside the timed region: replicas `reps` of the timed output vs the
    CPU oracle's comp_from_factors (compression.cpp:215-220) of the
    generating factors (pipeline.cpp:182-193) with the reference ensemble."""
    from oracle.oracle import Restated, rel_diff
    o = Restated()
    f = o.generate_dense(dims, cfg["R"], cfg["factor_seed"])
    ens = o.ensemble_cols(dims, red, P, cfg["S"], derive(cfg["seed"], 11))
    yh = y.detach().cpu().numpy()
    n = int(np.prod(red))
    errs = {}
    for p in reps:
        want = o.comp_from_factors(*f, ens[0][p], ens[1][p], ens[2][p])
        errs[int(p)] = rel_diff(want, yh[p * n:(p + 1) * n].reshape(red, order="F"))
    return {"oracle": "comp_from_factors (oracle/xts_oracle.c)", "replicas": sorted(errs),
            "max_rel_err": max(errs.values())}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cfg = dict(C2)
    rates = []
    for _ in range(max(1, args.steps)):
        r, sample = cpu_reference_rate(cfg, max(2.0, args.cpu_seconds / max(1, args.steps)), threads)
        rates.append(r)
    v = float(np.median(rates))
    line = {"impl": "reference", "metric": "input tensor elements compressed/sec", "value": v,
            "unit": "elements/s", "higher_is_better": True, "n_gpus": args.gpus, "steps": len(rates),
            "warmup": 0, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2: dense 2000^3 rank-20, streamed blocks, P=32 replicas of 64^3 (CPU sample)"},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    maybe_spawn(args)
    if args.cpu_smoke:
        run_cpu_smoke(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    import paper_2311_13693_b200 as xt

    cfg = dict(C2)
    K = args.K
    cfg["Ktot"] = K * world
    dims = (cfg["I"], cfg["J"], cfg["Ktot"])
    red = (cfg["L"], cfg["M"], cfg["N"])
    P = cfg["P"]
    k0 = rank * K
    t_plan = time.perf_counter()
    prec = {"bf16": xt.PREC_BF16, "fp16": xt.PREC_FP16, "fp16x3": xt.PREC_FP16X3}[args.precision]
    comp3 = prec == xt.PREC_FP16X3
    plan = xt.Plan(dims, red, P, cfg["S"], derive(cfg["seed"], 11), precision=prec)
    t_plan = time.perf_counter() - t_plan
    # the compensated mode splits fp32 X into its fp16 (hi, lo') planes on the device
    X, _ = make_block(torch, xt, cfg, k0, K, dev, {"fp16": torch.float16, "bf16": torch.bfloat16,
                                                     "fp16x3": torch.float32}[args.precision])
    torch.cuda.synchronize()
    ysz = P * int(np.prod(red))
    y = torch.zeros(ysz, dtype=torch.float32, device=dev)
    # a dedicated stream: the legacy default stream's handle is 0, which the
    # C ABI reads as "use the library's own per-thread stream"
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    elems_rank = cfg["I"] * cfg["J"] * K

    def step():
        plan.compress(X, y=y, offset=(0, 0, k0), stream=stream)
        if world > 1:
            dist.reduce(y, dst=0)

    plan.set_profiling(True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    plan.profile(reset=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = xt.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = xt.launch_count() - launches0
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    prof = plan.profile(reset=True)
    value = elems_rank * world * args.steps / (ms / 1e3)

    burst, sustained, hbm, src = peaks()
    fused_avg_ms = prof["fused_ms"] / max(1, prof["fused_launches"])
    flops_per_launch = prof["fused_flops"] / max(1, prof["fused_launches"])
    achieved = flops_per_launch / (fused_avg_ms / 1e3) / 1e12
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        try:
            traffic = json.loads(tj.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": sustained, "unit": "TFLOP/s",
                "frac": round(achieved / sustained, 4), "traffic": traffic if args.precision == "bf16" else None,
                "kernel": "ttm_pair_kernel (fused mode-1 + mode-2, tcgen05 kind::f16, cta_group::2)",
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside back-to-back steps)",
                "algorithmic_flops_per_launch": flops_per_launch,
                "kernel_share_of_step": round(prof["fused_ms"] / ms, 4) if ms > 0 else None,
                "mode3_ms_per_step": prof["mode3_ms"] / args.steps}
    if comp3:
        # three products per mode: the tensor cores execute 3x the useful flops
        roofline["flops"] = "useful (algorithmic); issued = 3x"
        roofline["issued_achieved"] = round(3 * achieved, 2)
        roofline["issued_frac"] = round(3 * achieved / sustained, 4)
        roofline["kernel"] = "ttm_pair_kernel compensated (fp16 hi/lo x3, tcgen05 kind::f16, cta_group::2)"

    # ---- e2e through the C ABI with host buffers ----
    def run_e2e(host_dtype, Ke, steps):
        tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[host_dtype]
        xh = torch.empty((Ke, cfg["J"], cfg["I"]), dtype=tdt, pin_memory=True)
        for k in range(0, Ke, 100):
            xh[k:k + 100].copy_(X.permute(2, 1, 0)[k:min(k + 100, Ke)].to(tdt))
        xh_v = xh.permute(2, 1, 0)
        yh = torch.zeros(ysz, dtype=torch.float32, pin_memory=True)

        def e2e_step():
            plan.compress(xh_v, y=yh, offset=(0, 0, k0))
            if world > 1:
                yd = yh.to(dev)
                dist.reduce(yd, dst=0)
                yh.copy_(yd.cpu())

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        narrow = os.environ.get("XTSG_HOST_NARROW", "1") != "0" and not comp3 and host_dtype != "bf16"
        out = {"value": cfg["I"] * cfg["J"] * Ke * world * steps / dt, "unit": "elements/s",
               "slices_per_rank": Ke, "steps": steps,
               "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
               "d2h_bytes_per_step": int(yh.numel() * 4),
               "host_dtype": host_dtype, "ms_per_step": dt / steps * 1e3,
               "pcie_h2d_bytes_per_step": int(xh.numel() * (2 if narrow else xh.element_size())),
               "note": ("f32/f64 host input is narrowed to bf16 on the host (RNE, multi-threaded) before the DMA"
                        if narrow else "host input copied as is; converted/split on the device")}
        del xh
        return out

    e2e = e2e_f64 = None
    if not args.no_e2e:
        # host memory is shared by the node's ranks: the e2e sample per rank
        # shrinks with N (the metric is a rate; per-rank pinned input <= 32 GB)
        e2e = run_e2e(args.e2e_dtype, max(100, K // world), args.e2e_steps)
        # the drop-in's own boundary type (Tensor3::values is fp64,
        # tensor.hpp:30-44): a quarter-size sample (8 GB pinned per rank)
        if args.e2e_dtype != "f64":
            e2e_f64 = run_e2e("f64", max(100, K // (4 * world)), max(2, args.e2e_steps // 2))

    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = parity_check(y, cfg, dims, red, P, (0, P - 1))
        except Exception as e:  # oracle build absent
            parity = {"error": str(e)}

    cp = None
    if rank == 0 and not args.no_cp_time:
        try:
            cp = cp_time_c1()
        except Exception as e:
            cp = {"error": str(e)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            v, sample = cpu_reference_rate(cfg, args.cpu_seconds, threads)
            cpu = {"value": v, "unit": "elements/s", "cores": threads, "kind": "reference", "sample": sample}
        except Exception as e:  # reference build absent on this box
            cpu = {"value": None, "unit": "elements/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    c3 = None
    if not args.no_c3:
        # free the C2 plan and block first: the C3 slabs need the HBM
        plan.close()
        del X
        torch.cuda.empty_cache()
        try:
            c3 = cp_time_c3(xt, torch, world, rank, dev)
        except Exception as e:
            c3 = {"error": str(e)}

    c4 = None
    if world == 1 and not args.no_c4:
        if args.no_c3:
            plan.close()
            del X
            torch.cuda.empty_cache()
        try:
            c4 = sparse_c4(xt, torch, dev)
        except Exception as e:
            c4 = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": "input tensor elements compressed/sec", "value": value, "unit": "elements/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (rank-20 reconstruct(A,B,C) from the reference's generate() streams)",
            "config": {"workload": "C2: dense 2000^3 rank-20, streamed blocks, P=32 replicas of 64^3, S=40",
                       "dims_per_rank": [cfg["I"], cfg["J"], K], "reduced": list(red), "replicas": P,
                       "shared_rows": cfg["S"], "parallelism": f"mode-3 slabs x{world}",
                       "l2": "inputs (16 GB bf16 per rank) larger than L2; no flush",
                       "plan_create_s": round(t_plan, 3)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_f64_host": e2e_f64,
            "gpu_launches": int(launches),
            "cp_time": cp, "cp_time_c3": c3, "sparse_c4": c4, "parity": parity,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if args.no_c3 and not (world == 1 and not args.no_c4):
        plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
