#!/usr/bin/env python
"""Benchmark: Schur-complement PCG solves/s on B200 (BASELINE.json metric), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5_2d_N2048_darcy] [--impl reference]

A "step" is one dd_pcg_solve over one batch of the workload (every column driven to rtol 1e-10):
the whole hot path per PCG iteration — the Schur apply (2D default: ONE grouped DMMA GEMM
Y[:, c] = H_p X[:, c] with H_p = K_p S_unit + γ_p F formed at setup; 3D: the PCG runs in the
parity-ordered sine domain of the face and each apply streams the class-sparse packed-symmetric
Ĥ = T(γ F + K S_unit)Tᵀ, interior solve folded in at setup) and the RA pole sum (2D: the fused
kernel doing the pole sum, the PCG updates and the dot products; 3D: the face systems' Chebyshev
steps in one cooperative launch, then the PCG updates).
Default workload: config 5 (2D, 2048 cells/side, the 16-point (K, μ⁻¹) Darcy sweep x 32 RHS = 512
independent solves per step; the largest single-GPU configuration of BASELINE.json, standing in
for the Appendix sweep).
Multi-GPU (torchrun, one rank per GPU): 2D configs split the FIXED batch over the ranks (strong
scaling, no data-path collective) in 32-column single-parameter blocks balanced by LPT on pilot
iteration counts; config 4 splits the RA systems over the ranks with one NCCL allreduce per
preconditioner apply and row-shards F with one NCCL allgather per Schur apply (strong).  value = the job's solves / max-over-ranks device time.
`--emulate-ranks W` (one GPU) adds a PREDICTION of the W-rank value: each rank's shard run alone.
Timing: W warm-up steps, then K steps each bracketed by CUDA events (recorded inside libdd
on its stream), with a 512 MiB L2 flush between steps outside the timed spans; barrier +
synchronize on both sides of the timed region; max over ranks.  Every timed solve must return
DD_OK (all columns converged) or the run fails.
`--impl reference`: the CPU oracle (this tier's reference arm) timed on host cores on a
bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2211_15308_b200 import configs, inputs, rafit  # noqa: E402

METRIC = "Schur PCG solves/s"
UNIT = "solves/s"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def live_columns(iters, compact: bool, bn: int = 64, min_tiles: int = 6):
    """Columns each Schur apply of one solve multiplies: all of them without compaction, else the
    columns of the bn-wide tiles that still hold an active column (iters[j] >= k at apply k)."""
    iters = np.asarray(iters); C = len(iters); kmax = int(iters.max()) if C else 0
    tiles = (C + bn - 1) // bn
    if not compact or (C + 63) // 64 < min_tiles:        # the library's threshold counts 64-column tiles
        return [C] * kmax
    tile_it = np.array([iters[t * bn:(t + 1) * bn].max() for t in range(tiles)])
    width = np.array([min(bn, C - t * bn) for t in range(tiles)])
    return [int(width[tile_it >= k].sum()) for k in range(1, kmax + 1)]


def fit_ras(cfg, t=-0.5, sigma=0.0):
    lo, hi = rafit.interval_1d(cfg.N) if cfg.dim == 2 else rafit.interval_face(cfg.N)
    return [rafit.fit_ra(K, g, lo, hi, cfg.n_poles, t=t, sigma=sigma) for K, g in cfg.params]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("DD_BENCH_CLOCK_MS", "200") == "0":     # diagnostics only: no sampling
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("DD_BENCH_CLOCK_MS", "200")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        under = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(cfg, ras, B, colp, per_param: int, t: float = -0.5, sigma: float = 0.0):
    """Time the CPU oracle (mode tier: scipy DST + LAPACK banded Cholesky pole solves, PCG per
    column) on `per_param` columns of every parameter set.  Returns (solves, seconds)."""
    from oracle import pcg as opcg
    from oracle import problem as oprob
    Mo = oprob.ModeProblem2D(cfg.N, t=t, sigma=sigma)
    t0 = time.perf_counter()
    solves = 0
    for p, (K, g) in enumerate(cfg.params):
        sel = np.nonzero(colp == p)[0][:per_param]
        ra = ras[p]
        for c in sel:
            opcg.pcg(lambda v: Mo.apply_S(K, g, v), lambda v: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c],
                     rtol=cfg.rtol, maxit=cfg.maxit)
            solves += 1
    return solves, time.perf_counter() - t0


def host_info():
    """CPU model, usable cores and BLAS of the host the oracle runs on (SURVEY §8(d) oracle timing)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [f"{i.get('internal_api')} {i.get('version')} x{i.get('num_threads')}" for i in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0)), "blas": blas}


def cores_used():
    try:
        from threadpoolctl import threadpool_info
        th = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        th = 1
    return int(min(th, len(os.sched_getaffinity(0))))


# ----------------------------------------------------------------------------- roofline inputs
def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def fp64_peak():
    m = load_json(os.path.join(ROOT, "MEASURED_FP64.json"))
    if m and m.get("dmma_tflops"):
        return float(m["dmma_tflops"]), "MEASURED_FP64.json dmma_tflops (DMMA issue-bound probe, this pool)"
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    bf16 = float(mp.get("bf16_tflops", 1590.0))
    return bf16 * 40.0 / 2250.0, "bf16 measured x nominal FP64/bf16 ratio (40/2250)"


def traffic_for(cfg_name, kernel):
    t = load_json(os.path.join(ROOT, "profiles", "traffic.json")) or {}
    v = t.get(cfg_name, {}).get(kernel)
    return float(v) if v is not None else None


# ----------------------------------------------------------------------------- roofline model
def step_model_2d(cfg, grouped: bool, assembled: bool, frac_ra: bool, cols_per_apply, n_live_groups, peaks,
                  pair: bool = False):
    """Algorithmic work of one PCG iteration per kernel class, for the live columns:
    Schur GEMM  F = 2 n^2 c (grouped; 4 n^2 c assembled / factored K2, 2 n^2 c more for K1),
                B = 8 n^2 (per live parameter group for grouped; the [F|G] / [S|F] operand once otherwise)
                    + 16 n c (X in, Y out);
    pole sum + PCG updates  F = 7 (m+1) n c + 12 n c (Thomas-minimal sweeps + accumulate, updates
                and dots), B = 56 n c (p, q, x, r in; x, r, p out).
    Returns {class: (flops, bytes, roofline seconds)} averaged over the solve's iterations."""
    n, m = cfg.n, cfg.n_poles
    c = float(np.mean(cols_per_apply)) if cols_per_apply else 0.0
    g = float(np.mean(n_live_groups)) if n_live_groups else 0.0
    p64, pdf, bw = peaks["dmma"] * 1e12, peaks["dfma"] * 1e12, peaks["hbm"] * 1e9
    if grouped:
        fg = 2.0 * n * n * c
        # H_p blocks: one n^2 operator per live parameter group; shared-pair kernel: G and F once
        bg = (16.0 * n * n if pair else 8.0 * n * n * g) + 16.0 * n * c
    else:
        fg = (2.0 if frac_ra else 4.0) * n * n * c
        bg = 8.0 * n * n * (1 if frac_ra else 2) + 24.0 * n * c
    fd = 0.0 if assembled else 2.0 * n * n * c
    bd = 0.0 if assembled else 8.0 * n * n + 16.0 * n * c
    fp = (7.0 * (m + 1) + 12.0) * n * c
    bp = 56.0 * n * c
    out = {"gemm_schur": (fg, bg, max(fg / p64, bg / bw)), "polesum_pcg": (fp, bp, max(fp / pdf, bp / bw))}
    if fd:
        out["gemm_dst"] = (fd, bd, max(fd / p64, bd / bw))
    return out


def peaks_all():
    m = load_json(os.path.join(ROOT, "MEASURED_FP64.json")) or {}
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    dmma, src = fp64_peak()
    return {"dmma": dmma, "dmma_src": src, "dfma": float(m.get("dfma_tflops", dmma * 0.917)),
            "hbm": float(mp.get("hbm_gbs", 6454.0)),
            "hbm_src": "MEASURED_PEAKS.json hbm_gbs" if mp else "fallback 6454 GB/s (B200_PROFILING.md)"}


def pilot_iterations(S, cfg, B_all, colp_all, dev):
    """PCG iteration count of every parameter set from ONE right-hand side each (its first): the
    cost model of the strong-scaling block shard.  Deterministic, so every rank computes the same
    partition without communicating.  Outside the timed region."""
    import torch
    first = np.array([int(np.nonzero(colp_all == p)[0][0]) for p in range(len(cfg.params))])
    r = S.pcg_solve(torch.as_tensor(B_all[first], device=dev), colp_all[first], rtol=cfg.rtol, maxit=cfg.maxit)
    if r.status != 0:
        raise SystemExit(f"pilot solve failed: status {r.status}")
    return [int(v) for v in r.iters]


def check_solve(r, what):
    """Every timed / e2e solve must converge on every column (no DD_ENOCONV / DD_ENOTSPD counted as
    a solve)."""
    if r.status != 0:
        raise SystemExit(f"{what}: solve status {r.status} (not DD_OK); refusing to report solves/s")


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=configs.HEADLINE.name)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--frac-mode", default="dense", choices=["dense", "ra"],
                    help="fractional term: dense F (Eq.(7)) or RA-evaluated (Remark 1, NEXT-2)")
    ap.add_argument("--t", type=float, default=-0.5, help="fractional exponent t of γ L^t (Eq.(9); NEXT-3)")
    ap.add_argument("--shifted", action="store_true", help="L = -Δ_Γ + I_Γ (Eq.(9); NEXT-3)")
    ap.add_argument("--mode", default="schur", choices=["schur", "bulk", "bulk-pcg"],
                    help="schur: interface PCG (headline); bulk: full DD solve on bulk RHS (NEXT-1); "
                         "bulk-pcg: PCG on the bulk system with the Eq.(5) DD preconditioner (the paper's protocol)")
    ap.add_argument("--pole-split", default="auto", choices=["auto", "on", "off"],
                    help="3D (config 4, SURVEY §8(e)): all ranks solve the same columns, the RA systems are split "
                         "across ranks and the partial sums allreduced over NCCL each preconditioner apply "
                         "(strong scaling).  auto = on under torchrun for config 4")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="PREDICTION on one GPU: run each of W ranks' shards alone, one after another, and report "
                         "the max-over-ranks time as a predicted W-GPU value (not a measurement of W GPUs)")
    ap.add_argument("--schur", default=None, choices=["grouped", "assembled", "factored"],
                    help="2D Schur apply (dd_set_schur_mode): grouped = one GEMM with H_p = K_p G + gamma_p F per "
                         "parameter set (default, dense F); assembled = one [F|G] GEMM (default in RA mode); "
                         "factored = per-apply fast diagonalisation K1 + K2")
    args = ap.parse_args()
    if args.schur is None:
        args.schur = "grouped" if args.frac_mode == "dense" else "assembled"
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = configs.BY_NAME[args.config]
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if args.mode in ("bulk", "bulk-pcg"):
        return run_bulk(args, cfg, world, rank)
    return run_schur(args, cfg, world, rank)


def run_schur(args, cfg, world, rank):
    import torch
    import torch.distributed as dist
    from paper_2211_15308_b200 import binding
    from paper_2211_15308_b200 import dist as ddist_mod

    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sigma = 1.0 if args.shifted else 0.0
    ras = fit_ras(cfg, args.t, sigma)
    split = cfg.dim == 3 and (args.pole_split == "on" or (args.pole_split == "auto" and world > 1 and cfg.pole_split))
    ddist = None
    if split:
        uid = binding.nccl_unique_id() if rank == 0 else None
        if world > 1:
            uid = ddist_mod.broadcast_bytes(uid, 128, device=dev)
        ddist = (rank, world, 1, uid if world > 1 else None)   # DD_SHARD_POLES
    frac = binding.Frac(t=args.t, shifted=args.shifted)
    if args.frac_mode == "ra":
        lo, hi = rafit.interval_1d(cfg.N) if cfg.dim == 2 else rafit.interval_face(cfg.N)
        frac = binding.Frac(t=args.t, shifted=args.shifted, mode="ra",
                            fra=rafit.fit_power(args.t, lo, hi, cfg.n_poles, sigma))
    # ---- the batch.  2D: the config's FIXED batch (every parameter set's seeded RHS) split over the
    # ranks in 32-column single-parameter blocks (strong scaling); 3D pole split: every
    # rank the same columns; 3D otherwise: replicas (each rank its own seeded columns, weak scaling)
    if cfg.dim == 2:
        B_all, colp_all = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
        scaling = "strong"
    else:
        B_all, colp_all = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param,
                                       seed_offset=0 if split else rank * len(cfg.params))
        scaling = "strong" if split else "weak"
    C_all = B_all.shape[0]
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=C_all, device=local, frac=frac, dist=ddist)
    if cfg.dim == 2:
        S.set_schur_mode(args.schur)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t_setup) * 1e3      # once per mesh and parameter sets (row a-1)
    shard = {}
    pilot = None
    if cfg.dim == 2:
        pilot = pilot_iterations(S, cfg, B_all, colp_all, dev)
        cols, colp = ddist_mod.block_shard(len(cfg.params), cfg.rhs_per_param, rank, world, pilot)
        B = np.ascontiguousarray(B_all[cols]) if len(cols) else np.zeros((0, cfg.n_gamma))
        shard = {"unit": "32-column single-parameter blocks, LPT on pilot PCG iterations x width",
                 "pilot_iters_by_param": pilot, "rank0_columns": int(len(cols))}
    else:
        B, colp = B_all, colp_all
    C = B.shape[0]
    solves_per_step = C_all if (cfg.dim == 2 or split) else C_all * world
    Bt = torch.as_tensor(B, device=dev)
    cp = torch.as_tensor(np.asarray(colp, dtype=np.int32), device=dev)
    X = torch.empty_like(Bt)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        r = S.pcg_solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=cfg.maxit)
        check_solve(r, "timed solve")
        return r

    for _ in range(args.warmup):
        flush.fill_(1.0)
        if C:
            step()
    iters_all = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    S.launch_count()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                      # L2 flush outside the timed span
            if C:
                r = step()
                step_ms.append(S.last_solve_ms())
                iters_all.append(r.iters.copy())
            else:
                step_ms.append(0.0)
        torch.cuda.synchronize()
    launches = S.launch_count()
    qc = S.query_config()              # launch configuration of the timed solves
    if world > 1:
        dist.barrier()
    total_ms = float(sum(step_ms))
    max_ms = ddist_mod.max_over_ranks(total_ms, device=dev)
    value = solves_per_step * args.steps / (max_ms / 1e3)

    # ---- instrumented pass: per-kernel-class device time (CUDA events on libdd's stream)
    prof = {k: (0.0, 0) for k in binding.KCLASS}
    nprof = max(2, min(args.steps, 5))
    if C:
        S.profile(True)
        for _ in range(nprof):
            flush.fill_(1.0)
            step()
        prof = S.profile_read()
        S.profile(False)
    inner_its = S.inner_iterations() if cfg.dim == 3 and C else None

    # ---- e2e through the host-buffer ABI call (pinned host memory, H2D + D2H inside)
    Bh = torch.as_tensor(B).pin_memory().numpy()
    Xh = torch.empty(B.shape, dtype=torch.float64).pin_memory().numpy()
    e2e_t = []
    if C:
        check_solve(S.pcg_solve_host(Bh, colp, rtol=cfg.rtol, maxit=cfg.maxit, x_out=Xh), "e2e solve")
        torch.cuda.synchronize()
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            check_solve(S.pcg_solve_host(Bh, colp, rtol=cfg.rtol, maxit=cfg.maxit, x_out=Xh), "e2e solve")
            e2e_t.append(time.perf_counter() - t0)
    n_e2e = max(3, min(args.steps, 10))
    e2e_s = ddist_mod.max_over_ranks(float(sum(e2e_t)), device=dev)
    e2e_value = solves_per_step * n_e2e / e2e_s if e2e_s > 0 else None

    # ---- precond applies/s (secondary metric of BASELINE.json)
    pa_ms = 0.0
    reps = 20
    if C:
        Z = torch.empty_like(Bt)
        for _ in range(3):
            S.apply_precond(Bt, cp, z=Z)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(S.stream)
        for _ in range(reps):
            S.apply_precond(Bt, cp, z=Z)
        e1.record(S.stream)
        torch.cuda.synchronize()
        pa_ms = e0.elapsed_time(e1)
    pa_ms = ddist_mod.max_over_ranks(pa_ms, device=dev)
    pa_per_s = solves_per_step * reps / (pa_ms / 1e3) if pa_ms > 0 else None

    pred = None
    if args.emulate_ranks > 1 and world == 1:
        pred = emulate_ranks(args, cfg, ras, frac, B_all, colp_all, pilot, dev, flush)

    if rank == 0:
        line = schur_line(args, cfg, world, S, ras, B, colp, C, C_all, solves_per_step, split, scaling, shard,
                          setup_ms, value, max_ms, iters_all, launches, qc, prof, nprof, inner_its, clk,
                          e2e_value, pa_per_s)
        if pred is not None:
            line["scaling_prediction"] = pred
        print(json.dumps(line), flush=True)
    S.close()
    if world > 1:
        dist.destroy_process_group()


def schur_line(args, cfg, world, S, ras, B, colp, C, C_all, solves_per_step, split, scaling, shard, setup_ms,
               value, max_ms, iters_all, launches, qc, prof, nprof, inner_its, clk, e2e_value, pa_per_s):
    n = cfg.n
    its = np.concatenate(iters_all) if iters_all else np.zeros(1)
    last = iters_all[-1] if iters_all else np.zeros(0, dtype=int)
    by_param = [[K, g, int(last[colp == p].max()), round(float(last[colp == p].mean()), 2)]
                for p, (K, g) in enumerate(cfg.params) if np.any(colp == p)]
    pk = peaks_all()
    total_prof_ms = sum(v[0] for v in prof.values()) or 1.0
    share = {k: round(v[0] / total_prof_ms, 4) for k, v in prof.items()}
    avg_us = {k: round(v[0] / v[1] * 1e3, 2) if v[1] else None for k, v in prof.items()}
    if cfg.dim == 2:
        assembled = qc["splitk_dst"] in (-1, -2, -3)    # one GEMM per apply, no K1 (dd_set_schur_mode)
        grouped = qc["splitk_dst"] in (-2, -3)          # K-dim n: H_p = K_p G + gamma_p F
        pair = qc["splitk_dst"] == -3                   # ... formed in registers from the shared (G, F)
        compact = os.environ.get("DD_NO_COMPACT", "0")[:1] != "1"
        bn = 32 if grouped else 64
        cols_per_apply = live_columns(last, compact=compact, bn=bn)
        groups = live_columns(last, compact=compact, bn=bn)
        n_groups = [int(np.ceil(c / 32.0)) for c in groups]
        model = step_model_2d(cfg, grouped, assembled, args.frac_mode == "ra", cols_per_apply, n_groups, pk, pair)
        iters_per_solve = len(cols_per_apply)
        per_iter_meas = {k: (prof[k][0] / prof[k][1] * 1e-3) if prof[k][1] else 0.0 for k in model}
        classes = {}
        for k, (fl, by, tr) in model.items():
            meas = per_iter_meas.get(k, 0.0)
            bound = "tensor" if k.startswith("gemm") and fl / (pk["dmma"] * 1e12) >= by / (pk["hbm"] * 1e9) else (
                "fp64" if fl / (pk["dfma"] * 1e12) >= by / (pk["hbm"] * 1e9) else "hbm")
            classes[k] = {"bound": bound, "flops_per_launch": fl, "bytes_per_launch": by,
                          "roofline_us": round(tr * 1e6, 2), "measured_us": round(meas * 1e6, 2),
                          "frac": round(tr / meas, 4) if meas else None}
        dom = max(model, key=lambda k: prof[k][0])
        fl, by, _ = model[dom]
        t_dom = per_iter_meas[dom]
        if dom.startswith("gemm"):
            ach = fl / t_dom / 1e12 if t_dom else None
            roof = {"bound": "tensor", "achieved": round(ach, 3) if ach else None, "peak": pk["dmma"], "unit": "TFLOP/s",
                    "frac": round(ach / pk["dmma"], 4) if ach else None, "peak_source": pk["dmma_src"]}
        else:
            ach = by / t_dom / 1e9 if t_dom else None
            roof = {"bound": "hbm", "achieved": round(ach, 1) if ach else None, "peak": pk["hbm"], "unit": "GB/s",
                    "frac": round(ach / pk["hbm"], 4) if ach else None, "peak_source": pk["hbm_src"]}
        if pair:
            kname = ("gemm_schur grouped from the shared pair ((K_p G + gamma_p F) x X_p, operator fragments formed "
                     "in registers from G, F tiles; stream-K DMMA fp64)")
        elif grouped:
            kname = "gemm_schur grouped (H_p x X_p per parameter set, H_p = K_p G + gamma_p F formed at setup, DMMA fp64)"
        elif assembled:
            kname = ("gemm_schur ([F|G] x [gamma X; K X], DMMA fp64; G = S_unit formed at setup)"
                     if args.frac_mode == "dense" else "gemm_schur (G x K X + U, DMMA fp64; U = gamma M r_F M x by pole sum)")
        else:
            kname = ("gemm_schur ([S_dst|F] x [T; gamma X], DMMA fp64)" if args.frac_mode == "dense"
                     else "gemm_schur (S_dst x T' + U, DMMA fp64; U = gamma M r_F M x by pole sum)")
        if dom != "gemm_schur":
            kname = "polesum_pcg (fused PCG update + RA pole sum + dots, k_pcg_iter)"
        step_roof = sum(v[2] for v in model.values())
        step_meas = sum(per_iter_meas.values())
        roof.update({"kernel": kname, "class": dom,
                     "schur_mode": ("grouped_pair" if pair else "grouped") if grouped else ("assembled" if assembled else "factored"),
                     "flops_per_launch": fl, "bytes_per_launch": by,
                     "mean_live_columns": round(float(np.mean(cols_per_apply)), 2) if cols_per_apply else 0,
                     "applies_per_solve": iters_per_solve,
                     "launches_per_solve": round(prof[dom][1] / nprof, 2),
                     "classes": classes,
                     "step": {"roofline_us_per_iter": round(step_roof * 1e6, 2),
                              "measured_us_per_iter": round(step_meas * 1e6, 2),
                              "frac": round(step_roof / step_meas, 4) if step_meas else None,
                              "model": "sum over kernel classes of max(F/P, B/BW), algorithmic F, B (DESIGN.md §6)"}})
        tkey = "gemm_schur_" + roof["schur_mode"] if dom == "gemm_schur" else dom
    else:
        hbm = pk["hbm"]
        # F stream: the packed-symmetric upper 128 x 128 blocks (default on one rank; DD_FX_PACKED=0 or a
        # row-sharded multi-rank split streams the full row-major F); padded face length NP = ldf^2
        ldf = -(-n // 16) * 16
        NP = ldf * ldf
        packed = os.environ.get("DD_FX_PACKED", "1") != "0" and not (split and world > 1) and NP % 128 == 0
        nbk = NP // 128
        f_elems = nbk * (nbk + 1) // 2 * 128 * 128 if packed else cfg.n_gamma * cfg.n_gamma
        # class-sparse: the folded sine-domain H̃ at ldf = 128 is block-diagonal in the face parity
        # classes, so each 64-row half of a stored block keeps one 64-column quadrant (half the bytes)
        class_sparse = (packed and ldf == 128 and (n + 1) // 2 == 64 and os.environ.get("DD_FX_FOLD", "1") != "0"
                        and os.environ.get("DD_FX_CLASS_SPARSE", "1") != "0")
        if class_sparse:
            f_elems //= 2
        bytes_fx = 8.0 * f_elems + 3 * 8.0 * cfg.n_gamma * C
        g2_ms, g2_n = prof["gemm_schur"]
        ps_ms, ps_n = prof["polesum_pcg"]
        # RA mode (Remark 1) has no F stream: its gemm_schur class holds the two consistent-mass
        # products around the r_F pole sum, not an F read — no bandwidth figure
        ach = bytes_fx / (g2_ms / g2_n / 1e3) / 1e9 if g2_n and args.frac_mode != "ra" else None
        iters_solve = float(np.max(last)) if len(last) else 0.0
        # inner solver (polesum_pcg class), per operator application and (system, column) pair: the
        # two slab passes of D̂ V D̂^T with D̂ = [[0, E], [E', 0]] in the parity-ordered sine domain —
        # n^2 outputs x n/2 nonzero terms x 2 flops each, 2 n^3 algorithmic flops — and the vector
        # traffic: Chebyshev (default) x̂ read + T written (pass 1), T, x̂, d̂ read + x̂, d̂ written
        # (pass 2, fused step) = 7 x 8 B per face entry; CG (DD_INNER_CG=1) 2 passes + the 3-sweep
        # update = 16 x 8 B per entry
        cheb = os.environ.get("DD_INNER_CG", "0") != "1"
        nsys = len(ras[0].poles) + 1
        applies = iters_solve + 1
        npair = nsys * C / (world if split else 1)
        f_in = (inner_its or 0) * npair * (2.0 * n ** 3) * applies
        b_in = (inner_its or 0) * npair * ((56.0 if cheb else 128.0) * n * n) * applies
        t_in = ps_ms / 1e3 / nprof if ps_n else None
        inner_roof = max(f_in / (pk["dmma"] * 1e12), b_in / (hbm * 1e9))
        ra_mode = args.frac_mode == "ra"
        classes = {"gemm_schur": {"bound": "hbm", "bytes_per_launch": None if ra_mode else bytes_fx,
                                  "share_of_step": share.get("gemm_schur"),
                                  "f_storage": "none (RA-evaluated F)" if ra_mode else (
                                      ("packed_symmetric_class_sparse" if class_sparse else "packed_symmetric")
                                      if packed else "full"),
                                  "frac": round(ach / hbm, 4) if ach else None},
                   "polesum_pcg": {"bound": "tensor" if f_in / (pk["dmma"] * 1e12) >= b_in / (hbm * 1e9) else "hbm",
                                   "what": ("face inner Chebyshev (slab DMMA operator passes, fused step epilogue)" if cheb
                                            else "face inner CG (slab DMMA operator passes + vector updates)") + " per solve",
                                   "inner_solver": "chebyshev" if cheb else "cg",
                                   "inner_iterations_per_apply": inner_its, "pairs": npair,
                                   "flops_per_solve": f_in, "bytes_per_solve": b_in,
                                   "roofline_ms_per_solve": round(inner_roof * 1e3, 3),
                                   "measured_ms_per_solve": round(t_in * 1e3, 3) if t_in else None,
                                   "frac": round(inner_roof / t_in, 4) if t_in else None,
                                   "share_of_step": share.get("polesum_pcg")}}
        dom = max(("gemm_schur", "polesum_pcg"), key=lambda k: prof[k][0])
        if dom == "polesum_pcg" and t_in:
            # achieved / peak / unit follow the bound the algorithmic count picks, so that
            # frac = achieved / peak (= roofline time / measured time)
            hb = classes["polesum_pcg"]["bound"] == "hbm"
            roof = {"bound": classes["polesum_pcg"]["bound"], "class": "polesum_pcg",
                    "kernel": "3D face inner " + ("Chebyshev" if cheb else "CG") +
                              " (sine-diagonal preconditioned, batched over (system, column) pairs)",
                    "achieved": round(b_in / t_in / 1e9, 1) if hb else round(f_in / t_in / 1e12, 3),
                    "peak": hbm if hb else pk["dmma"], "unit": "GB/s" if hb else "TFLOP/s",
                    "frac": classes["polesum_pcg"]["frac"], "peak_source": pk["hbm_src"] if hb else pk["dmma_src"],
                    "achieved_fp64_tflops": round(f_in / t_in / 1e12, 3),
                    "frac_of_dmma_peak": round(f_in / t_in / 1e12 / pk["dmma"], 4)}
        else:
            roof = {"bound": "hbm", "class": "gemm_schur",
                    "kernel": ("gemm_schur (gamma F x, packed-symmetric F: direct + transposed DMMA per stored block"
                               " + fixed-order partial reduce)" if packed else
                               "gemm_schur (gamma F x, full F stream, stream-K DMMA, BN=8)"),
                    "achieved": round(ach, 1) if ach else None, "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4) if ach else None, "peak_source": pk["hbm_src"],
                    "bytes_per_launch": bytes_fx}
        roof["classes"] = classes
        roof["f_stream"] = {"achieved_gbs": round(ach, 1) if ach else None, "frac": round(ach / hbm, 4) if ach else None,
                            "frac_vs_nominal_8000gbs": round(ach / 8000.0, 4) if ach else None}
        fkey = ("gemm_schur_packed_cs" if class_sparse else "gemm_schur_packed") if packed else "gemm_schur"
        ikey = ("cheb_step" if os.environ.get("DD_CHEB_FUSED", "1") != "0" and n == 127 else "cheb_two_pass") if cheb \
            else "inner_update"
        tkey = fkey if roof["class"] == "gemm_schur" else ikey
        if args.frac_mode == "ra":
            roof["note"] = "RA mode: no dense F; the face inner solver (r_F and P systems) carries the step"
    roof.update({"traffic": traffic_for(cfg.name, tkey), "traffic_key": tkey,
                 "avg_launch_us": avg_us.get(roof.get("class", "gemm_schur")),
                 "share_of_step": share, "avg_us": avg_us})
    if cfg.dim == 3:
        roof["traffic_f_stream"] = traffic_for(cfg.name, fkey) if args.frac_mode != "ra" else None
    if split:
        par = f"RA systems split over {world} rank(s), NCCL allreduce of the partial sums per preconditioner apply"
    elif cfg.dim == 2:
        par = (f"fixed batch of {C_all} solves split over {world} rank(s) in 32-column single-parameter blocks "
               f"(LPT on pilot iterations), no collective")
    else:
        par = f"replicas: each of {world} rank(s) solves its own {C} columns, no collective"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "dim": cfg.dim, "cells_per_side": cfg.N, "n_gamma": cfg.n_gamma,
                   "param_sets": len(cfg.params), "rhs_per_param": cfg.rhs_per_param,
                   "solves_per_step": solves_per_step, "rank0_solves_per_step": C,
                   "poles": cfg.n_poles, "rtol": cfg.rtol, "l2": "flushed (512 MiB write) between timed steps",
                   "schur_apply": args.schur if cfg.dim == 2 else "factored (3D)",
                   "setup_ms_untimed": round(setup_ms, 1), "parallelism": par, "shard": shard,
                   "fractional_term": "dense F (Eq.(7))" if args.frac_mode == "dense"
                   else f"RA-evaluated (Remark 1), {cfg.n_poles} poles",
                   "t": args.t, "L": "-Δ_Γ + I" if args.shifted else "-Δ_Γ",
                   "ra_max_rel_err": max(r.rel_err for r in ras),
                   "mean_pcg_iters": round(float(its.mean()), 3), "max_pcg_iters": int(its.max()),
                   "iters_by_param": {"fields": ["K", "mu_inv", "max", "mean"], "rows": by_param}},
        "precond_applies_per_s": round(pa_per_s, 1) if pa_per_s else None,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "roofline": roof,
        "launch_config": qc,
        "e2e": {"value": round(e2e_value, 3) if e2e_value else None, "unit": UNIT,
                "h2d_bytes_per_step": int(B.nbytes + C * 4), "d2h_bytes_per_step": int(B.nbytes + C * 12)},
    }
    if not args.no_cpu_baseline and world == 1:
        if cfg.dim == 3:
            line["cpu_baseline"] = oracle_baseline_3d(cfg, ras, B)
        else:
            per = max(1, int(os.environ.get("DD_ORACLE_PER_PARAM", "64")))
            solves, secs = oracle_sample(cfg, ras, B, colp, per, args.t, 1.0 if args.shifted else 0.0)
            line["cpu_baseline"] = {"value": round(solves / secs, 4), "unit": UNIT, "cores": cores_used(),
                                    "kind": "oracle",
                                    "sample": f"{solves} of the {C} solves ({per} per parameter set max), oracle mode "
                                              f"tier (scipy DST + LAPACK banded Cholesky), {secs:.1f} s",
                                    "host": host_info()}
    return line


def oracle_baseline_3d(cfg, ras, B):
    """Config 4 on the host: the oracle's setup (P1 face pair, the dense 16129^2 generalised
    eigensolve for F = (MU) Λ^-1/2 (MU)^T) — untimed, reported, as the library's setup is — then the
    oracle's PCG (dense F matvec, mode-tier S_unit, sparse-direct shifted solves) on ONE of the
    columns, timed: solves/s = 1 / that time.  Needs ~16 GB of host memory and minutes of setup."""
    from oracle import fem, pcg as opcg, ra as ora, schur as osch, spectral
    n = cfg.n; ng = n * n
    K, g = cfg.params[0]; fit = ras[0]
    t0 = time.perf_counter()
    A, M = fem.trace_pair_face(cfg.N)
    G = spectral.GEVP(A.toarray(), M.toarray())
    F = G.power(-0.5)
    del G
    s = osch.schur_modes_3d(cfg.N)
    setup_s = time.perf_counter() - t0

    def apply_S(x):
        Y = x.reshape(n, n)
        Yh = osch.dst_ortho(osch.dst_ortho(Y, axis=0), axis=1)
        Y = osch.dst_ortho(osch.dst_ortho(s * Yh, axis=0), axis=1)
        return K * Y.ravel() + g * (F @ x)

    t1 = time.perf_counter()
    x, it, rel, hist, conv = opcg.pcg(apply_S, lambda v: ora.apply_ra(A, M, fit.c0, fit.poles, fit.residues, v), B[0],
                                      rtol=cfg.rtol, maxit=cfg.maxit)
    secs = time.perf_counter() - t1
    return {"value": round(1.0 / secs, 5), "unit": UNIT, "cores": cores_used(), "kind": "oracle",
            "sample": f"1 of the {B.shape[0]} solves (column 0, {it} iterations) by the oracle's PCG: dense F matvec, "
                      f"mode-tier S_unit, sparse-direct LU per shifted system; {secs:.1f} s",
            "oracle_setup_s_untimed": round(setup_s, 1), "host": host_info()}


def emulate_ranks(args, cfg, ras, frac, B_all, colp_all, pilot, dev, flush):
    """PREDICTION of the W-GPU value on ONE GPU: each rank's shard is run alone, one after another,
    and the predicted step time is the max over ranks (2D, strong scaling: no collective on the
    path).  3D pole split: the replicated Schur apply plus each rank's partial preconditioner apply
    are timed, the allreduce is not (one GPU): t_step ~ iters x (schur + max_r precond_r) + precond,
    reported with the allreduce cost left out and said so."""
    import torch
    from paper_2211_15308_b200 import binding
    from paper_2211_15308_b200 import dist as ddist_mod
    W = args.emulate_ranks
    out = {"kind": "prediction (ranks run one after another on one GPU; not a W-GPU measurement)", "world": W}
    if cfg.dim == 2:
        per = []
        S = binding.Solver(2, cfg.N, cfg.params, ras, max_cols=B_all.shape[0], device=torch.device(dev).index, frac=frac)
        S.set_schur_mode(args.schur)
        try:
            for r in range(W):
                cols, colp = ddist_mod.block_shard(len(cfg.params), cfg.rhs_per_param, r, W, pilot)
                if not len(cols):
                    per.append(0.0)
                    continue
                Bt = torch.as_tensor(np.ascontiguousarray(B_all[cols]), device=dev)
                cp = torch.as_tensor(colp, device=dev)
                for _ in range(2):
                    flush.fill_(1.0)
                    check_solve(S.pcg_solve(Bt, cp, rtol=cfg.rtol, maxit=cfg.maxit), "emulated rank")
                ms = []
                for _ in range(max(3, args.steps)):
                    flush.fill_(1.0)
                    check_solve(S.pcg_solve(Bt, cp, rtol=cfg.rtol, maxit=cfg.maxit), "emulated rank")
                    ms.append(S.last_solve_ms())
                per.append(float(np.median(ms)))
        finally:
            S.close()
        out.update({"rank_ms_per_step": [round(v, 4) for v in per],
                    "predicted_value": round(B_all.shape[0] / (max(per) / 1e3), 3), "unit": UNIT})
        return out
    # 3D pole split
    Bt = torch.as_tensor(B_all, device=dev)
    cp = torch.as_tensor(colp_all, device=dev)
    full = binding.Solver(3, cfg.N, cfg.params, ras, max_cols=B_all.shape[0], device=torch.device(dev).index, frac=frac)
    try:
        r = full.pcg_solve(Bt, cp, rtol=cfg.rtol, maxit=cfg.maxit)
        iters = int(r.iters.max())
        t_solve1 = full.last_solve_ms()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        full.apply_schur(Bt, cp)
        e0.record(full.stream)
        for _ in range(5):
            full.apply_schur(Bt, cp)
        e1.record(full.stream)
        torch.cuda.synchronize()
        t_schur = e0.elapsed_time(e1) / 5
    finally:
        full.close()
    per, per_s = [], []
    for rk in range(W):
        S = binding.Solver(3, cfg.N, cfg.params, ras, max_cols=B_all.shape[0], device=torch.device(dev).index,
                           frac=frac, dist=(rk, W, 1, None))
        try:
            for what, lst in (("precond", per), ("schur", per_s)):
                fn = S.apply_precond if what == "precond" else S.apply_schur
                fn(Bt, cp)
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(S.stream)
                for _ in range(3):
                    fn(Bt, cp)
                e1.record(S.stream)
                torch.cuda.synchronize()
                lst.append(e0.elapsed_time(e1) / 3)
        finally:
            S.close()
    # each rank: its F rows (row-sharded stream) + the replicated slab passes, then its share of the
    # pole sum; the step waits for the slowest rank at each of the two collectives
    t_step = iters * (max(per_s) + max(per)) + max(per)
    t_step_repl = iters * (t_schur + max(per)) + max(per)
    out.update({"iters": iters, "schur_apply_ms_1gpu": round(t_schur, 3), "rank_schur_ms_row_sharded_F": [round(v, 3) for v in per_s],
                "rank_precond_ms": [round(v, 3) for v in per],
                "predicted_ms_per_solve_batch": round(t_step, 3), "measured_1gpu_ms": round(t_solve1, 3),
                "predicted_value": round(B_all.shape[0] / (t_step / 1e3), 3), "unit": UNIT,
                "predicted_value_replicated_F": round(B_all.shape[0] / (t_step_repl / 1e3), 3),
                "excludes": "per PCG iteration the NCCL allreduce of the partial pole sums and the allgather of the "
                            "F rows (16129 x 8 fp64 each) — one GPU available"})
    return out


def run_bulk(args, cfg, world, rank):
    """NEXT-1: full DD solve on bulk right-hand sides (dd_bulk_solve): metric bulk solves/s;
    the slab transforms (4 batched n x n x n DMMA GEMMs per RHS) bound it."""
    import torch
    from paper_2211_15308_b200 import binding
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    ras = fit_ras(cfg)
    n = cfg.n
    C = cfg.n_cols
    rng = np.random.default_rng(1000 + rank)
    nb = n * n + n if cfg.dim == 2 else n ** 3 + n * n
    Bb = rng.uniform(-1.0, 1.0, (C, nb))
    colp = (np.arange(C) // cfg.rhs_per_param).astype(np.int32)
    frac = None
    if args.frac_mode == "ra":
        # Remark 1: the operator's fractional term evaluated by RA as well
        lo, hi = rafit.interval_1d(cfg.N) if cfg.dim == 2 else rafit.interval_face(cfg.N)
        frac = binding.Frac(mode="ra", fra=rafit.fit_power(-0.5, lo, hi, cfg.n_poles, 0.0))
    S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=C, device=local, frac=frac)
    Bt = torch.as_tensor(Bb, device=f"cuda:{local}")
    X = torch.empty_like(Bt)
    cp = torch.as_tensor(colp, device=f"cuda:{local}")
    solve = S.bulk_solve if args.mode == "bulk" else S.bulk_pcg_solve
    for _ in range(args.warmup):
        solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=cfg.maxit)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(S.stream)
        for _ in range(args.steps):
            r = solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=cfg.maxit)
        e1.record(S.stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    S.profile(True)
    S.bulk_solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=0)      # maxit 0: gemm_dst holds the 4 slab passes only
    prof = S.profile_read()
    S.profile(False)
    ldf = (n + 15) // 16 * 16
    pass_ms, pass_n = prof["gemm_dst"]
    if cfg.dim == 2:
        fl_pass = 2.0 * n * n * ldf * C                       # one slab pass over the C fields
        ach = fl_pass / (pass_ms / pass_n / 1e3) / 1e12 if pass_n else None
        kname = "bulk slab pass (S Y per field, batched DMMA)"
    else:
        # 3D: every DMMA launch of one bulk solve (the class holds them all): the forward and inverse
        # full-field transforms (face passes over n layers + the normal-axis pass) and four face passes
        NP = ldf * ldf
        fl_pass = C * (2 * (2 * n * (2.0 * n * n * ldf) + 2.0 * NP * n * ldf) + 4 * 2.0 * n * n * ldf)
        ach = fl_pass / (pass_ms / 1e3) / 1e12 if pass_ms else None
        kname = "3D bulk transforms (face passes + normal-axis pass, batched DMMA), per solve"
    peak, peak_src = fp64_peak()
    if rank == 0:
        print(json.dumps({
            "metric": "DD bulk solves/s" if args.mode == "bulk" else "bulk PCG (Eq.(5) DD preconditioner) solves/s",
            "value": round(C / (ms / 1e3), 3), "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name + ("_bulk" if args.mode == "bulk" else "_bulk_pcg")
                                   + ("_frac_ra" if args.frac_mode == "ra" else ""),
                       "bulk_unknowns_per_solve": nb, "solves_per_step": C,
                       "mean_pcg_iters": float(np.mean(r.iters)),
                       "l2": "inputs (4.3 GB of fields) exceed L2" if cfg.dim == 2 else "fields of 133 MB per 8 columns"},
            "clocks": clk.summary(),
            "roofline": {"bound": "tensor", "kernel": kname,
                         "achieved": round(ach, 3) if ach else None, "peak": peak, "unit": "TFLOP/s",
                         "frac": round(ach / peak, 4) if ach else None, "peak_source": peak_src,
                         "flops_per_launch": fl_pass, "avg_launch_us": round(pass_ms / pass_n * 1e3, 1) if pass_n else None,
                         "traffic": None,
                         "share_of_step": {k: round(v[0] / sum(x[0] for x in prof.values()), 4) for k, v in prof.items()}},
        }), flush=True)
    S.close()


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    ras = fit_ras(cfg)
    B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
    per = max(1, int(os.environ.get("DD_ORACLE_PER_PARAM", "16")))
    for _ in range(args.warmup):
        oracle_sample(cfg, ras, B, colp, 1)
    tot_s, tot_n = 0.0, 0
    for _ in range(args.steps):
        n, s = oracle_sample(cfg, ras, B, colp, per)
        tot_s += s; tot_n += n
    v = tot_n / tot_s
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_s / args.steps * 1e3, 3),
            # the same fixed sample whatever the launch width (rank 0 only): strong, like this arm's own line
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "solves_per_step": per * len(cfg.params)},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores_used(), "kind": "oracle",
                             "sample": f"{per} solves per parameter set per step (of {cfg.rhs_per_param}), oracle mode tier",
                             "host": host_info()},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
