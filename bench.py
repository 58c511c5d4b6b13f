#!/usr/bin/env python
"""Benchmark: Schur-complement PCG solves/s on B200 (BASELINE.json metric), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2_2d_N1024_sweep] [--impl reference]

A "step" is one dd_pcg_solve over one batch of the workload (every column driven to
rtol 1e-10): the whole hot path (Schur apply = DST GEMM + [S_dst|F] GEMM, RA pole sum, fused
PCG updates) per iteration.  At N=1 the workload is BASELINE.json configs[1] (2D, 1024
cells/side, 4 parameter sets x 64 RHS = 256 solves per step).
Multi-GPU (torchrun): independent (K, mu, RHS) columns shard with no data-path collective —
each rank solves its own full batch (weak scaling, seeds offset by rank); value = all ranks'
solves / max-over-ranks time.
Timing: W warm-up steps, then K steps each bracketed by CUDA events (recorded inside libdd
on its stream), with a 512 MiB L2 flush between steps outside the timed spans; barrier +
synchronize on both sides of the timed region; max over ranks.
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
    ap.add_argument("--pole-split", action="store_true",
                    help="3D (config 4, SURVEY §8(e)): all ranks solve the same columns, the RA poles are split "
                         "across ranks and the partial sums allreduced over NCCL each preconditioner apply "
                         "(strong scaling); default: columns per rank (weak scaling, no collective)")
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
    local = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if args.mode in ("bulk", "bulk-pcg"):
        return run_bulk(args, cfg, world, rank)

    import torch
    import torch.distributed as dist
    from paper_2211_15308_b200 import binding

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sigma = 1.0 if args.shifted else 0.0
    ras = fit_ras(cfg, args.t, sigma)
    split = bool(args.pole_split and cfg.dim == 3)
    # pole split: every rank holds the same columns (the exchange is inside the preconditioner)
    B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param,
                           seed_offset=0 if split else rank * len(cfg.params))
    C = B.shape[0]
    ddist = None
    if split:
        from paper_2211_15308_b200 import dist as ddist_mod
        uid = binding.nccl_unique_id() if rank == 0 else None
        if world > 1:
            uid = ddist_mod.broadcast_bytes(uid, 128, device=f"cuda:{local}")
        ddist = (rank, world, 1, uid if world > 1 else None)   # DD_SHARD_POLES
    frac = binding.Frac(t=args.t, shifted=args.shifted)
    if args.frac_mode == "ra":
        lo, hi = rafit.interval_1d(cfg.N) if cfg.dim == 2 else rafit.interval_face(cfg.N)
        frac = binding.Frac(t=args.t, shifted=args.shifted, mode="ra",
                            fra=rafit.fit_power(args.t, lo, hi, cfg.n_poles, sigma))
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=C, device=local, frac=frac, dist=ddist)
    if cfg.dim == 2:
        S.set_schur_mode(args.schur)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t_setup) * 1e3      # once per mesh and parameter sets (row a-1)
    Bt = torch.as_tensor(B, device=f"cuda:{local}")
    cp = torch.as_tensor(colp.astype(np.int32), device=f"cuda:{local}")
    X = torch.empty_like(Bt)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def step():
        return S.pcg_solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=cfg.maxit)

    for _ in range(args.warmup):
        flush.fill_(1.0)
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
            r = step()
            step_ms.append(S.last_solve_ms())
            iters_all.append(r.iters.copy())
        torch.cuda.synchronize()
    launches = S.launch_count()
    qc = S.query_config()              # launch configuration of the timed solves
    if world > 1:
        dist.barrier()
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    solves_total = C * args.steps * (1 if split else world)
    value = solves_total / (max_ms / 1e3)

    # ---- instrumented pass: per-kernel-class device time (CUDA events on libdd's stream)
    S.profile(True)
    nprof = max(2, min(args.steps, 5))
    for _ in range(nprof):
        flush.fill_(1.0)
        step()
    prof = S.profile_read()
    S.profile(False)

    # ---- e2e through the host-buffer ABI call (pinned host memory, H2D + D2H inside)
    Bh = torch.as_tensor(B).pin_memory().numpy()
    Xh = torch.empty(B.shape, dtype=torch.float64).pin_memory().numpy()
    S.pcg_solve_host(Bh, colp, rtol=cfg.rtol, maxit=cfg.maxit, x_out=Xh)
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S.pcg_solve_host(Bh, colp, rtol=cfg.rtol, maxit=cfg.maxit, x_out=Xh)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = float(sum(e2e_t))
    te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = C * len(e2e_t) * (1 if split else world) / float(te.item())

    # ---- precond applies/s (secondary metric of BASELINE.json)
    Z = torch.empty_like(Bt)
    for _ in range(3):
        S.apply_precond(Bt, cp, z=Z)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(S.stream)
    for _ in range(reps):
        S.apply_precond(Bt, cp, z=Z)
    e1.record(S.stream)
    torch.cuda.synchronize()
    pa_per_s = C * reps * (1 if split else world) / (e0.elapsed_time(e1) / 1e3)

    if rank == 0:
        n = cfg.n
        its = np.concatenate(iters_all)
        mean_it = float(its.mean())
        last = iters_all[-1]
        by_param = [[K, g, int(last[colp == p].max()), round(float(last[colp == p].mean()), 2)]
                    for p, (K, g) in enumerate(cfg.params)]
        peak, peak_src = fp64_peak()
        g2_ms, g2_n = prof["gemm_schur"]
        g1_ms, g1_n = prof["gemm_dst"]
        ps_ms, ps_n = prof["polesum_pcg"]
        total_prof_ms = sum(v[0] for v in prof.values())
        if cfg.dim == 2:
            # [S_dst | F] (n x 2n) times (2n x C), algorithmic; RA mode (Remark 1): S_dst T' only
            assembled = qc["splitk_dst"] in (-1, -2)    # one GEMM per apply, no K1 (dd_set_schur_mode)
            grouped = qc["splitk_dst"] == -2            # K-dim n: H_p = K_p G + gamma_p F
            # Live-tile compaction (>= 6 tiles of 64 columns): the apply at iteration k runs only the
            # column tiles (32 wide for the grouped GEMM, else 64) holding a column with iters >= k, so
            # the algorithmic work per launch is counted over those columns (the profiled solves repeat
            # the timed ones: same inputs, same iterations).
            cols_per_apply = live_columns(last, compact=(os.environ.get("DD_NO_COMPACT", "0")[:1] != "1"),
                                          bn=32 if grouped else 64)
            c_eff = float(np.mean(cols_per_apply))
            flops_g2 = 2.0 * n * (2 * n) * c_eff if (args.frac_mode == "dense" and not grouped) else 2.0 * n * n * c_eff
            flops_g1 = 0.0 if assembled else 2.0 * n * n * c_eff
            ach_g2 = flops_g2 / (g2_ms / g2_n / 1e3) / 1e12 if g2_n else None
            step_flops = (flops_g1 + flops_g2) * len(cols_per_apply)
            if grouped:
                kname = "gemm_schur grouped (H_p x X_p per parameter set, H_p = K_p G + gamma_p F formed at setup, DMMA fp64)"
            elif assembled:
                kname = ("gemm_schur ([F|G] x [gamma X; K X], DMMA fp64; G = S_unit formed at setup)"
                         if args.frac_mode == "dense" else
                         "gemm_schur (G x K X + U, DMMA fp64; U = gamma M r_F M x by pole sum)")
            else:
                kname = ("gemm_schur ([S_dst|F] x [T; gamma X], DMMA fp64)" if args.frac_mode == "dense"
                         else "gemm_schur (S_dst x T' + U, DMMA fp64; U = gamma M r_F M x by pole sum)")
            roof = {"bound": "tensor", "kernel": kname,
                    "schur_mode": "grouped" if grouped else ("assembled" if assembled else "factored"),
                    "achieved": round(ach_g2, 3) if ach_g2 else None, "peak": peak, "unit": "TFLOP/s",
                    "frac": round(ach_g2 / peak, 4) if ach_g2 else None, "peak_source": peak_src,
                    "flops_per_launch": flops_g2, "mean_live_columns": round(c_eff, 2),
                    "applies_per_solve": len(cols_per_apply), "launches_per_solve": round(g2_n / nprof, 2),
                    "step_fp64_frac": round(step_flops / (total_prof_ms / nprof / 1e3) / 1e12 / peak, 4)}
        elif args.frac_mode == "ra":
            # 3D, Remark 1: no dense F; the step is the face inner CG (slab DMMA passes + vector updates)
            roof = {"bound": "tensor", "kernel": "3D RA mode: face inner-CG slab passes + updates (class polesum_pcg)",
                    "achieved": None, "peak": fp64_peak()[0], "unit": "TFLOP/s", "frac": None,
                    "peak_source": fp64_peak()[1],
                    "note": "no single dominant kernel: inner-CG GEMM passes and memory-bound updates share the step"}
        else:
            # 3D: the dense fractional term F (n_Γ^2 fp64) is streamed once per Schur apply: HBM-bound
            mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
            hbm = float(mp.get("hbm_gbs", 6650.0))
            bytes_fx = 8.0 * cfg.n_gamma * cfg.n_gamma + 3 * 8.0 * cfg.n_gamma * C
            ach = bytes_fx / (g2_ms / g2_n / 1e3) / 1e9 if g2_n else None
            roof = {"bound": "hbm", "kernel": "gemm_schur (gamma F x + sine back-transform, stream-K DMMA, BN=8)",
                    "achieved": round(ach, 1) if ach else None, "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4) if ach else None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if mp else "fallback 6650 GB/s",
                    "bytes_per_launch": bytes_fx,
                    # also against the north star's nominal 8.0 TB/s
                    "frac_vs_nominal_8000gbs": round(ach / 8000.0, 4) if ach else None}
        tkey = "gemm_schur" if cfg.dim == 3 else "gemm_schur_" + roof.get("schur_mode", "factored")
        roof.update({"traffic": traffic_for(cfg.name, tkey), "traffic_key": tkey,
                     "avg_launch_us": round(g2_ms / g2_n * 1e3, 2) if g2_n else None,
                     "share_of_step": {k: round(v[0] / total_prof_ms, 4) for k, v in prof.items()},
                     "avg_us": {k: round(v[0] / v[1] * 1e3, 2) if v[1] else None for k, v in prof.items()}})
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if split else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "dim": cfg.dim, "cells_per_side": cfg.N, "n_gamma": cfg.n_gamma,
                       "param_sets": len(cfg.params), "rhs_per_param": cfg.rhs_per_param, "solves_per_step": C,
                       "poles": cfg.n_poles, "rtol": cfg.rtol, "l2": "flushed (512 MiB write) between timed steps",
                       "schur_apply": args.schur if cfg.dim == 2 else "factored (3D)",
                       "setup_ms_untimed": round(setup_ms, 1),
                       "parallelism": (f"RA poles split over {world} rank(s), NCCL allreduce of the partial "
                                       f"sums per preconditioner apply" if split else
                                       f"columns sharded, {world} rank(s), no collective"),
                       "fractional_term": "dense F (Eq.(7))" if args.frac_mode == "dense"
                       else f"RA-evaluated (Remark 1), {cfg.n_poles} poles",
                       "t": args.t, "L": "-Δ_Γ + I" if args.shifted else "-Δ_Γ",
                       "ra_max_rel_err": max(r.rel_err for r in ras),
                       "mean_pcg_iters": round(mean_it, 3), "max_pcg_iters": int(its.max()),
                       "iters_by_param": {"fields": ["K", "mu_inv", "max", "mean"], "rows": by_param}},
            "precond_applies_per_s": round(pa_per_s, 1),
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "roofline": roof,
            "launch_config": qc,
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT,
                    "h2d_bytes_per_step": int(B.nbytes + C * 4), "d2h_bytes_per_step": int(B.nbytes + C * 12)},
        }
        if cfg.dim == 3:
            line["cpu_baseline"] = None
            line["cpu_baseline_note"] = ("not run: the dense oracle at n_Gamma = 16129 needs ~5e14 flop of elimination "
                                         "plus a 16129^2 generalised eigensolve (tens of minutes on the host)")
        elif not args.no_cpu_baseline and world == 1:
            per = max(1, int(os.environ.get("DD_ORACLE_PER_PARAM", "64")))
            solves, secs = oracle_sample(cfg, ras, B, colp, per, args.t, 1.0 if args.shifted else 0.0)
            line["cpu_baseline"] = {"value": round(solves / secs, 4), "unit": UNIT, "cores": cores_used(),
                                    "kind": "oracle",
                                    "sample": f"{solves} of the {C} solves ({per} per parameter set), oracle mode tier "
                                              f"(scipy DST + LAPACK banded Cholesky), {secs:.1f} s",
                                    "host": host_info()}
        print(json.dumps(line), flush=True)
    S.close()
    if world > 1:
        dist.destroy_process_group()


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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "solves_per_step": per * len(cfg.params)},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores_used(), "kind": "oracle",
                             "sample": f"{per} solves per parameter set per step (of {cfg.rhs_per_param}), oracle mode tier",
                             "host": host_info()},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
