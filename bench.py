"""bench.py -- time-to-1e-8 of SP / SP-RK-RGS / SP-SCD on one B200 through the C ABI (libils.so).

Contract (driver): python bench.py --gpus N --steps K --warmup W [--impl reference]
prints ONE JSON line on rank 0.

A "step" is one pass of the whole hot path over the workload:
  ils_create (ingest: layout, column norms, sampling tables, A1^T b1)            row a0
  ils_sp_solve  to ||x-x_ref|| <= tol  (DMMA Gram + Cholesky + P, fused K1 stream)  rows a1 a2 a7
  ils_rk_solve  to tol (K1 stream + persistent RK-RGS, Philox index stream)      rows a1 a3 a4 a5 a7
  ils_rgs_solve to tol (K1 stream + persistent SP-SCD, Feistel subsets)          rows a1 a3 a5 a6 a7
  ils_destroy
value = device time of one step in ms (= sum over the three methods of time-to-tolerance, setup
and ingest included; lower is better). The default workload is BASELINE.json configs[1] (c1).
Inputs are resident in HBM when the timed region starts; L2 is flushed (256 MiB write) between
timed steps. e2e repeats the step with pinned HOST buffers (H2D of A, b, x_ref and D2H of x inside
the timed region). cpu_baseline times the CPU oracle (test infrastructure) on a bounded sample.

Multi-GPU: the single-instance path does not shard ("replicas only"): --gpus N
runs N independent replicas (weak scaling), value = max over ranks of ms per step. The batched
config (c4) partitions instances: rank r solves its own 4096 instances (data seeds r*4096 + i,
instance_partition()), no data-path collective (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "time-to-1e-8 rel err per method (SP/RK/RGS); achieved HBM GB/s vs 8 TB/s"
HBM_NOMINAL_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0
FALLBACK_BF16_TFLOPS = 1590.0
# fp64 DMMA: no measured peak on this pool; B200 nominal FP64 tensor 40 TFLOP/s vs 2250 bf16
# dense -> measured bf16 x 40/2250 (the guide's rule for another dtype's peak).
FP64_OVER_BF16 = 40.0 / 2250.0
KINDS = {0: "sp_persistent_kernel (K1 stream + P apply)",
         1: "rk_rgs_la_kernel (K2a: 16-CTA look-ahead SP-RK-RGS, one launch per inner solve with its checks, at c1)",
         2: "scd_kernel (K2b)", 3: "setup: gemm_dmma_kernel + potf2_trtri_kernel (K3)"}


def workload_desc(cfg: str) -> str:
    return {
        "c0": "c0 tiny dense p=200 q=100 n=50, A2 0.3N(0,1), b=Ax*, tol 1e-10",
        "c1": "c1 medium dense p=8000 q=2000 n=1000, A2 0.5N(0,1), b=Ax*+0.01N(0,1), tol 1e-8 vs oracle Cholesky x_ref",
        "c2": "c2 ill-conditioned dense p=40000 q=10000 n=4000, s log-spaced 1..1e3, b=Ax*, tol 1e-8",
        "c3": "c3 sparse CSR p=500000 q=100000 n=20000, 10 nnz/row, A2 0.3N(0,1), b=Ax*+1e-3N(0,1), tol 1e-8 vs oracle Cholesky x_ref",
        "c4": "c4 batched 4096 x (p=96 q=32 n=32), tol 1e-10 per instance",
    }[cfg]


def config_dict(cfg: str, methods, world: int) -> dict:
    """The line's `config` (identical for the GPU arm and the reference arm)."""
    return {"workload": workload_desc(cfg), "methods": list(methods),
            "parallelism": ("instance-partition" if cfg == "c4" else "replicas") if world > 1 else "single-gpu",
            "l2": "flushed between timed steps (256 MiB write)"}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, 1400.0, "fallback"


def inner_tol_for(tol: float) -> float:
    return 1e-12 if tol <= 1e-10 else 1e-10


# RK / RGS on c2 and c3 need ~1e10 / ~1e6-1e7 latency-bound inner steps per outer iteration
# (DESIGN.md §8): the bench times SP there; tools/probe_perf.py reports capped runs.
DEFAULT_METHODS = {"c0": "sp,rk,rgs", "c1": "sp,rk,rgs", "c2": "sp", "c3": "sp", "c4": "sp,rk,rgs"}


def instance_partition(rank: int, world: int, batch: int) -> tuple:
    """Batched config under N ranks: rank r owns instances [r*batch, (r+1)*batch) of the global
    seeded family (instance i has data seed i), so ranks hold disjoint instances and the job solves
    world*batch instances (weak scaling, no collective on the data path)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * batch, (rank + 1) * batch


def load_problem(cfg: str, rank: int = 0, world: int = 1):
    """Seeded synthetic workload (workloads/) and its x_ref: x* for consistent configs, else the
    oracle-written file workloads/xref/<cfg>_seed0.npy (tools/make_xref.py)."""
    from workloads import CONFIGS, fingerprint, make_problem
    if cfg == "c4":
        lo, _ = instance_partition(rank, world, CONFIGS["c4"]["batch"])
        pr = make_problem(cfg, seed=lo)
        return pr, pr.xstar
    base = os.path.join(ROOT, "workloads", "xref", f"{cfg}_seed0")
    meta = None
    if os.path.exists(base + ".json"):
        with open(base + ".json") as f:
            meta = json.load(f)
    pr = make_problem(cfg, seed=(meta or {}).get("data_seed", 0))
    if pr.consistent:
        return pr, pr.xstar
    if meta is None or meta["fingerprint"] != fingerprint(pr if hasattr(pr, "scipy") else pr.A, pr.b):
        raise RuntimeError(f"x_ref file {base}.npy does not match the generated {cfg} data; rerun tools/make_xref.py")
    return pr, np.load(base + ".npy")


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.f is None:
            return None
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [s.strip() for s in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------ GPU arm
class Runner:
    """Runs one step of the hot path through the C ABI (paper_2203_15340_b200.ils)."""

    def __init__(self, cfg, pr, xref, methods, torch, dev, host=False):
        from paper_2203_15340_b200 import ils
        self.ils, self.torch, self.dev, self.cfg, self.pr = ils, torch, dev, cfg, pr
        self.methods = methods
        self.batched = cfg == "c4"
        self.sparse = hasattr(pr, "scipy")
        self.B = pr.batch if self.batched else 1
        self.n = pr.n
        self.tol = pr.tol
        self.itol = inner_tol_for(pr.tol)
        self.host = host
        t = torch
        if self.sparse:
            src = {k: np.ascontiguousarray(getattr(pr, k)) for k in ("vals", "row_ptr", "col_idx")}
            if host:
                self.A, self.rp, self.ci = (t.from_numpy(src[k]).pin_memory() for k in ("vals", "row_ptr", "col_idx"))
            else:
                self.A, self.rp, self.ci = (t.from_numpy(src[k]).to(dev) for k in ("vals", "row_ptr", "col_idx"))
        if host:   # pinned host buffers: the library stages them to HBM inside the call
            if not self.sparse:
                self.A = t.from_numpy(np.ascontiguousarray(pr.A)).pin_memory()
            self.b = t.from_numpy(np.ascontiguousarray(pr.b)).pin_memory()
            self.xref = t.from_numpy(np.ascontiguousarray(xref, dtype=np.float64).reshape(-1)).pin_memory()
            self.x = {m: t.zeros(self.B * self.n, dtype=t.float64).pin_memory() for m in methods}
        else:
            if not self.sparse:
                self.A = t.from_numpy(np.ascontiguousarray(pr.A)).to(dev)
            self.b = t.from_numpy(np.ascontiguousarray(pr.b)).to(dev)
            self.xref = t.from_numpy(np.ascontiguousarray(xref, dtype=np.float64).reshape(-1)).to(dev)
            self.x = {m: t.zeros(self.B * self.n, dtype=t.float64, device=dev) for m in methods}
        self.xref_host = np.ascontiguousarray(xref, dtype=np.float64).reshape(self.B, self.n)
        self.h2d = self.A.numel() * 8 + self.b.numel() * 8 + len(methods) * self.xref.numel() * 8
        if self.sparse:
            self.h2d += self.rp.numel() * 8 + self.ci.numel() * 4
        self.d2h = len(methods) * self.B * self.n * 8

    def step(self):
        ils, t = self.ils, self.torch
        stream = t.cuda.current_stream().cuda_stream
        evs = [t.cuda.Event(enable_timing=True) for _ in range(len(self.methods) + 2)]
        evs[0].record()
        if self.sparse:
            h = ils.ils_create(self.A, self.b, self.pr.p, self.pr.q, self.n, stream=stream, row_ptr=self.rp,
                               col_idx=self.ci)
        elif self.batched:
            h = ils.ils_create(self.A, self.b, self.pr.p, self.pr.q, self.n, batch=self.B, stream=stream)
        else:
            h = ils.ils_create(self.A, self.b, self.pr.p, self.pr.q, self.n, stream=stream)
        evs[1].record()
        out = {}
        try:
            for i, m in enumerate(self.methods):
                o = ils.ils_default_opts(x_ref=self.xref.data_ptr(), inner_tol=self.itol, max_inner=1_000_000)
                fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve, "rgs": ils.ils_rgs_solve}[m]
                st, rep = fn(h, None, self.x[m], self.tol, 1000, o)
                evs[2 + i].record()
                out[m] = (st, rep.as_dict())
        finally:
            ils.ils_destroy(h)
        t.cuda.synchronize()
        create_ms = evs[0].elapsed_time(evs[1])
        per = {}
        prev = evs[1]
        for i, m in enumerate(self.methods):
            per[m] = dict(out[m][1], status=out[m][0], ms=prev.elapsed_time(evs[2 + i]))
            prev = evs[2 + i]
        total = evs[0].elapsed_time(evs[-1 if len(self.methods) else 1])
        return total, create_ms, per

    def errors(self):
        res = {}
        for m in self.methods:
            x = self.x[m].cpu().numpy().reshape(self.B, self.n)
            e = np.linalg.norm(x - self.xref_host, axis=1) / np.linalg.norm(self.xref_host, axis=1)
            res[m] = float(e.max())
        return res


def max_over_ranks(value: float, device) -> float:
    """Whole-job time = the slowest rank (contract: max over ranks). One all-reduce (MAX) of a
    scalar; a no-op for a single process. Works for nccl (cuda device) and gloo (cpu)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def flush_l2(buf):
    buf.add_(1)   # 256 MiB read+write > 126 MB L2


def summarise_methods(steps, cfg, pr, peak_hbm):
    """Per-method means over the timed steps (ms, counts, iters/s, algorithmic GB/s)."""
    out = {}
    for m in steps[0][2]:
        rows = [s[2][m] for s in steps]
        ms = statistics.mean(r["ms"] for r in rows)
        solve = statistics.mean(r["solve_ms"] for r in rows)
        setup = statistics.mean(r["setup_ms"] for r in rows)
        outer = rows[-1]["outer_iters"]
        inner = rows[-1]["inner_iters_total"]
        byt = rows[-1]["bytes_touched"]
        gbs = byt / (solve * 1e-3) / 1e9 if solve > 0 else None
        d = {"ms": round(ms, 4), "setup_ms": round(setup, 4), "solve_ms": round(solve, 4), "outer": outer,
             "inner": inner, "converged": bool(rows[-1]["converged"]), "final_metric": rows[-1]["final_metric"],
             "algorithmic_GBps": round(gbs, 2) if gbs else None,
             "frac_of_8TBps": round(gbs / HBM_NOMINAL_GBS, 5) if gbs else None,
             "frac_of_measured_hbm": round(gbs / peak_hbm, 5) if gbs else None,
             "kernel_launches": rows[-1]["kernel_launches"]}
        if m == "sp":
            d["outer_iters_per_s"] = round(outer / (solve * 1e-3), 1) if solve > 0 else None
        else:
            d["inner_steps_per_s"] = round(inner / (solve * 1e-3), 1) if solve > 0 else None
        out[m] = d
    return out


def roofline(steps, peak_hbm, peak_bf16, traffic_map, cfg):
    """Dominant kernel class by device time over the timed steps (CUDA events on the launching stream)."""
    ms = [0.0] * 4
    work = [0.0] * 4
    n = [0] * 4
    for s in steps:
        for m, r in s[2].items():
            for c in range(4):
                ms[c] += r["hot_ms"][c]
                work[c] += r["hot_work"][c]
                n[c] += r["hot_launches"][c]
    c = max(range(4), key=lambda i: ms[i])
    if ms[c] <= 0 or n[c] == 0:
        return None
    per_launch_ms = ms[c] / n[c]
    per_launch_work = work[c] / n[c]
    step_ms = sum(s[0] for s in steps)
    if c == 3:
        peak, note = peak_bf16 * FP64_OVER_BF16, "fp64 DMMA: measured bf16 burst x 40/2250 (nominal ratio)"
        try:   # a measured fp64 tensor peak on this pool (cuBLAS DGEMM), if recorded
            with open(os.path.join(ROOT, "profiles", "measured_fp64.json")) as f:
                m = json.load(f)
            if m.get("dgemm_tflops", 0) > peak:
                peak, note = float(m["dgemm_tflops"]), "fp64 DMMA: measured cuBLAS DGEMM on this pool (profiles/measured_fp64.json)"
        except (OSError, ValueError):
            pass
        ach = per_launch_work / (per_launch_ms * 1e-3) / 1e12
        d = {"bound": "tensor", "unit": "TFLOP/s", "peak_note": note}
    else:
        peak = peak_hbm
        ach = per_launch_work / (per_launch_ms * 1e-3) / 1e9
        d = {"bound": "hbm", "unit": "GB/s", "peak_note": "measured hbm_gbs (MEASURED_PEAKS.json)"}
    if c == 1:
        d["limiter"] = ("latency: one 16-CTA DSMEM all-to-all per 4 inner steps (~1000-1300 cycles floor, "
                        "tools/mb/dsmem_bench2.cu), two blocks deep in flight; per step the compute warps' "
                        "products -> recurrence -> axpy chain; the columns are L2-resident at c1 (DESIGN.md §7). "
                        "Per launch = one inner solve: algorithmic bytes 16p per step + 8n^2 per in-kernel check, "
                        "time = CUDA events around the launch (kernel time, no host gaps)")
    elif c == 2:
        d["limiter"] = "latency: one dependent A1bar row load plus a CTA argmax per inner step (DESIGN.md §7)"
    tr = traffic_map.get(f"{cfg}:{c}") if traffic_map else None
    tr_note = None
    if isinstance(tr, dict):
        tr_note = tr.get("note")
        tr = tr.get("dram_bytes_per_launch")
    d.update({"kernel": KINDS[c], "achieved": round(ach, 3), "peak": round(peak, 2), "frac": round(ach / peak, 5),
              "traffic": tr, "traffic_note": tr_note, "launches": n[c], "avg_launch_ms": round(per_launch_ms, 5),
              "algorithmic_per_launch": per_launch_work, "share_of_step": round(ms[c] / step_ms, 4)})
    return d


def validity(steps, errs, tol):
    """(valid, reason): every timed step of every method returned ILS_OK and the final iterates are
    within the config tolerance of x_ref; a capped (ILS_NOT_CONVERGED) run is not a time-to-tolerance."""
    bad = []
    for m in steps[0][2]:
        sts = sorted({int(s[2][m]["status"]) for s in steps})
        if sts != [0]:
            bad.append(f"{m}: status {sts}")
        if not (errs[m] <= tol):
            bad.append(f"{m}: rel err {errs[m]:.3e} > tol {tol:g}")
    return (not bad), "; ".join(bad) or None


def config_block(cfgs, torch, dev, peak_hbm, flushbuf, steps=3, warmup=2):
    """Compact results of the other BASELINE.json configs in the same run (same timing rules: inputs
    resident in HBM, L2 flushed between steps, CUDA events on the launching stream). For c2 the
    K1 + P stream of SP (`sp_persistent_kernel`, one launch for all outer steps) is reported against
    the measured HBM peak with the algorithmic bytes 8q(n+1) + 8n^2 per outer step;
    for c4 the batched methods' effective GB/s of A touched (on-chip served, not an HBM claim)."""
    out = {}
    for cfg in cfgs:
        t_gen = time.perf_counter()
        pr, xref = load_problem(cfg)
        gen_s = time.perf_counter() - t_gen
        methods = DEFAULT_METHODS[cfg].split(",")
        run = Runner(cfg, pr, xref, methods, torch, dev)
        for _ in range(warmup):
            flush_l2(flushbuf)
            run.step()
        sts = []
        for _ in range(steps):
            flush_l2(flushbuf)
            torch.cuda.synchronize()
            sts.append(run.step())
        errs = run.errors()
        per = summarise_methods(sts, cfg, pr, peak_hbm)
        ok, why = validity(sts, errs, pr.tol)
        blk = {"workload": workload_desc(cfg), "steps": steps, "ms": round(statistics.mean(x[0] for x in sts), 4),
               "valid": ok, "invalid_reason": why, "generate_s": round(gen_s, 1), "per_method": {}}
        for m, d in per.items():
            keep = {k: d[k] for k in ("ms", "setup_ms", "solve_ms", "outer", "inner", "converged",
                                      "algorithmic_GBps", "frac_of_measured_hbm") if k in d}
            keep["max_rel_err_vs_xref"] = errs[m]
            blk["per_method"][m] = keep
        if cfg == "c2" and "sp" in methods:
            ms = sum(x[2]["sp"]["hot_ms"][0] for x in sts)
            work = sum(x[2]["sp"]["hot_work"][0] for x in sts)
            if ms > 0:
                gbs = work / (ms * 1e-3) / 1e9
                o = sts[-1][2]["sp"]["outer_iters"]
                blk["k1p_stream"] = {
                    "kernel": "sp_persistent_kernel (K1 fused A2 stream + P apply, all outer steps in one launch)",
                    "GBps": round(gbs, 1), "frac_of_measured_hbm": round(gbs / peak_hbm, 4),
                    "frac_of_8TBps": round(gbs / HBM_NOMINAL_GBS, 4), "peak_hbm_gbs": peak_hbm,
                    "bytes_per_outer": 8.0 * pr.q * (pr.n + 1) + 8.0 * pr.n * pr.n, "outer": o,
                    "kernel_ms_per_solve": round(ms / len(sts), 4),
                    "note": "algorithmic bytes 8q(n+1) (A2 rows + b2) + 8n^2 (P) per outer step / kernel time "
                            "(CUDA events around the launch on the handle's stream); A2 + P = 450 MB per step, "
                            "far above the 126 MB L2"}
            try:
                with open(os.path.join(ROOT, "profiles", "c2_rho.json")) as f:
                    blk["rho_sp"] = json.load(f)
            except OSError:
                pass
        out[cfg] = blk
        del run
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------------------ oracle
def oracle_sample(cfg, pr, xref, counts, methods, budget_s=20.0):
    """CPU oracle (test infrastructure) on a bounded sample of the workload, extrapolated to the
    full time-to-tolerance with the iteration counts `counts` {method: (outer, inner_total)}.
    Returns (total_ms, per_method_ms, sample description, cores)."""
    from oracle import ils_oracle as O
    from oracle import index_stream as ix
    from threadpoolctl import threadpool_limits
    cores = 1   # the oracle is timed single-threaded (BLAS pinned to one thread, north_star)
    with threadpool_limits(limits=1):
        return _oracle_sample(O, ix, cfg, pr, xref, counts, methods, budget_s, cores)


def _oracle_sample(O, ix, cfg, pr, xref, counts, methods, budget_s, cores):
    if hasattr(pr, "scipy"):
        S = pr.scipy()
        A1, A2, b1, b2 = S[:pr.p], S[pr.p:], pr.b[:pr.p], pr.b[pr.p:]
        methods = [m for m in methods if m == "sp"]
    else:
        A1, A2, b1, b2 = pr.A1, pr.A2, pr.b1, pr.b2
    n = pr.n
    itol = inner_tol_for(pr.tol)
    per = {}
    notes = []
    t_all = time.perf_counter()
    for m in methods:
        outer, inner = counts[m]
        if m == "sp":
            t0 = time.perf_counter()
            O.sp_solve(A1, A2, b1, b2, tol=pr.tol, x_ref=xref, max_iter=max(outer, 1))
            per[m] = (time.perf_counter() - t0) * 1e3
            notes.append(f"sp: full oracle solve ({outer} outer)")
            continue
        t0 = time.perf_counter()
        A1T = np.ascontiguousarray(A1.T)
        N = ix.column_norms_sq(A1)
        _, S = ix.weights_prefix(N)
        G = A1.T @ A1 if m == "rgs" else None
        setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        bhat = O.sp_rhs(A1, A2, b1, b2, np.zeros(n))
        rhs = time.perf_counter() - t0
        T = int(min(max(inner, 1), 4 * n if m == "rk" else 2 * n))
        t0 = time.perf_counter()
        if m == "rk":
            O.rk_rgs_inner(A1T, N, S, bhat, 0, 0, T, n, 0.0)
        else:
            O.scd_inner(G, N, S, bhat, 0, 0, T, n, 0.0)
        per_step = (time.perf_counter() - t0) / T
        per[m] = (setup + outer * (rhs + 0.0) + inner * per_step) * 1e3
        notes.append(f"{m}: setup + {outer} x rhs + {inner} inner steps extrapolated from {T} timed oracle steps")
        if time.perf_counter() - t_all > budget_s:
            break
    return sum(per.values()), per, "; ".join(notes), cores


def oracle_counts(cfg, methods):
    """Iteration counts of the oracle's full solves (profiles/oracle_<cfg>_counts.json, written by
    tools/oracle_counts.py), used to extrapolate bounded oracle samples."""
    path = os.path.join(ROOT, "profiles", f"oracle_{cfg}_counts.json")
    with open(path) as f:
        d = json.load(f)
    return {m: (d[m]["outer"], d[m]["inner_total"]) for m in methods if m in d}


def run_reference(a, rank, world):
    if rank != 0:
        return
    cfg = a.config
    methods = a.methods.split(",")
    pr, xref = load_problem(cfg)
    if cfg == "c4":
        print(json.dumps({"impl": "reference", "unavailable": "oracle arm for the batched config is not wired"}))
        return
    try:
        counts = oracle_counts(cfg, methods)
    except FileNotFoundError:
        print(json.dumps({"impl": "reference", "unavailable": f"profiles/oracle_{cfg}_counts.json missing (tools/oracle_counts.py)"}))
        return
    for _ in range(a.warmup):
        oracle_sample(cfg, pr, xref, counts, methods, budget_s=5.0)
    vals, walls = [], []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        tot, per, note, cores = oracle_sample(cfg, pr, xref, counts, methods)
        walls.append((time.perf_counter() - t0) * 1e3)
        vals.append(tot)
    v = statistics.mean(vals)
    line = {"metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(v, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, methods, world),
            "per_method_ms": {m: round(x, 2) for m, x in per.items()},
            "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": note + f"; wall per sample step {statistics.mean(walls):.0f} ms"},
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--methods", default=None, help="default: per config (DEFAULT_METHODS)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--extra-configs", default="c0,c2,c3,c4",
                    help="other configs measured in the same run (compact block); '' to skip")
    a = ap.parse_args()
    if a.methods is None:
        a.methods = DEFAULT_METHODS[a.config]
    if a.warmup < 3:
        a.warmup = 3   # contract: W >= 3 warm-up steps
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product has no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2203_15340_b200 import ils
    ils.load_library()
    peak_hbm, peak_bf16, _, peak_src = load_peaks()
    cfg = a.config
    methods = a.methods.split(",")
    pr, xref = load_problem(cfg, rank, world)
    run = Runner(cfg, pr, xref, methods, torch, dev)
    flushbuf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        flush_l2(flushbuf)
        run.step()
    barrier()
    l0 = ils.ils_kernel_launch_count()
    steps = []
    with ClockSampler(local) as clk:
        for _ in range(a.steps):
            flush_l2(flushbuf)
            torch.cuda.synchronize()
            steps.append(run.step())
    barrier()
    launches = ils.ils_kernel_launch_count() - l0
    clocks = clk.summary()
    errs = run.errors()
    step_ms = statistics.mean(s[0] for s in steps)
    value = max_over_ranks(step_ms, dev)

    e2e = None
    if not a.no_e2e:
        hrun = Runner(cfg, pr, xref, methods, torch, dev, host=True)
        hrun.step()
        barrier()
        es = []
        for _ in range(a.steps):
            flush_l2(flushbuf)
            torch.cuda.synchronize()
            es.append(hrun.step()[0])
        barrier()
        ev = max_over_ranks(statistics.mean(es), dev)
        e2e = {"value": round(ev, 4), "unit": "ms", "h2d_bytes_per_step": hrun.h2d,
               "d2h_bytes_per_step": hrun.d2h}
        del hrun

    traffic_map = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic_map = json.load(f)
    per = summarise_methods(steps, cfg, pr, peak_hbm)
    for m in per:
        per[m]["max_rel_err_vs_xref"] = errs[m]
    valid, why = validity(steps, errs, pr.tol)
    extra = None
    if rank == 0 and world == 1 and a.extra_configs:
        del run
        torch.cuda.empty_cache()
        extra = config_block([c for c in a.extra_configs.split(",") if c and c != cfg], torch, dev, peak_hbm,
                             flushbuf)
    line = {"metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(value, 4), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, methods, world),
            "create_ms": round(statistics.mean(s[1] for s in steps), 4),
            "valid": valid, "invalid_reason": why,
            "per_method": per,
            "configs": extra,
            "roofline": roofline(steps, peak_hbm, peak_bf16, traffic_map, cfg),
            "peaks_source": peak_src,
            "gpu_launches": launches, "clocks": clocks, "e2e": e2e}
    if rank == 0 and world == 1 and not a.no_cpu_baseline and cfg != "c4":
        counts = {m: (per[m]["outer"], per[m]["inner"]) for m in methods}
        tot, pm, note, cores = oracle_sample(cfg, pr, xref, counts, methods)
        line["cpu_baseline"] = {"value": round(tot, 2), "unit": "ms", "cores": cores, "kind": "oracle",
                                "sample": note, "per_method_ms": {m: round(v, 1) for m, v in pm.items()}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
