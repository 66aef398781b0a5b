#!/usr/bin/env python
"""PB-SpGEMM benchmark (BASELINE.json metric: SpGEMM mults/sec + HBM GB/s as
a fraction of the memory roofline).

A *step* is one full C = A·A multiplication (symbolic + expand + sort/merge/
CSR) of the workload on device-resident inputs. Default workload: C2 (ER
n=2^20, d=16), the config BASELINE.json quotes its multiply count on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
    python bench.py --impl reference ...   # the reference's CPU path (oracle/_ref)

N>1 (torchrun), the path shards by output rows with no exchange step
(SURVEY.md §8e):
  --scaling strong (default): rank 0 builds A, broadcasts A (CSC) and B (CSR)
      once over NCCL at setup; every rank cuts the rows into N flop-balanced
      bands on its device (the balanced_starts rule; identical cuts, no
      exchange), builds its CSC row slab of A on the device, and each step
      multiplies that slab by all of B. Config 5 (C5a / C5b) is the scaling
      run of BASELINE.json; C2 at N=1 equals the BENCH line.
  --scaling weak: rank r multiplies its own C2-sized row block A_r (seed 1+r)
      by the shared B, so per-GPU work is fixed as N grows.
A band whose tuples exceed HBM runs as bounded-memory rounds (sub-bands cut
and sliced on the device inside every step). No collective runs in the timed
region; the step time is the max over ranks; afterwards an all-gather of the
band nnz places every band in the global CSR and an order-free checksum of C
is summed over ranks.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

M = None  # paper_2002_11302_b200.matrices, imported by the GPU arm only

FALLBACK_HBM_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def model_bytes(nnz_a, nnz_b, flop, nnz_c, b=16.0):
    """The reference's traffic model (roofline.hpp:56-63, report.hpp:42-51), b=16."""
    expand = b * (nnz_a + nnz_b + flop)
    sort = b * (flop + nnz_c)
    return expand, sort, expand + sort


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled around the timed region
    (B200_PROFILING.md clocks line). Started before warm-up so the first
    sample exists when timing begins; rows are time-stamped and the ones
    inside [start, stop] (plus the nearest on each side) are summarised."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def wait_first(self, timeout=5.0):
        t = time.time()
        while self.proc and not self.rows and time.time() - t < timeout:
            time.sleep(0.02)

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()
        time.sleep(0.12)  # one more sample after the region

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        rows = self.rows
        if self.t0 is not None and self.t1 is not None and rows:
            inside = [r for r in rows if self.t0 <= r[0] <= self.t1]
            before = [r for r in rows if r[0] < self.t0][-1:]
            after = [r for r in rows if r[0] > self.t1][:1]
            rows = before + inside + after
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[1][0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1][1]) for r in rows) if v is not None]
        pw = [v for v in (num(r[1][2]) for r in rows) if v is not None]
        reasons = sorted({self.NAMES[i] for _, r in rows for i in range(4)
                          if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "reasons": reasons,
                "samples": len(rows),
                "window_s": (self.t1 - self.t0) if self.t0 and self.t1 else None}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


MATRIX_PATH = None  # --matrix: a Matrix Market file squared instead of a config


def data_desc() -> str:
    if MATRIX_PATH:
        return f"Matrix Market file {Path(MATRIX_PATH).name}"
    return "synthetic (seeded, SURVEY.md §8d generators)"


def workload_name(cfg_name: str) -> str:
    if MATRIX_PATH:
        return f"matrix {Path(MATRIX_PATH).name}: C = A*A (mm_read, duplicates summed)"
    return f"{cfg_name}: {CONFIG_NAMES[cfg_name]}"


def build_inputs(cfg_name: str, seed: int = 1):
    """The config's matrix as (CSC, CSR): generated on the GPU when one is
    present (pbg_generate_begin, bit-identical to the host build), else on
    the host. With --matrix, the file's matrix (the reference bench's
    --matrix squaring path, spgemm_bench.cpp:55-58)."""
    t = time.time()
    if MATRIX_PATH:
        a_csr = M.matrix_from_mtx(MATRIX_PATH)
        log(f"[bench] {MATRIX_PATH}: {a_csr.nrows}x{a_csr.ncols} nnz={a_csr.nnz} read in "
            f"{time.time() - t:.1f}s")
        return M.csr_to_csc(a_csr), a_csr
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    if gpu:
        local = int(os.environ.get("PBG_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        a_csc, a_csr = M.make_config_gpu(cfg_name, seed, device=local)
    else:
        a_csc, a_csr = M.make_config(cfg_name, seed)
    log(f"[bench] {cfg_name}: n={a_csr.nrows} nnz={a_csr.nnz} inputs built in {time.time() - t:.1f}s")
    return a_csc, a_csr


# The configs: generator kind, scale, edge factor. Kept here so
# the reference arm needs nothing from the product package.
CONFIGS = {
    "C1": ("er", 16, 4), "C2": ("er", 20, 16), "C3": ("rmat", 20, 16),
    "C4": ("stencil", 128, None), "C5a": ("er", 24, 8), "C5b": ("rmat", 24, 8),
    "R16": ("rmat", 16, 16), "R18": ("rmat", 18, 16), "S64": ("stencil", 64, None),
    "E22": ("er", 22, 8),
}
CONFIG_NAMES = {
    "C1": "ER n=2^16 d=4, C=A*A, fp64 U[0,1)",
    "C2": "ER n=2^20 d=16, C=A*A, fp64 U[0,1)",
    "C3": "RMAT scale 20 ef 16 (a,b,c,d=.57,.19,.19,.05, dedup, no self-loops), C=A*A, fp64 U[0,1)",
    "C4": "27-point stencil 128^3 (26 / -1), C=A*A",
    "C5a": "ER n=2^24 d=8, C=A*A, fp64 U[0,1)",
    "C5b": "RMAT scale 24 ef 8 (dedup, no self-loops), C=A*A, fp64 U[0,1)",
    "R16": "dev: RMAT scale 16 ef 16, C=A*A",
    "R18": "dev: RMAT scale 18 ef 16, C=A*A",
    "S64": "dev: 27-point stencil 64^3, C=A*A",
    "E22": "dev: ER n=2^22 d=8, C=A*A",
}
VALUE_SEED_XOR = 0x5EED5EED5EED5EED
L2_NOTE = "inputs+tuples larger than L2 (tuples alone are 12 B x flop)"


def reference_config(cfg_name: str, seed: int = 1):
    """The config built by the reference library alone (oracle/_ref:
    gen_er / gen_rmat / coo_to_csc / coo_to_csr + the SplitMix64 values),
    pinned equal to the product's inputs by tests/test_oracle.py."""
    import oracle
    if MATRIX_PATH:
        return oracle.RefConfig("mtx", path=MATRIX_PATH)
    kind, scale, ef = CONFIGS[cfg_name]
    return oracle.RefConfig(kind, scale, ef or 0, seed, seed ^ VALUE_SEED_XOR)


def time_reference(rc, steps: int, warmup: int, budget_s: float, nthreads: int):
    """The reference's own pb_multiply (oracle/_ref: unmodified sources,
    OpenMP with nthreads) on the whole config, timed by its own PhaseReport
    t_total (bench.cpp:84-93,130-138 take the median of t_total). Only when
    (steps + warmup) full multiplies would exceed budget_s does each step
    run a flop-balanced leading row band instead (said in `sample`)."""
    # estimate the full step from a 1/16-flop band (fixed costs make this an
    # over-estimate, so a config that fits is never cut)
    frac = 1.0
    if rc.flop > 0:
        rc.band(1.0 / 16)
        t, _, _ = rc.multiply(nthreads)
        est = t[5] * 16
        if est * (steps + warmup) > budget_s:
            frac = max(1e-4, budget_s / (steps + warmup) / est)
    r1, band_flop = rc.band(frac)
    for _ in range(warmup):
        rc.multiply(nthreads)
    times, phases, nnz_c, flop = [], [], 0, 0
    for _ in range(steps):
        t, flop, nnz_c = rc.multiply(nthreads)
        times.append(float(t[5]))
        phases.append(t)
    med = statistics.median(times)
    full = r1 == rc.nrows
    sample = ((f"whole config (100%: {flop} of {rc.flop} mults)" if full else
               f"rows [0,{r1}) of {rc.nrows} ({band_flop} of {rc.flop} mults, "
               f"{100.0 * band_flop / max(rc.flop, 1):.1f}%: the whole config would exceed the "
               f"{budget_s:.0f} s budget)") +
              f", median PbResult.phases.t_total of {steps} after {warmup} warm-up")
    mid = phases[times.index(med)] if med in times else phases[len(phases) // 2]
    return {"value": flop / med if med > 0 else None, "unit": "mult/s", "cores": nthreads,
            "kind": "reference", "sample": sample, "seconds_per_step": med, "times": times,
            "full": full, "flop": flop, "nnz_c": nnz_c,
            "phases_s": dict(zip(("symbolic", "expand", "sort", "compress", "convert", "total"),
                                 (float(x) for x in mid)))}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_PROC_BIND", "close")
    nthreads = os.cpu_count() or 1
    t = time.time()
    rc = reference_config(args.config)
    log(f"[bench] {args.config}: n={rc.nrows} nnz={rc.nnz_a} flop={rc.flop} reference inputs "
        f"in {time.time() - t:.1f}s")
    res = time_reference(rc, args.steps, args.warmup, args.ref_budget, nthreads)
    peak, _ = peak_hbm()
    _, _, b_tot = model_bytes(rc.nnz_a, rc.nnz_b, res["flop"], res["nnz_c"])
    t_step = res["seconds_per_step"]
    line = {
        "metric": "SpGEMM mults/sec", "value": res["value"], "unit": "mult/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": data_desc(),
        "config": {"workload": workload_name(args.config), "n": rc.nrows, "nnz_a": rc.nnz_a,
                   "flop": res["flop"], "nnz_c": res["nnz_c"], "model_bytes": b_tot,
                   "model_GBps": b_tot / t_step / 1e9 if t_step else None,
                   "model_frac_of_peak_per_gpu": None, "l2": L2_NOTE,
                   "partition": "host CPU, OpenMP (rank 0 only)"},
        "impl": "reference",
        "same_config": res["full"],
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "mult/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "phases_s": res["phases_s"],
    }
    print(json.dumps(line), flush=True)
    rc.close()
    return 0


def host_ram_bytes() -> int:
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 0


def run_gpu_arm(args):
    global M
    import torch
    import torch.distributed as dist

    from paper_2002_11302_b200 import api
    from paper_2002_11302_b200 import matrices

    M = matrices
    ws, rank, local = dist_env()
    # test hooks: PBG_BENCH_DEVICE pins every rank to one device and
    # PBG_BENCH_BACKEND=gloo replaces NCCL, so the N>1 control flow can be
    # exercised on a single GPU (no kernel waits on another rank's kernel)
    local = int(os.environ.get("PBG_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("PBG_BENCH_BACKEND", "nccl")
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    weak = ws > 1 and args.scaling == "weak"
    bdev = dev if backend == "nccl" else torch.device("cpu")  # where collectives' tensors live

    def to_dev(x, dt):
        return torch.from_numpy(np.ascontiguousarray(x).view(dt)).to(dev)

    # ---- inputs (setup, untimed). strong (default): rank 0 builds A once and
    # broadcasts A (CSC, for the row slabs) and B (CSR) over NCCL; every rank
    # then cuts the rows into ws flop-balanced bands ON THE DEVICE (identical
    # cuts everywhere, no exchange) and takes band `rank`. weak: rank r
    # multiplies its own A_r (seed 1+r) by the shared B.
    n = k_a = k_b = 0
    if weak or ws == 1 or rank == 0:
        a_csc, a_csr = build_inputs(args.config, seed=1)
        n, k_a, k_b = a_csc.nrows, a_csc.nnz, a_csr.nnz
    if ws > 1 and not weak:
        meta = torch.tensor([n, k_a, a_csr.nnz] if rank == 0 else [0, 0, 0], dtype=torch.int64,
                            device=bdev)
        dist.broadcast(meta, 0)
        n, k_a, k_b = (int(x) for x in meta.tolist())
        if rank == 0:
            At = [to_dev(a_csc.colptr, np.int64), to_dev(a_csc.rowids, np.int32),
                  to_dev(a_csc.values, np.float64)]
            Bt = [to_dev(a_csr.rowptr, np.int64), to_dev(a_csr.colids, np.int32),
                  to_dev(a_csr.values, np.float64)]
        else:
            At = [torch.empty(n + 1, dtype=torch.int64, device=dev),
                  torch.empty(k_a, dtype=torch.int32, device=dev),
                  torch.empty(k_a, dtype=torch.float64, device=dev)]
            Bt = [torch.empty(n + 1, dtype=torch.int64, device=dev),
                  torch.empty(k_b, dtype=torch.int32, device=dev),
                  torch.empty(k_b, dtype=torch.float64, device=dev)]
        t0 = time.time()
        for t in At + Bt:  # NCCL broadcast over NVLink (gloo: through the host)
            if backend == "nccl":
                dist.broadcast(t, 0)
            else:
                h = t.cpu()
                dist.broadcast(h, 0)
                t.copy_(h)
        torch.cuda.synchronize()
        t_bcast = time.time() - t0
    else:
        if weak and rank > 0:
            a_csc = build_inputs(args.config, seed=1 + rank)[0]
        At = [to_dev(a_csc.colptr, np.int64), to_dev(a_csc.rowids, np.int32),
              to_dev(a_csc.values, np.float64)]
        Bt = [to_dev(a_csr.rowptr, np.int64), to_dev(a_csr.colids, np.int32),
              to_dev(a_csr.values, np.float64)]
        k_a, t_bcast = At[1].numel(), 0.0
    torch.cuda.synchronize()
    ctx = api.DeviceContext(local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    va = api.DeviceContext.view(n, n, *At)
    vb = api.DeviceContext.view(n, n, *Bt)
    if ws > 1 and not weak:
        cuts, _ = ctx.band_cuts(va, vb, ws, sp)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    else:
        r0, r1 = 0, n
    _, band_flop = ctx.band_cuts(va, vb, 1, sp, rows=(r0, r1))
    # bounded-memory rounds: a band whose tuples (+ C bound) exceed the HBM
    # budget runs as R flop-balanced sub-bands, cut and sliced on the device
    # inside every step (as the host path's rounds)
    free_b, _ = torch.cuda.mem_get_info(dev)
    budget = max(1, int(0.7 * (free_b - 2 * (k_b * 12 + k_a * 12))))
    per_tuple = 40  # tuples 12 + C bound 12 + heavy-row scratch 12 + grow-only headroom
    if args.max_round_tuples:
        rounds = max(1, -(-band_flop // args.max_round_tuples))
    else:
        rounds = max(1, -(-band_flop * per_tuple // budget))
    if rounds > 1:
        sub, _ = ctx.band_cuts(va, vb, rounds, sp, rows=(r0, r1))
        sub = [int(x) for x in sub]
        log(f"[bench] rank {rank}: rows [{r0},{r1}) in {rounds} bounded-memory rounds of "
            f"~{band_flop // rounds} mults")
        va_step, slab_keep = None, None
    elif (r0, r1) != (0, n):
        slab_keep, va_step = ctx.row_slab(va, r0, r1, sp)  # this rank's row slab of A
    else:
        slab_keep, va_step = None, va
    torch.cuda.synchronize()
    cfg = api.PbConfig(device=local)
    sums_keys = ("flop", "nnz_c", "t_symbolic", "t_expand", "t_sort", "t_total", "t_count",
                 "t_sortmerge_kernel", "tuples_into_sort", "merged_total")

    def one_step():
        """One multiply of this rank's rows (all its rounds); phase times summed."""
        if rounds == 1:
            _, rep = ctx.multiply(va_step, vb, cfg, sp)
            return dict(rep), ctx.launches()
        tot, launches = None, 0
        for q in range(rounds):
            if sub[q] == sub[q + 1]:
                continue
            _, rep = ctx.multiply_band(va, vb, sub[q], sub[q + 1], cfg, sp)
            launches += ctx.launches()
            if tot is None:
                tot = dict(rep)
            else:
                for key in sums_keys:
                    tot[key] += rep[key]
        return tot, launches

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    for _ in range(args.warmup):
        one_step()
    if sampler:
        sampler.wait_first()
        sampler.mark_start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    step_reps = []
    for _ in range(args.steps):
        rep, nl = one_step()
        launches += nl
        step_reps.append(rep)
    ev1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark_stop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    t_local = ev0.elapsed_time(ev1) * 1e-3 / max(args.steps, 1)

    flop_local = step_reps[-1]["flop"]
    nnz_local = step_reps[-1]["nnz_c"]
    # identity of this rank's product (single round: its C is still in the
    # context): nnz + order-free hashes, summed over ranks below
    ck = ctx.checksum(row_base=r0) if rounds == 1 else (nnz_local, 0, 0, 0.0)
    t_sort = statistics.mean(r["t_sortmerge_kernel"] for r in step_reps)
    t_count = statistics.mean(r["t_count"] for r in step_reps)
    t_exp = statistics.mean(r["t_expand"] for r in step_reps)
    t_sym = statistics.mean(r["t_symbolic"] for r in step_reps)
    stats = torch.tensor([t_local, t_sort, t_exp, t_sym, t_count], dtype=torch.float64, device=bdev)
    sums = torch.tensor([flop_local, nnz_local, slab_keep[1].numel() if slab_keep else k_a],
                        dtype=torch.float64, device=bdev)
    # 64-bit order-free hashes as 32-bit halves: int64 sums over ranks cannot overflow
    hashes = torch.tensor([ck[1] & 0xffffffff, ck[1] >> 32, ck[2] & 0xffffffff, ck[2] >> 32],
                          dtype=torch.int64, device=bdev)
    nnz_a_local = slab_keep[1].numel() if slab_keep else k_a
    all_t = None
    if ws > 1:
        # per-rank band times and nnz (the band-nnz exchange that places each
        # band in the global CSR: an all-gather of ws u64)
        g_t = [torch.zeros(1, dtype=torch.float64, device=bdev) for _ in range(ws)]
        dist.all_gather(g_t, torch.tensor([t_local], dtype=torch.float64, device=bdev))
        all_t = [float(x.item()) for x in g_t]
        g_n = [torch.zeros(1, dtype=torch.int64, device=bdev) for _ in range(ws)]
        dist.all_gather(g_n, torch.tensor([nnz_local], dtype=torch.int64, device=bdev))
        band_nnz = [int(x.item()) for x in g_n]
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(hashes, op=dist.ReduceOp.SUM)
    else:
        band_nnz = [nnz_local]
    t_step, t_sort_max, t_exp_max, t_sym_max, t_count_max = stats.tolist()
    flop, nnz_c, nnz_a = (int(x) for x in sums.tolist())

    # e2e through the public API with host buffers (pinned): H2D of this
    # rank's A rows and B, the multiply, D2H of its C rows, every step
    e2e = None
    c_bytes = nnz_local * 12 + (r1 - r0 + 1) * 8
    if args.e2e_steps > 0 and (nnz_local != band_nnz[rank] or c_bytes > 0.7 * host_ram_bytes()):
        e2e = {"value": None, "unit": "mult/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": f"skipped: C ({c_bytes / 1e9:.0f} GB) does not fit host memory; "
                       "checksum-and-discard mode"}
    elif args.e2e_steps > 0:
        if slab_keep is not None:
            a_band_cp = slab_keep[0].cpu().numpy().view(np.uint64)
            a_band = M.CscMatrix(r1 - r0, n, a_band_cp, slab_keep[1].cpu().numpy().view(np.uint32),
                                 slab_keep[2].cpu().numpy())
        elif (r0, r1) != (0, n):
            (cp, ri, vv), _ = ctx.row_slab(va, r0, r1, sp)
            a_band = M.CscMatrix(r1 - r0, n, cp.cpu().numpy().view(np.uint64),
                                 ri.cpu().numpy().view(np.uint32), vv.cpu().numpy())
        else:
            a_band = M.CscMatrix(n, n, At[0].cpu().numpy().view(np.uint64),
                                 At[1].cpu().numpy().view(np.uint32), At[2].cpu().numpy())
        b_host = M.CsrMatrix(n, n, Bt[0].cpu().numpy().view(np.uint64),
                             Bt[1].cpu().numpy().view(np.uint32), Bt[2].cpu().numpy())

        def pinned(x, tdt, dt):
            t = torch.empty(x.size, dtype=tdt, pin_memory=True)
            t.numpy().view(dt)[:] = x
            return t.numpy().view(dt)
        ah = M.CscMatrix(a_band.nrows, n, pinned(a_band.colptr, torch.int64, np.uint64),
                         pinned(a_band.rowids, torch.int32, np.uint32),
                         pinned(a_band.values, torch.float64, np.float64))
        bh = M.CsrMatrix(n, n, pinned(b_host.rowptr, torch.int64, np.uint64),
                         pinned(b_host.colids, torch.int32, np.uint32),
                         pinned(b_host.values, torch.float64, np.float64))
        out = (torch.empty(a_band.nrows + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
               torch.empty(max(nnz_local, 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
               torch.empty(max(nnz_local, 1), dtype=torch.float64, pin_memory=True).numpy())
        hcfg = api.PbConfig(device=local)
        api.pb_multiply(ah, bh, hcfg, symbolic=False, out=out)  # warm
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            res = api.pb_multiply(ah, bh, hcfg, symbolic=False, out=out)
        te = (time.perf_counter() - t0) / args.e2e_steps
        h2d = (ah.colptr.nbytes + ah.rowids.nbytes + ah.values.nbytes + bh.rowptr.nbytes +
               bh.colids.nbytes + bh.values.nbytes)
        d2h = (a_band.nrows + 1) * 8 + res.c.nnz * 12
        st = torch.tensor([te, h2d, d2h], dtype=torch.float64, device=bdev)
        if ws > 1:
            t_max = st[:1].clone()
            dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
            dist.all_reduce(st, op=dist.ReduceOp.SUM)
            st[0] = t_max[0]
        te, h2d, d2h = st.tolist()
        e2e = {"value": flop / te, "unit": "mult/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": te * 1e3,
               "rounds": int(res.report.get("nrounds", 1))}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    def hsum(i):  # recombine the summed halves of a 64-bit hash (mod 2^64)
        return (int(hashes[i].item()) + (int(hashes[i + 1].item()) << 32)) % (1 << 64)

    peak, peak_src = peak_hbm()
    b_exp, b_sort, b_tot = model_bytes(nnz_a, k_b, flop, nnz_c)
    # dominant kernel = the longer of expand and sort/merge (rank 0's own band);
    # the sort/merge phase includes the distinct-count pass that places its output
    my_b_exp, my_b_sort, _ = model_bytes(nnz_a_local, k_b, flop_local, nnz_local)
    t_sm_phase = t_sort + t_count
    kern = ("k_sortmerge", my_b_sort, t_sort) if t_sort >= t_exp else ("k_expand", my_b_exp, t_exp)
    achieved = kern[1] / kern[2] / 1e9
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{args.config}.json"
    if tf.exists():
        try:
            td = json.loads(tf.read_text())
            traffic = td.get(kern[0])
            traffic_src = td.get("source")
        except Exception:
            traffic, traffic_src = None, None
    roofline = {"bound": "hbm", "kernel": kern[0], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_src if traffic is not None else None,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": kern[1],
                "avg_launch_s": kern[2],
                "per_phase": {
                    "expand": {"model_bytes": my_b_exp, "s": t_exp,
                               "GBps": my_b_exp / t_exp / 1e9 if t_exp else None,
                               "frac": my_b_exp / t_exp / 1e9 / peak if t_exp else None},
                    "sort_merge": {"model_bytes": my_b_sort, "s": t_sm_phase,
                                   "includes": "k_bincount (distinct count + offsets) + k_sortmerge",
                                   "GBps": my_b_sort / t_sm_phase / 1e9 if t_sm_phase else None,
                                   "frac": my_b_sort / t_sm_phase / 1e9 / peak if t_sm_phase else None},
                    "sortmerge_kernel_alone": {"s": t_sort,
                                               "frac": my_b_sort / t_sort / 1e9 / peak if t_sort else None},
                    "symbolic_s": t_sym, "bin_count_s": t_count}}
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            rcfg = reference_config(args.config)
            res_c = time_reference(rcfg, 3, 1, args.cpu_budget, os.cpu_count() or 1)
            rcfg.close()
            cpu = {k: res_c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the baseline is reported, not required
            cpu = {"value": None, "unit": "mult/s", "cores": 0, "kind": "reference",
                   "sample": f"failed: {e}"}
    partition = ((f"weak: rank r multiplies its own {args.config}-sized row block A_r (seed 1+r) "
                  f"of the row-stacked A by the shared B" if weak else
                  f"strong: {ws} flop-balanced row bands (cut on the device), A and B broadcast "
                  f"once over {backend} at setup ({t_bcast:.2f} s)")
                 if ws > 1 else "single GPU")
    if rounds > 1:
        partition += f", {rounds} bounded-memory rounds per rank (device-side cuts and slabs)"
    line = {
        "metric": "SpGEMM mults/sec", "value": flop / t_step, "unit": "mult/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64",
        "data": data_desc(),
        "config": {"workload": workload_name(args.config),
                   "n": n, "nnz_a": nnz_a, "flop": flop, "nnz_c": nnz_c,
                   "model_bytes": b_tot, "model_GBps": b_tot / t_step / 1e9,
                   "model_frac_of_peak_per_gpu": b_tot / t_step / 1e9 / (peak * ws),
                   "l2": L2_NOTE, "partition": partition},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "phases_ms": {"symbolic": t_sym_max * 1e3, "expand": t_exp_max * 1e3,
                      "bin_count": t_count_max * 1e3, "sort_merge": t_sort_max * 1e3},
        "c_checksum": {"nnz": nnz_c, "row_hash": hsum(0), "rowcol_hash": hsum(2)}
        if rounds == 1 else None,
    }
    if ws > 1:
        line["per_rank_ms"] = [t * 1e3 for t in all_t]
        line["band_nnz"] = band_nnz
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--matrix", default=None,
                    help="Matrix Market file: square it (C = A*A) instead of a synthetic config")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--ref-budget", type=float, default=240.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: total work fixed, flop-balanced row bands of one A with A and B "
                         "broadcast once (strong, default: SURVEY.md §8e) or per-GPU work fixed "
                         "(weak, opt-in)")
    ap.add_argument("--max-round-tuples", type=int, default=0,
                    help="force bounded-memory rounds of at most this many mults")
    args = ap.parse_args()
    if args.matrix:
        global MATRIX_PATH
        MATRIX_PATH = args.matrix
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
