#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 eigenvector–eigenvalue identity.

Default workload (BASELINE.json metric "|v_ij|^2 components/sec + % FP64 peak;
end-to-end n=4096 time at 1/2/4/8 GPUs"): config C4, the full all_magnitudes
pipeline (identity.cpp:294-316) on one n = 4096 GOE matrix
A = (G + G^T)/sqrt(2n) (random_symmetric(42, 4096).scaled(sqrt(2/4096))),
i.e. lambda(A) + 4096 minor spectra + the 4096^2 identity products.  Under
torchrun the minor index j is sharded over ranks (rank r owns rows
[r n/N, (r+1) n/N) of out[j*n+i]); lambda(A) is recomputed per rank and the
rows are all-gathered with NCCL (the path's only exchange).  Strong scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C1|C2|C3|C4|C5] [--no-cpu-baseline]

Prints ONE JSON line on rank 0.  `value` is device-timed with CUDA events on
the library's stream (inputs resident in HBM), max over ranks; `e2e` goes
through the public API with host buffers (H2D of A and D2H of |v|^2 inside the
timed region); `roofline` is the stage-1 band-reduction kernel (the dominant
launch) against the measured FP64 DMMA peak; `cpu_baseline` times the oracle
port on a bounded sample on this host.  --impl reference times the unmodified
reference (oracle/_ref, compiled from /root/reference/proj/src) instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_FP64_MEASURED_TFLOPS = 37.09   # tools/fp64_peak.cu DMMA m8n8k4 on this pool
P_FP64_SOURCE = "measured: tools/fp64_peak.cu, DMMA m8n8k4 f64 (profiles/r01_fp64_peak.json)"
METRIC = "|v_ij|^2 components/sec"
UNIT = "components/s"


# ----------------------------------------------------------------- inputs
def goe_matrix(n: int, seed: int = 42) -> np.ndarray:
    """random_symmetric(seed, n).scaled(sqrt(2/n)) — SURVEY §8 d4 (the
    reference's seeded generator, provided by the product library)."""
    from paper_2002_04989_b200 import random_symmetric
    return random_symmetric(seed, n) * math.sqrt(2.0 / n)


def c3_matrix(n: int = 1024, seed: int = 3) -> np.ndarray:
    """A = Q diag(linspace(-1,1)) Q^T, Q from QR of a seeded Gaussian, sign-fixed
    by diag(R), then build(kSymmetrize)."""
    from paper_2002_04989_b200.engine import seeded_draws
    g = seeded_draws(seed, n * n).reshape(n, n)
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))[None, :]
    lam = -1.0 + 2.0 * np.arange(n) / (n - 1)
    a = (q * lam[None, :]) @ q.T
    iu = np.triu_indices(n, 1)
    mid = 0.5 * (a[iu] + a.T[iu])
    a[iu] = mid
    a.T[iu] = mid
    return np.ascontiguousarray(a)


def f_tri(n: int, rows: int) -> float:
    """(4/3)[n^3 + rows (n-1)^3]: Householder flops of A and `rows` minors."""
    return 4.0 / 3.0 * (n ** 3 + rows * (n - 1) ** 3)


def f_id(n: int, rows: int) -> float:
    """4 n (n-1) per row: identity-stage flops (identity.cpp:68,70,209-210)."""
    return 4.0 * rows * n * (n - 1)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- dist
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = "nccl"

    def init(self, backend: str):
        self.backend = backend
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            # one rank per GPU; with --dist-backend gloo several ranks may
            # share a GPU to exercise the multi-rank flow (host collectives)
            ndev = max(torch.cuda.device_count(), 1)
            self.local = self.local % ndev
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------- CPU legs
def cpu_baseline_c4(n: int, a: np.ndarray, lam: np.ndarray, mu_rows: np.ndarray,
                    budget_s: float = 12.0) -> dict:
    """Oracle port (oracle/oracle.c) on a bounded sample of C4, extrapolated:
    the first S Householder steps (tred1, eigensolve.cpp:24-61) of K
    concurrent minors scaled by the exact per-step cost model sum (l+1)^2,
    plus the identity stage for K columns (identity.cpp:185-238)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle
    orc = Oracle()
    K = os.cpu_count() or 1
    m = n - 1
    minors = [orc.minor(a, j) for j in range(K)]

    def run(steps):
        t = time.perf_counter()
        with ThreadPoolExecutor(K) as ex:
            list(ex.map(lambda mm: orc.tridiagonalize(mm, max_steps=steps), minors))
        return time.perf_counter() - t

    def frac(steps):  # sampled share of the tred1 step cost
        sizes = np.arange(1, m, dtype=np.float64)  # l+1 for steps i = m-1..1
        tot = float(np.sum(sizes ** 2))
        smp = float(np.sum(sizes[::-1][:steps] ** 2))
        return smp / tot

    steps = 16
    t = run(steps)
    if t < budget_s * 0.4:
        steps = int(min(m - 1, steps * budget_s * 0.6 / max(t, 1e-3)))
        t = run(steps)
    t_minor_batch = t / frac(steps)        # K full tridiagonalisations, concurrent
    t0 = time.perf_counter()
    orc.identity_rows(lam, mu_rows[:K], threads=K)
    t_id = time.perf_counter() - t0        # identity for K columns
    total = math.ceil((n + 1) / K) * t_minor_batch + (n / K) * t_id
    return {"value": n * n / total, "unit": UNIT, "cores": K, "kind": "port",
            "sample": (f"oracle port: first {steps} of {m - 1} tred1 steps of {K} "
                       f"concurrent {m}x{m} minors + identity for {K} columns; "
                       f"extrapolated to n+1 solves and n columns by the "
                       f"sum (l+1)^2 step-cost model (QL omitted: <1%)"),
            "extrapolated_seconds": total}


def reference_arm(args, cfg_desc: dict) -> dict:
    """--impl reference: the unmodified reference (oracle/_ref) on this host."""
    from oracle.oracle import Reference
    ref = Reference()
    K = os.cpu_count() or 1
    wl = args.config
    if wl in ("C4", "C3"):
        n = 4096 if wl == "C4" else 1024
        a = goe_matrix(n) if wl == "C4" else c3_matrix(n)
        if wl == "C3":
            # full reference pipeline
            for _ in range(args.warmup):
                ref.all_magnitudes(goe_matrix(64))
            times = []
            for _ in range(args.steps):
                t = time.perf_counter()
                ref.all_magnitudes(a, workers=K)
                times.append(time.perf_counter() - t)
            tmean = statistics.mean(times)
            value = n * n / tmean
            sample = f"full all_magnitudes n={n} on {K} workers"
        else:
            lam = np.linalg.eigvalsh(a)  # untimed input prep for the identity sample
            for _ in range(args.warmup):  # bounded warm-up: small full pipeline
                ref.all_magnitudes(goe_matrix(64))
            times = []
            js = list(range(K))
            for s in range(args.steps):
                jj = [(j + s * K) % n for j in js]
                t = time.perf_counter()
                mu = ref.minor_spectra(a, jj, workers=K)
                t_solve = time.perf_counter() - t
                t = time.perf_counter()
                ref.identity_rows(lam, mu, workers=K)
                t_id = time.perf_counter() - t
                times.append(math.ceil((n + 1) / K) * t_solve + (n / K) * t_id)
            tmean = statistics.mean(times)
            value = n * n / tmean
            sample = (f"per step: {K} concurrent reference minor solves "
                      f"(eigenvalues(minor_matrix(j)), ThreadPool of {K}) + reference "
                      f"identity for those {K} columns; extrapolated to n+1 solves and "
                      f"n columns (eig(A) counted at minor cost; warm-up steps run "
                      f"all_magnitudes at n=64)")
    elif wl in ("C1", "C2"):
        n = 64 if wl == "C1" else 32
        count = 1 if wl == "C1" else 4096
        from oracle.oracle import Oracle
        orc = Oracle()
        mats = [orc.random_symmetric(1 if wl == "C1" else b, n) for b in range(count)]
        from concurrent.futures import ThreadPoolExecutor
        for _ in range(args.warmup):
            ref.all_magnitudes(mats[0], workers=1)
        times = []
        for _ in range(args.steps):
            t = time.perf_counter()
            if count == 1:
                ref.all_magnitudes(mats[0], workers=K)
            else:
                with ThreadPoolExecutor(K) as ex:
                    list(ex.map(lambda m_: ref.all_magnitudes(m_, workers=1), mats))
            times.append(time.perf_counter() - t)
        tmean = statistics.mean(times)
        value = count * n * n / tmean
        sample = f"full: {count} x all_magnitudes n={n}"
    else:  # C5: identity only, sampled columns
        n = 32768
        from oracle.oracle import Oracle
        orc = Oracle()
        lam = orc.c5_lambda(5, n)
        times = []
        for s in range(args.steps):
            rows = list(range(s * K, (s + 1) * K))
            mu = orc.c5_mu_rows(5, lam, rows)
            t = time.perf_counter()
            ref.identity_rows(lam, mu, workers=K)
            times.append((time.perf_counter() - t) * n / K)
        tmean = statistics.mean(times)
        value = n * n / tmean
        sample = f"reference identity for {K} columns per step, x n/{K}"
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmean * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg_desc,
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": K,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------- our arm
def config_desc(wl: str, world: int) -> dict:
    d = {
        "C1": {"workload": "C1: n=64 random_symmetric(1,64), full pipeline", "n": 64},
        "C2": {"workload": "C2: 4096 x n=32 random_symmetric(b,32), full pipeline",
               "n": 32, "matrices": 4096},
        "C3": {"workload": "C3: n=1024 Q diag(linspace(-1,1)) Q^T, full pipeline", "n": 1024},
        "C4": {"workload": ("C4: n=4096 GOE (G+G^T)/sqrt(2n) seed 42, full pipeline "
                            "(lambda(A) + 4096 minor spectra + identity), minor index j "
                            "sharded over ranks + NCCL all-gather of rows"), "n": 4096},
        "C5": {"workload": ("C5: identity stage only, n=32768, synthetic interlacing "
                            "spectra (seed 5), rows sharded over ranks"), "n": 32768},
    }[wl]
    d = dict(d)
    d["parallelism"] = f"j-shard x{world}"
    d["l2"] = "inputs/working set larger than L2 (126 MB) for C4/C5; C1-C3 re-run from HBM"
    return d


def our_arm(args, dist: Dist, cfg_desc: dict) -> dict | None:
    import torch

    from paper_2002_04989_b200 import IdentityConfig, IdentityEngine
    from paper_2002_04989_b200.shard import gather_rows, shard_range
    torch.cuda.set_device(dist.local)
    eng = IdentityEngine(IdentityConfig(), device=dist.local)
    dev = eng.device
    stream = torch.cuda.ExternalStream(dev.stream(), device=f"cuda:{dist.local}")
    wl = args.config
    world, rank = dist.world, dist.rank
    n = cfg_desc["n"]

    # ---- inputs in HBM
    lam_host = mu_host = None
    from paper_2002_04989_b200 import random_symmetric
    from paper_2002_04989_b200.engine import c5_lambda
    if wl in ("C1", "C3", "C4"):
        a_host = {"C1": lambda: random_symmetric(1, 64),
                  "C3": lambda: c3_matrix(1024), "C4": lambda: goe_matrix(4096)}[wl]()
        a_dev = torch.from_numpy(a_host).to(f"cuda:{dist.local}")
        j0, j1 = shard_range(n, world, rank)
        rows = j1 - j0
        out_dev = torch.empty((rows, n), dtype=torch.float64, device=a_dev.device)
        lam_dev = torch.empty(n, dtype=torch.float64, device=a_dev.device)
        mu_dev = torch.empty((max(rows, 1), n - 1), dtype=torch.float64, device=a_dev.device)
        full = None
        units = n * n

        def step():
            nonlocal full
            eng.all_magnitudes_device(a_dev.data_ptr(), n, j0, j1, out_dev.data_ptr(),
                                      lam_dev.data_ptr(), mu_dev.data_ptr())
            if world > 1:
                if dist.backend == "nccl":
                    with torch.cuda.stream(stream):
                        full = gather_rows(out_dev, n, world, dist.pg)
                else:  # host collective (gloo): the rows travel through the CPU
                    stream.synchronize()
                    full = gather_rows(out_dev.cpu(), n, world, dist.pg)
        flops = f_tri(n, rows) + f_id(n, rows)
    elif wl == "C2":
        count = 4096
        b0, b1 = shard_range(count, world, rank)
        a_host = np.stack([random_symmetric(b, 32) for b in range(b0, b1)])
        a_dev = torch.from_numpy(a_host).to(f"cuda:{dist.local}")
        out_dev = torch.empty((b1 - b0, 32 * 32), dtype=torch.float64, device=a_dev.device)
        units = count * 32 * 32

        def step():
            eng.batched_device(a_dev.data_ptr(), b1 - b0, 32, out_dev.data_ptr())
        rows = n
        flops = (b1 - b0) * (f_tri(32, 32) + f_id(32, 32))
    else:  # C5
        lam_host = c5_lambda(5, n)
        lam_dev = torch.from_numpy(lam_host).to(f"cuda:{dist.local}")
        j0, j1 = shard_range(n, world, rank)
        rows = j1 - j0
        mu_dev = torch.empty((rows, n - 1), dtype=torch.float64, device=lam_dev.device)
        eng.c5_mu_device(5, lam_dev.data_ptr(), n, j0, j1, mu_dev.data_ptr())
        out_dev = torch.empty((rows, n), dtype=torch.float64, device=lam_dev.device)
        units = n * n

        def step():
            eng.identity_device(lam_dev.data_ptr(), mu_dev.data_ptr(), n, j0, j1,
                                out_dev.data_ptr())
        flops = f_id(n, rows)

    # ---- warm-up, then K timed steps (device clock on the library stream)
    for _ in range(args.warmup):
        step()
    eng.sync()
    dev.set_profiling(True)
    stage1_ms = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = dev.launch_count()
    clocks.start()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        if wl in ("C3", "C4"):
            stream.synchronize()
            stage1_ms.append(dev.stage_times()["stage1"])
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = dev.launch_count() - launches0
    dist.barrier()
    eng.sync()
    dev.set_profiling(False)
    t_total = dist.max(ev0.elapsed_time(ev1) / 1e3)
    value = units * args.steps / t_total
    ms_step = t_total / args.steps * 1e3

    # ---- end to end through the public API with host buffers
    e2e = None
    e2e_steps = max(1, args.steps // 2)
    if wl in ("C1", "C3", "C4"):
        if world == 1:
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.all_magnitudes(a_host)   # H2D A, pipeline, D2H |v|^2
            te = time.perf_counter() - t
            float(res[0])
            e2e = {"value": units * e2e_steps / te, "unit": UNIT,
                   "h2d_bytes_per_step": a_host.nbytes,
                   "d2h_bytes_per_step": res.nbytes + n * 8}
        else:
            pin = torch.from_numpy(a_host).pin_memory()
            out_pin = torch.empty((n, n), dtype=torch.float64).pin_memory()
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(e2e_steps):
                with torch.cuda.stream(stream):
                    a_dev.copy_(pin, non_blocking=True)
                step()
                with torch.cuda.stream(stream):
                    out_pin.copy_(full, non_blocking=True)
            if dist.backend != "nccl":
                torch.cuda.synchronize()
            e1.record(stream)
            e1.synchronize()
            te = dist.max(e0.elapsed_time(e1) / 1e3)
            e2e = {"value": units * e2e_steps / te, "unit": UNIT,
                   "h2d_bytes_per_step": a_host.nbytes, "d2h_bytes_per_step": n * n * 8}
    elif wl == "C2":
        if world == 1:
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.all_magnitudes_batched(a_host)
            te = time.perf_counter() - t
            e2e = {"value": units * e2e_steps / te, "unit": UNIT,
                   "h2d_bytes_per_step": a_host.nbytes, "d2h_bytes_per_step": res.nbytes}
    else:
        if world == 1:
            mu_host = mu_dev.cpu().numpy()
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.identity(lam_host, mu_host)
            te = time.perf_counter() - t
            e2e = {"value": units * e2e_steps / te, "unit": UNIT,
                   "h2d_bytes_per_step": lam_host.nbytes + mu_host.nbytes,
                   "d2h_bytes_per_step": res.nbytes}

    # ---- roofline of the dominant kernel
    if wl in ("C3", "C4"):
        t1 = statistics.mean(stage1_ms) / 1e3
        achieved = f_tri(n, rows) / t1 / 1e12
        # DRAM bytes per solve of the stage-1 kernel at n = 4096 from one ncu
        # --set full capture of 296 solves (profiles/
        # r01h_band_4096_wide_raw_summary.csv: 2.053 TB read + 1.231 TB
        # written), scaled to this launch's solve count
        traffic = (2.052512e12 + 1.230878e12) / 296 * (rows + 1) if n == 4096 else None
        roof = {"bound": "tensor", "kernel": "band_reduce_kernel (stage 1, dense->band, DMMA)",
                "achieved": achieved, "peak": P_FP64_MEASURED_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / P_FP64_MEASURED_TFLOPS, "traffic": traffic,
                "traffic_note": ("ncu dram__bytes_read+write per solve x solves; "
                                 "HBM rate = traffic / launch time"),
                "hbm_GBps": (traffic / t1 / 1e9) if traffic else None,
                "ceiling_note": ("cuBLAS DGEMM on the stage-1 update shapes reaches 18.9 "
                                 "(n=32 SYMM) / 20.3 (k=64 SYR2K) TFLOP/s on this B200 "
                                 "(profiles/r01_cublas_dgemm_ceilings.txt)"),
                "peak_source": P_FP64_SOURCE,
                "algorithmic": "F_tri = (4/3)[n^3 + rows (n-1)^3] flops per launch",
                "launch_ms": t1 * 1e3, "share_of_step": t1 * 1e3 / ms_step}
    else:
        achieved = flops / (ms_step / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "whole step", "achieved": achieved,
                "peak": P_FP64_MEASURED_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / P_FP64_MEASURED_TFLOPS, "traffic": None,
                "peak_source": P_FP64_SOURCE,
                "algorithmic": "F_tri + F_id (C2) or F_id = 4 n^2 (n-1) (C5) per step"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg_desc,
            "matrices_per_sec": (1e3 / ms_step) * (4096 if wl == "C2" else 1),
            "fp64_frac_whole_step": flops * world / (ms_step / 1e3) / 1e12 / (
                P_FP64_MEASURED_TFLOPS * world),
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "roofline": roof}
    if wl in ("C3", "C4"):
        line["stage_ms"] = dev.stage_times()

    # ---- CPU baseline (rank 0, N = 1 only)
    if world == 1 and not args.no_cpu_baseline and wl == "C4":
        lam_h = lam_dev.cpu().numpy()
        mu_h = mu_dev[: os.cpu_count() or 1].cpu().numpy()
        line["cpu_baseline"] = cpu_baseline_c4(n, a_host, lam_h, mu_h)
    elif world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = None
    return line if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4", "C5"], default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo lets several ranks share one GPU (flow testing only)")
    args = ap.parse_args()
    dist = Dist()
    cfg = config_desc(args.config, dist.world)
    if args.impl == "reference":
        if dist.rank != 0:
            return 0
        print(json.dumps(reference_arm(args, cfg)), flush=True)
        return 0
    dist.init(args.dist_backend)
    try:
        line = our_arm(args, dist, cfg)
    finally:
        dist.close()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
