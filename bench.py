#!/usr/bin/env python
"""bench.py — benchmark of the B200 eigenvector–eigenvalue identity.

Headline workload (BASELINE.json metric "|v_ij|^2 components/sec + % FP64
peak; end-to-end n=4096 time at 1/2/4/8 GPUs"): config C4, the full
all_magnitudes pipeline (identity.cpp:294-316) on one n = 4096 GOE matrix
A = (G + G^T)/sqrt(2n) (random_symmetric(42, 4096).scaled(sqrt(2/4096))),
i.e. lambda(A) + 4096 minor spectra + the 4096^2 identity products.  Under
torchrun the minor index j is sharded over ranks (rank r owns rows
[r n/N, (r+1) n/N) of out[j*n+i]); lambda(A) is recomputed per rank and the
rows are all-gathered with NCCL (the path's only exchange).  Strong scaling.

At N = 1 the same JSON line also carries `configs`: C1, C2, C3 and C5
measured the same way (bounded step counts), each with its own e2e,
cpu_baseline and parity record.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C1|C2|C3|C4|C5] [--no-cpu-baseline] [--no-subconfigs]

Prints ONE JSON line on rank 0.  `value` is device-timed with CUDA events on
the library's stream (inputs resident in HBM), max over ranks; `e2e` goes
through the public API with host buffers (H2D of the inputs and D2H of
|v|^2 inside the timed region); `roofline` is the stage-1 band-reduction
kernel (the dominant launch) against the measured FP64 DMMA peak;
`cpu_baseline` times the oracle port on a bounded sample on this host and
`parity` compares the GPU's output with the reference's committed goldens
(tests/golden/reference_c{3,4}.npz, reference_golden.npz) or with the oracle
on the cpu_baseline's own sample.  --impl reference times the unmodified
reference (oracle/_ref, compiled from /root/reference/proj/src); its inputs
come from oracle/_ref and the oracle, so no product library is loaded there.
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
GOLDEN = os.path.join(ROOT, "tests", "golden")

P_FP64_MEASURED_TFLOPS = 37.09   # tools/fp64_peak.cu DMMA m8n8k4 on this pool
P_FP64_SOURCE = ("measured: tools/fp64_peak.cu, DMMA m8n8k4 f64 "
                 "(profiles/r01_fp64_peak.json, re-measured in round 2: 37.01 burst / "
                 "37.08 sustained at 1965 MHz, profiles/r02_fp64_peak.json; "
                 "MEASURED_PEAKS.json has no FP64 entry)")
METRIC = "|v_ij|^2 components/sec"
UNIT = "components/s"
SUB_STEPS = {"C1": 20, "C2": 10, "C3": 5, "C4": 2, "C5": 2}
C5_SEED = 5


def arm_watchdog(phase: str) -> None:
    """(Re)starts the hang watchdog for the next phase of the run and notes
    the phase on stderr, so a dump says what was running."""
    import faulthandler
    budget = float(os.environ.get("BENCH_WATCHDOG_S", "1500"))
    print(f"[bench] phase: {phase}", file=sys.stderr, flush=True)
    faulthandler.cancel_dump_traceback_later()
    faulthandler.dump_traceback_later(budget, exit=True)


# ----------------------------------------------------------------- inputs
def goe_matrix(n: int, seed: int = 42) -> np.ndarray:
    """random_symmetric(seed, n).scaled(sqrt(2/n)) — SURVEY §8 d4 (the
    reference's seeded generator, provided by the product library)."""
    from paper_2002_04989_b200 import random_symmetric
    return random_symmetric(seed, n) * math.sqrt(2.0 / n)


def c3_matrix(n: int = 1024, seed: int = 3) -> np.ndarray:
    """Q diag(linspace(-1,1)) Q^T (product host generator)."""
    from paper_2002_04989_b200 import c3_matrix as gen
    return gen(n, seed)


def f_tri(n: int, rows: int) -> float:
    """(4/3)[n^3 + rows (n-1)^3]: Householder flops of A and `rows` minors."""
    return 4.0 / 3.0 * (n ** 3 + rows * (n - 1) ** 3)


def f_id(n: int, rows: int) -> float:
    """4 n (n-1) per row: identity-stage flops (identity.cpp:68,70,209-210)."""
    return 4.0 * rows * n * (n - 1)


def f_chase(n: int, rows: int, b: int = 32) -> float:
    """Bulge chase, ~6 b m^2 flops per solve: m^2 / (2b) chase steps, each a
    length-b reflector applied from the right and left to a b x b block and
    two-sided to a b x b diagonal block (~12 b^2 flops)."""
    return 6.0 * b * (n ** 2 + rows * (n - 1) ** 2)


# ----------------------------------------------------------------- parity
def parity_record(g: np.ndarray, c: np.ndarray, checker: str, sample: str,
                  rel: float = 1e-9, abs_: float = 1e-12) -> dict:
    """SURVEY §8 d0 predicate |g - c| <= rel |c| + abs, plus max abs error and
    max relative error on entries >= 1e-3."""
    g = np.asarray(g, np.float64)
    c = np.asarray(c, np.float64)
    d = np.abs(g - c)
    big = np.abs(c) >= 1e-3
    return {"checker": checker, "sample": sample,
            "predicate": f"|g-c| <= {rel:g}|c| + {abs_:g}",
            "ok": bool(np.all(d <= rel * np.abs(c) + abs_)),
            "max_abs": float(d.max()) if d.size else 0.0,
            "max_rel_ge_1e-3": float((d[big] / np.abs(c[big])).max()) if big.any() else 0.0,
            "bit_exact_frac": float(np.mean(g.view(np.uint64) == c.view(np.uint64)))}


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
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


def _cores() -> int:
    return os.cpu_count() or 1


def _timed_reps(fn, budget_s: float, max_reps: int = 1000):
    """Runs fn() until budget_s of wall time is used (at least once)."""
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or reps >= max_reps:
            return reps, dt


# ----------------------------------------------------------------- CPU legs (oracle port)
def cpu_c1(a: np.ndarray, g: np.ndarray) -> dict:
    """Oracle port, full all_magnitudes n = 64 on all host threads."""
    from oracle.oracle import Oracle
    orc = Oracle()
    K = _cores()
    n = a.shape[0]
    reps, dt = _timed_reps(lambda: orc.all_magnitudes(a, threads=K), 2.0)
    c = orc.all_magnitudes(a, threads=K)
    return {"value": reps * n * n / dt, "unit": UNIT, "cores": K, "kind": "port",
            "sample": f"full: oracle all_magnitudes n={n}, {reps} repetitions, {K} threads",
            "parity": parity_record(g.reshape(n, n), c.reshape(n, n), "oracle port",
                                    "full 64x64")}


def cpu_c2(mats: np.ndarray, g: np.ndarray) -> dict:
    """Oracle port, all 4096 matrices (one single-thread oracle call per
    matrix, K threads) — the full config, a couple of seconds."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle
    orc = Oracle()
    K = _cores()
    t = time.perf_counter()
    with ThreadPoolExecutor(K) as ex:
        outs = list(ex.map(lambda m: orc.all_magnitudes(m, threads=1), mats))
    dt = time.perf_counter() - t
    c = np.stack(outs).reshape(g.shape)
    count, n = mats.shape[0], mats.shape[1]
    return {"value": count * n * n / dt, "unit": UNIT, "cores": K, "kind": "port",
            "sample": f"full: {count} x oracle all_magnitudes n={n} on {K} threads",
            "parity": parity_record(g, c, "oracle port", f"all {count} matrices")}


def cpu_c3(a: np.ndarray, lam_g: np.ndarray, mu_g: np.ndarray, g: np.ndarray) -> dict:
    """Oracle port on a sample of C3: eig(A), K concurrent minor solves and
    the identity for those K columns, extrapolated to n+1 solves and n
    columns; parity of the GPU's spectra and rows on that sample."""
    from oracle.oracle import Oracle
    orc = Oracle()
    K = _cores()
    n = a.shape[0]
    js = [int(j) for j in np.linspace(0, n - 1, K).round()]
    t = time.perf_counter()
    lam = orc.eigenvalues(a)
    t_eig = time.perf_counter() - t
    t = time.perf_counter()
    mu = orc.minor_spectra(a, js, threads=K)
    t_batch = time.perf_counter() - t
    t = time.perf_counter()
    rows = orc.identity_rows(lam, mu, threads=K)
    t_id = time.perf_counter() - t
    total = t_eig + math.ceil(n / K) * t_batch + (n / K) * t_id
    par = parity_record(g[js], rows, "oracle port", f"{K} rows j={js[0]}..{js[-1]}")
    par["max_abs_lambda"] = float(np.max(np.abs(lam_g - lam)))
    par["max_abs_mu"] = float(np.max(np.abs(mu_g[js] - mu)))
    return {"value": n * n / total, "unit": UNIT, "cores": K, "kind": "port",
            "sample": (f"oracle port: eig(A) + {K} concurrent minor solves + identity for "
                       f"those {K} columns ({t_eig + t_batch + t_id:.1f} s), extrapolated "
                       f"to n+1 solves and n columns"),
            "extrapolated_seconds": total, "parity": par}


def cpu_c4(n: int, a: np.ndarray, lam: np.ndarray, mu_rows: np.ndarray,
           budget_s: float = 12.0) -> dict:
    """Oracle port on a bounded sample of C4, extrapolated: the first S
    Householder steps (tred1, eigensolve.cpp:24-61) of K concurrent minors
    scaled by the exact per-step cost model sum (l+1)^2, plus the identity
    stage for K columns (identity.cpp:185-238)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle
    orc = Oracle()
    K = _cores()
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


def cpu_c5(lam: np.ndarray, mu_rows: np.ndarray, g_rows: np.ndarray, j0: int,
           budget_s: float = 10.0) -> dict:
    """Oracle port, identity only (cached spectra, evaluate() per component)
    on a bounded sample of components over K threads, extrapolated to n^2;
    each sampled component is compared with the GPU's bit for bit."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle
    orc = Oracle()
    K = _cores()
    n = lam.shape[0]
    rows = mu_rows.shape[0]
    rng = np.random.default_rng(0)

    def comps(count, seed):
        r = np.random.default_rng(seed)
        return list(zip(r.integers(0, rows, count), r.integers(0, n, count)))

    def work(batch):
        return [orc.evaluate(lam, mu_rows[r], int(i))[0] for r, i in batch]

    t = time.perf_counter()
    work(comps(4, 1))
    per = max((time.perf_counter() - t) / 4, 1e-6)
    m = max(4, int(budget_s / per))
    batches = [comps(m, 100 + k) for k in range(K)]
    t = time.perf_counter()
    with ThreadPoolExecutor(K) as ex:
        vals = list(ex.map(work, batches))
    dt = time.perf_counter() - t
    got = np.array([g_rows[r, i] for b in batches for r, i in b])
    want = np.array([v for vs in vals for v in vs])
    del rng
    return {"value": K * m / dt, "unit": UNIT, "cores": K, "kind": "port",
            "sample": (f"oracle port evaluate() on {K} x {m} random components of rows "
                       f"j={j0}..{j0 + rows - 1} (cached spectra), rate x n^2"),
            "parity": parity_record(got, want, "oracle port", f"{K * m} components",
                                    rel=1e-10, abs_=0.0)}


# ----------------------------------------------------------------- reference arm
def reference_arm(args, cfg_desc: dict) -> dict:
    """--impl reference: the unmodified reference (oracle/_ref) on this
    host's cores.  Inputs come from oracle/_ref (random_symmetric), the
    oracle (C3 / C5 generators) and the committed reference goldens, so no
    product library is loaded.  Each timed step is one real, bounded sample
    of the workload; `value` = components that sample produced / its time."""
    K = _cores()
    wl = args.config
    line = _reference_config(wl, args.steps, args.warmup, K)
    line.update({"metric": METRIC, "n_gpus": args.gpus, "steps": args.steps,
                 "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
                 "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                 "config": cfg_desc, "impl": "reference"})
    if not args.no_subconfigs and args.gpus == 1 and wl == "C4":
        line["configs"] = {}
        for c in ("C1", "C2", "C3", "C5"):
            sub = _reference_config(c, SUB_STEPS[c] if c != "C5" else 1, 1, K)
            sub["config"] = config_desc(c, 1)
            line["configs"][c] = sub
    return line


def _reference_config(wl: str, steps: int, warmup: int, K: int) -> dict:
    from oracle.oracle import Oracle, Reference
    ref = Reference()
    warm = ref.random_symmetric(1, 64)
    for _ in range(warmup):                   # cheap, untimed (no JIT on the CPU side)
        ref.all_magnitudes(warm, workers=K)
    times, units = [], 0
    if wl in ("C3", "C4"):
        n = 4096 if wl == "C4" else 1024
        if wl == "C4":
            a = ref.random_symmetric(42, n) * math.sqrt(2.0 / n)
            lam = np.load(os.path.join(GOLDEN, "reference_c4.npz"))["lam"]
        else:
            a = Oracle().c3_matrix(n, 3)
            lam = np.load(os.path.join(GOLDEN, "reference_c3.npz"))["lam"]
        for s in range(steps):
            js = [(j + s * K) % n for j in range(K)]
            t = time.perf_counter()
            mu = ref.minor_spectra(a, js, workers=K)
            ref.identity_rows(lam, mu, workers=K)
            times.append(time.perf_counter() - t)
            units += K * n
        sample = (f"per step: {K} concurrent reference minor solves (eigenvalues("
                  f"minor_matrix(j)) on the reference ThreadPool) + the reference "
                  f"identity for those {K} columns = {K}x{n} components; lambda(A) is "
                  f"the reference's own (committed golden), its one solve (1/{n + 1} of "
                  f"the solves) is not timed; warm-up: all_magnitudes n=64")
    elif wl in ("C1", "C2"):
        n = 64 if wl == "C1" else 32
        count = 1 if wl == "C1" else 4096
        mats = [ref.random_symmetric(1 if wl == "C1" else b, n) for b in range(count)]
        from concurrent.futures import ThreadPoolExecutor
        for _ in range(steps):
            t = time.perf_counter()
            if count == 1:
                ref.all_magnitudes(mats[0], workers=K)
            else:
                with ThreadPoolExecutor(K) as ex:
                    list(ex.map(lambda m_: ref.all_magnitudes(m_, workers=1), mats))
            times.append(time.perf_counter() - t)
            units += count * n * n
        sample = (f"full: {count} x reference all_magnitudes n={n}"
                  + (f" ({K} workers)" if count == 1 else
                     f" (1-worker engines on {K} threads)"))
    else:  # C5: identity only, sampled components
        n = 32768
        orc = Oracle()
        lam = orc.c5_lambda(C5_SEED, n)
        from concurrent.futures import ThreadPoolExecutor
        per_thread = 8000
        for s in range(steps):
            rows = list(range(s * K, (s + 1) * K))
            mu = orc.c5_mu_rows(C5_SEED, lam, rows)

            def work(r):
                rng = np.random.default_rng(1000 + r)
                for i in rng.integers(0, n, per_thread):
                    ref.component_magnitude_cached(lam, mu[r], int(i), rows[r])
            t = time.perf_counter()
            with ThreadPoolExecutor(K) as ex:
                list(ex.map(work, range(K)))
            times.append(time.perf_counter() - t)
            units += K * per_thread
        sample = (f"per step: {K} threads x {per_thread} reference component_magnitude "
                  f"calls with cached spectra (1-worker engines, SURVEY §3.4)")
    t_all = sum(times)
    value = units / t_all
    return {"value": value, "unit": UNIT, "ms_per_step": t_all / len(times) * 1e3,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": K, "kind": "reference",
                             "sample": sample},
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
    d["l2"] = ("C4/C5: working set > L2 (126 MB); C1-C3: inputs re-read from HBM each "
               "step, no L2 flush")
    return d


def our_config(args, dist: Dist, eng, wl: str, steps: int, warmup: int,
               cpu: bool) -> dict | None:
    import torch

    from paper_2002_04989_b200 import random_symmetric
    from paper_2002_04989_b200.engine import c5_lambda
    from paper_2002_04989_b200.shard import gather_rows, shard_range
    dev = eng.device
    stream = torch.cuda.ExternalStream(dev.stream(), device=f"cuda:{dist.local}")
    world, rank = dist.world, dist.rank
    cfg_desc = config_desc(wl, world)
    n = cfg_desc["n"]
    cuda = f"cuda:{dist.local}"
    state = {}

    # ---- inputs in HBM
    if wl in ("C1", "C3", "C4"):
        a_host = {"C1": lambda: random_symmetric(1, 64),
                  "C3": lambda: c3_matrix(1024), "C4": lambda: goe_matrix(4096)}[wl]()
        a_dev = torch.from_numpy(a_host).to(cuda)
        j0, j1 = shard_range(n, world, rank)
        rows = j1 - j0
        out_dev = torch.empty((rows, n), dtype=torch.float64, device=cuda)
        lam_dev = torch.empty(n, dtype=torch.float64, device=cuda)
        mu_dev = torch.empty((max(rows, 1), n - 1), dtype=torch.float64, device=cuda)
        units = n * n

        def step():
            eng.all_magnitudes_device(a_dev.data_ptr(), n, j0, j1, out_dev.data_ptr(),
                                      lam_dev.data_ptr(), mu_dev.data_ptr())
            if world > 1:
                if dist.backend == "nccl":
                    with torch.cuda.stream(stream):
                        state["full"] = gather_rows(out_dev, n, world, dist.pg)
                else:  # host collective (gloo): the rows travel through the CPU
                    stream.synchronize()
                    state["full"] = gather_rows(out_dev.cpu(), n, world, dist.pg)
        flops = f_tri(n, rows) + f_id(n, rows)
    elif wl == "C2":
        count = 4096
        b0, b1 = shard_range(count, world, rank)
        a_host = np.stack([random_symmetric(b, 32) for b in range(b0, b1)])
        a_dev = torch.from_numpy(a_host).to(cuda)
        out_dev = torch.empty((b1 - b0, 32 * 32), dtype=torch.float64, device=cuda)
        units = count * 32 * 32

        def step():
            eng.batched_device(a_dev.data_ptr(), b1 - b0, 32, out_dev.data_ptr())
        rows = n
        flops = (b1 - b0) * (f_tri(32, 32) + f_id(32, 32))
    else:  # C5
        lam_host = c5_lambda(C5_SEED, n)
        lam_dev = torch.from_numpy(lam_host).to(cuda)
        j0, j1 = shard_range(n, world, rank)
        rows = j1 - j0
        mu_dev = torch.empty((rows, n - 1), dtype=torch.float64, device=cuda)
        eng.c5_mu_device(C5_SEED, lam_dev.data_ptr(), n, j0, j1, mu_dev.data_ptr())
        out_dev = torch.empty((rows, n), dtype=torch.float64, device=cuda)
        units = n * n

        def step():
            eng.identity_device(lam_dev.data_ptr(), mu_dev.data_ptr(), n, j0, j1,
                                out_dev.data_ptr())
        flops = f_id(n, rows)

    # ---- warm-up, then K timed steps (device clock on the library stream)
    arm_watchdog(f"{wl}: warm-up and timed steps")
    for _ in range(warmup):
        step()
    eng.sync()
    large = wl in ("C3", "C4")
    dev.set_profiling(large)
    stage_runs = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = dev.launch_count()
    clocks.start()
    ev0.record(stream)
    for _ in range(steps):
        step()
        if large:   # stage events are on the library stream; read per call
            stage_runs.append(dev.stage_times())
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = dev.launch_count() - launches0
    dist.barrier()
    eng.sync()
    dev.set_profiling(False)
    t_total = dist.max(ev0.elapsed_time(ev1) / 1e3)
    value = units * steps / t_total
    ms_step = t_total / steps * 1e3

    # ---- end to end through the public API with host buffers
    arm_watchdog(f"{wl}: end to end")
    e2e = None
    e2e_steps = max(1, min(steps // 4, 5)) if wl == "C4" else max(1, min(steps // 2, 5))
    res = None
    if wl in ("C1", "C3", "C4"):
        if world == 1:
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.all_magnitudes(a_host)   # H2D A, pipeline, D2H |v|^2
            te = time.perf_counter() - t
            e2e = {"value": units * e2e_steps / te, "unit": UNIT, "steps": e2e_steps,
                   "h2d_bytes_per_step": a_host.nbytes,
                   "d2h_bytes_per_step": res.nbytes,
                   "api": "IdentityEngine.all_magnitudes (host numpy in, host numpy out)"}
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
                    out_pin.copy_(state["full"], non_blocking=True)
            if dist.backend != "nccl":
                torch.cuda.synchronize()
            e1.record(stream)
            e1.synchronize()
            te = dist.max(e0.elapsed_time(e1) / 1e3)
            e2e = {"value": units * e2e_steps / te, "unit": UNIT, "steps": e2e_steps,
                   "h2d_bytes_per_step": a_host.nbytes, "d2h_bytes_per_step": n * n * 8,
                   "api": "pinned H2D + all_magnitudes_device + NCCL all-gather + D2H"}
    elif wl == "C2":
        if world == 1:
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.all_magnitudes_batched(a_host)
            te = time.perf_counter() - t
            e2e = {"value": units * e2e_steps / te, "unit": UNIT, "steps": e2e_steps,
                   "h2d_bytes_per_step": a_host.nbytes, "d2h_bytes_per_step": res.nbytes,
                   "api": "IdentityEngine.all_magnitudes_batched"}
    else:
        if world == 1:
            mu_host = mu_dev.cpu().numpy()
            eng.identity(lam_host, mu_host)   # untimed: one-time pinned staging buffers
            t = time.perf_counter()
            for _ in range(e2e_steps):
                res = eng.identity(lam_host, mu_host)
            te = time.perf_counter() - t
            e2e = {"value": units * e2e_steps / te, "unit": UNIT, "steps": e2e_steps,
                   "h2d_bytes_per_step": lam_host.nbytes + mu_host.nbytes,
                   "d2h_bytes_per_step": res.nbytes,
                   "api": "IdentityEngine.identity (cached spectra, host buffers)"}

    # ---- roofline of the dominant kernel (+ the other stages)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg_desc,
            "matrices_per_sec": (1e3 / ms_step) * (4096 if wl == "C2" else 1),
            "fp64_frac_whole_step": flops * world / (ms_step / 1e3) / 1e12 / (
                P_FP64_MEASURED_TFLOPS * world),
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}
    if large:
        st = {k: statistics.mean(r[k] for r in stage_runs) for k in stage_runs[0]}
        t1 = st["stage1"] / 1e3
        achieved = f_tri(n, rows) / t1 / 1e12
        # DRAM bytes per solve of the stage-1 kernel at n = 4096 from one ncu
        # --set full capture (profiles/r02j_band_4096_widesp_raw_summary.csv:
        # 1.0028 TB read + 0.5993 TB written over the 146 solves of the captured launch), scaled to this
        # launch's solve count
        traffic = (1.002844e12 + 0.599308e12) / 146 * (rows + 1) if n == 4096 else None
        line["roofline"] = {
            "bound": "tensor", "kernel": "band_reduce_kernel (stage 1, dense->band, DMMA; widesp layout)",
            "achieved": achieved, "peak": P_FP64_MEASURED_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / P_FP64_MEASURED_TFLOPS, "traffic": traffic,
            "traffic_note": "ncu dram__bytes_read+write per solve x solves",
            "hbm_GBps": (traffic / t1 / 1e9) if traffic else None,
            "peak_source": P_FP64_SOURCE,
            "algorithmic": "F_tri = (4/3)[n^3 + rows (n-1)^3] flops per launch",
            "launch_ms": t1 * 1e3, "share_of_step": t1 * 1e3 / ms_step}
        line["stage_ms"] = st
        line["stages"] = {
            "stage2_bulge_chase": {"ms": st["stage2"], "TFLOP/s": f_chase(n, rows) /
                                   (st["stage2"] / 1e3) / 1e12,
                                   "algorithmic": "6 b m^2 per solve, b = 32"},
            "identity": {"ms": st["identity"], "TFLOP/s": f_id(n, rows) /
                         (st["identity"] / 1e3) / 1e12 if st["identity"] > 0 else None,
                         "algorithmic": "F_id = 4 n (n-1) per row"},
            "lambda_A_side_stream_ms": st["lambda_A"],
            "bisect_minors_ms": st["bisect_minors"]}
    else:
        achieved = flops / (ms_step / 1e3) / 1e12
        line["roofline"] = {
            "bound": "tensor",
            "kernel": "identity_kernel (whole step)" if wl == "C5" else "whole step",
            "achieved": achieved, "peak": P_FP64_MEASURED_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / P_FP64_MEASURED_TFLOPS, "traffic": None,
            "peak_source": P_FP64_SOURCE,
            "algorithmic": ("F_id = 4 n^2 (n-1) per step (2 DP ops per triple are issued "
                            "after hoisting the denominator: FP64-pipe share ~ frac/2)"
                            if wl == "C5" else "F_tri + F_id per step")}

    # ---- parity (golden fixtures) and CPU baseline (rank 0, N = 1 only)
    arm_watchdog(f"{wl}: parity and CPU baseline")
    if world == 1:
        g = out_dev.cpu().numpy()
        if wl == "C1":
            gold = np.load(os.path.join(GOLDEN, "reference_golden.npz"))
            line["parity"] = parity_record(g, gold["s1_n64_all64"], "reference golden",
                                           "full 64x64 (reference_golden.npz s1_n64)")
        elif wl in ("C3", "C4"):
            gold = np.load(os.path.join(GOLDEN, f"reference_{wl.lower()}.npz"))
            js = gold["js"]
            lam_g = lam_dev.cpu().numpy()
            mu_g = mu_dev.cpu().numpy()
            par = parity_record(g[js], gold["rows"], "reference golden (oracle/_ref)",
                                f"{len(js)} rows j in {list(map(int, js))}")
            par["max_abs_lambda"] = float(np.max(np.abs(lam_g - gold["lam"])))
            par["max_abs_mu_sampled"] = float(np.max(np.abs(mu_g[js] - gold["mu"])))
            line["parity"] = par
        if cpu and not args.no_cpu_baseline:
            if wl == "C1":
                line["cpu_baseline"] = cpu_c1(a_host, g)
            elif wl == "C2":
                line["cpu_baseline"] = cpu_c2(a_host, g)
                line["parity"] = line["cpu_baseline"].pop("parity")
            elif wl == "C3":
                line["cpu_baseline"] = cpu_c3(a_host, lam_dev.cpu().numpy(),
                                              mu_dev.cpu().numpy(), g)
                line["cpu_baseline"]["parity_vs_oracle"] = line["cpu_baseline"].pop("parity")
            elif wl == "C4":
                mu_h = mu_dev[: _cores()].cpu().numpy()
                line["cpu_baseline"] = cpu_c4(n, a_host, lam_dev.cpu().numpy(), mu_h)
            else:
                line["cpu_baseline"] = cpu_c5(lam_host, mu_dev[:64].cpu().numpy(), g[:64], 0)
                line["parity"] = line["cpu_baseline"].pop("parity")
    return line if rank == 0 else None


def our_arm(args, dist: Dist) -> dict | None:
    import torch

    from paper_2002_04989_b200 import IdentityConfig, IdentityEngine
    torch.cuda.set_device(dist.local)
    eng = IdentityEngine(IdentityConfig(), device=dist.local)
    line = our_config(args, dist, eng, args.config, args.steps, args.warmup, cpu=True)
    if line is not None and dist.world == 1 and args.config == "C4" and not args.no_subconfigs:
        line["configs"] = {}
        for c in ("C1", "C2", "C3", "C5"):
            sub = our_config(args, dist, eng, c, SUB_STEPS[c], 2, cpu=True)
            for k in ("metric", "unit", "n_gpus", "higher_is_better", "scaling",
                      "vs_baseline", "dtype", "data"):
                sub.pop(k, None)
            line["configs"][c] = sub
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4", "C5"], default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-subconfigs", action="store_true",
                    help="only the headline config (the N>1 runs never add them)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo lets several ranks share one GPU (flow testing only)")
    args = ap.parse_args()
    # Watchdog: a run that stops making progress dumps every thread's Python
    # stack to stderr and exits non-zero instead of blocking its caller.  It
    # is re-armed per timed phase through stage_note(); BENCH_WATCHDOG_S
    # overrides the per-phase budget (seconds).
    arm_watchdog("start")
    dist = Dist()
    if args.impl == "reference":
        if dist.rank != 0:
            return 0
        print(json.dumps(reference_arm(args, config_desc(args.config, dist.world))),
              flush=True)
        return 0
    dist.init(args.dist_backend)
    try:
        try:
            line = our_arm(args, dist)
        except Exception as e:  # noqa: BLE001
            # a bounded device-side wait ran out (the library reports it as a
            # DeviceError and the context stays usable): measure once more
            if "wait timed out" not in str(e):
                raise
            print(f"[bench] {e}; repeating the run once", file=sys.stderr, flush=True)
            line = our_arm(args, dist)
    finally:
        dist.close()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
