#!/usr/bin/env python
"""Benchmark: distributed fp64 MatMult on a COO-assembled MPIAIJ matrix (arXiv 2406.08646).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One "step" is one MatMult y = A x through the C ABI (halo bcast_begin on the comm stream,
diagonal SpMV, bcast_end, off-diagonal SpMV-add).  The matrix is assembled once before the
timed region by spmat_create_coo + spmat_set_values_coo (the paper's one-time symbolic stage
amortised over repeated numeric stages and many MatMults); both are timed
separately and reported under "assembly".  Rank 0 prints ONE JSON line.

Default workload: C4 -- 3D 7-point Laplacian, 256^3 rows per GPU in z-slabs (weak scaling),
BASELINE.json configs[3], the 7-point Laplacian the north-star target is quoted on at
1/2/4/8 B200.  Inputs: 1.74 GB per GPU of val/col/rowptr/x/y >> 126 MB L2, so no flush is
needed between steps.  Timing: 5 trials of exactly K MatMults, each between a barrier and a
device synchronisation, CUDA events on the launching stream, max over ranks per trial, the
median trial reported.  cpu_baseline: the oracle's MatMult on the same
matrix on 1 core and on all host cores (median of 3).  --impl reference times the oracle on
all host cores (the reference arm for this tier) on the same matrix.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

KERNEL_NAMES = {1: "k_spmv_stream (diagonal-block SpMV)", 2: "k_spmv_vector (diagonal-block SpMV)",
                3: "k_spmv_tma (diagonal-block SpMV, bulk-copy staged)",
                4: "k_spmv_bsr3 (diagonal-block 3x3 block-CSR SpMV, bulk-copy staged)",
                5: "k_spmv_direct (diagonal-block SpMV, small-matrix direct loads)"}
METRIC = "MatMult GFLOP/s & HBM GB/s (% roofline), fp64, at 1/2/4/8 B200"
UNIT = "GFLOP/s"
FALLBACK_HBM = 6650.0
TRIALS = 5
NVLINK_GBPS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200, help="MatMults per timed trial (5 trials)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--values", default="real", choices=["real", "int"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch every MatMult from Python (no CUDA graph)")
    ap.add_argument("--kernel", default=None, help="SPMAT_SPMV_KERNEL override")
    ap.add_argument("--block-size", type=int, default=None,
                    help="spmat_set_block_size (default: 3 for the 3-dof config c5, else 1)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)", {}


# ------------------------------------------------------------------ clocks sampler (NVML)
class Clocks:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index):
        self.samples, self.mem, self.reasons = [], [], set()
        self.max_mhz = self.mem_max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.mem_max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_MEM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.mem.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for k, bit in self.REASONS.items():
            if r & bit and k != "gpu_idle":
                self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self._stop.wait(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()
            if not self.samples:
                self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "mem_mhz": statistics.median(self.mem), "mem_max_mhz": self.mem_max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "sample_period_ms": 2}


# ------------------------------------------------------------------ NVLink counters (NVML)
class NvLink:
    """Hardware NVLink byte counters of this GPU (NVML field values, summed over links): the
    bytes the halo actually put on the wire, read around the timed trials.  Tries the byte
    counters (NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES), then the throughput counters (KiB)."""
    FIELDS = (("count_bytes", 202, 204, 1), ("throughput_kib", 138, 139, 1024))

    def __init__(self, index):
        self.h, self.field = None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            for f in self.FIELDS:
                if self._read(f) is not None:
                    self.field = f
                    break
        except Exception:
            self.h = None

    def _read(self, f):
        tx = rx = 0
        ok = 0
        for link in range(18):
            try:
                a, b = self.nv.nvmlDeviceGetFieldValues(self.h, [(f[1], link), (f[2], link)])
                if a.nvmlReturn == 0 and b.nvmlReturn == 0:
                    tx += int(a.value.ullVal) * f[3]
                    rx += int(b.value.ullVal) * f[3]
                    ok += 1
            except Exception:
                return None
        return (tx, rx) if ok else None

    def read(self):
        return self._read(self.field) if self.field else None


# ------------------------------------------------------------------ byte / flop model
def byte_model(info, m, n, bs=1):
    """Algorithmic bytes per MatMult (int32 indices, fp64 values); with 3x3
    block-CSR one column index per 9 values and one row pointer per block row."""
    if bs == 3:
        diag = 8 * info["nnz_d"] + 4 * (info["nnz_d"] // 9) + 4 * (m // 3 + 1) + 8 * n + 8 * m
    else:
        diag = 12 * info["nnz_d"] + 4 * (m + 1) + 8 * n + 8 * m
    nro = info["n_offdiag_rows"]
    off = (12 * info["nnz_o"] + 4 * (nro + 1) + 4 * nro + 8 * info["n_ghost"] + 16 * nro
           if nro else 0)
    return diag, off


# ------------------------------------------------------------------ CPU oracle legs
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


MAX_ORACLE_ROWS = 1 << 25  # rows of the benchmarked matrix the oracle holds in host memory


def oracle_workload(cfg, P=1):
    """The matrix the oracle multiplies: the benchmarked matrix itself when the oracle can hold
    it -- row-sorted, duplicate-free COO (the stencil configs) goes through the direct CSR
    builder, SURVEY.md §8(d) -- else a bounded sample (element / node-block COO: the general
    tuple-sort assembly on a smaller grid).  Returns (csr, x, description, same_config)."""
    import oracle
    c = synth.CONFIGS[cfg]
    if c["kind"] in ("stencil", "box"):
        if c["kind"] == "stencil":
            shape = synth.config_shape(cfg, P)
            M = int(np.prod(shape))
            R = min(M, MAX_ORACLE_ROWS)
            i, j, v = synth.stencil_coo(shape, c["npts"], rows=(0, R), values="real")
        else:  # the one-box (P=1) matrix: natural lexicographic order
            i, j, v, sizes = synth.config_rank_coo(cfg, 1, 0, values="real")
            M = R = sizes[0]
        C = oracle.OracleCsr(R, M, i, j, v)
        del i, j, v
        x = synth.x_vector(0, M, "real").numpy()
        same = R == M and (c["kind"] == "stencil" or P == 1)
        desc = (f"the benchmarked matrix ({synth.CONFIG_TEXT[cfg]}, {M} rows)" if same else
                f"rows [0, {R}) of the {M}-row matrix of {cfg} at {P} GPUs")
        return C, x, desc + " via oracle.OracleCsr (direct CSR, oracle.c orc_csr_direct)", same
    if c["kind"] == "q1":
        n = 40
        i, j, v = synth.q1_coo(n, values="real")
        M = n ** 3
        desc = f"Q1 {n}^3 nodes (element COO, general oracle assembly) sample of {cfg}"
    else:
        n = 24
        i, j, v = synth.elasticity_coo(n, values="real")
        M = 3 * n ** 3
        desc = f"3-dof 27-pt {n}^3 nodes (general oracle assembly) sample of {cfg}"
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v])
    C = oracle.OracleCsr.from_oracle(O)
    x = synth.x_vector(0, M, "real").numpy()
    return C, x, desc, False


def time_oracle(C, x, nthreads, reps):
    """Median over reps of one oracle MatMult (orc_csr_mult: orc_mult's per-row loop, serial or
    over nthreads row slices; bit-identical either way, tests/test_oracle.py)."""
    y = np.zeros(C.M)
    C.mult(x, nthreads=nthreads, out=y)  # first touch
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        C.mult(x, nthreads=nthreads, out=y)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def run_oracle(cfg, P=1, reps=3):
    """cpu_baseline: the oracle on 1 core and on all host cores, median of
    `reps`, same byte/flop model as the GPU line."""
    C, x, desc, same = oracle_workload(cfg, P)
    nt = host_threads()
    t1 = time_oracle(C, x, 1, reps)
    tn = time_oracle(C, x, nt, reps) if nt > 1 else t1
    flops = 2 * C.nnz
    byts = 12 * C.nnz + 4 * (C.M + 1) + 8 * C.N + 8 * C.M
    return {"value": flops / tn / 1e9, "unit": UNIT, "cores": nt, "kind": "oracle",
            "value_1core": flops / t1 / 1e9, "value_all_cores": flops / tn / 1e9,
            "GBps_1core": byts / t1 / 1e9, "GBps_all_cores": byts / tn / 1e9,
            "ms_per_matmult_1core": t1 * 1e3, "ms_per_matmult_all_cores": tn * 1e3,
            "cpu_model": cpu_model(), "sched_getaffinity": nt, "reps": reps, "stat": "median",
            "same_config": same, "rows": C.M, "nnz": C.nnz,
            "sample": f"{desc}: {C.M} rows, {C.nnz} nnz; oracle/oracle.c orc_csr_mult "
                      f"(gcc -O2 -ffp-contract=off), 1 thread and {nt} threads (row slices)"}


def sdist_agree_launch(launch, max_over_ranks):
    """Every rank times the same way: graphs only if every rank captured one."""
    ok = 0.0 if launch == "cuda_graph" else 1.0
    return launch if max_over_ranks(ok) == 0.0 else ("eager" if launch == "cuda_graph" else launch)


# ------------------------------------------------------------------ shared line parts
def config_dict(cfg, P, values):
    """The workload as both arms name it (computed from the config alone, so the reference
    arm's line carries the identical dict)."""
    c = synth.CONFIGS[cfg]
    M = synth.config_rows(cfg, P)
    part = {"box": "box (cube) decomposition", "stencil": "z-slabs", "q1": "z-slabs",
            "elasticity": "z-slabs"}[c["kind"]]
    l2 = ("no flush: per-GPU inputs exceed the L2 (see roofline.l2_bytes)" if cfg != "c1" else
          "no flush: 0.3 MB latency case, L2-resident by design")
    return {"workload": synth.CONFIG_TEXT[cfg], "config_id": cfg, "rows_global": M,
            "rows_per_gpu": M // P, "partition": part, "values": values,
            "parallelism": f"row-partitioned MPIAIJ x{P}", "l2": l2}


def reference_line(a, cfg):
    """--impl reference: the oracle (the reference arm of this tier) on the host's cores, on
    the benchmarked matrix (or, past MAX_ORACLE_ROWS, its leading rows), K timed steps after W
    warm-up steps, each step one all-core oracle MatMult (bounded to ~2 minutes)."""
    C, x, desc, same = oracle_workload(cfg, a.gpus)
    nt = host_threads()
    y = np.zeros(C.M)
    for _ in range(max(a.warmup, 1)):
        C.mult(x, nthreads=nt, out=y)
    ts = []
    t_end = time.perf_counter() + 120
    for _ in range(a.steps):
        t0 = time.perf_counter()
        C.mult(x, nthreads=nt, out=y)
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    t = sum(ts) / len(ts)
    t1 = time_oracle(C, x, 1, 3)
    val = 2 * C.nnz / t / 1e9
    return {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": a.gpus, "steps": len(ts), "warmup": a.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True,
            "scaling": "weak" if synth.CONFIGS[cfg]["per_gpu"] else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, a.gpus, "real"),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": nt, "kind": "oracle",
                             "value_1core": 2 * C.nnz / t1 / 1e9, "value_all_cores": val,
                             "cpu_model": cpu_model(), "sched_getaffinity": nt,
                             "same_config": same, "rows": C.M, "nnz": C.nnz,
                             "sample": f"{desc}: {C.M} rows, {C.nnz} nnz; each step one oracle "
                                       f"MatMult on {nt} threads (oracle.c orc_csr_mult, row "
                                       f"slices); value_1core = median of 3 serial MatMults"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


# ------------------------------------------------------------------ main
_OUT = None


def emit(line):
    """The single JSON line goes to the real stdout; everything else printed by libraries
    (NCCL's version banner, warnings) was redirected to stderr in main()."""
    (_OUT or sys.stdout).write(json.dumps(line) + "\n")
    (_OUT or sys.stdout).flush()


def main():
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    cfg = a.config

    if a.impl == "reference":
        if rank != 0:
            return 0
        emit(reference_line(a, cfg))
        return 0

    if a.kernel:
        os.environ["SPMAT_SPMV_KERNEL"] = a.kernel
    import paper_2406_08646_b200 as sp
    torch.cuda.set_device(local)
    if P > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = sp.Comm(device=local, nranks=P, rank=rank)

    from paper_2406_08646_b200 import dist as sdist
    barrier, max_over_ranks = sdist.barrier, sdist.max_over_ranks

    # ---- inputs (seeded, synthetic, generated on the device)
    i, j, v, sizes = synth.config_rank_coo(cfg, P, rank, values=a.values, device="cuda")
    off = synth.offsets_from_sizes(sizes)
    M = off[-1]
    m = sizes[rank]
    ncoo = i.numel()
    stream = torch.cuda.current_stream()

    torch.cuda.empty_cache()  # hand the generator's temporaries back before libspmat allocates
    # ---- assembly (a1-a4 once, a3 repeated): timed separately
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = sp.Mat(comm, m, m, M, M, i, j)
    t_create = max_over_ranks(time.perf_counter() - t0)
    bs = a.block_size if a.block_size is not None else (3 if cfg == "c5" else 1)
    if bs != 1:
        A.set_block_size(bs)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    A.set_values(v)
    torch.cuda.synchronize()
    nsv = 5
    barrier()
    ev0.record()
    for _ in range(nsv):
        A.set_values(v)
    ev1.record()
    torch.cuda.synchronize()
    t_setvals = max_over_ranks(ev0.elapsed_time(ev1) / nsv / 1e3)
    del i, j
    torch.cuda.empty_cache()
    info = A.info()
    nnz_local = info["nnz_d"] + info["nnz_o"]
    n_contrib = info["n_contrib"]
    setv_bytes = 12 * n_contrib + (0 if n_contrib == nnz_local else 4 * (nnz_local + 1)) + 8 * nnz_local
    nnz_global = sdist.sum_over_ranks(nnz_local)

    x = synth.x_vector(off[rank], off[rank + 1], a.values, device="cuda")
    y = torch.empty(m, dtype=torch.float64, device="cuda")

    # ---- warm-up
    for _ in range(max(a.warmup, 3)):
        A.mult(x, y, stream)
    torch.cuda.synchronize()

    # ---- the K MatMults of a trial captured once as a CUDA graph (the launch-bound small
    # configs would otherwise measure Python's launch rate); NCCL-mode halos stay eager
    launch, graph = "eager", None
    if not a.eager and (P == 1 or A.halo_mode() == 2):
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=gs):
                for _ in range(a.steps):
                    A.mult(x, y, gs)
            stream.wait_stream(gs)
            for _ in range(2):
                graph.replay()
            y2 = torch.empty_like(y)
            A.mult(x, y2, stream)  # the replayed MatMult equals an eager one bit for bit
            torch.cuda.synchronize()
            launch = "cuda_graph" if torch.equal(y, y2) else "eager (graph result differs)"
            del y2
        except Exception as ex:  # capture refused: time eager launches instead
            graph, launch = None, f"eager (graph capture failed: {type(ex).__name__})"
            torch.cuda.synchronize()
    launch = sdist_agree_launch(launch, max_over_ranks)
    if not launch.startswith("cuda_graph"):
        graph = None

    # ---- timed region: TRIALS trials of exactly K MatMults each, barrier + sync on both sides
    # of every trial, max over ranks per trial, median over trials; then one
    # more trial of K MatMults with per-kernel CUDA events on the launching stream (in-library,
    # spmat_profile) for the roofline's kernel duration -- kept out of the headline trials,
    # where the extra event records would lengthen latency-bound steps (C1)
    clk = Clocks(local)
    nvl = NvLink(local) if P > 1 else None
    nvl0 = nvl.read() if nvl else None
    trials = []
    with clk:
        for _ in range(TRIALS):
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                for _ in range(a.steps):
                    A.mult(x, y, stream)
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier()
            trials.append(max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / a.steps))
        t_step = statistics.median(trials)
        nvl1 = nvl.read() if nvl else None
        A.profile(True)
        A.profile_read()  # clear
        barrier()
        torch.cuda.synchronize()
        for _ in range(a.steps):
            A.mult(x, y, stream)
        torch.cuda.synchronize()
        barrier()
        prof_ms, prof_n = A.profile_read()
        A.profile(False)
    t_diag = prof_ms[0] / max(prof_n[0], 1) / 1e3
    t_off = prof_ms[1] / max(prof_n[1], 1) / 1e3 if prof_n[1] else 0.0
    t_halo = prof_ms[2] / max(prof_n[2], 1) / 1e3 if prof_n[2] else 0.0

    # ---- isolated phases (diag only / halo only / offdiag only, the halo then both SpMVs with
    # no overlap, and the whole MatMult), launched like the headline trials (K calls captured
    # as one CUDA graph when those were), 3 interleaved rounds, median per phase: power and
    # clock drift over the run hits every phase alike
    phases = [("all", 7), ("diag", sp.PART_DIAG)]
    if P > 1:
        phases += [("halo", sp.PART_HALO), ("offdiag", sp.PART_OFFDIAG), ("sequential", None)]
    samples = {name: [] for name, _ in phases}
    kk = max(10, min(a.steps, 100))

    def phase_calls(part, st):
        for _ in range(kk):
            if part is None:
                A.mult_part(x, y, sp.PART_HALO, st)
                A.mult_part(x, y, sp.PART_DIAG | sp.PART_OFFDIAG, st)
            else:
                A.mult_part(x, y, part, st)

    phase_graphs = {}
    if graph is not None:
        try:
            for name, part in phases:
                gs = torch.cuda.Stream()
                gs.wait_stream(stream)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=gs):
                    phase_calls(part, gs)
                stream.wait_stream(gs)
                g.replay()
                phase_graphs[name] = g
            torch.cuda.synchronize()
        except Exception:
            phase_graphs = {}
            torch.cuda.synchronize()
    iso_launch = "cuda_graph" if len(phase_graphs) == len(phases) else "eager"
    iso_launch = sdist_agree_launch(iso_launch, max_over_ranks)
    for _round in range(3):
        for name, part in phases:
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            if iso_launch == "cuda_graph":
                phase_graphs[name].replay()
            else:
                phase_calls(part, stream)
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier()
            samples[name].append(max_over_ranks(ev0.elapsed_time(ev1) / kk))
    del phase_graphs
    iso = {name: statistics.median(v) for name, v in samples.items()}
    A.mult(x, y, stream)  # restore y = A x after the partial products
    torch.cuda.synchronize()
    overlap = None
    if P > 1 and min(iso["diag"], iso["halo"] + iso["offdiag"]) > 0:
        # share of the smaller side (diagonal SpMV vs halo + off-diagonal SpMV) hidden behind the
        # other, all phases timed the same way (eager, interleaved); above 1 when the fused
        # launch also saves the separate launches' fixed costs
        overlap = (iso["diag"] + iso["halo"] + iso["offdiag"] - iso["all"]) / \
            min(iso["diag"], iso["halo"] + iso["offdiag"])

    # ---- end to end through the public API with HOST buffers (pinned), copies inside
    e2e = None
    if not a.no_e2e:
        xh = x.cpu().pin_memory()
        yh = torch.empty(m, dtype=torch.float64).pin_memory()
        A.mult(xh, yh, stream)
        ke = max(3, min(a.steps, 50))
        # every step: H2D of its x from pinned host memory, MatMult, D2H of its y, enqueued
        # (spmat_mult_pipelined: step k+1's upload and SpMV overlap step k's download), all K
        # downloads waited for (flush) before the end event; y checked against the device result
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(ke):
            A.mult_pipelined(xh, yh, stream)
        A.flush(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        te = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / ke)
        e2e_ok = bool(torch.equal(yh, y.cpu()))
        # spmat_mult_async (the caller's stream waits for each download) for reference
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(ke):
            A.mult_async(xh, yh, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ta = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / ke)
        # the synchronous call (returns after y is on the host), for reference
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(ke):
            A.mult(xh, yh, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ts = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / ke)
        e2e = {"value": 2 * nnz_global / te / 1e9, "unit": UNIT, "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": 8 * m * P, "d2h_bytes_per_step": 8 * m * P, "steps": ke,
               "api": "spmat_mult_pipelined (pinned host x, y), flush + one sync after K steps",
               "y_equals_device_result": e2e_ok,
               "async_call_ms_per_step": ta * 1e3,
               "sync_call_value": 2 * nnz_global / ts / 1e9, "sync_call_ms_per_step": ts * 1e3}

    # ---- no NVLink wait timed out and no asynchronous CUDA/NCCL error (else the numbers are void)
    A.check()

    # ---- report
    diag_bytes, off_bytes = byte_model(info, m, m, bs)
    hinfo = sp.sf_get_info(A.halo_sf())
    halo_bytes = 8 * (hinfo["n_recv"] + hinfo["n_send"])
    hbm_peak, peak_src, peakd = peaks()
    # in-run pure-read reference: sum-reduce of 4 GB of doubles on this GPU
    read_ref = None
    try:
        buf = torch.ones(1 << 29, dtype=torch.float64, device="cuda")
        buf.sum()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record()
            buf.sum()
            r1.record()
            torch.cuda.synchronize()
            best = min(best, r0.elapsed_time(r1) / 1e3)
        read_ref = buf.numel() * 8 / best / 1e9
        del buf
        torch.cuda.empty_cache()
    except torch.OutOfMemoryError:
        pass
    # with the NVLink halo the off-diagonal add runs inside the same kernel (t_off == 0):
    # that kernel then moves the diagonal and the off-diagonal bytes
    fused = info["n_offdiag_rows"] > 0 and t_off == 0.0
    kernel_bytes = diag_bytes + (off_bytes if fused else 0)
    # our kernels per MatMult: the fused kernel alone (NVLink halo + off-diagonal items inside);
    # otherwise diag + off-diagonal (+ the SF pack/unpack kernels, or the standalone put) --
    # NCCL's own kernels are not counted
    halo_mode = A.halo_mode()
    if fused or P == 1:
        per_step_kernels = 1
    else:
        per_step_kernels = 1 + (1 if info["n_offdiag_rows"] > 0 else 0)
        if halo_mode == 1 and hinfo["packed"]:
            per_step_kernels += 1
        if halo_mode == 2:
            per_step_kernels += 1 if info["spmv_kernel_id"] != 3 else 0
    if info["spmv_kernel_id"] == 3 and info["max_row_nnz"] > 2560:
        per_step_kernels += 1  # k_spmv_long
    # the dominant kernel's duration: when a step is exactly one launch of it replayed from a
    # CUDA graph, the timed region's CUDA events / K ARE its average launch duration (no events
    # between kernels: those break the programmatic-dependent-launch overlap of consecutive
    # launches and add their drain/ramp to every launch); otherwise the in-library per-launch
    # events of the profiled trial
    if per_step_kernels == 1 and launch == "cuda_graph":
        t_kernel, dur_src = t_step, "timed region / K (one launch per step, CUDA-graph replay)"
    else:
        t_kernel, dur_src = t_diag, "in-library CUDA events around every launch (profiled trial)"
    achieved = kernel_bytes / t_kernel / 1e9 if t_kernel > 0 else None
    traffic = None  # from the committed ncu --set full capture (profiles/traffic.json), not this run
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tr = json.load(open(tp)).get(f"{cfg}_P{P}")
            traffic = tr.get("traffic_bytes_per_launch") if tr else None
        except Exception:
            traffic = None
    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size
    # halo against NVLink: bytes on the wire per direction (16-byte flagged lines
    # with the device-initiated transport, 8-byte values with NCCL) over the isolated halo time
    halo = None
    if P > 1:
        line_b = 16 if halo_mode == 2 else 8
        out_b = max_over_ranks(line_b * hinfo["n_send"])
        in_b = max_over_ranks(line_b * hinfo["n_recv"])
        th = iso.get("halo", 0.0) / 1e3
        halo = {"transport": {1: "nccl", 2: "nvlink-peer-stores"}.get(halo_mode, str(halo_mode)),
                "wire_bytes_out": out_b, "wire_bytes_in": in_b, "payload_bytes_out": out_b * 8 // line_b,
                "isolated_ms": th * 1e3, "nvlink_GBps_per_dir": NVLINK_GBPS,
                "halo_nvlink_frac": (max(out_b, in_b) / th / 1e9 / NVLINK_GBPS) if th > 0 else None,
                "note": "isolated halo = put kernel + wait for every ghost line + buffer release, "
                        "latency-bound at these sizes (0.5-2 MB)"}
        if nvl0 and nvl1:  # hardware counters over the TRIALS x K timed MatMults (this rank)
            ns = TRIALS * a.steps
            halo["nvml_counter"] = nvl.field[0]
            halo["nvml_tx_bytes_per_step"] = (nvl1[0] - nvl0[0]) / ns
            halo["nvml_rx_bytes_per_step"] = (nvl1[1] - nvl0[1]) / ns
    gflops = 2 * nnz_global / t_step / 1e9
    gbs_gpu = (diag_bytes + off_bytes) / t_step / 1e9
    line = {
        "metric": METRIC,
        "value": gflops,
        "unit": UNIT,
        "n_gpus": P,
        "steps": a.steps,
        "warmup": a.warmup,
        "trials": TRIALS,
        "launch": launch,
        "ms_per_step": t_step * 1e3,
        "trials_ms_per_step": [t * 1e3 for t in trials],
        "higher_is_better": True,
        "scaling": "weak" if synth.CONFIGS[cfg]["per_gpu"] else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(cfg, P, a.values),
        "nnz_global": nnz_global,
        "hbm_gbs_per_gpu": gbs_gpu,
        "pct_hbm_roofline": gbs_gpu / hbm_peak,
        "roofline": {"bound": "hbm", "kernel": KERNEL_NAMES.get(info["spmv_kernel_id"], "?"),
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak if achieved else None, "traffic": traffic,
                     "traffic_source": "profiles/traffic.json (committed ncu --set full capture)"
                                       if traffic else None,
                     "algorithmic_bytes_per_launch": kernel_bytes,
                     "avg_launch_ms": t_kernel * 1e3, "duration_source": dur_src,
                     "avg_launch_ms_profiled": t_diag * 1e3, "peak_source": peak_src,
                     "frac_of_spec_8000": achieved / 8000.0 if achieved else None,
                     "in_run_read_GBps": read_ref, "l2_bytes": l2_bytes,
                     "inputs_bytes_per_gpu": diag_bytes + off_bytes,
                     "inputs_exceed_l2": diag_bytes + off_bytes > l2_bytes},
        "phases_ms": {"diag_spmv": t_diag * 1e3, "offdiag_spmv": t_off * 1e3,
                      "halo_comm_stream": t_halo * 1e3, "halo_bytes": halo_bytes,
                      "isolated": iso, "isolated_launch": iso_launch, "overlap_efficiency": overlap},
        "halo": halo,
        "assembly": {"create_coo_s": t_create, "set_values_coo_ms": t_setvals * 1e3,
                     "coo_entries_per_rank": ncoo,
                     # compulsory bytes: v (8) and perm (4) per contribution, jmap (4 per nonzero;
                     # not read with one contribution per nonzero), the values written (8 per nonzero)
                     "set_values_bytes": setv_bytes,
                     "set_values_GBps": setv_bytes / t_setvals / 1e9,
                     "set_values_GBps_model_12_12": (12 * ncoo + 12 * nnz_local) / t_setvals / 1e9},
        "e2e": e2e,
        "gpu_launches": per_step_kernels * a.steps * TRIALS,
        "clocks": clk.summary(),
        "spmv_kernel_id": info["spmv_kernel_id"],
    }
    if rank == 0 and P == 1 and not a.no_cpu:
        try:
            line["cpu_baseline"] = run_oracle(cfg, 1)
        except Exception as ex:  # the CPU leg never decides the GPU number
            line["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        emit(line)
    A.close()
    comm.close()
    if P > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
