#!/usr/bin/env python
"""bench.py -- B200 benchmark of the Gray-code Ryser/Glynn permanent (arXiv 1904.06229).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

N > 1 is launched by the driver as `torchrun --nproc-per-node N ... bench.py --gpus N ...` (one rank per
GPU, NCCL).  Rank 0 prints ONE JSON line.

Workloads (BASELINE.json configs; synthetic inputs from paper_1904_06229_b200/inputs.py):
  cfg5 (default): one 44x44 complex Gaussian matrix, 2^43 Gray terms, range-sharded over the N GPUs with
                  one NCCL all-gather of the double-double partials -- the metric's headline case.
  cfg4: 32x32 block of a 1024x1024 Haar unitary, 2^31 terms, range-sharded.
  cfg1: one 16x16 complex Gaussian (latency-bound).
  cfg2: 10^5 submatrices of an n^2 x n^2 Haar unitary for each n in {8,12,16,20}; batched perms/s.
  cfg3: 64 Bernoulli 0-1 matrices of order 24; exact int128; perms/s.
  cfg3s: one 0-1 matrix of order 33, exact int128 via 2^33 Eq. (3) terms, rank space sharded; terms/s.
  cfgbd: 10^4 band matrices, n = 100, k = 5, App. C transfer method (NEXT-4); perms/s.
  cfgsp: one sparse 48x48 complex matrix (4% + a matching), App. B restricted enumeration (NEXT-3); sets/s.
  cfgpm: 1024 Bernoulli +-1 matrices of order 24 (Sec. V ensemble); exact; perms/s.
  cfgens: 10^4 Ginibre + 10^4 circular matrices of order 24 (Secs. III-IV ensembles; NEXT-2), X = |per|/sqrt(n!)
          streamed per matrix; perms/s and the sample moments of X.
  cfgw: 10^4 Boson-sampling output patterns with collisions (20 photons, 20 modes), weighted Ryser
        Eq. (4) (not a BASELINE config); perms/s.

A step is one pass of the whole hot path over the config's input: walk + in-GPU reduction + (N > 1)
the all-gather + ordered combine.  `value` is timed with CUDA events on the compute stream from the
first kernel to the end of the collective (inputs already in HBM); `e2e` times the same steps through
the public API from pinned host input to the host result (H2D and D2H inside).  The roofline object
uses the walk kernel's own duration, taken with CUDA events that the library records around that
launch.  `--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
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

METRIC = "Gray-code terms/sec and % FP64 peak at n=44 on 1/2/4/8 B200; batched perms/sec"
SMS_NOMINAL = 148
FP64_LANES_PER_SM = 64           # FP64 FMA units per SM (B200)
SM_MAX_MHZ = 1965.0


def fp64_nominal_tflops(sm_mhz: float = SM_MAX_MHZ, sms: int = SMS_NOMINAL) -> float:
    return sms * FP64_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12


INT_LANES_PER_SM = 128           # 4 SMSPs x (16-lane fma pipe + 16-lane alu pipe) = 1 warp-instr/clk/SMSP


def int_nominal_tops(sm_mhz: float = SM_MAX_MHZ, sms: int = SMS_NOMINAL) -> float:
    """Integer-op peak (T ops/s): every SMSP issues one 32-lane integer instruction per clock, split
    over the fma pipe (IMAD) and the alu pipe (IADD3/LOP3), each 16 lanes wide (B300_MICROARCH
    "Pipe rates": rt_SMSP = 2 for both)."""
    return sms * INT_LANES_PER_SM * sm_mhz * 1e6 / 1e12


def ncu_traffic(cfg: str):
    """DRAM bytes (read + write) per launch of the config's dominant kernel from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f).get(cfg)
        return None if t is None else float(t["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


# ------------------------------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING recipe's clocks line).

    NVML in-process (pynvml) every 2 ms, so that even a timed region of a few tens of milliseconds carries
    samples; `nvidia-smi -lms 200` as the fallback when NVML is unavailable."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    # NVML clocks-event reason bits
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                   "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int, period_s: float = float(os.environ.get("PERM_BENCH_CLOCK_MS", "2")) * 1e-3):
        self.gpu = gpu_index
        self.period = period_s
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []    # (sm MHz, max sm MHz, reason bits)
        self.thread = None
        self.stop = threading.Event()
        self.source = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while True:
                    try:
                        self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), mx,
                                             int(reasons(h))))
                    except pynvml.NVMLError:
                        pass
                    if self.stop.wait(self.period):
                        break

            self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), mx, int(reasons(h))))
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi below
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            self.source = "nvidia-smi"
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.source == "nvml":
            self.stop.set()
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        if self.source == "nvml":
            for f, m, bits in list(self.samples):
                sm.append(f)
                mx.append(m)
                reasons.update(nm for nm, b in self.REASON_BITS.items() if bits & b)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------------------------------ helpers

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def flush_l2(buf):
    buf.fill_(1)   # 256 MiB write > 126 MB L2


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure_fp64_peak(pb, torch) -> float:
    """Live FP64 DFMA probe: TFLOP/s of independent DFMA chains on all SMs."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.empty(sms * 8 * 256, dtype=torch.float64, device="cuda")
    iters = 20000
    pb.perm_fp64_probe(sms * 8, 256, 100, sink)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        s.record()
        pb.perm_fp64_probe(sms * 8, 256, iters, sink)
        e.record()
        torch.cuda.synchronize()
        best = max(best, sms * 8 * 256 * iters * 64 / (s.elapsed_time(e) * 1e-3) / 1e12)
    return best


# ------------------------------------------------------------------------------------------ CPU oracle

def oracle_rate_cfg(cfg: str, seconds: float = 12.0) -> dict:
    """Time the CPU oracle (oracle/, as it stands) on a bounded sample of the workload.  Returns the
    rate in the workload's metric unit and a description of the sample."""
    import oracle
    from paper_1904_06229_b200 import inputs
    cores = oracle.num_threads()
    if cfg in ("cfg5", "cfg4", "cfg1"):
        A = {"cfg5": inputs.cfg5, "cfg4": inputs.cfg4, "cfg1": inputs.cfg1}[cfg]()
        n = A.shape[0]
        total = 1 << (n - 1)
        span = min(total, 1 << 14)
        while True:
            t0 = time.perf_counter()
            oracle.subpermanent(A, total // 3, min(span, total - total // 3) if total > 1 else 1,
                                parts=4 * cores)
            dt = time.perf_counter() - t0
            if dt > seconds / 8 or span >= total:
                break
            span = min(total, span * 4)
        if dt < seconds / 2 and span < total:
            span = min(total, int(span * seconds / max(dt, 1e-3)))
            t0 = time.perf_counter()
            oracle.subpermanent(A, 0, span, parts=4 * cores)
            dt = time.perf_counter() - t0
        # 1-core rate: the serial App. A subpermanent (parts = 1) on a proportionally smaller span
        span1 = max(1, min(total, int(span / cores / 3)))
        t0 = time.perf_counter()
        oracle.subpermanent(A, 0, span1, parts=1)
        dt1 = time.perf_counter() - t0
        return {"value": span / dt, "unit": "terms/s", "cores": cores, "kind": "oracle",
                "value_1core": span1 / dt1,
                "sample": f"App. A subpermanent (binary128) over {span} of the {total} Gray ranks of the {cfg} "
                          f"matrix, {dt:.1f} s on {cores} host threads (1 core: {span1} ranks in {dt1:.1f} s); "
                          f"rate extrapolates linearly"}
    if cfg == "cfg2":
        rates, parts = [], []
        for n in (8, 12, 16, 20):
            A = inputs.cfg2(n, 200 if n <= 12 else 4)
            t0 = time.perf_counter()
            k = 0
            while time.perf_counter() - t0 < seconds / 4 and k < A.shape[0]:
                step = min(A.shape[0] - k, 50 if n <= 12 else 1)
                if n <= 12:
                    oracle.ryser_batch(A[k:k + step])
                else:
                    oracle.permanent_hr(A[k])
                k += step
            dt = time.perf_counter() - t0
            rates.append(dt / k)
            parts.append(f"n={n}: {k} matrices in {dt:.1f} s")
        per_step = sum(r * 100000 for r in rates)      # seconds for 4 x 10^5 permanents
        return {"value": 400000 / per_step, "unit": "perms/s", "cores": cores, "kind": "oracle",
                "sample": "Eq. (3)/App. A binary128 oracle on the first config-2 submatrices; " + "; ".join(parts)}
    if cfg == "cfgens":
        Gm, Cm = inputs.cfgens(count=64)
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < seconds and k < 64:
            oracle.ryser_batch(np.stack([Gm[k], Cm[k]]))
            k += 1
        dt = time.perf_counter() - t0
        return {"value": 2 * k / dt, "unit": "perms/s", "cores": cores, "kind": "oracle",
                "sample": f"Eq. (3) binary128 oracle on the first {k} Ginibre + {k} circular cfgens matrices, {dt:.1f} s"}
    if cfg == "cfg3":
        A = inputs.cfg3()
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < seconds and k < A.shape[0]:
            oracle.ryser_i01(A[k])
            k += 1
        dt = time.perf_counter() - t0
        return {"value": k / dt, "unit": "perms/s", "cores": cores, "kind": "oracle",
                "sample": f"Eq. (3) int128 oracle on {k} of the 64 config-3 matrices, {dt:.1f} s"}
    if cfg == "cfg3s":
        A = inputs.bernoulli01((1, 33, 33), 33)[0]
        B = np.ascontiguousarray(A[:24, :24])
        t0 = time.perf_counter()
        oracle.ryser_i01(B)
        dt = time.perf_counter() - t0
        return {"value": (1 << 24) / dt, "unit": "terms/s", "cores": cores, "kind": "oracle",
                "sample": f"Eq. (3) int128 oracle on the leading 24x24 block of the cfg3s matrix (2^24 terms in "
                          f"{dt:.1f} s); the rate per term extrapolates to the 2^33 terms at n = 33 within n/24"}
    if cfg == "cfgbd":
        A = inputs.cfgbd(64)
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < seconds and k < A.shape[0]:
            oracle.band(A[k], 5)
            k += 1
        dt = time.perf_counter() - t0
        return {"value": k / dt, "unit": "perms/s", "cores": 1, "kind": "oracle",
                "sample": f"App. C binary128 oracle (literal polynomial, single-threaded) on {k} cfgbd matrices, {dt:.1f} s"}
    if cfg == "cfgsp":
        A = inputs.cfgsp()
        A20 = inputs.sparse_gaussian(24, 0.04 * 48 / 24, inputs.SEEDS["cfgsp"])
        t0 = time.perf_counter()
        _, cnt = oracle.sparse(A20)
        dt = time.perf_counter() - t0
        return {"value": cnt / dt, "unit": "terms/s", "cores": cores, "kind": "oracle",
                "sample": f"App. B binary128 oracle (sparsepermanent) on a 24x24 matrix of the same recipe "
                          f"({cnt} restricted sets in {dt:.1f} s; the 48x48 instance is out of its reach)"}
    if cfg == "cfgpm":
        A = inputs.bernoulli_pm1((1024, 24, 24), inputs.SEEDS["cfgpm"])
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < seconds and k < A.shape[0]:
            oracle.ryser_i8(A[k])
            k += 1
        dt = time.perf_counter() - t0
        return {"value": k / dt, "unit": "perms/s", "cores": cores, "kind": "oracle",
                "sample": f"Eq. (3) int128 oracle on the first {k} of the 1024 cfgpm matrices, {dt:.1f} s"}
    if cfg == "cfgw":
        C, M = inputs.cfgw()
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < seconds and k < C.shape[0]:
            oracle.ryser_weighted(C[k], M[k])
            k += 1
        dt = time.perf_counter() - t0
        return {"value": k / dt, "unit": "perms/s", "cores": cores, "kind": "oracle",
                "sample": f"Eq. (4) binary128 oracle on the first {k} of the 10^4 cfgw patterns, {dt:.1f} s"}
    raise ValueError(cfg)


# ------------------------------------------------------------------------------------------ GPU arm

def run_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    # Launched by torchrun (even with one rank): one process per GPU over NCCL.  PERM_BENCH_DIST_BACKEND=gloo
    # is a functional test hook only (several ranks sharing the box's one GPU, results checked, timings
    # meaningless).
    dist_on = world > 1 or ("MASTER_ADDR" in os.environ and "RANK" in os.environ)
    if dist_on:
        backend = os.environ.get("PERM_BENCH_DIST_BACKEND", "nccl")
        dev = local % torch.cuda.device_count() if backend != "nccl" else local
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    device = torch.device("cuda", torch.cuda.current_device())
    import paper_1904_06229_b200 as pb
    from paper_1904_06229_b200 import inputs, shard

    pb.lib()
    stream = torch.cuda.current_stream()
    l2buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    cfg = args.config

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    result = {}
    warm_step = None
    gpu_launches_per_step = 0
    h2d = d2h = 0
    walk_launches_per_step = 0
    roofline_units = None          # (flops per walk launch)

    if cfg in ("cfg5", "cfg4", "cfg1"):
        A_np = {"cfg5": inputs.cfg5, "cfg4": inputs.cfg4, "cfg1": inputs.cfg1}[cfg]()
        n = A_np.shape[0]
        total = 1 << (n - 1)
        b = pb.chunk_log2(n)
        chunks = 1 << (n - 1 - b)
        c0, c1 = shard.chunk_span(n, world, rank, b)            # whole aligned chunks per GPU
        wave = pb.chunk_walkers(n, b)                           # chunks one launch walks per round
        # One permanent per step when it takes seconds at most; otherwise ONE permanent per run, its chunk
        # range cut into K steps of whole rounds (each step: walk + tree + all-gather of the nodes).
        est_s = total / world / 6.0e10
        perm_steps = args.steps_per_perm or (args.steps if est_s > 4.0 else 1)
        if args.steps % perm_steps:
            raise SystemExit("--steps must be a multiple of --steps-per-perm")
        slices = shard.step_slices(c0, c1, perm_steps, wave)
        warm = (c0, min(c1, c0 + wave))                        # warm-up: one round of the rank's first chunks
        max_slice = max([s1 - s0 for s0, s1 in slices] + [warm[1] - warm[0], 1])
        A_pin = torch.from_numpy(A_np).pin_memory()
        parts = torch.empty((max_slice, 4), dtype=torch.float64, device=device)
        ws_a = torch.empty(n * n * 16, dtype=torch.uint8, device=device)
        tree_ws = torch.empty(pb.tree_workspace_bytes(max_slice), dtype=torch.uint8, device=device)
        nodes = torch.empty((pb.TREE_MAX_NODES, 6), dtype=torch.int64, device=device)
        gathered = torch.empty((world * pb.TREE_MAX_NODES, 6), dtype=torch.int64, device=device)
        gathered_host = torch.empty((world * pb.TREE_MAX_NODES, 6), dtype=torch.int64).pin_memory()
        ew0, ew1, ec1, es0, es1 = ev(), ev(), ev(), ev(), ev()
        h2d, d2h = A_np.nbytes, gathered_host.numel() * 8
        walk_launches_per_step = 1
        collected: list = []
        step_idx = [0]
        terms_walked = [0]
        launch_count = [0]

        # One process and a whole permanent per step: the single-call public API perm_c128 (for n <= 16 one
        # cluster launch; else the chunk walk + tree inside the library -- the same chunks and tree, same bits).
        single = not dist_on and perm_steps == 1
        out_dev = torch.empty(1, dtype=torch.complex128, device=device)
        out_host = torch.empty(1, dtype=torch.complex128).pin_memory()
        ws_single = pb.make_workspace(n, device=device) if single else None
        if single:
            d2h = 16

        # A small permanent (n <= 16: one cluster launch in the library) is latency-bound: its step is replayed
        # from CUDA graphs captured once -- `dev`: the kernel on the device-resident matrix; `e2e`: H2D of the
        # pinned host matrix + kernel + D2H of per(A).  Captured after the warm-up call (function attributes set).
        graphs = {}
        A_dev_single = A_pin.to(device) if single else None

        def capture_graphs():
            pb.perm_c128(A_dev_single, workspace=ws_single, out=out_dev, stream=stream)
            torch.cuda.synchronize()
            # events recorded INSIDE the graphs (event-record nodes) bracket the library call, so a step's
            # device time excludes the graph-launch latency of the otherwise idle device
            x = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
            gd, ge = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gd):
                cs = torch.cuda.current_stream()
                x[0].record(cs)
                pb.perm_c128(A_dev_single, workspace=ws_single, out=out_dev, stream=cs)
                x[1].record(cs)
            nl = pb.last_launches()
            with torch.cuda.graph(ge):
                cs = torch.cuda.current_stream()
                x[2].record(cs)
                pb.perm_c128(A_pin, workspace=ws_single, out=out_dev, stream=cs)
                out_host.copy_(out_dev, non_blocking=True)
                x[3].record(cs)
            torch.cuda.synchronize()
            graphs.update(dev=gd, e2e=ge, launches=nl, ev=x)

        def step_graph(sl=None):
            warmup = sl is not None
            if not graphs:
                capture_graphs()
            graphs["dev"].replay()
            graphs["e2e"].replay()
            torch.cuda.synchronize()
            if warmup:
                return {}
            launch_count[0] += 2 * graphs["launches"]
            terms_walked[0] += total
            step_idx[0] += 1
            x = graphs["ev"]
            d = x[0].elapsed_time(x[1])
            return {"dev": d, "e2e": x[2].elapsed_time(x[3]), "walk": d, "result": complex(out_host.item())}

        def step_single(sl=None):
            if n <= 16:
                return step_graph(sl)
            warmup = sl is not None
            es0.record(stream)
            pb.perm_c128(A_pin, workspace=ws_single, out=out_dev, stream=stream, events=(ew0, ew1))
            nl = pb.last_launches()
            ec1.record(stream)
            out_host.copy_(out_dev, non_blocking=True)
            es1.record(stream)
            torch.cuda.synchronize()
            if not warmup:
                launch_count[0] += nl
                terms_walked[0] += total
                step_idx[0] += 1
            return {"dev": ew0.elapsed_time(ec1), "e2e": es0.elapsed_time(es1), "walk": ew0.elapsed_time(ew1),
                    "result": complex(out_host.item())}

        def step(sl=None):
            if single:
                return step_single(sl)
            warmup = sl is not None
            s0, s1 = sl if warmup else slices[step_idx[0] % perm_steps]
            es0.record(stream)                                  # e2e: from the H2D of A (inside the call)
            pb.perm_c128_chunks(A_pin, s0, s1, partials=parts, workspace=ws_a, stream=stream, events=(ew0, ew1))
            nl = pb.last_launches()
            pb.perm_c128_tree(parts, s0, s1, nodes=nodes, workspace=tree_ws, stream=stream)
            nl += pb.last_launches()
            if dist_on:
                dist.all_gather_into_tensor(gathered, nodes)
                src = gathered
            else:
                src = nodes
            ec1.record(stream)
            gathered_host[: src.shape[0]].copy_(src, non_blocking=True)
            es1.record(stream)
            torch.cuda.synchronize()
            val = None
            if not warmup:
                launch_count[0] += nl
                terms_walked[0] += (s1 - s0) << b
                collected.append(gathered_host[: src.shape[0]].numpy().copy())
                if step_idx[0] % perm_steps == perm_steps - 1:
                    val = shard.combine_nodes(np.concatenate(collected), n)
                    collected.clear()
                step_idx[0] += 1
            return {"dev": ew0.elapsed_time(ec1), "e2e": es0.elapsed_time(es1), "walk": ew0.elapsed_time(ew1),
                    "result": val}

        warm_step = lambda: step(warm)
        unit = "terms/s"
        gpu_launches_per_step = None                            # counted below from the library
        workload = {"cfg5": "one 44x44 complex Gaussian matrix (re, im ~ N(0,1/2), seed 44): per(A) via 2^43 Gray terms",
                    "cfg4": "32x32 leading block of a 1024x1024 Haar unitary (seed 1024): per(A) via 2^31 Gray terms",
                    "cfg1": "one 16x16 complex Gaussian matrix (seed 16): per(A) via 2^15 Gray terms"}[cfg]
        config = {"workload": workload, "n": n, "chunk_log2": b, "chunks": chunks,
                  "parallelism": f"Gray-chunk range x{world}",
                  "permanents_per_run": args.steps // perm_steps,
                  "steps_per_permanent": perm_steps,
                  "terms_per_step": (total // perm_steps if perm_steps > 1 else total),
                  "slicing": ("one full permanent per run: the rank's chunk span cut into K steps of whole "
                              f"rounds of {wave} chunks; every step walks its slice, reduces it by the canonical "
                              "chunk tree and all-gathers the tree nodes; the last step merges all nodes -> per(A)"
                              if perm_steps > 1 else "one full permanent per step"),
                  "api": ("perm_c128 (one call per permanent" + (", replayed from CUDA graphs: device-resident "
                          "graph for value, H2D + call + D2H graph for e2e; timing events recorded inside the graphs "
                          "around the call)" if n <= 16 else ")") if single else
                          "perm_c128_chunks + perm_c128_tree per step, all-gather of the tree nodes, "
                          "perm_c128_tree_combine + perm_c128_finalize"),
                  "chunks_rank0": shard.chunk_span(n, world, 0, b)[1], "input_bytes": A_np.nbytes,
                  "l2": "compute-bound (input 31 KB); L2 flushed between steps (256 MiB write)"}
        scaling = "strong"
    elif cfg == "cfg2":
        ns = (8, 12, 16, 20)
        count = 100000
        mats = {n: inputs.cfg2(n, count) for n in ns}
        # weak scaling: every rank processes its contiguous share of each batch
        host = {}
        dev_in = {}
        outs = {}
        for n in ns:
            b0, b1 = shard.rank_span(count, world, rank)
            host[n] = torch.from_numpy(np.ascontiguousarray(mats[n][b0:b1])).pin_memory()
            dev_in[n] = host[n].to(device)
            outs[n] = (torch.empty(b1 - b0, dtype=torch.complex128, device=device),
                       torch.empty(b1 - b0, dtype=torch.float64, device=device))
        abs2_host = {n: torch.empty(outs[n][1].shape[0], dtype=torch.float64).pin_memory() for n in ns}
        e0, e1, e2 = ev(), ev(), ev()
        h2d = sum(h.numel() * 16 for h in host.values())
        d2h = sum(a.numel() * 8 for a in abs2_host.values())
        walk_launches_per_step = len(ns)
        roofline_units = None

        def step():
            # device-resident pass
            e0.record(stream)
            for n in ns:
                pb.perm_c128_batched(dev_in[n], per=outs[n][0], abs2=outs[n][1], stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            # end-to-end pass through the public API from pinned host memory
            es = torch.cuda.Event(enable_timing=True)
            ee = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            for n in ns:
                dev_in[n].copy_(host[n], non_blocking=True)
                pb.perm_c128_batched(dev_in[n], per=outs[n][0], abs2=outs[n][1], stream=stream)
                abs2_host[n].copy_(outs[n][1], non_blocking=True)
            ee.record(stream)
            torch.cuda.synchronize()
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": float(abs2_host[20][0])}

        units_per_step = count * len(ns)
        unit = "perms/s"
        gpu_launches_per_step = 2 * len(ns)
        config = {"workload": "Boson-sampling |per|^2 of 10^5 submatrices (distinct rows/cols) of an n^2 x n^2 "
                              "Haar unitary for each n in {8,12,16,20}", "batch_per_n": count,
                  "parallelism": f"batch x{world}", "l2": "inputs 1.4 GB > L2"}
        scaling = "weak" if world > 1 else "strong"
        if world > 1:
            units_per_step = count * len(ns)   # every rank does its share of the same global batch
    elif cfg == "cfgens":
        # NEXT-2: the Sec. III-IV ensembles streamed through the batched kernel with the X = |per|/sqrt(n!) output
        Gm, Cm = inputs.cfgens()
        B, n = Gm.shape[0], Gm.shape[1]
        b0, b1 = shard.rank_span(B, world, rank)
        hosts = [torch.from_numpy(np.ascontiguousarray(M[b0:b1])).pin_memory() for M in (Gm, Cm)]
        ens_dev = [h.to(device) for h in hosts]
        xs = [torch.empty(b1 - b0, dtype=torch.float64, device=device) for _ in hosts]
        xs_host = [torch.empty(b1 - b0, dtype=torch.float64).pin_memory() for _ in hosts]
        e0, e1 = ev(), ev()
        h2d = sum(h.numel() * 16 for h in hosts)
        d2h = sum(x.numel() * 8 for x in xs_host)
        walk_launches_per_step = 2
        ens_stats = {}

        def step():
            e0.record(stream)
            for dv, x in zip(ens_dev, xs):
                pb.perm_c128_batched_x(dv, x=x, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            es = torch.cuda.Event(enable_timing=True)
            ee = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            for h, dv, x, xh in zip(hosts, ens_dev, xs, xs_host):
                dv.copy_(h, non_blocking=True)
                pb.perm_c128_batched_x(dv, x=x, stream=stream)
                xh.copy_(x, non_blocking=True)
            ee.record(stream)
            torch.cuda.synchronize()
            for name, xh in zip(("ginibre", "circular"), xs_host):
                X = xh.numpy()
                ens_stats[name] = {"mean_X": float(X.mean()), "mean_X2": float((X ** 2).mean()),
                                   "mean_X4": float((X ** 4).mean()), "count": int(X.size)}
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": ens_stats["circular"]["mean_X2"]}

        units_per_step = 2 * B
        unit = "perms/s"
        gpu_launches_per_step = 2 * 2
        config = {"workload": f"Sec. III-IV ensembles: {B} Ginibre + {B} circular (exp(i theta)) matrices of order {n} "
                              f"(seeds {inputs.SEEDS['cfgens_g']}, {inputs.SEEDS['cfgens_c']}), X = |per|/sqrt(n!) "
                              "streamed per matrix", "batch": 2 * B, "n": n, "parallelism": f"batch x{world}",
                  "l2": "inputs 184 MB > L2"}
        scaling = "weak" if world > 1 else "strong"
    elif cfg in ("cfg3", "cfgpm"):
        pm1 = cfg == "cfgpm"
        A_np = inputs.bernoulli_pm1((1024, 24, 24), inputs.SEEDS["cfgpm"]) if pm1 else inputs.cfg3()
        B, n = A_np.shape[0], A_np.shape[1]
        b0, b1 = shard.rank_span(B, world, rank)
        host = torch.from_numpy(np.ascontiguousarray(A_np[b0:b1])).pin_memory()
        dev_in = host.to(device)
        out = torch.empty((b1 - b0, 2), dtype=torch.int64, device=device)
        out_host = torch.empty((b1 - b0, 2), dtype=torch.int64).pin_memory()
        ws = torch.empty(pb.int01_workspace_bytes(n, b1 - b0), dtype=torch.uint8, device=device)
        e0, e1 = ev(), ev()
        h2d, d2h = host.numel(), out_host.numel() * 8
        walk_launches_per_step = 1
        fn = pb.perm_pm1 if pm1 else pb.perm_int01

        def step():
            e0.record(stream)
            fn(dev_in, workspace=ws, out=out, stream=stream, as_int=False)
            e1.record(stream)
            torch.cuda.synchronize()
            es = torch.cuda.Event(enable_timing=True)
            ee = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            dev_in.copy_(host, non_blocking=True)
            fn(dev_in, workspace=ws, out=out, stream=stream, as_int=False)
            out_host.copy_(out, non_blocking=True)
            ee.record(stream)
            torch.cuda.synchronize()
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": int(out_host[0, 0])}

        units_per_step = B
        unit = "perms/s"
        gpu_launches_per_step = 2 * 2
        config = {"workload": ("1024 Bernoulli +-1 matrices of order 24 (Sec. V ensemble, seed 2425), exact int128 "
                               "permanents" if pm1 else
                               "64 Bernoulli(1/2) 0-1 matrices of order 24 (seed 24), exact int128 permanents"),
                  "parallelism": f"batch x{world}", "l2": "input 0.6 MB; compute-bound" if pm1 else "input 37 KB; compute-bound"}
        scaling = "weak" if world > 1 else "strong"
    elif cfg == "cfg3s":
        # one exact 0-1 permanent of order 33 (2^33 terms of Eq. (3)), the rank space sharded over ranks
        n = 33
        A_np = inputs.bernoulli01((1, n, n), 33)[0]
        total = shard.int01_rank_space(n)
        k0, k1 = shard.rank_span(total, world, rank)
        host = torch.from_numpy(np.ascontiguousarray(A_np)).pin_memory()
        dev_in = host.to(device)
        gathered = torch.empty(2 * world, dtype=torch.int64, device=device)
        e0, e1 = ev(), ev()
        h2d, d2h = host.numel(), 16 * world
        walk_launches_per_step = 1
        nlaunch = [0]

        def step():
            es = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            dev_in.copy_(host, non_blocking=True)
            e0.record(stream)
            raw = pb.perm_int01_range(dev_in, k0, k1, stream=stream)      # synchronizes the stream
            nlaunch[0] = pb.last_launches()
            part = torch.from_numpy(shard.pack_i128(raw)).to(device, non_blocking=False)
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(gathered, part)
                src = gathered
            else:
                src = part
            e1.record(stream)
            val = shard.combine_int01(src.cpu().numpy(), n)
            ee = torch.cuda.Event(enable_timing=True)
            ee.record(stream)
            torch.cuda.synchronize()
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": val}

        units_per_step = total
        unit = "terms/s"
        gpu_launches_per_step = 0                      # counted from the library after the warm-up
        config = {"workload": "one Bernoulli(1/2) 0-1 matrix of order 33 (seed 33): exact per(A) via the 2^33 "
                              "terms of Eq. (3) in int128, rank space sharded",
                  "n": n, "terms_per_step": total, "parallelism": f"Gray-range x{world}",
                  "l2": "input 1 KB; compute-bound"}
        scaling = "strong"
    elif cfg == "cfgbd":
        kb = 5
        A_np = inputs.cfgbd()
        Bn, n = A_np.shape[0], A_np.shape[1]
        b0, b1 = shard.rank_span(Bn, world, rank)
        host = torch.from_numpy(np.ascontiguousarray(pb.band_storage(A_np[b0:b1], kb))).pin_memory()
        dev_in = host.to(device)
        per_d = torch.empty(b1 - b0, dtype=torch.complex128, device=device)
        abs2_d = torch.empty(b1 - b0, dtype=torch.float64, device=device)
        abs2_h = torch.empty(b1 - b0, dtype=torch.float64).pin_memory()
        e0, e1 = ev(), ev()
        h2d, d2h = host.numel() * 16, abs2_h.numel() * 8
        walk_launches_per_step = 1
        # transitions per row of the App. C transfer matrix: every new state has k+1 predecessors unless
        # the window's top column is the one just used (then 1)
        trans = sum((1 if (t >> (2 * kb - 1)) & 1 else kb + 1) for t in range(1 << (2 * kb))
                    if bin(t).count("1") == kb)
        band_flops = (b1 - b0) * n * trans * 8.0

        def step():
            e0.record(stream)
            pb.perm_c128_band_batched(dev_in, kb, per=per_d, abs2=abs2_d, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            es = torch.cuda.Event(enable_timing=True)
            ee = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            dev_in.copy_(host, non_blocking=True)
            pb.perm_c128_band_batched(dev_in, kb, per=per_d, abs2=abs2_d, stream=stream)
            abs2_h.copy_(abs2_d, non_blocking=True)
            ee.record(stream)
            torch.cuda.synchronize()
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": float(abs2_h[0])}

        units_per_step = Bn
        unit = "perms/s"
        gpu_launches_per_step = 2
        config = {"workload": "10^4 complex Gaussian matrices of order 100 and bandwidth 5 (seed 1005), App. C "
                              "transfer method", "batch": Bn, "n": n, "k": kb, "parallelism": f"batch x{world}",
                  "l2": "inputs 176 MB > L2"}
        scaling = "weak" if world > 1 else "strong"
    elif cfg == "cfgsp":
        A_np = inputs.cfgsp()
        n = A_np.shape[0]
        plan = pb.perm_sparse_plan(A_np)
        A_pin = torch.from_numpy(A_np).pin_memory()
        A_dev = A_pin.to(device)
        h2d, d2h = A_np.nbytes, 16
        walk_launches_per_step = 1
        sets = plan["sets"]
        _, sp_info = pb.perm_c128_sparse(A_dev, stream=stream, info=True)    # planning call: the walk it picks
        sp_group = sp_info["group_cols"]

        def step():
            es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            es.record(stream)
            val = pb.perm_c128_sparse(A_dev, stream=stream)      # synchronizes
            ee.record(stream)
            torch.cuda.synchronize()
            e2s, e2e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2s.record(stream)
            val = pb.perm_c128_sparse(A_pin, stream=stream)      # host input: H2D inside the call
            e2e.record(stream)
            torch.cuda.synchronize()
            return {"dev": es.elapsed_time(ee), "e2e": e2s.elapsed_time(e2e), "walk": es.elapsed_time(ee),
                    "result": val}

        units_per_step = sets
        unit = "terms/s"
        gpu_launches_per_step = 2 * 2
        config = {"workload": "one sparse 48x48 complex matrix (density 4% + a perfect matching, seed 4848): per(A) "
                              "by App. B restricted enumeration", "n": n, "terms_per_step": sets,
                  "dense_terms": float(2 ** (n - 1)), "partition": {"d": len(plan["S"]), "T": plan["nt"]},
                  "parallelism": "sets x1", "l2": "input 37 KB; compute-bound"}
        scaling = "strong"
    elif cfg == "cfgw":
        C_np, M_np = inputs.cfgw()
        B, n, R = C_np.shape
        b0, b1 = shard.rank_span(B, world, rank)
        hostC = torch.from_numpy(np.ascontiguousarray(C_np[b0:b1])).pin_memory()
        hostM = torch.from_numpy(np.ascontiguousarray(M_np[b0:b1])).pin_memory()
        devC, devM = hostC.to(device), hostM.to(device)
        per_d = torch.empty(b1 - b0, dtype=torch.complex128, device=device)
        abs2_d = torch.empty(b1 - b0, dtype=torch.float64, device=device)
        abs2_h = torch.empty(b1 - b0, dtype=torch.float64).pin_memory()
        e0, e1 = ev(), ev()
        h2d, d2h = hostC.numel() * 16 + hostM.numel() * 4, abs2_h.numel() * 8
        terms_w = float(np.sum(np.prod(M_np[b0:b1].astype(np.float64) + 1.0, axis=1)))
        walk_launches_per_step = 1
        nlaunch = [2]

        def step():
            e0.record(stream)
            pb.perm_c128_weighted_batched(devC, devM, per=per_d, abs2=abs2_d, stream=stream)
            nlaunch[0] = pb.last_launches()                    # order kernel + weighted kernel
            e1.record(stream)
            torch.cuda.synchronize()
            es = torch.cuda.Event(enable_timing=True)
            ee = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            devC.copy_(hostC, non_blocking=True)
            devM.copy_(hostM, non_blocking=True)
            pb.perm_c128_weighted_batched(devC, devM, per=per_d, abs2=abs2_d, stream=stream)
            abs2_h.copy_(abs2_d, non_blocking=True)
            ee.record(stream)
            torch.cuda.synchronize()
            return {"dev": e0.elapsed_time(e1), "e2e": es.elapsed_time(ee), "walk": e0.elapsed_time(e1),
                    "result": float(abs2_h[0])}

        units_per_step = B
        unit = "perms/s"
        gpu_launches_per_step = 2
        config = {"workload": "10^4 Boson-sampling output patterns with collisions: 20 photons in the 20 modes of a "
                              "Haar unitary (seed 2424), weighted Ryser Eq. (4)", "batch": B, "n": n,
                  "terms_per_step": terms_w * world, "parallelism": f"batch x{world}",
                  "l2": "inputs 64 MB; compute-bound"}
        scaling = "weak" if world > 1 else "strong"
    else:
        raise SystemExit(f"unknown config {cfg}")

    # warm-up (untimed)
    for _ in range(args.warmup):
        (warm_step or step)()
        flush_l2(l2buf)
    torch.cuda.synchronize()
    peak_meas = measure_fp64_peak(pb, torch) if rank == 0 else None

    # timed region: barrier + synchronize on both sides
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    devs, e2es, walks, res = [], [], [], None
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        pending = []
        for _ in range(args.steps):
            r = step()
            if "lazy" in r:
                pending.append(r["lazy"])
            else:
                pending.append(lambda r=r: r)
            flush_l2(l2buf)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        for f in pending:
            r = f()
            devs.append(r["dev"])
            e2es.append(r["e2e"])
            walks.append(r["walk"])
            if r["result"] is not None:
                res = r["result"]
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms = max_over_ranks(sum(devs), world, device)
    e2e_ms = max_over_ranks(sum(e2es), world, device)
    walk_ms_local = sum(walks) / len(walks)
    walk_ms = max_over_ranks(walk_ms_local, world, device)
    clocks = clk.summary()
    if cfg in ("cfg5", "cfg4", "cfg1"):
        # roofline of the walk kernel: algorithmic flops of rank 0's walk launches / their event-timed duration
        roofline_units = 8.0 * n * terms_walked[0] / args.steps
        walk_ms = sum(walks) / len(walks)
        units_per_step = total / perm_steps

    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return
    K = args.steps
    value = units_per_step * K / (dev_ms * 1e-3)
    e2e_val = units_per_step * K / (e2e_ms * 1e-3)
    out = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": K, "warmup": args.warmup,
           "ms_per_step": dev_ms / K, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
           "dtype": "int128" if cfg in ("cfg3", "cfgpm", "cfg3s") else "f64",
           "data": "synthetic (seeded generators, paper_1904_06229_b200/inputs.py)",
           "config": config}
    nominal = fp64_nominal_tflops()
    if roofline_units is not None:
        achieved = roofline_units / (walk_ms * 1e-3) / 1e12
        out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                           "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                           "kernel": ((f"walk_small_kernel<{n}> (one cluster launch: walk + tree)" if n <= 16
                                       else f"walk_kernel_c<{n}, unit column>" if n == 32
                                       else f"walk_kernel_cm<{n}, unit column>" if 33 <= n <= 48 else f"walk_kernel<{n}>")
                                      + " (FP64 vector pipe)"),
                           "algorithmic": ("8n flops per Gray term x terms per launch (rank 0)" +
                                           (" (the unit-column walk executes 5n - 2 FP64 instructions per term "
                                            "instead of 6n - 4: ceiling 0.81 instead of 0.68 of peak at n = 44; "
                                            "DESIGN.md 5.1)" if 32 <= n <= 48 else "")),
                           "peak_note": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz",
                           "peak_measured_probe": peak_meas, "frac_of_measured": achieved / peak_meas,
                           "walk_ms_per_launch": walk_ms}
        if cfg == "cfg5":
            out["fp64_peak_frac"] = achieved / nominal
    else:
        # batched / int: report the device time of the batch kernels against the FP64 (or INT) pipe
        if cfg == "cfgbd":
            achieved = band_flops / (dev_ms / K * 1e-3) / 1e12
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                               "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                               "kernel": "band_kernel (FP64 complex MACs from shared memory)",
                               "algorithmic": "8 flops per transfer-matrix transition x transitions per row x n rows",
                               "peak_measured_probe": peak_meas}
        elif cfg == "cfgsp":
            # the shared-rows group walk, per block of 2^G sets: the column flip 2n, Z and the block
            # product n - M - 1 complex multiplies (6 flops), the fused accumulate 8, 2^G products of M rows, the
            # 2^G - 1 shifted row sums (2M) and signed sums (2); the term-by-term walk: 8n per set
            Mr = 4
            fpset = ((2 * n + 6 * (n - Mr - 1) + 8 + 2 ** sp_group * 6 * (Mr - 1) + (2 ** sp_group - 1) * (2 * Mr + 2))
                     / 2 ** sp_group) if sp_group else 8 * n
            fl = sets * fpset
            achieved = fl / (dev_ms / K * 1e-3) / 1e12
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                               "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                               "kernel": (f"sparse_kernel_c<48, G = {sp_group}> (shared-rows group walk)"
                                          if sp_group else "sparse_kernel_c<48> (FP64 vector pipe)"),
                               "algorithmic": (f"{fpset:.1f} flops per restricted set J (group walk, G = {sp_group}, "
                                               f"M = {Mr}; the term-by-term walk's 8n = {8 * n} would read "
                                               f"{sets * 8 * n / (dev_ms / K * 1e-3) / 1e12 / nominal:.3f})"
                                               if sp_group else "8n flops per restricted set J")
                                              + " x 2^|T| prod (2^|S_l| - 1) sets",
                               "peak_measured_probe": peak_meas}
        elif cfg == "cfgw":
            fl = terms_w * 8 * 20
            achieved = fl / (dev_ms / K * 1e-3) / 1e12
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                               "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                               "kernel": "weighted_kernel<20> (FP64 vector pipe)",
                               "algorithmic": "8n flops per Eq. (4) term x prod_k (m_k+1) terms per pattern",
                               "peak_measured_probe": peak_meas}
        elif cfg == "cfgens":
            fl = 2 * (b1 - b0) * (1 << (n - 1)) * 8 * n
            achieved = fl / (dev_ms / K * 1e-3) / 1e12
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                               "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                               "kernel": f"batched_kernel<{n}> x2 (FP64 vector pipe)",
                               "algorithmic": "8n flops per Gray term x 2^(n-1) terms x matrices",
                               "peak_measured_probe": peak_meas}
            out["ensemble"] = ens_stats
        elif cfg == "cfg2":
            fl = sum(100000 / world * (1 << (n - 1)) * 8 * n for n in (8, 12, 16, 20))
            achieved = fl / (dev_ms / K * 1e-3) / 1e12
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                               "frac": achieved / nominal, "traffic": ncu_traffic(cfg),
                               "kernel": "batched_kernel<n> x4 (unit-column walk for n >= 14; FP64 vector pipe)",
                               "algorithmic": "8n flops per Gray term x 2^(n-1) terms x 10^5 per n",
                               "peak_measured_probe": peak_meas}
        else:
            # algorithmic integer ops per Gray term: n row-sum adds + (n-1) multiplies + 1 signed add
            n3 = 33 if cfg == "cfg3s" else 24
            ops = (units_per_step / world * 2 * n3 if cfg == "cfg3s"
                   else units_per_step / world * (1 << (n3 - 1)) * 2 * n3)
            kname = {"cfgpm": "int01_kernel<24, pm1> (quad-factored walk; INT fma + alu pipes)",
                     "cfg3s": "int01_kernel<33> (Eq. (3) branch, pair-factored walk; INT fma + alu pipes)"}.get(
                         cfg, "int01_kernel<24> (pair-factored walk; INT fma + alu pipes)")
            achieved = ops / (dev_ms / K * 1e-3) / 1e12
            ipeak = int_nominal_tops()
            out["roofline"] = {"bound": "alu", "achieved": achieved, "peak": ipeak, "unit": "Tops/s",
                               "frac": achieved / ipeak, "traffic": ncu_traffic(cfg),
                               "kernel": kname,
                               "algorithmic": ("2n integer ops per Gray term x 2^n terms / ranks" if cfg == "cfg3s" else
                                               "2n integer ops per Gray term x 2^(n-1) terms x matrices") +
                                              " (the plain walk's count: the pair/quad-factored walks need fewer "
                                              "operations per term, so frac is an effective rate; DESIGN.md 5.3)",
                               "peak_note": "derived: 148 SMs x 128 int lanes/clk (issue-bound) x 1965 MHz"}
    out["e2e"] = {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if cfg == "cfg3s":
        gpu_launches_per_step = nlaunch[0]             # range pieces + the summing kernel (library count)
    if cfg == "cfgw":
        gpu_launches_per_step = 2 * nlaunch[0]         # device-timed + e2e calls, library count each
    if cfg in ("cfg5", "cfg4", "cfg1"):
        gpu_launches_per_step = launch_count[0] / K
    out["gpu_launches"] = int(round(gpu_launches_per_step * K))
    out["clocks"] = clocks
    out["wall_s_timed_region"] = t_wall
    out["result_sample"] = str(res)
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = oracle_rate_cfg(cfg, seconds=args.cpu_seconds)
    print(json.dumps(out), flush=True)
    if dist_on:
        dist.destroy_process_group()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return          # the reference arm runs on rank 0 only
    cfg = args.config
    unit = "perms/s" if cfg in ("cfg2", "cfg3", "cfgw", "cfgpm", "cfgbd", "cfgens") else "terms/s"
    for _ in range(max(0, args.warmup)):
        oracle_rate_cfg(cfg, seconds=1.0)
    rates, samples = [], []
    t0 = time.perf_counter()
    # each step is a bounded sample; its length shrinks with K so that the whole arm ends within a few minutes
    per_step = min(args.cpu_seconds, max(1.5, 150.0 / max(1, args.steps)))
    for _ in range(args.steps):
        r = oracle_rate_cfg(cfg, seconds=per_step)
        rates.append(r["value"])
        samples.append(r)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    last = samples[-1]
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "binary128",
           "data": "synthetic (seeded generators, paper_1904_06229_b200/inputs.py)",
           "config": {"workload": cfg, "reference": "CPU oracle (oracle/oracle.c), bounded sample per step"},
           "cpu_baseline": {"value": value, "unit": unit, "cores": last["cores"], "kind": "oracle",
                            "sample": last["sample"]},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg3s", "cfg4", "cfg5", "cfgw", "cfgpm",
                                                          "cfgsp", "cfgbd", "cfgens"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--steps-per-perm", type=int, default=0,
                    help="cfg5/cfg4/cfg1: steps one permanent is sliced into (default: K when a permanent takes more "
                         "than a few seconds at this GPU count, i.e. one permanent per run; else 1, a permanent per step)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
