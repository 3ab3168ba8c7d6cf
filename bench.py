#!/usr/bin/env python
"""PM+ hashing benchmark (BASELINE.json metric: "PM+ hashed GB/s (32/64-bit out)").

Default: every BASELINE.json config that is a throughput workload, one JSON line
each, the headline last:
    fixed4k   configs[2]  2^20 x 4096 B, PM+64                       (>= 1 GB)
    long16g   configs[3]  one 16 GiB string, PM+64                   (>= 1 GB)
    mixed     configs[4]  byte-balanced shard r of 8 of 2^22 log-uniform
                          [1 B, 1 MiB] strings (~37 GiB), PM+32        (>= 1 GB)
    tiny      configs[0]  1,000 strings U[1,64] B, PM+64 (latency path)
    hashtable configs[1]  2^24 strings U[8,64] B, PM+64 AND PM+32     <- headline (last line)
--workload NAME runs one of them.

One step = the whole hot path over one batch: the library call(s) that turn
the device-resident batch into digests (hashtable: pmp_hash_batch_multi with
both schedules, one fused pass).  value = payload bytes x digest widths, all
ranks / max-over-ranks device time (CUDA events, inputs larger than L2, so no
flush between steps; tiny is L2-resident and says so).

Multi-GPU (torchrun): hashtable / fixed4k / tiny: the ONE global batch is
sharded by payload bytes (parallel.shard_batch), no collective on the data
path -> "scaling": "strong" (--weak: every rank hashes its own batch of the
recipe, data seed + 256 rank).  long16g: block-aligned ranges of the one string,
one all-gather of 16-byte partials (strong).  mixed: rank r hashes shard r of 8
(configs[4] is sized for 8 GPUs; one GPU holds one shard) -> weak.

Each line carries roofline (dominant kernel, live CUDA-event launch times from
a separate profiled pass after the timed region), e2e (the same metric through
the public host-memory API: pmp_hash_batch_host / pmp_hash_long_host, copies
inside the timed region), clocks (NVML during the timed region) and
cpu_baseline (the oracle, median of 3 bounded samples on the host cores).

--impl reference: the CPU oracle (oracle/, plain C) timed on bounded samples of
the same workloads on the host cores (the paper ships no code; per the task
the reference arm is the oracle).
"""
from __future__ import annotations

import argparse
import contextlib
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

import datagen  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback
ORDER = ["fixed4k", "long16g", "mixed", "tiny", "hashtable"]   # headline last


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: NVML polled every ~1 ms in a thread; falls back to nvidia-smi."""

    REASONS = {  # NVML clocks-event reason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nv is not None:
                    nv = self._nv
                    sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                    try:
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    except Exception:
                        rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                    self.samples.append((sm, self.max_mhz, rs))
                    self._stop.wait(0.001)
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    a, b = [float(x) for x in out.split(",")]
                    self.samples.append((a, b, 0))
                    self._stop.wait(0.05)
            except Exception:
                self._stop.wait(0.01)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(x[0]) for x in self.samples]
        mask = 0
        for x in self.samples:
            mask |= int(x[2])
        reasons = sorted(v for k, v in self.REASONS.items() if mask & k)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(self.samples[0][1]),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nv is not None else "nvidia-smi"}


# ----------------------------------------------------------------- workloads
def metric_of(wl):
    return f"PM+ hashed GB/s ({'/'.join(str(b) for b in wl.bits)}-bit out)"


def dtype_of(wl):
    return "u64+u32" if len(wl.bits) > 1 else f"u{wl.bits[0]}"


def scaling_of(wl, weak):
    if wl.long:
        return "strong"
    if wl.name == "mixed" or weak:
        return "weak"
    return "strong"


def make_batch(wl, rank, world=1, weak=False, n=None):
    """Host lengths / offsets of this rank's strings and the data seed / first
    payload byte they start at.  Returns (seed, lens, offsets rebased to the
    rank's first byte, b0 = that byte's position in the global payload).

    mixed: byte-balanced shard r of 8 of the one global corpus (configs[4] is
    sized for 8 GPUs).  weak: the rank's own batch of the recipe (data seed +
    256 rank).  Otherwise (strong scaling): byte-balanced shard r of `world` of
    the one global batch.  ``n`` truncates the rank's strings (oracle samples)."""
    from paper_1609_09840_b200 import parallel

    if wl.name == "mixed" or (not weak and world > 1):
        lens = wl.lengths()
        offs_all = datagen.offsets_from_lengths(lens)
        parts = 8 if wl.name == "mixed" else world
        lo, hi = parallel.shard_batch(offs_all, parts)[rank % parts]
        if n is not None:
            hi = min(hi, lo + n)
        sub, b0, _ = parallel.rebase_offsets(offs_all, lo, hi)
        return wl.seed, lens[lo:hi], sub, b0
    nn = wl.n if n is None else min(n, wl.n)
    seed = wl.seed + (256 * rank if weak else 0)
    lens = datagen.lengths(wl.kind, seed, wl.n, wl.lo, wl.hi)[:nn]
    return seed, lens, datagen.offsets_from_lengths(lens), 0


def workload_config(wl, world, weak, variant="tree"):
    sc = scaling_of(wl, weak)
    c = {"workload": wl.name, "baseline_config": {"tiny": 0, "hashtable": 1, "fixed4k": 2, "long16g": 3,
                                                 "mixed": 4}[wl.name],
         "strings": wl.n, "len_bytes": [wl.lo, wl.hi],
         "len_dist": {0: "fixed", 1: "uniform", 2: "log-uniform"}[wl.kind], "bits": list(wl.bits),
         "key_seed": wl.seed,
         "parallelism": (f"split{world}" if wl.long else
                         f"shard{world}" if sc == "strong" else f"dp{world}"),
         "l2": ("inputs larger than L2 (126 MB); no flush needed" if wl.name != "tiny" else
                "48 KB batch, L2-resident between steps (latency workload, no flush)")}
    if wl.long:
        c["strings"] = 1
        c["string_bytes"] = wl.lo
    if wl.name == "mixed":
        c["strings"] = "shard r of 8 of 2^22 (~2^19 per rank, ~37 GiB)"
    if variant != "tree":
        c["variant"] = "two-level: multilinear chunks + polynomial in r (8(f4), reading Q19)"
    return c


# ----------------------------------------------------------------- oracle (cpu_baseline / reference arm)
class OracleSample:
    """A bounded prefix sample of the workload for the oracle (all host
    threads), sized once by calibration to ~budget_s per run."""

    def __init__(self, wl, budget_s, variant="tree"):
        import oracle

        self.oracle = oracle
        self.wl = wl
        self.variant = variant
        self.threads = os.cpu_count() or 1
        self.keys = {b: oracle.keygen(wl.seed, b) for b in wl.bits}
        if wl.long:
            nb = 16 << 20
            pay = datagen.payload_host(wl.seed, 0, nb)
            dt = self._run_long(pay)
            self.nbytes = int(min(wl.lo, max(nb, nb * budget_s / max(dt, 1e-6))) // 1024 * 1024)
            self.pay = datagen.payload_host(wl.seed, 0, self.nbytes)
            self.desc = f"first {self.nbytes} B of the 16 GiB string hashed as one string"
            return
        seed, lens, offs, b0 = make_batch(wl, 0, n=min(wl.n, 1 << 22))
        n_cal = min(1 << 15 if wl.name != "mixed" else 1 << 9, offs.size - 1)
        pay = datagen.payload_host(seed, b0, int(offs[n_cal]))
        dt = self._run_batch(pay, offs[:n_cal + 1])
        n_s = int(min(offs.size - 1, max(n_cal, n_cal * budget_s / max(dt, 1e-6))))
        self.offs = offs[:n_s + 1]
        self.pay = datagen.payload_host(seed, b0, int(offs[n_s]))
        self.nbytes = int(offs[n_s]) * len(wl.bits)
        self.desc = f"first {n_s} strings of the workload ({int(offs[n_s])} B), widths {list(wl.bits)}"

    def _run_long(self, pay):
        o = self.oracle
        t0 = time.perf_counter()
        (o.hash2 if self.variant == "two-level" else o.hash_long)(self.keys[64], pay, nthreads=self.threads)
        return time.perf_counter() - t0

    def _run_batch(self, pay, offs):
        hb = self.oracle.hash2_batch if self.variant == "two-level" else self.oracle.hash_batch
        t0 = time.perf_counter()
        for b in self.wl.bits:
            hb(self.keys[b], pay, offs, nthreads=self.threads)
        return time.perf_counter() - t0

    def run(self):
        """One timed run: (GB/s, seconds)."""
        dt = self._run_long(self.pay) if self.wl.long else self._run_batch(self.pay, self.offs)
        return self.nbytes / dt / 1e9, dt


def oracle_single_thread(wl, variant="tree"):
    """One host thread of the oracle on a small sample (a
    single-core figure beside the paper's bytes/cycle/core)."""
    import oracle

    bits = wl.bits[0]
    k = oracle.keygen(wl.seed, bits)
    if wl.long:
        nb = 8 << 20
        pay = datagen.payload_host(wl.seed, 0, nb)
        t0 = time.perf_counter()
        (oracle.hash2 if variant == "two-level" else oracle.hash_long)(k, pay, nthreads=1)
        dt = time.perf_counter() - t0
    else:
        lens = wl.lengths(min(wl.n, 1 << 16)).astype(np.uint64)
        offs = datagen.offsets_from_lengths(lens)
        n = lens.size
        if wl.name in ("mixed", "fixed4k"):
            n = min(n, int(np.searchsorted(offs, 32 << 20)))
        offs = offs[: n + 1]
        pay = datagen.payload_host(wl.seed, 0, int(offs[-1]))
        t0 = time.perf_counter()
        (oracle.hash2_batch if variant == "two-level" else oracle.hash_batch)(k, pay, offs, nthreads=1)
        dt = time.perf_counter() - t0
        nb = int(offs[-1])
    mhz = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("cpu MHz"):
                    mhz = float(ln.split(":", 1)[1])
                    break
    except OSError:
        pass
    gbs = nb / dt / 1e9
    return {"value": gbs, "unit": "GB/s", "width": bits, "sample_bytes": nb,
            "bytes_per_cycle": (gbs * 1e9 / (mhz * 1e6)) if mhz else None, "cpu_mhz": mhz}


def host_cpu():
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("physical id"):
                    sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "sockets": len(sockets) or None}


def cpu_baseline(wl, variant="tree", runs=3, budget_s=3.0):
    """The oracle as it stands on the host cores: median of `runs` runs of one
    bounded sample (the same sampler as --impl reference)."""
    try:
        smp = OracleSample(wl, budget_s, variant)
        res = [smp.run() for _ in range(runs)]
        v = statistics.median(r[0] for r in res)
        return {"value": v, "unit": "GB/s", "cores": smp.threads, "kind": "oracle", "sample": smp.desc,
                "runs": [round(r[0], 4) for r in res], "seconds_per_run": statistics.median(r[1] for r in res),
                "host": host_cpu(), "single_thread": oracle_single_thread(wl, variant)}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": f"failed: {e}"}


def run_reference(args, names):
    """The reference arm: the oracle, timed on the host cores, one line per
    workload in the GPU arm's order (headline last).  Rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    per_step = max(0.3, min(4.0, 150.0 / (len(names) * (args.warmup + args.steps))))
    for name in names:
        wl = datagen.WORKLOADS[name]
        smp = OracleSample(wl, per_step, args.variant)
        rates, times = [], []
        for i in range(args.warmup + args.steps):
            r, dt = smp.run()
            if i >= args.warmup:
                rates.append(r)
                times.append(dt)
        v = statistics.median(rates)
        line = {"impl": "reference", "metric": metric_of(wl), "value": v, "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(times),
                "higher_is_better": True, "scaling": scaling_of(wl, args.weak), "vs_baseline": None,
                "dtype": dtype_of(wl), "data": "synthetic (seeded xoshiro256** bytes)",
                "config": workload_config(wl, args.gpus, args.weak, args.variant),
                "cpu_baseline": {"value": v, "unit": "GB/s", "cores": smp.threads, "kind": "oracle",
                                 "sample": smp.desc, "host": host_cpu()},
                "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU arm
class Ctx:
    """Process-wide state: ranks, device, stream, collectives."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # PMP_BENCH_BACKEND=gloo: a plumbing test for several ranks sharing one
        # GPU (collectives on CPU tensors); real multi-GPU runs use NCCL.
        self.backend = os.environ.get("PMP_BENCH_BACKEND", "nccl")
        if self.backend != "nccl":
            local = local % max(torch.cuda.device_count(), 1)
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        if self.world > 1:
            if self.backend == "nccl":
                # NCCL's INIT lines (rank count, NVLS / P2P transport) go to stderr
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)
            dist.barrier()
        self.cdev = self.dev if self.backend == "nccl" else torch.device("cpu")
        self.stream = torch.cuda.current_stream()
        self.sp = int(self.stream.cuda_stream)

    def max_over_ranks(self, x):
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.cdev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x):
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.cdev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def all_ok(self, ok):
        """True on every rank iff `ok` on every rank (a failed rank must still
        take part in the collectives that follow)."""
        t = self.torch.tensor([1 if ok else 0], dtype=self.torch.int64, device=self.cdev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return bool(t.item())

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()


class Work:
    """One workload on this rank: device buffers, the step, and what the
    roofline needs.  Attributes: step(), payload_bytes (this rank, x widths),
    dominant, alg_bytes_per_launch, e2e()."""


def prepare_long(args, wl, ctx, pmp, keys):
    torch = ctx.torch
    v2 = args.variant == "two-level"
    total = wl.lo
    begins = pmp.pmp_long_split(64, total, ctx.world)
    lo, hi = begins[ctx.rank], begins[ctx.rank + 1]
    assert lo % datagen.PAGE == 0
    d_data = torch.empty(hi - lo + 16, dtype=torch.uint8, device=ctx.dev)
    d_full = d_data[: hi - lo]
    datagen.fill_device(wl.seed, d_full.data_ptr(), hi - lo, ctx.sp, start=lo)
    parts = torch.zeros(2 * ctx.world, dtype=torch.int64, device=ctx.dev)
    out = torch.zeros(1, dtype=torch.int64, device=ctx.dev)
    sth = pmp.pmp_stream_new(keys[64].handle) if args.stream_mib else 0
    piece = args.stream_mib << 20
    from paper_1609_09840_b200 import parallel

    w = Work()

    def step_stream():
        pmp._check(pmp.pmp_stream_reset(sth, ctx.sp), "reset")
        for pos in range(0, hi - lo, piece):
            pmp._check(pmp.pmp_stream_update(sth, d_full.data_ptr() + pos, min(piece, hi - lo - pos), ctx.sp),
                       "update")
        pmp._check(pmp.pmp_stream_final(sth, out.data_ptr(), ctx.sp), "final")

    def step():
        if args.stream_mib:
            assert ctx.world == 1, "--stream-mib measures one GPU"
            return step_stream()
        part_fn = pmp.pmp_hash2_long_partial if v2 else pmp.pmp_hash_long_partial
        mine = parts[2 * ctx.rank:2 * ctx.rank + 2]
        pmp._check(part_fn(keys[64].handle, d_full.data_ptr(), hi - lo, lo, total, mine.data_ptr(), ctx.sp),
                   "partial")
        if ctx.world > 1:
            parts.copy_(parallel.gather_partials(mine.clone(), ctx.world))
        if v2:
            pmp._check(pmp.pmp_hash2_long_combine(keys[64].handle, parts.data_ptr(), ctx.world, out.data_ptr(),
                                                  ctx.sp), "combine")
        else:
            pmp._check(pmp.pmp_hash_long_combine(keys[64].handle, parts.data_ptr(), ctx.world, total,
                                                 out.data_ptr(), ctx.sp), "combine")

    w.step = step
    w.payload_bytes = hi - lo
    w.dominant = "k_stream_node" if args.stream_mib else ("k_poly_node" if v2 else "k_node")
    w.alg_bytes_per_launch = min(piece, hi - lo) if args.stream_mib else hi - lo
    w.traffic_key = w.dominant
    w.bufs = [d_data, parts, out]

    def e2e():
        """The string from pinned HOST memory: world == 1 -> pmp_hash_long_host
        (pieces copied H2D on internal streams, overlapped with the incremental
        device state); world > 1 -> each rank copies its range H2D and runs the
        partial / all-gather / combine.  Digest read back to the host."""
        if args.variant != "tree" or args.stream_mib:
            return None
        err = None
        try:
            h = torch.empty(hi - lo, dtype=torch.uint8, pin_memory=True)
            h.copy_(d_full)
            torch.cuda.synchronize()
        except Exception as ex:  # pinned host memory can run out on a shared node
            err = repr(ex)[:200]
        if not ctx.all_ok(err is None):
            return {"value": None, "unit": "GB/s", "error": err or "another rank failed"}
        dig = np.zeros(1, dtype=np.uint64)

        def one():
            if ctx.world == 1:
                pmp._check(pmp.lib().pmp_hash_long_host(keys[64].handle, h.data_ptr(), total, dig.ctypes.data,
                                                        args.e2e_piece_mib << 20, ctx.sp), "pmp_hash_long_host")
            else:
                d_full.copy_(h, non_blocking=True)
                step()
                dig[0] = int(out.cpu().numpy().view(np.uint64)[0])

        one()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ctx.stream)
        for _ in range(args.e2e_steps):
            one()
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = ctx.max_over_ranks(ev0.elapsed_time(ev1) / args.e2e_steps)
        del h
        return {"value": total / (ms / 1000) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": hi - lo,
                "d2h_bytes_per_step": 8, "ms_per_step": ms,
                "path": (f"pmp_hash_long_host (pinned host string, {args.e2e_piece_mib or 256} MiB pieces copied H2D on 3 internal streams, "
                         "overlapped with the incremental device state)" if ctx.world == 1 else
                         "pinned host range -> H2D -> pmp_hash_long_partial -> all-gather -> combine -> host")}

    w.e2e = e2e
    return w


def prepare_batch(args, wl, ctx, pmp, keys):
    torch = ctx.torch
    v2 = args.variant == "two-level"
    seed, lens, offs, b0 = make_batch(wl, ctx.rank, ctx.world, args.weak)
    n = lens.size
    total_bytes = int(offs[-1])
    lead = b0 % datagen.PAGE
    d_buf = torch.empty(total_bytes + lead + 16, dtype=torch.uint8, device=ctx.dev)
    datagen.fill_device(seed, d_buf.data_ptr(), total_bytes + lead, ctx.sp, start=b0 - lead)
    d_pay = d_buf[lead:]
    d_off = torch.from_numpy(offs.view(np.int64)).to(ctx.dev)
    outs = {b: torch.empty(max(n, 1), dtype=torch.int64 if b == 64 else torch.int32, device=ctx.dev)
            for b in wl.bits}
    counts = torch.zeros(max(args.buckets, 1), dtype=torch.int32, device=ctx.dev)
    assert not args.partition or args.buckets, "--partition needs --buckets M"
    if args.partition:
        p_starts = torch.empty(args.buckets + 1, dtype=torch.int64, device=ctx.dev)
        p_perm = torch.empty(max(n, 1), dtype=torch.int32, device=ctx.dev)
    fused = len(wl.bits) == 2 and not args.buckets and not args.separate_widths
    multi_fn = pmp.pmp_hash2_batch_multi if v2 else pmp.pmp_hash_batch_multi

    def step():
        if fused:  # both outputs of the batch in one pass over the short strings
            pmp._check(multi_fn([keys[b].handle for b in wl.bits], d_pay.data_ptr(), d_off.data_ptr(), n,
                                [outs[b].data_ptr() for b in wl.bits], ctx.sp), "pmp_hash_batch_multi")
            return
        for b in wl.bits:
            if args.buckets:
                pmp._check(pmp.pmp_hash_batch_buckets(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n,
                                                      args.buckets, outs[b].data_ptr(), counts.data_ptr(), ctx.sp),
                           "pmp_hash_batch_buckets")
                if args.partition:
                    pmp._check(pmp.pmp_bucket_partition(outs[b].data_ptr(), n, args.buckets, 0,
                                                        p_starts.data_ptr(), p_perm.data_ptr(), ctx.sp),
                               "pmp_bucket_partition")
            else:
                fn = pmp.pmp_hash2_batch if v2 else pmp.pmp_hash_batch
                pmp._check(fn(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n, outs[b].data_ptr(), ctx.sp),
                           "pmp_hash_batch")

    w = Work()
    w.step = step
    w.payload_bytes = total_bytes * len(wl.bits)
    small = not v2 and n <= 4096
    w.dominant = "k_small" if small else ("k_short" if wl.hi <= 127 else "k_wstring")
    w.traffic_key = w.dominant + ("+dual" if fused and w.dominant == "k_short" else "")
    # algorithmic bytes per dominant launch: payload + offsets + digests (fused: both
    # widths' digests in one launch; otherwise the average over the widths' launches)
    if fused and w.dominant in ("k_short", "k_small"):
        w.alg_bytes_per_launch = total_bytes + 8 * (n + 1) + n * sum(b // 8 for b in wl.bits)
    else:
        w.alg_bytes_per_launch = total_bytes + 8 * (n + 1) + n * sum(b // 8 for b in wl.bits) / len(wl.bits)
    w.bufs = [d_buf, d_off, outs, counts]

    def e2e():
        """The same batch from pinned HOST memory through pmp_hash_batch_host
        (tree) -- pieces copied H2D, hashed and copied back D2H on 3 internal
        streams -- digests in host memory at the end of every step."""
        # several ranks of one node pin their host copies at once: above 8 GiB per
        # rank, time a string-aligned prefix of the rank's strings (same rate, said so)
        n_e, tb_e = n, total_bytes
        cap = 8 << 30
        if ctx.world > 1 and total_bytes > cap:
            n_e = max(1, int(np.searchsorted(offs, np.uint64(cap), side="right")) - 1)
            tb_e = int(offs[n_e])
        err = None
        try:
            h_pay = torch.empty(max(tb_e, 1), dtype=torch.uint8, pin_memory=True)
            h_pay[:tb_e].copy_(d_pay[:tb_e])
            h_off = torch.from_numpy(offs[:n_e + 1].view(np.int64)).pin_memory()
            h_out = {b: torch.empty(n_e, dtype=outs[b].dtype).pin_memory() for b in wl.bits}
            torch.cuda.synchronize()
        except Exception as ex:  # pinned host memory can run out on a shared node
            err = repr(ex)[:200]
        if not ctx.all_ok(err is None):
            return {"value": None, "unit": "GB/s", "error": err or "another rank failed"}
        host_api = not v2
        d_out = outs

        def one():
            if host_api:
                pmp._check(pmp.pmp_hash_batch_host([keys[b].handle for b in wl.bits], h_pay.data_ptr(),
                                                   h_off.data_ptr(), n_e, [h_out[b].data_ptr() for b in wl.bits],
                                                   args.e2e_piece_mib << 20, ctx.sp), "e2e hash")
                return
            d_pay[:tb_e].copy_(h_pay[:tb_e], non_blocking=True)
            d_off[:n_e + 1].copy_(h_off, non_blocking=True)
            for b in wl.bits:
                pmp._check(pmp.pmp_hash2_batch(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n_e,
                                               d_out[b].data_ptr(), ctx.sp), "e2e hash")
                h_out[b].copy_(d_out[b][:n_e], non_blocking=True)

        one()
        torch.cuda.synchronize()
        steps = args.e2e_steps if wl.name != "tiny" else 50
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ctx.stream)
        for _ in range(steps):
            one()
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = ctx.max_over_ranks(ev0.elapsed_time(ev1) / steps)
        moved = ctx.sum_over_ranks(tb_e * len(wl.bits))
        del h_pay
        return {"value": moved / (ms / 1000) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": tb_e + 8 * (n_e + 1),
                "d2h_bytes_per_step": n_e * sum(b // 8 for b in wl.bits), "ms_per_step": ms,
                **({"sample": f"first {n_e} of the rank's {n} strings ({tb_e} B): pinned host memory of "
                              f"{ctx.world} ranks per node"} if n_e < n else {}),
                "path": (f"pmp_hash_batch_host (pinned host buffers, {'both widths in one pass, ' if fused else ''}"
                         f"{args.e2e_piece_mib or 64} MiB pieces: H2D / hash / D2H overlapped on 3 streams)" if host_api else
                         "pinned host -> cudaMemcpyAsync -> pmp_hash2_batch (both widths) -> host")}

    w.e2e = e2e
    return w


def bench_one(args, wl, ctx, pmp, clean_first=True):
    torch = ctx.torch
    keys = {b: pmp.Keys.generate(wl.seed, b) for b in wl.bits}
    v2 = args.variant == "two-level"
    assert not (v2 and (args.buckets or args.stream_mib)), "--variant two-level: plain digests only"
    w = prepare_long(args, wl, ctx, pmp, keys) if wl.long else prepare_batch(args, wl, ctx, pmp, keys)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        w.step()
    torch.cuda.synchronize()
    # ---- per-kernel launch times: a profiled pass with CUDA events around every
    # launch (pmp_prof_*, on the launch stream), kept OUT of the timed region
    # (the events add gaps between launches); its clocks are sampled too
    prof_steps = max(3, min(args.steps, 20))
    pmp.pmp_prof_reset()
    pmp.pmp_prof_enable(True)
    with ClockSampler(ctx.local) as pclk:
        for _ in range(prof_steps):
            w.step()
        torch.cuda.synchronize()
    pmp.pmp_prof_enable(False)
    k_ms, k_cnt = pmp.pmp_prof_read(w.dominant)
    kernel_ms = {name: pmp.pmp_prof_read(name) for name in
                 ("k_short", "k_small", "k_wstring", "k_histogram", "k_node", "k_level", "k_combine", "k_stream",
                  "k_poly", "k_part")}
    time.sleep(0.3)   # let the power controller settle after the profiled pass
    ctx.barrier()
    torch.cuda.synchronize()
    # ---- timed region: the steps only (library instrumentation off)
    l0 = pmp.pmp_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.local) as clk:
        # throughput workloads: a device-side head start (a sleep kernel before
        # ev0, outside the timed region) so the host has queued the steps before
        # the device reaches them -- the K steps then run back to back and a
        # host-side stall (thread scheduling, the clock sampler) cannot open a
        # gap between them (one of five hashtable runs showed 0.352 instead of
        # 0.269 ms per step with identical kernel times).  The latency path
        # (tiny) is timed as the host issues it.
        if wl.name != "tiny":
            torch.cuda._sleep(int((10.0 + 0.1 * args.steps) * 1e-3 * 2.0e9))
        ev0.record(ctx.stream)
        for _ in range(args.steps):
            w.step()
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
    launches = pmp.pmp_launch_count() - l0
    ms_max = ctx.max_over_ranks(ev0.elapsed_time(ev1))
    ms_per_step = ms_max / args.steps
    moved = wl.lo if wl.long else ctx.sum_over_ranks(w.payload_bytes)   # long: the one string, once
    value = moved / (ms_per_step / 1000) / 1e9
    e2e = None
    if not args.no_e2e:
        e2e = w.e2e()
    line = None
    if ctx.rank == 0:
        peak, peak_src = hbm_peak()
        avg_ms = k_ms / max(k_cnt, 1)
        achieved = w.alg_bytes_per_launch / (avg_ms / 1000) / 1e9 if k_cnt else None
        traffic = load_profile(wl.name, w.traffic_key)
        pipes = load_profile(wl.name, w.traffic_key, "pipes.json")
        clocks = clk.summary()
        cpu = None if args.no_cpu else cpu_baseline(wl, args.variant)
        cfg = dict(workload_config(wl, ctx.world, args.weak, args.variant))
        if args.buckets:
            cfg["output"] = f"buckets mod {args.buckets} + histogram" + (" + partition" if args.partition else "")
        if args.stream_mib:
            cfg["api"] = f"pmp_stream_update in {args.stream_mib} MiB pieces"
        line = {
            "metric": metric_of(wl), "value": value, "unit": "GB/s", "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling_of(wl, args.weak), "vs_baseline": None, "dtype": dtype_of(wl),
            "data": "synthetic (seeded xoshiro256** bytes, generated on device)", "config": cfg,
            # bytes hashed per width (the headline counts every (byte, schedule) pair)
            "payload_gbs_per_width": value / len(wl.bits),
            "bytes_per_gpu_cycle": (value / ctx.world * 1e9) / (clocks["sm_mhz"] * 1e6) if clocks.get("sm_mhz") else None,
            "roofline": {"bound": "hbm", "kernel": w.dominant, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         # the measured peak is a read+write COPY rate; a read-only stream
                         # (the long string) can exceed it -- the nominal 8 TB/s beside it
                         "frac_of_nominal_8000": (achieved / 8000.0) if achieved else None,
                         "alg_bytes_per_launch": w.alg_bytes_per_launch, "avg_launch_ms": avg_ms,
                         "launches_profiled": k_cnt, "profiled_steps": prof_steps,
                         "profiled_pass_clocks": pclk.summary(),
                         # issue / integer-pipe utilisation of this kernel from the committed
                         # ncu capture (profiles/pipes.json), for the IMAD side of the roofline
                         "ncu_pipes": pipes},
            "clocks": clocks,
            "gpu_launches": launches,
            "kernel_ms_per_step": {k: v[0] / prof_steps for k, v in kernel_ms.items() if v[1]},
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    for k in keys.values():
        k.close()
    del w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    ctx.barrier()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pmp", choices=["pmp", "reference"])
    ap.add_argument("--workload", default="all", choices=["all"] + sorted(datagen.WORKLOADS),
                    help="all (default): fixed4k, long16g, mixed, tiny, then the hashtable headline last")
    ap.add_argument("--weak", action="store_true",
                    help="batch workloads at N > 1: every rank hashes its own batch (weak scaling) "
                         "instead of a shard of the one global batch (strong)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--stream-mib", type=int, default=0,
                    help="long16g only (SURVEY 8(f1)): feed the string through pmp_stream_update in pieces of this many MiB")
    ap.add_argument("--buckets", type=int, default=0,
                    help="hash-table consumer (SURVEY 8(f3)): write digest mod M + histogram instead of digests")
    ap.add_argument("--partition", action="store_true",
                    help="with --buckets: also group the string indices by bucket (pmp_bucket_partition)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--variant", default="tree", choices=["tree", "two-level"],
                    help="two-level: the multilinear + polynomial variant (8(f4), pmp_hash2_*)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--separate-widths", action="store_true",
                    help="hash the two widths of configs[1] with two pmp_hash_batch calls instead of one fused pass")
    ap.add_argument("--e2e-piece-mib", type=int, default=0,
                    help="piece size of the host-resident e2e paths (0: library default, 64 MiB batch / 256 MiB long)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    names = ORDER if args.workload == "all" else [args.workload]
    if args.impl == "reference":
        return run_reference(args, names)

    import paper_1609_09840_b200 as pmp
    from paper_1609_09840_b200 import _build

    if _build.needs_build() and int(os.environ.get("RANK", "0")) == 0:
        _build.build()
    ctx = Ctx()
    for name in names:
        wl = datagen.WORKLOADS[name]
        if args.stream_mib and not wl.long:
            continue
        if (args.buckets or args.separate_widths) and wl.long:
            continue
        bench_one(args, wl, ctx, pmp)
    if ctx.world > 1:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    return 0


def load_profile(workload, kernel, name="traffic.json"):
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
