#!/usr/bin/env python
"""PM+ hashing benchmark (BASELINE.json metric: "PM+ hashed GB/s (32/64-bit out)").

Default workload = BASELINE.json configs[1] ("hashtable"): 2^24 strings with
lengths U[8,64] bytes, packed contiguously with uint64 offsets, hashed with
BOTH 64-bit and 32-bit PM+ (keys from seed 2).  One step = pmp_hash_batch with
the PM+64 keys + pmp_hash_batch with the PM+32 keys over the resident batch.
value = payload bytes hashed (both widths, all ranks) / max-over-ranks time.

Multi-GPU (torchrun): each rank hashes its own batch of the same recipe
(data seed 2 + 256*rank, same keys): weak scaling, no collective on the data
path.  --workload long16g splits one 16 GiB string across ranks with one NCCL
all-gather of 16-byte partials (strong scaling).

--impl reference: the CPU oracle (oracle/, plain C) timed on a bounded sample
of the same workload on the host cores (there is no other reference program:
the paper ships no code).
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

import datagen  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: NVML polled every ~1 ms in a thread (the region is tens of ms);
    falls back to nvidia-smi."""

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
def make_batch(wl, rank, n=None):
    """Host lengths/offsets for this rank's batch.

    hashtable/fixed4k/tiny: each rank hashes its own batch of the recipe (data
    seed + 256*rank).  mixed (configs[4], ~295 GiB, sized for 8 GPUs): rank r
    hashes byte-balanced shard r of 8 of the one global corpus; returns
    offsets rebased to the shard and the shard's first payload byte."""
    if wl.name == "mixed":
        from paper_1609_09840_b200 import parallel

        lens = wl.lengths()
        offs_all = datagen.offsets_from_lengths(lens)
        lo, hi = parallel.shard_batch(offs_all, 8)[rank % 8]
        if n is not None:
            hi = min(hi, lo + n)
        sub, b0, _ = parallel.rebase_offsets(offs_all, lo, hi)
        return wl.seed, lens[lo:hi], sub, b0
    n = wl.n if n is None else n
    seed = wl.seed + 256 * rank
    lens = datagen.lengths(wl.kind, seed, n, wl.lo, wl.hi)
    offs = datagen.offsets_from_lengths(lens)
    return seed, lens, offs, 0


def oracle_sample_rate(wl, seed, offs, bits_list, budget_s=12.0, max_threads=None, base=0, variant="tree"):
    """Oracle GB/s on a bounded prefix sample of the batch (all host threads)."""
    import oracle

    hb = oracle.hash2_batch if variant == "two-level" else oracle.hash_batch
    threads = max_threads or os.cpu_count() or 1
    keys = {b: oracle.keygen(wl.seed, b) for b in bits_list}
    # calibrate on 2^15 strings, then size the sample to ~budget_s
    n_cal = min(1 << 15, offs.size - 1)
    if wl.name == "mixed":
        n_cal = min(1 << 9, offs.size - 1)
    pay = datagen.payload_host(seed, base, int(offs[n_cal]))
    t0 = time.perf_counter()
    for b in bits_list:
        hb(keys[b], pay, offs[:n_cal + 1], nthreads=threads)
    dt = time.perf_counter() - t0
    n_s = int(min(offs.size - 1, max(n_cal, n_cal * budget_s / max(dt, 1e-6))))
    pay = datagen.payload_host(seed, base, int(offs[n_s]))
    t0 = time.perf_counter()
    for b in bits_list:
        hb(keys[b], pay, offs[:n_s + 1], nthreads=threads)
    dt = time.perf_counter() - t0
    nbytes = int(offs[n_s]) * len(bits_list)
    return nbytes / dt / 1e9, threads, f"first {n_s} strings of the batch ({int(offs[n_s])} B), widths {bits_list}", dt


def oracle_single_thread(wl, variant="tree", budget_s=2.0):
    """One host thread of the oracle on a small sample of the workload (SURVEY
    8(d): a single-core figure beside the paper's bytes/cycle/core; the oracle
    is the literal slow program, not the paper's tuned code)."""
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
        lens = wl.lengths()[: 1 << 16].astype(np.uint64)
        offs = datagen.offsets_from_lengths(lens)
        n = 1 << 16
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


def oracle_long_rate(wl, nbytes_sample, budget_s=12.0, variant="tree"):
    import oracle

    threads = os.cpu_count() or 1
    k = oracle.keygen(wl.seed, 64)
    pay = datagen.payload_host(wl.seed, 0, nbytes_sample)
    t0 = time.perf_counter()
    if variant == "two-level":
        oracle.hash2(k, pay, nthreads=threads)
    else:
        oracle.hash_long(k, pay, nthreads=threads)
    dt = time.perf_counter() - t0
    return nbytes_sample / dt / 1e9, threads, f"first {nbytes_sample} B of the 16 GiB string hashed as one string", dt


# ----------------------------------------------------------------- reference arm
def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    unit = "GB/s"
    times, rates = [], []
    desc = cores = None
    if wl.long:
        for i in range(args.warmup + args.steps):
            r, cores, desc, dt = oracle_long_rate(wl, 64 << 20, variant=args.variant)
            if i >= args.warmup:
                rates.append(r)
                times.append(dt)
    else:
        seed, lens, offs, b0 = make_batch(wl, 0, n=min(wl.n, 1 << 22))
        for i in range(args.warmup + args.steps):
            r, cores, desc, dt = oracle_sample_rate(wl, seed, offs, list(wl.bits), budget_s=4.0, base=b0,
                                                    variant=args.variant)
            if i >= args.warmup:
                rates.append(r)
                times.append(dt)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": f"PM+ hashed GB/s ({'/'.join(str(b) for b in wl.bits)}-bit out)",
            "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.median(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64+u32" if len(wl.bits) > 1 else f"u{wl.bits[0]}",
            "data": "synthetic (seeded xoshiro256** bytes)", "config": workload_config(wl, args.gpus, args.variant),
            "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "oracle", "sample": desc,
                             "host": host_cpu()},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(wl, gpus, variant="tree"):
    c = {"workload": wl.name, "strings_per_gpu": wl.n if wl.name != "mixed" else "shard of 8 (~2^19)",
         "len_bytes": [wl.lo, wl.hi],
         "len_dist": {0: "fixed", 1: "uniform", 2: "log-uniform"}[wl.kind], "bits": list(wl.bits),
         "key_seed": wl.seed, "parallelism": f"dp{gpus}" if not wl.long else f"split{gpus}",
         "l2": "inputs larger than L2 (126 MB); no flush needed"}
    if wl.long:
        c["strings_per_gpu"] = None
        c["string_bytes"] = wl.lo
    if variant != "tree":
        c["variant"] = "two-level: multilinear chunks + polynomial in r (8(f4), reading Q19)"
    return c


# ----------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pmp", choices=["pmp", "reference"])
    ap.add_argument("--workload", default="hashtable", choices=sorted(datagen.WORKLOADS))
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
    ap.add_argument("--e2e-piece-mib", type=int, default=64, help="piece size of the host-resident e2e path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = datagen.WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    import paper_1609_09840_b200 as pmp
    from paper_1609_09840_b200 import _build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if _build.needs_build() and rank == 0:
        _build.build()
    # PMP_BENCH_BACKEND=gloo is a plumbing test for several ranks sharing one
    # GPU (collectives on CPU tensors); real multi-GPU runs use NCCL.
    backend = os.environ.get("PMP_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        dist.barrier()
    cdev = dev if backend == "nccl" else torch.device("cpu")  # device of collective tensors
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)

    keys = {b: pmp.Keys.generate(wl.seed, b) for b in wl.bits}
    outs = {}
    v2 = args.variant == "two-level"
    assert not (v2 and (args.buckets or args.stream_mib)), "--variant two-level: plain digests only"
    fused_dual = False
    if wl.long:
        total = wl.lo
        begins = pmp.pmp_long_split(64, total, world)
        lo, hi = begins[rank], begins[rank + 1]
        d_data = torch.empty(hi - lo + 16, dtype=torch.uint8, device=dev)
        # rank's slice of the string: regenerate its pages (page-aligned since lo % 4096 == 0)
        assert lo % datagen.PAGE == 0
        d_full = d_data[: hi - lo]
        fill_slice(wl.seed, d_full, lo, sp)
        parts = torch.zeros(2 * world, dtype=torch.int64, device=dev)
        out = torch.zeros(1, dtype=torch.int64, device=dev)
        payload_bytes = total

        sth = pmp.pmp_stream_new(keys[64].handle) if args.stream_mib else 0
        piece = args.stream_mib << 20

        def step_stream():
            pmp._check(pmp.pmp_stream_reset(sth, sp), "reset")
            for pos in range(0, hi - lo, piece):
                pmp._check(pmp.pmp_stream_update(sth, d_full.data_ptr() + pos, min(piece, hi - lo - pos), sp),
                           "update")
            pmp._check(pmp.pmp_stream_final(sth, out.data_ptr(), sp), "final")

        def step():
            if args.stream_mib:
                assert world == 1, "--stream-mib measures one GPU"
                return step_stream()
            part_fn = pmp.pmp_hash2_long_partial if v2 else pmp.pmp_hash_long_partial
            pmp._check(part_fn(keys[64].handle, d_full.data_ptr(), hi - lo, lo, total,
                               parts[2 * rank:2 * rank + 2].data_ptr(), sp), "partial")
            if world > 1:
                if backend == "nccl":
                    dist.all_gather_into_tensor(parts, parts[2 * rank:2 * rank + 2].clone())
                else:
                    host = parts.cpu()
                    dist.all_gather_into_tensor(host, host[2 * rank:2 * rank + 2].clone())
                    parts.copy_(host)
            if v2:
                pmp._check(pmp.pmp_hash2_long_combine(keys[64].handle, parts.data_ptr(), world, out.data_ptr(), sp),
                           "combine")
            else:
                pmp._check(pmp.pmp_hash_long_combine(keys[64].handle, parts.data_ptr(), world, total,
                                                     out.data_ptr(), sp), "combine")
        dominant = "k_stream_node" if args.stream_mib else ("k_poly_node" if v2 else "k_node")
        alg_bytes_per_launch = min(piece, hi - lo) if args.stream_mib else hi - lo
        n = 1
    else:
        seed, lens, offs, b0 = make_batch(wl, rank)
        n = lens.size
        total_bytes = int(offs[-1])
        lead = b0 % datagen.PAGE
        d_buf = torch.empty(total_bytes + lead + 16, dtype=torch.uint8, device=dev)
        datagen.fill_device(seed, d_buf.data_ptr(), total_bytes + lead, sp, start=b0 - lead)
        d_pay = d_buf[lead:]
        d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
        for b in wl.bits:
            outs[b] = torch.empty(n, dtype=torch.int64 if b == 64 else torch.int32, device=dev)
        payload_bytes = total_bytes * len(wl.bits)

        counts = torch.zeros(max(args.buckets, 1), dtype=torch.int32, device=dev)
        assert not args.partition or args.buckets, "--partition needs --buckets M"
        if args.partition:
            p_starts = torch.empty(args.buckets + 1, dtype=torch.int64, device=dev)
            p_perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)

        fused = len(wl.bits) == 2 and not args.buckets and not args.separate_widths
        fused_dual = fused
        multi_fn = pmp.pmp_hash2_batch_multi if v2 else pmp.pmp_hash_batch_multi

        def step():
            if fused:  # both outputs of the batch in one pass over the short strings (pmp_hash_batch_multi)
                pmp._check(multi_fn([keys[b].handle for b in wl.bits], d_pay.data_ptr(),
                                    d_off.data_ptr(), n, [outs[b].data_ptr() for b in wl.bits], sp),
                           "pmp_hash_batch_multi")
                return
            for b in wl.bits:
                if args.buckets:
                    pmp._check(pmp.pmp_hash_batch_buckets(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n,
                                                          args.buckets, outs[b].data_ptr(), counts.data_ptr(), sp),
                               "pmp_hash_batch_buckets")
                    if args.partition:
                        pmp._check(pmp.pmp_bucket_partition(outs[b].data_ptr(), n, args.buckets, 0,
                                                            p_starts.data_ptr(), p_perm.data_ptr(), sp),
                                   "pmp_bucket_partition")
                else:
                    fn = pmp.pmp_hash2_batch if v2 else pmp.pmp_hash_batch
                    pmp._check(fn(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n,
                                  outs[b].data_ptr(), sp), "pmp_hash_batch")
        dominant = "k_short" if wl.hi <= 127 else "k_wstring"
        # algorithmic bytes per dominant launch: payload + offsets + digests (fused: both
        # widths' digests in one launch; otherwise the average over the widths' launches)
        if fused and dominant == "k_short":
            alg_bytes_per_launch = total_bytes + 8 * (n + 1) + n * sum(b // 8 for b in wl.bits)
        else:
            alg_bytes_per_launch = total_bytes + 8 * (n + 1) + n * sum(b // 8 for b in wl.bits) / len(wl.bits)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = pmp.pmp_launch_count()
    pmp.pmp_prof_reset()
    pmp.pmp_prof_enable(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    pmp.pmp_prof_enable(False)
    launches = pmp.pmp_launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    k_ms, k_cnt = pmp.pmp_prof_read(dominant)
    kernel_ms = {name: pmp.pmp_prof_read(name) for name in ("k_short", "k_wstring", "k_histogram", "k_node", "k_level", "k_combine",
                                                             "k_stream", "k_poly", "k_part")}
    t = torch.tensor([ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    if wl.long:
        value = payload_bytes / (ms_per_step / 1000) / 1e9
    else:
        value = payload_bytes * world / (ms_per_step / 1000) / 1e9

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, pmp, keys, dev, stream, rank, world, cdev)

    line = None
    if rank == 0:
        peak, peak_src = hbm_peak()
        avg_ms = k_ms / max(k_cnt, 1)
        achieved = alg_bytes_per_launch / (avg_ms / 1000) / 1e9 if k_cnt else None
        traffic = load_traffic(wl.name, dominant + ("+dual" if fused_dual else ""))
        pipes = load_traffic(wl.name, dominant + ("+dual" if fused_dual else ""), "pipes.json")
        clocks = clk.summary()
        cpu = None
        if not args.no_cpu:
            cpu = cpu_baseline(wl, args.variant)
        line = {
            "metric": f"PM+ hashed GB/s ({'/'.join(str(b) for b in wl.bits)}-bit out)",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if wl.long else "weak", "vs_baseline": None,
            "dtype": "u64+u32" if len(wl.bits) > 1 else f"u{wl.bits[0]}",
            "data": "synthetic (seeded xoshiro256** bytes, generated on device)",
            "config": dict(workload_config(wl, world, args.variant), **({"output": f"buckets mod {args.buckets} + histogram"
                                                                     + (" + partition" if args.partition else "")}
                                                          if args.buckets else {}),
                           **({"api": f"pmp_stream_update in {args.stream_mib} MiB pieces"} if args.stream_mib else {})),
            "bytes_per_gpu_cycle": (value / world * 1e9) / (clocks["sm_mhz"] * 1e6) if clocks.get("sm_mhz") else None,
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes_per_launch, "avg_launch_ms": avg_ms,
                         "launches_timed": k_cnt,
                         # integer-pipe / issue utilisation of this kernel from the committed
                         # ncu capture (profiles/pipes.json), for the IMAD side of the roofline
                         "ncu_pipes": pipes},
            "clocks": clocks,
            "gpu_launches": launches,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kernel_ms.items() if v[1]},
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def fill_slice(seed, d_buf, start, sp):
    """Regenerate payload bytes [start, start + len) of the stream on device."""
    datagen.fill_device(seed, d_buf.data_ptr(), d_buf.numel(), sp, start=start)


def run_e2e(args, wl, pmp, keys, dev, stream, rank, world, cdev):
    import torch

    if wl.long:
        return None
    seed, lens, offs, b0 = make_batch(wl, rank)
    n = lens.size
    total = int(offs[-1])
    h_pay = torch.from_numpy(datagen.payload_host(seed, b0, total)).pin_memory()
    h_off = torch.from_numpy(offs.view(np.int64)).pin_memory()
    d_pay = torch.empty(total + 16, dtype=torch.uint8, device=dev)
    d_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    d_out = {b: torch.empty(n, dtype=torch.int64 if b == 64 else torch.int32, device=dev) for b in wl.bits}
    h_out = {b: torch.empty(n, dtype=d_out[b].dtype).pin_memory() for b in wl.bits}
    sp = int(stream.cuda_stream)

    host_api = args.variant == "tree"

    def step():
        if host_api:  # the public host-resident call: pieces stream H2D / hash / D2H overlapped
            pmp._check(pmp.pmp_hash_batch_host([keys[b].handle for b in wl.bits], h_pay.data_ptr(),
                                               h_off.data_ptr(), n, [h_out[b].data_ptr() for b in wl.bits],
                                               args.e2e_piece_mib << 20, sp), "e2e hash")
            return
        d_pay[:total].copy_(h_pay, non_blocking=True)
        d_off.copy_(h_off, non_blocking=True)
        for b in wl.bits:
            pmp._check(pmp.pmp_hash2_batch(keys[b].handle, d_pay.data_ptr(), d_off.data_ptr(), n,
                                           d_out[b].data_ptr(), sp), "e2e hash")
            h_out[b].copy_(d_out[b], non_blocking=True)

    step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.e2e_steps
    t = torch.tensor([ms], dtype=torch.float64, device=cdev)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": total * len(wl.bits) * world / (ms / 1000) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": total + 8 * (n + 1),
            "d2h_bytes_per_step": n * sum(b // 8 for b in wl.bits), "ms_per_step": ms,
            "path": (f"pmp_hash_batch_host (pinned host buffers, both widths in one pass, "
                     f"{args.e2e_piece_mib} MiB pieces: H2D / hash / D2H overlapped on 3 streams)" if host_api else
                     "pinned host -> cudaMemcpyAsync -> pmp_hash2_batch (both widths) -> host")}


def cpu_baseline(wl, variant="tree"):
    try:
        if wl.long:
            v, cores, desc, dt = oracle_long_rate(wl, 256 << 20, variant=variant)
        else:
            seed, lens, offs, b0 = make_batch(wl, 0, n=min(wl.n, 1 << 23))
            v, cores, desc, dt = oracle_sample_rate(wl, seed, offs, list(wl.bits), budget_s=10.0, base=b0,
                                                    variant=variant)
        return {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": desc,
                "seconds": dt, "host": host_cpu(), "single_thread": oracle_single_thread(wl, variant)}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": f"failed: {e}"}


def host_cpu():
    """CPU model, logical CPUs and sockets of the host the oracle ran on."""
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


def load_traffic(workload, kernel, name="traffic.json"):
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
