#!/usr/bin/env python3
"""Benchmark: RS(2^16, 2^15) GF(2^16) encode + erasure-decode on B200.

Default workload (`--workload codec`, the BASELINE.json headline): one step =
encode 4096 codewords (config 3: 256 MiB of uint16 message, parity written
separately) + erasure-decode 4096 codewords with one shared pattern of 2^15
erased positions (config 4a), per GPU.  Multi-GPU is weak scaling: rank r owns
codewords [r*4096, (r+1)*4096), no collective on the data path;
the timed region is bracketed by barrier + synchronize and the reported time
is the max over ranks.

  value      = message bytes encoded + decoded (2 * k * 2 B per codeword, all
               ranks) / max-over-ranks step time, GB/s (1e9)
  e2e        = the same metric through the public API with pinned HOST
               buffers (H2D of message / received words and D2H of parity /
               decoded messages inside the timed region)
  roofline   = dominant kernel (pass_kernel, the encode's 5 tile passes):
               algorithmic bytes per launch (4 B per symbol-position: 2 B read +
               2 B write, SURVEY §8d "transform pass: 4h bytes per polynomial")
               / average launch duration (CUDA events on the launch stream), vs
               measured HBM copy bandwidth
  cpu_baseline = the C oracle (restated reference algorithm) on the host cores,
               rank 0, bounded sample

Other §8 rows (auxiliary lines, same JSON keys):
  --workload stripe --rate 1/2|3/4|15/16   config 5: 4 KiB packets, 32 GiB of
               message split over the GPUs (strong scaling), per-stripe-group
               erasure patterns of n-k packets
  --workload transform                     config 2: forward + inverse +
               derivative, h = 2^16, 1024 polynomials per GPU
  --workload pcw                           config 4b: decode 4096 codewords with
               per-codeword patterns
  --workload r8                            config 1: (256,128), 64 codewords

`--impl reference` times the reference's CPU path (oracle port, all host
threads) on the same config and prints the reference-arm JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)



# Rank plumbing is local to bench.py: the reference arm must not import the
# product package (whose __init__ maps liblch.so).
def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(values, device=None):
    """Element-wise max over all ranks (identity for one rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def gather_to_rank0(obj):
    """List of every rank's `obj` on rank 0 (None elsewhere); [obj] for one rank."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(obj, out, dst=0)
    return out


def codeword_shard(rank: int, world: int, per_rank: int) -> tuple[int, int]:
    """Weak scaling (configs 3/4): rank r owns codewords [r B, (r + 1) B)."""
    return rank * per_rank, (rank + 1) * per_rank


def group_shard(rank: int, world: int, total: int) -> tuple[int, int]:
    """Strong scaling (config 5): contiguous split of the stripe groups."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)

# NCCL for the driver's multi-GPU runs; LCH_DIST_BACKEND=gloo runs the same
# multi-rank logic (CPU collectives) e.g. with several ranks on one device.
DIST_BACKEND = os.environ.get("LCH_DIST_BACKEND", "nccl")


def dist_device():
    return "cuda" if DIST_BACKEND == "nccl" else "cpu"

R_BITS, N, K = 16, 1 << 16, 1 << 15
BATCH = 4096
SEED_MSG, SEED_ERA = 1404345803, 1404345804
SEED_CFG = {1: 1404345801, 2: 1404345802, 5: 1404345805}
METRIC = "RS(2^16,2^15) GF(2^16) encode & erasure-decode GB/s; % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
STRIPE = {"1/2": (1 << 15, 256), "3/4": (49152, 168), "15/16": (61440, 136)}  # k, groups
PKT = 2048
DATA = "synthetic (seeded counter-based generator, SURVEY §8d)"


def hbm_peak():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML every
    5 ms (nvidia_ml_py), else `nvidia-smi` every 100 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set(reasons))
        self._stop = threading.Event()
        self._th = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._phys_index(index))
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    @staticmethod
    def _phys_index(index: int) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[index])
            except Exception:
                return index
        return index

    def _sample_nvml(self):
        pynvml, h = self._nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
        self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))

    def _sample_smi(self):
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            f = [x.strip() for x in out.stdout.strip().split(",")]
            sm = float(f[0]) if f[0].replace(".", "").isdigit() else None
            mx = float(f[1]) if f[1].replace(".", "").isdigit() else None
            act = {nm for nm, v in zip(self.REASONS, f[4:8]) if v.strip().lower() == "active"}
            if sm is not None:
                self.samples.append((sm, mx or sm, act))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                self._nvml = None
            self._stop.wait(0.005 if self._nvml else 0.1)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)
        if not self.samples:  # a region shorter than one sample: take one now
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        reasons = set()
        for _, _, r in self.samples:
            reasons |= r
        return {"sm_mhz": float(np.median([x[0] for x in self.samples])),
                "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted(reasons), "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU legs (oracle = restated reference; bounded samples)

def _oracle_codec_seconds(orc, msgs, mask, nthreads):
    """(encode s, decode s) of the C oracle on `msgs` (configs 3 + 4a)."""
    t0 = time.perf_counter()
    par = orc.encode_batch(K, msgs, nthreads)
    t1 = time.perf_counter()
    rx = np.concatenate([msgs, par], axis=1)
    rx[:, mask == 1] = 0
    t2 = time.perf_counter()
    out = orc.decode_batch(K, rx, mask, nthreads)
    t3 = time.perf_counter()
    assert np.array_equal(out, msgs), "oracle round trip failed"
    return t1 - t0, t3 - t2


CPU_SAMPLE_CW = 256  # 256 codewords for configs 3 / 4a


def cpu_codec(sample_cw: int, nthreads: int, one_core_cw: int = 0, python_ref_cw: int = 0):
    """The oracle (C restatement of the reference algorithm) on a bounded
    sample of configs 3 + 4a: all host threads (`value`), optionally one core
    (`one_core`) and the reference's own Python BatchCodec (`reference_python`,
    when baseline/_ref is staged)."""
    from oracle import oracle as O
    orc = O.Oracle(16)
    msgs = O.gen_symbols(SEED_MSG, 16, 0, sample_cw, K)
    mask = O.gen_erasures(SEED_ERA, N, N - K, 0, 1)[0]
    es, ds = _oracle_codec_seconds(orc, msgs, mask, nthreads)
    res = {"value": round(sample_cw * 2 * K * 2 / (es + ds) / 1e9, 6), "unit": "GB/s",
           "cores": nthreads, "kind": "port",
           "sample": f"{sample_cw} codewords encode + {sample_cw} shared-pattern decodes "
                     f"(RS(2^16,2^15)), C oracle, {nthreads} threads",
           "sample_codewords": sample_cw, "encode_s": round(es, 3), "decode_s": round(ds, 3)}
    if one_core_cw:
        es1, ds1 = _oracle_codec_seconds(orc, msgs[:one_core_cw], mask, 1)
        res["one_core"] = {"value": round(one_core_cw * 2 * K * 2 / (es1 + ds1) / 1e9, 6), "unit": "GB/s",
                           "cores": 1, "sample_codewords": one_core_cw,
                           "encode_s": round(es1, 3), "decode_s": round(ds1, 3)}
    if python_ref_cw:
        pr = python_reference_codec(python_ref_cw)
        if pr:
            res["reference_python"] = pr
    return res


def python_reference_codec(sample_cw: int):
    """The reference's own BatchCodec (pure Python + numpy, batch.py:110-153)
    on one core, from the staged baseline/_ref (None if absent).  Its output
    is checked against the oracle's."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "binfec")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from binfec.basis import build_basis_tables
    from binfec.batch import BatchCodec
    from binfec.field import tables_for
    from binfec.rs import CodeParams
    from oracle import oracle as O
    t0 = time.perf_counter()
    codec = BatchCodec(CodeParams(16, K), build_basis_tables(tables_for(16), N))
    setup = time.perf_counter() - t0
    msgs = O.gen_symbols(SEED_MSG, 16, 0, sample_cw, K)
    mask = O.gen_erasures(SEED_ERA, N, N - K, 0, 1)[0]
    erased = set(np.nonzero(mask)[0].tolist())
    codec.decode(codec.encode(msgs[:1]), erased)  # warm the FWHT(log) cache (walsh.py:64-74)
    t0 = time.perf_counter()
    cw = codec.encode(msgs)
    t1 = time.perf_counter()
    out = codec.decode(cw, erased)
    t2 = time.perf_counter()
    orc = O.Oracle(16)
    assert np.array_equal(cw[:, K:], orc.encode_batch(K, msgs, 1)[:, :]), "reference != oracle"
    assert np.array_equal(out, msgs)
    return {"value": round(sample_cw * 2 * K * 2 / (t2 - t0) / 1e9, 6), "unit": "GB/s", "cores": 1,
            "kind": "reference", "sample_codewords": sample_cw,
            "sample": f"binfec.BatchCodec encode + decode of {sample_cw} codewords (baseline/_ref, "
                      "unmodified reference, one core)",
            "encode_s": round(t1 - t0, 3), "decode_s": round(t2 - t1, 3), "setup_s": round(setup, 3)}


def cpu_stripe(k: int, lanes: int, nthreads: int):
    """Config 5 lanes (one lane = one codeword) through the general-k oracle."""
    from oracle import oracle as O
    orc = O.Oracle(16)
    msgs = O.gen_symbols(SEED_CFG[5], 16, 0, lanes, k)
    mask = O.gen_erasures(SEED_CFG[5] ^ 0xE, N, N - k, 0, 1)[0]
    t0 = time.perf_counter()
    par = orc.encode_any_batch(k, msgs, nthreads)
    t1 = time.perf_counter()
    rx = np.concatenate([msgs, par], axis=1)
    rx[:, mask == 1] = 0
    t2 = time.perf_counter()
    out = orc.decode_any_batch(k, rx, mask, nthreads)
    t3 = time.perf_counter()
    assert np.array_equal(out, msgs), "oracle round trip failed"
    sec = (t1 - t0) + (t3 - t2)
    return {"value": round(lanes * 2 * k * 2 / sec / 1e9, 6), "unit": "GB/s", "cores": nthreads,
            "kind": "port",
            "sample": f"{lanes} packet lanes (codewords) of RS(2^16,{k}) encode + decode with "
                      f"{N - k} erasures, C oracle, {nthreads} threads"}


def cpu_transform(polys: int, nthreads: int):
    from oracle import oracle as O
    orc = O.Oracle(16)
    a = O.gen_symbols(SEED_CFG[2], 16, 0, polys, N)
    t0 = time.perf_counter()
    orc.transform_batch(a, 0, False, nthreads)
    orc.transform_batch(a, 0, True, nthreads)
    for b in range(polys):
        orc.derivative(a[b])
    sec = time.perf_counter() - t0
    return {"value": round(3 * polys * 4 * N / sec / 1e9, 6), "unit": "GB/s", "cores": nthreads,
            "kind": "port",
            "sample": f"{polys} polynomials h=2^16 forward + inverse ({nthreads} threads) + "
                      "derivative (1 thread), C oracle"}


def cpu_pcw(cws: int, nthreads: int):
    from oracle import oracle as O
    orc = O.Oracle(16)
    msgs = O.gen_symbols(SEED_MSG, 16, 0, cws, K)
    masks = O.gen_erasures(SEED_ERA, N, N - K, 0, cws)
    par = orc.encode_batch(K, msgs, nthreads)
    rx = np.concatenate([msgs, par], axis=1)
    rx[masks == 1] = 0
    t0 = time.perf_counter()
    out = orc.decode_batch(K, rx, masks, nthreads)
    sec = time.perf_counter() - t0
    assert np.array_equal(out, msgs)
    return {"value": round(cws * K * 2 / sec / 1e9, 6), "unit": "GB/s", "cores": nthreads,
            "kind": "port",
            "sample": f"{cws} per-codeword-pattern decodes RS(2^16,2^15), C oracle, {nthreads} threads"}


def cpu_r8(nthreads: int):
    from oracle import oracle as O
    orc = O.Oracle(8)
    msgs = O.gen_symbols(SEED_CFG[1], 8, 0, 64, 128)
    masks = O.gen_erasures(SEED_CFG[1] ^ 0xE, 256, 128, 0, 64)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        par = orc.encode_batch(128, msgs, 1)
        rx = np.concatenate([msgs, par], axis=1)
        out = orc.decode_batch(128, rx, masks, 1)
    sec = (time.perf_counter() - t0) / reps
    assert np.array_equal(out, msgs)
    return {"value": round(2 * 64 * 128 / sec / 1e9, 6), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": "64 codewords (256,128) encode + per-codeword decode, C oracle, 1 thread"}


# ---------------------------------------------------------------------------

def workload_config(wl: str, args, world: int) -> dict:
    """The `config` of a workload's JSON line (identical for both arms)."""
    if wl == "codec":
        return {"workload": "cfg3+cfg4a: RS(2^16,2^15) encode 4096 cw + shared-pattern decode "
                            "4096 cw (2^15 erasures) per GPU",
                "batch_per_gpu": args.batch, "n": N, "k": K, "parallelism": f"codeword-shard x{world}",
                "l2": "inputs larger than L2 (256 MiB message, 512 MiB received per GPU)"}
    if wl == "stripe":
        k, total = STRIPE[args.rate]
        total = args.groups or total
        lo, hi = group_shard(0, world, total)
        return {"workload": f"cfg5: storage stripes RS(2^16,{k}) (k/n={args.rate}), 4 KiB packets "
                            f"(P={PKT}), {total} stripe groups = {total * PKT * k * 2 / 2**30:.1f} GiB of "
                            "message over all GPUs; encode + decode with per-group patterns of n-k "
                            "erased packets",
                "k": k, "n": N, "packet_len": PKT, "groups_total": total, "groups_per_gpu": hi - lo,
                "parallelism": f"stripe-group shard x{world}", "l2": "inputs larger than L2"}
    if wl == "transform":
        return {"workload": "cfg2: forward + inverse + derivative, h=2^16, 1024 polynomials per GPU",
                "h": N, "batch_per_gpu": 1024, "parallelism": f"polynomial-shard x{world}"}
    if wl == "pcw":
        return {"workload": "cfg4b: RS(2^16,2^15) decode 4096 cw, per-codeword patterns of 2^15 erasures",
                "batch_per_gpu": args.batch, "n": N, "k": K, "parallelism": f"codeword-shard x{world}"}
    return {"workload": "cfg1: GF(2^8) (256,128) encode + per-codeword decode, 64 cw per GPU",
            "batch_per_gpu": 64, "n": 256, "k": 128}


def run_reference_arm(args):
    """The reference's CPU path on the host cores, on the GPU arm's exact
    config: each step times a bounded sample of the workload with all host
    threads (the reference is pure Python; its algorithm runs here as the C
    oracle port, oracle/lch_oracle.c, pinned to the reference's outputs), and
    the line reports the sample's measured rate and time per step."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    nth = cpu_threads()
    wl = args.workload
    if wl == "codec":
        sample = CPU_SAMPLE_CW
        step = lambda: cpu_codec(sample, nth)  # noqa: E731
        unit = f"{sample} codewords (of the {args.batch} per GPU) encode + shared-pattern decode"
    elif wl == "stripe":
        k, _ = STRIPE[args.rate]
        step = lambda: cpu_stripe(k, 64, nth)  # noqa: E731
        unit = "64 packet lanes (codewords) of one stripe group, encode + decode"
    elif wl == "transform":
        step = lambda: cpu_transform(max(nth, 8), nth)  # noqa: E731
        unit = f"{max(nth, 8)} of the 1024 polynomials, forward + inverse + derivative"
    elif wl == "pcw":
        step = lambda: cpu_pcw(max(nth, 16), nth)  # noqa: E731
        unit = f"{max(nth, 16)} of the {args.batch} codewords, per-codeword-pattern decode"
    else:
        step = lambda: cpu_r8(nth)  # noqa: E731
        unit = "all 64 codewords, encode + per-codeword decode"
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    vals = [step() for _ in range(args.steps)]
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    v = float(np.median([x["value"] for x in vals]))
    cb = dict(vals[-1])
    cb["value"] = round(v, 6)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
            "data": DATA, "config": workload_config(wl, args, args.gpus),
            "sample_per_step": unit + f" on {nth} host threads (ms_per_step is the sample's time)",
            "cpu_baseline": cb,
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if wl == "codec" and not args.no_cpu:
        pr = python_reference_codec(16)
        if pr:
            line["reference_python"] = pr
    print(json.dumps(line), flush=True)
    return 0


class Timer:
    """Per-phase CUDA-event timing of `steps` steps on the launch stream."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream

    def ev(self):
        return self.torch.cuda.Event(enable_timing=True)

    def run(self, phases, steps, warmup, world, local, lib, ctx):
        torch, dist = self.torch, None
        if world > 1:
            import torch.distributed as dist
        for _ in range(warmup):
            for _, fn in phases:
                fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n0 = lib.lch_launch_count(ctx)
        marks = []
        with ClockSampler(local) as clk:
            t0 = self.ev()
            t0.record(self.stream)
            for _ in range(steps):
                evs = [self.ev() for _ in range(len(phases) + 1)]
                evs[0].record(self.stream)
                for i, (_, fn) in enumerate(phases):
                    fn()
                    evs[i + 1].record(self.stream)
                marks.append(evs)
            t1 = self.ev()
            t1.record(self.stream)
            torch.cuda.synchronize()
        launches = lib.lch_launch_count(ctx) - n0
        step_ms = t0.elapsed_time(t1) / steps
        ph = [float(np.mean([m[i].elapsed_time(m[i + 1]) for m in marks])) for i in range(len(phases))]
        if world > 1:
            vals = max_over_ranks([step_ms] + ph, dist_device())
            step_ms, ph = vals[0], vals[1:]
        return step_ms, dict(zip([n for n, _ in phases], ph)), int(launches), clk.summary()


def read_profile():
    """Per-launch DRAM traffic and ALU-pipe occupancy of the pass kernel from
    the committed ncu capture (profiles/pass_kernel_traffic.json)."""
    tfile = os.path.join(ROOT, "profiles", "pass_kernel_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                return json.load(fh)
        except Exception:
            return {}
    return {}


def read_traffic():
    return read_profile().get("dram_bytes_per_launch")


def base_line(args, world, value, step_ms, cfg, launches, clocks, scaling="weak"):
    return {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u16",
            "data": DATA, "config": cfg, "gpu_launches": launches, "clocks": clocks}


def roofline(name, alg_bytes, ms, peak, peak_src, traffic=None):
    ach = alg_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": name, "achieved": round(ach, 2), "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": traffic, "algorithmic_bytes_per_launch": alg_bytes,
            "avg_launch_ms": round(ms, 4)}


# ---------------------------------------------------------------------------

def run_codec(args, torch, lch, _lib, world, rank, local):
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, encode_device
    B = args.batch
    ft = lch.tables_for(16)
    bt = lch.build_basis_tables(ft, N)
    cp = lch.CodeParams(16, K)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    cw0, _ = codeword_shard(rank, world, B)

    # inputs resident in HBM (weak scaling: each rank owns its own codewords)
    msg = torch.empty((B, K), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_gen_symbols(ctx, SEED_MSG, cw0, B, K, msg.data_ptr(), K,
                                        stream.cuda_stream))
    cw = torch.empty((B, N), dtype=torch.int16, device="cuda")
    cw[:, :K].copy_(msg)
    parity = cw[:, K:]
    emask = gen.erasure_masks(bt.ctx, SEED_ERA, N, N - K, 0, 1)  # shared pattern (cw index 0)
    bits = gen.mask_to_bits(emask)[0].contiguous()
    out = torch.empty((B, K), dtype=torch.int16, device="cuda")
    era_cols = torch.nonzero(emask[0]).flatten()

    def step_encode():
        encode_device(cp, bt, msg, parity)

    def step_decode():
        decode_device(cp, bt, cw, bits, out, N - K)

    # correctness gate (full batch): decode(encode(m)) == m
    step_encode()
    rx = cw.clone()
    rx[:, era_cols] = 0
    decode_device(cp, bt, rx, bits, out, N - K)
    torch.cuda.synchronize()
    if not bool(torch.equal(out, msg)):
        print(json.dumps({"error": "round trip failed", "rank": rank}), flush=True)
        return None

    phases = []
    if args.only in ("", "encode"):
        phases.append(("encode", step_encode))
    if args.only in ("", "decode"):
        phases.append(("decode", step_decode))
    step_ms, ph, launches, clocks = Timer(torch, stream).run(phases, args.steps, args.warmup, world,
                                                             local, _lib.lib, ctx)
    msg_bytes = B * K * 2
    value = world * len(phases) * msg_bytes / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    enc, dec = ph.get("encode"), ph.get("decode")
    codec_alg = 2 * N * B  # SURVEY §8d encode: read k + write n-k symbols (2 B each) per codeword
    dec_alg = (2 * (N - K) + 2 * K) * B  # decode: read n-|E| survivors + write k
    cfg = workload_config("codec", args, world)
    res = base_line(args, world, value, step_ms, cfg, launches, clocks)
    res.update({
        "encode_ms": round(enc, 4) if enc else None, "decode_ms": round(dec, 4) if dec else None,
        "encode_gbs": round(world * msg_bytes / (enc * 1e-3) / 1e9, 3) if enc else None,
        "decode_gbs": round(world * msg_bytes / (dec * 1e-3) / 1e9, 3) if dec else None,
        "encode_symbols_per_s": round(B * K * world / (enc * 1e-3), 1) if enc else None,
        "decode_symbols_per_s": round(B * K * world / (dec * 1e-3), 1) if dec else None,
        "encode_hbm_frac": round(codec_alg / (enc * 1e-3) / 1e9 / peak, 4) if enc else None,
        "decode_hbm_frac": round(dec_alg / (dec * 1e-3) / 1e9 / peak, 4) if dec else None,
    })
    if enc:
        # the encode's algorithmic bytes over the summed duration of
        # the dominant kernel's launches in it (all 5 launches of an RS(2^16,
        # 2^15) encode are pass_kernel instances, so that sum is the encode time)
        prof = read_profile()
        enc_traffic = sum(prof["per_launch"]) if prof.get("per_launch") else None
        res["roofline"] = roofline("pass_kernel<16,0x1100B> (the 5 launches of one encode)", codec_alg,
                                   enc, peak, peak_src, enc_traffic)
        res["roofline"]["traffic_note"] = ("ncu dram bytes read+write summed over the 5 launches of one encode "
                                           "(each pass streams its own 512 MiB)")
        res["roofline"]["launches_per_unit"] = 5
        res["roofline"]["unit_of_work"] = f"one encode of {B} codewords (2n B per codeword)"
        res["pass_dram_efficiency"] = {
            "what": "per-pass bytes (4 B per symbol-position: 2 B read + 2 B write) / mean pass time, "
                    "vs measured HBM peak -- how close each pass is to streaming, not codec progress",
            "achieved_gbs": round(4 * K * B / (enc / 5 * 1e-3) / 1e9, 1),
            "frac": round(4 * K * B / (enc / 5 * 1e-3) / 1e9 / peak, 4)}
    prof = read_profile()
    if enc:
        # the integer-ALU floor of the encode: 458,753
        # GF(2^16) multiplies per codeword at 157 LOP3 per
        # 1024 symbol-multiplies, plus the raw-tile bit transposes (~0.146
        # warp-instructions per symbol, in and out), at 2 cycles per warp-
        # instruction per SM sub-partition, 148 SMs, max SM clock
        clk = (res.get("clocks") or {}).get("sm_max_mhz") or 1965.0
        warp_instr = 458753 * B / 1024 * 157 + 2 * K * B * 0.146
        floor_ms = warp_instr / (148 * 4 * 0.5 * clk * 1e6) * 1e3
        res["compute_roofline"] = {
            "bound": "alu", "pipe": "integer ALU (LOP3 bit-sliced GF(2^16) multiplies)",
            "floor_ms": round(floor_ms, 4), "achieved_ms": round(enc, 4),
            "frac": round(floor_ms / enc, 4),
            "hbm_frac_ceiling": round(codec_alg / (floor_ms * 1e-3) / 1e9 / peak, 4),
            "what": "encode time at 100 % ALU pipe (the arithmetic floor of this bit-sliced design) over the "
                    "measured encode time; hbm_frac_ceiling = the HBM roofline fraction that floor allows"}
        if prof.get("alu_pipe_pct_per_launch"):
            alu = prof["alu_pipe_pct_per_launch"]
            res["compute_roofline"]["alu_busy_frac_ncu"] = round(sum(alu) / len(alu) / 100.0, 3)
            res["compute_roofline"]["source"] = prof.get("source", "ncu --set full (profiles/)")

    # e2e through the public host-buffer API (lch_encode_host / lch_decode_host:
    # chunked H2D / kernels / D2H overlapped on three streams), pinned buffers
    if not args.no_e2e:
        import torch.distributed as dist
        from paper_1404_3458_b200.rs import decode_host, encode_host
        h_msg = msg.cpu().pin_memory()
        h_par = torch.empty((B, N - K), dtype=torch.int16, pin_memory=True)
        h_rx = rx.cpu().pin_memory()
        h_out = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
        h_bits = bits.cpu().numpy().view(np.uint32).copy()

        def e2e_step():
            encode_host(cp, bt, h_msg, h_par)
            decode_host(cp, bt, h_rx, h_bits, h_out)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        def copied():
            import ctypes
            h2d, d2h = ctypes.c_uint64(0), ctypes.c_uint64(0)
            _lib.check(_lib.lib.lch_host_copy_bytes(ctx, ctypes.byref(h2d), ctypes.byref(d2h)))
            return h2d.value, d2h.value

        tm = Timer(torch, stream)
        a, b = tm.ev(), tm.ev()
        c0 = copied()
        a.record(stream)
        e2e_steps = max(1, min(args.steps, 5))
        for _ in range(e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        c1 = copied()
        e2e_ms = a.elapsed_time(b) / e2e_steps
        per_rank = gather_to_rank0(round(e2e_ms, 3))
        if world > 1:
            e2e_ms = max_over_ranks([e2e_ms], dist_device())[0]
        assert torch.equal(h_out, h_msg), "e2e round trip failed"
        assert torch.equal(h_par, parity.cpu()), "e2e parity differs from the device path"
        # bytes counted by the library from the copies it queued (a chunk of the
        # received words crosses PCIe compacted to its survivors, or as it is)
        res["e2e"] = {"value": round(world * 2 * msg_bytes / (e2e_ms * 1e-3) / 1e9, 3),
                      "unit": "GB/s", "h2d_bytes_per_step": (c1[0] - c0[0]) // e2e_steps,
                      "d2h_bytes_per_step": (c1[1] - c0[1]) // e2e_steps,
                      "ms_per_step": round(e2e_ms, 3), "ms_per_step_per_rank": per_rank,
                      "api": "lch_encode_host + lch_decode_host (pinned host buffers; chunked "
                             "H2D / kernel / D2H overlap on three streams, steps queued back to "
                             "back; a chunk of the received words is compacted to its survivors "
                             "on the host -- erased symbols, which the decoder ignores, then do "
                             "not cross PCIe -- while copies are still queued, and sent as it is "
                             "when the copy stream has run dry)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        nth = cpu_threads()
        res["cpu_baseline"] = cpu_codec(CPU_SAMPLE_CW, nth, one_core_cw=CPU_SAMPLE_CW, python_ref_cw=16)
    return res


def run_stripe(args, torch, lch, _lib, world, rank, local):
    """Config 5: codeword buffer [G, n, P] per GPU, message = positions [0, k)."""
    from paper_1404_3458_b200 import gen
    k, groups_total = STRIPE[args.rate]
    if args.groups:
        groups_total = args.groups
    g_lo, g_hi = group_shard(rank, world, groups_total)  # strong scaling: 32 GiB total
    G = g_hi - g_lo
    bt = lch.build_basis_tables(lch.tables_for(16), N)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    lanes = G * PKT
    cw = torch.empty((G, N, PKT), dtype=torch.int16, device="cuda")
    # message packets: lane g * P + t of group g is codeword (g_lo * P + lane)
    _lib.check(_lib.lib.lch_gen_packets(ctx, SEED_CFG[5], g_lo * PKT, lanes, k, cw.data_ptr(), N,
                                        PKT, s))
    out = torch.empty((G, k, PKT), dtype=torch.int16, device="cuda")
    masks = gen.erasure_masks(bt.ctx, SEED_CFG[5] ^ 0xE, N, N - k, g_lo, G)  # one per group
    bits = gen.mask_to_bits(masks).contiguous()
    counts = (torch.full((G,), N - k, dtype=torch.int64)).numpy()
    import ctypes
    cnt = (ctypes.c_int64 * G)(*[int(x) for x in counts])
    par_ptr = cw.data_ptr() + k * PKT * 2

    def step_encode():
        _lib.check(_lib.lib.lch_encode_k(ctx, cw.data_ptr(), N, par_ptr, N, lanes, k, PKT, s))

    def step_decode():
        _lib.check(_lib.lib.lch_decode_k(ctx, cw.data_ptr(), N, bits.data_ptr(), 0, out.data_ptr(), k,
                                         lanes, k, PKT, cnt, s))

    step_encode()
    step_decode()
    torch.cuda.synchronize()
    if not bool(torch.equal(out, cw[:, :k, :])):
        print(json.dumps({"error": "stripe round trip failed", "rank": rank}), flush=True)
        return None
    phases = [("encode", step_encode), ("decode", step_decode)]
    step_ms, ph, launches, clocks = Timer(torch, stream).run(phases, args.steps, args.warmup, world,
                                                             local, _lib.lib, ctx)
    msg_bytes = lanes * k * 2
    total_msg = groups_total * PKT * k * 2
    value = 2 * total_msg / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    enc, dec = ph["encode"], ph["decode"]
    cfg = workload_config("stripe", args, world)
    cfg["groups_per_gpu"] = G
    res = base_line(args, world, value, step_ms, cfg, launches, clocks, scaling="strong")
    res.update({
        "encode_ms": round(enc, 3), "decode_ms": round(dec, 3),
        "encode_gbs": round(world * msg_bytes / (enc * 1e-3) / 1e9, 3),
        "decode_gbs": round(world * msg_bytes / (dec * 1e-3) / 1e9, 3),
        "encode_hbm_frac": round(lanes * 2 * N / (enc * 1e-3) / 1e9 / peak, 4),
        "decode_hbm_frac": round(lanes * 2 * N / (dec * 1e-3) / 1e9 / peak, 4),
        "roofline": roofline("encode (whole pipeline, algorithmic 2n B per lane)", lanes * 2 * N, enc,
                             peak, peak_src),
        "e2e": None,
    })
    if not args.no_e2e:
        # host-buffer API (lch_encode_host / lch_decode_host, packet layout) on a
        # pinned subset of the stripe groups (pinning 32 GiB would dominate the run)
        import torch.distributed as dist
        import ctypes as C
        Ge = min(G, 8)
        h_cw = cw[:Ge].cpu().pin_memory()
        h_out = torch.empty((Ge, k, PKT), dtype=torch.int16, pin_memory=True)
        h_bits = bits[:Ge].cpu().numpy().view(np.uint32).copy()
        h_par = torch.empty((Ge, N - k, PKT), dtype=torch.int16, pin_memory=True)
        le = Ge * PKT

        def e2e_step():
            _lib.check(_lib.lib.lch_encode_host(ctx, h_cw.data_ptr(), N, h_par.data_ptr(), N - k, le, k, PKT, 0,
                                                s))
            _lib.check(_lib.lib.lch_decode_host(ctx, h_cw.data_ptr(), N, h_bits.ctypes.data, 0, h_out.data_ptr(),
                                                k, le, k, PKT, 0, s))

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        def copied():
            h2d, d2h = C.c_uint64(0), C.c_uint64(0)
            _lib.check(_lib.lib.lch_host_copy_bytes(ctx, C.byref(h2d), C.byref(d2h)))
            return h2d.value, d2h.value

        tm = Timer(torch, stream)
        a, b = tm.ev(), tm.ev()
        c0 = copied()
        a.record(stream)
        for _ in range(2):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        c1 = copied()
        e2e_ms = a.elapsed_time(b) / 2
        if world > 1:
            e2e_ms = max_over_ranks([e2e_ms], dist_device())[0]
        assert torch.equal(h_out, h_cw[:, :k]), "stripe e2e round trip failed"
        assert torch.equal(h_par, h_cw[:, k:]), "stripe e2e parity differs"
        res["e2e"] = {"value": round(world * 2 * le * k * 2 / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                      "h2d_bytes_per_step": (c1[0] - c0[0]) // 2,
                      "d2h_bytes_per_step": (c1[1] - c0[1]) // 2,
                      "ms_per_step": round(e2e_ms, 3),
                      "sample": f"{Ge} stripe groups per GPU ({Ge * PKT * k * 2 / 2**30:.2f} GiB of message), "
                                "pinned host buffers"}
    if rank == 0 and world == 1 and not args.no_cpu:
        nth = cpu_threads()
        res["cpu_baseline"] = cpu_stripe(k, max(8, min(nth, 64)), nth)
    return res


def run_transform_wl(args, torch, lch, _lib, world, rank, local):
    """Config 2: forward + inverse + derivative, h = 2^16, 1024 polynomials per GPU."""
    from paper_1404_3458_b200.derivative import run_derivative
    from paper_1404_3458_b200.transform import run_transform
    B = 1024
    bt = lch.build_basis_tables(lch.tables_for(16), N)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    a = torch.empty((B, N), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_gen_symbols(ctx, SEED_CFG[2], rank * B, B, N, a.data_ptr(), N,
                                        stream.cuda_stream))
    a0 = a.clone()
    d = torch.empty_like(a)
    run_transform(bt, a, 0, False)
    run_transform(bt, a, 0, True)
    torch.cuda.synchronize()
    if not bool(torch.equal(a, a0)):
        print(json.dumps({"error": "transform round trip failed"}), flush=True)
        return None
    phases = [("forward", lambda: run_transform(bt, a, 0, False)),
              ("inverse", lambda: run_transform(bt, a, 0, True)),
              ("derivative", lambda: run_derivative(bt, a, d))]
    step_ms, ph, launches, clocks = Timer(torch, stream).run(phases, args.steps, args.warmup, world,
                                                             local, _lib.lib, ctx)
    per = 4 * N * B  # 4h bytes per polynomial per pass
    value = world * 3 * per / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    cfg = workload_config("transform", args, world)
    res = base_line(args, world, value, step_ms, cfg, launches, clocks)
    res.update({f"{k}_ms": round(v, 4) for k, v in ph.items()})
    res.update({f"{k}_gbs": round(world * per / (v * 1e-3) / 1e9, 2) for k, v in ph.items()})
    res["roofline"] = roofline("forward transform (4 passes)", per, ph["forward"], peak, peak_src)
    res["e2e"] = None
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_transform(max(8, cpu_threads()), cpu_threads())
    return res


def run_pcw(args, torch, lch, _lib, world, rank, local):
    """Config 4b: decode 4096 codewords, one erasure pattern per codeword."""
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, encode_device
    B = args.batch
    bt = lch.build_basis_tables(lch.tables_for(16), N)
    cp = lch.CodeParams(16, K)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    msg = torch.empty((B, K), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_gen_symbols(ctx, SEED_MSG, rank * B, B, K, msg.data_ptr(), K,
                                        stream.cuda_stream))
    cw = torch.empty((B, N), dtype=torch.int16, device="cuda")
    cw[:, :K].copy_(msg)
    encode_device(cp, bt, msg, cw[:, K:])
    masks = gen.erasure_masks(bt.ctx, SEED_ERA, N, N - K, rank * B, B)
    bits = gen.mask_to_bits(masks).contiguous()
    cw[masks] = 0
    out = torch.empty((B, K), dtype=torch.int16, device="cuda")
    counts = [N - K] * B
    step = lambda: decode_device(cp, bt, cw, bits, out, counts)  # noqa: E731
    step()
    torch.cuda.synchronize()
    if not bool(torch.equal(out, msg)):
        print(json.dumps({"error": "pcw round trip failed"}), flush=True)
        return None
    step_ms, ph, launches, clocks = Timer(torch, stream).run([("decode", step)], args.steps,
                                                             args.warmup, world, local, _lib.lib, ctx)
    value = world * B * K * 2 / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    cfg = workload_config("pcw", args, world)
    res = base_line(args, world, value, step_ms, cfg, launches, clocks)
    alg = (2 * K + 2 * K + N // 8) * B
    res["roofline"] = roofline("decode pipeline (algorithmic: survivors + output + bitmask)", alg,
                               ph["decode"], peak, peak_src)
    res["e2e"] = None
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_pcw(max(8, min(cpu_threads(), 32)), cpu_threads())
    return res


def run_r8(args, torch, lch, _lib, world, rank, local):
    """Config 1: GF(2^8) (256,128), 64 codewords, 128 per-codeword erasures."""
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, encode_device
    B, n, k = 64, 256, 128
    bt = lch.build_basis_tables(lch.tables_for(8), n)
    cp = lch.CodeParams(8, k)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    msg = gen.symbols(bt.ctx, SEED_CFG[1], rank * B, B, k)
    cw = torch.empty((B, n), dtype=torch.int16, device="cuda")
    cw[:, :k].copy_(msg)
    masks = gen.erasure_masks(bt.ctx, SEED_CFG[1] ^ 0xE, n, n - k, rank * B, B)
    bits = gen.mask_to_bits(masks).contiguous()
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    counts = [n - k] * B

    def step_enc():
        encode_device(cp, bt, msg, cw[:, k:])

    def step_dec():
        decode_device(cp, bt, cw, bits, out, counts)

    step_enc()
    step_dec()
    torch.cuda.synchronize()
    if not bool(torch.equal(out, msg)):
        print(json.dumps({"error": "r8 round trip failed"}), flush=True)
        return None
    # 64 codewords are launch-latency bound: replay each phase as a CUDA graph
    # (one small-codeword kernel per phase, captured through the C ABI)
    graphs = []
    for fn in (step_enc, step_dec):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        graphs.append(g)
    torch.cuda.synchronize()
    out.zero_()
    graphs[0].replay()
    graphs[1].replay()
    torch.cuda.synchronize()
    if not bool(torch.equal(out, msg)):
        print(json.dumps({"error": "r8 graph round trip failed"}), flush=True)
        return None
    stream = torch.cuda.current_stream()
    step_ms, ph, launches, clocks = Timer(torch, stream).run(
        [("encode", graphs[0].replay), ("decode", graphs[1].replay)], args.steps, args.warmup, world,
        local, _lib.lib, ctx)
    launches = 2 * args.steps  # one kernel per phase inside the graphs
    value = world * 2 * B * k / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    cfg = workload_config("r8", args, world)
    cfg["note"] = "small-codeword kernel, one CTA per codeword, phases replayed as CUDA graphs"
    res = base_line(args, world, value, step_ms, cfg, launches, clocks)
    res.update({"encode_ms": round(ph["encode"], 4), "decode_ms": round(ph["decode"], 4)})
    res["roofline"] = roofline("encode (latency bound)", 2 * n * B, ph["encode"], peak, peak_src)
    res["e2e"] = None
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_r8(cpu_threads())
    return res


AUX_KEYS = ("value", "unit", "ms_per_step", "encode_ms", "decode_ms", "forward_ms", "inverse_ms",
            "derivative_ms", "encode_gbs", "decode_gbs", "forward_gbs", "inverse_gbs", "derivative_gbs",
            "encode_hbm_frac", "decode_hbm_frac", "gpu_launches", "scaling", "clocks")


def run_aux(args, torch, lch, _lib, world, rank, local):
    """The other BASELINE configs (1, 2, 4b, 5 at all three rates), each on its
    full per-GPU shape with a few steps, so the default run reports every
    config (each function gates its timing on a full-batch round trip)."""
    import copy
    res = {}
    todo = [("cfg1_r8", run_r8, {}), ("cfg2_transform", run_transform_wl, {}), ("cfg4b_pcw", run_pcw, {}),
            ("cfg5_rate_1_2", run_stripe, {"rate": "1/2"}), ("cfg5_rate_3_4", run_stripe, {"rate": "3/4"}),
            ("cfg5_rate_15_16", run_stripe, {"rate": "15/16"})]
    for name, fn, extra in todo:
        a = copy.copy(args)
        a.__dict__.update(steps=max(1, min(args.steps, 3)), warmup=3, no_cpu=True, no_e2e=True, **extra)
        try:
            r = fn(a, torch, lch, _lib, world, rank, local)
        except Exception as exc:  # report, keep the headline line
            r = {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if r is None:
            r = {"error": "round-trip check failed"}
        ent = {k: r[k] for k in AUX_KEYS if k in r}
        if "error" in r:
            ent["error"] = r["error"]
        if "config" in r:
            ent["workload"] = r["config"]["workload"]
        if r.get("roofline"):
            ent["roofline_frac"] = r["roofline"]["frac"]
        ent["steps"], ent["warmup"] = a.steps, a.warmup
        res[name] = ent
    return res


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks (one process per GPU, NCCL)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} but only {have} CUDA devices visible"}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lch", choices=["lch", "reference"])
    ap.add_argument("--workload", default="codec", choices=["codec", "stripe", "transform", "pcw", "r8"])
    ap.add_argument("--rate", default="1/2", choices=sorted(STRIPE))
    ap.add_argument("--groups", type=int, default=0, help="stripe groups (default: 32 GiB)")
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-aux", action="store_true", help="skip the other configs' keys")
    ap.add_argument("--only", default="", help="encode|decode (profiling runs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference_arm(args)

    launched = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not launched:
        return spawn_ranks(args.gpus)
    rank, world, local = env_rank()
    if launched and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        if DIST_BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(DIST_BACKEND)
    dev = torch.cuda.current_device()
    props = torch.cuda.get_device_properties(dev)
    # one line per rank (stderr): which device each rank drives, and the
    # communicator size it sees
    print(json.dumps({"rank": rank, "local_rank": local, "world_size": world, "device": dev,
                      "device_name": props.name, "pci_bus_id": getattr(props, "pci_bus_id", None),
                      "comm_size": dist.get_world_size() if dist.is_initialized() else 1,
                      "backend": DIST_BACKEND if world > 1 else None}), file=sys.stderr, flush=True)
    import paper_1404_3458_b200 as lch
    from paper_1404_3458_b200 import _lib

    fn = {"codec": run_codec, "stripe": run_stripe, "transform": run_transform_wl, "pcw": run_pcw,
          "r8": run_r8}[args.workload]
    res = fn(args, torch, lch, _lib, world, rank, local)
    if res is not None and args.workload == "codec" and not args.no_aux and not args.only:
        torch.cuda.empty_cache()
        res["other_configs"] = run_aux(args, torch, lch, _lib, world, rank, local)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if res is None:
        return 1
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
