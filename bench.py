#!/usr/bin/env python3
"""Benchmark: RS(2^16, 2^15) GF(2^16) encode + erasure-decode on B200.

One step = encode 4096 codewords (config 3: 256 MiB of uint16 message, parity
written separately) + erasure-decode 4096 codewords with one shared pattern of
2^15 erased positions (config 4a), per GPU.  Multi-GPU is weak scaling: rank
r owns codewords [r*4096, (r+1)*4096), no collective on the data
path; the timed region is bracketed by barrier + synchronize and the reported
time is the max over ranks.

  value      = message bytes encoded + decoded (2 * k * 2 B per codeword, all
               ranks) / max-over-ranks step time, GB/s (1e9)
  e2e        = the same metric through the public API with pinned HOST
               buffers (H2D of message / received words and D2H of parity /
               decoded messages inside the timed region)
  roofline   = dominant kernel (pass_kernel, the encode's 5 tile passes):
               algorithmic bytes per launch (4 B per symbol-position: 2 B read +
               2 B write, SURVEY §8d "transform pass: 4h bytes per polynomial")
               / average launch duration, vs measured HBM copy bandwidth
  cpu_baseline = the C oracle (restated reference algorithm) on the host cores,
               rank 0, bounded sample

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

R_BITS, N, K = 16, 1 << 16, 1 << 15
BATCH = 4096
SEED_MSG, SEED_ERA = 1404345803, 1404345804
METRIC = "RS(2^16,2^15) GF(2^16) encode & erasure-decode GB/s; % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference(sample_cw: int, nthreads: int):
    """Time the oracle (restated reference) encode + shared-pattern decode."""
    from oracle import oracle as O
    orc = O.Oracle(16)
    msgs = O.gen_symbols(SEED_MSG, 16, 0, sample_cw, K)
    mask = O.gen_erasures(SEED_ERA, N, N - K, 0, 1)[0]
    t0 = time.perf_counter()
    par = orc.encode_batch(K, msgs, nthreads)
    t1 = time.perf_counter()
    rx = np.concatenate([msgs, par], axis=1)
    rx[:, mask == 1] = 0
    t2 = time.perf_counter()
    out = orc.decode_batch(K, rx, mask, nthreads)
    t3 = time.perf_counter()
    assert np.array_equal(out, msgs), "oracle round trip failed"
    sec = (t1 - t0) + (t3 - t2)
    gbs = sample_cw * 2 * K * 2 / sec / 1e9
    return {"value": round(gbs, 6), "unit": "GB/s", "cores": nthreads, "kind": "port",
            "sample": f"{sample_cw} codewords encode + {sample_cw} shared-pattern decodes "
                      f"(RS(2^16,2^15)), C oracle, {nthreads} threads",
            "encode_s": round(t1 - t0, 3), "decode_s": round(t3 - t2, 3)}


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    nth = cpu_threads()
    sample = max(nth, 16)
    vals = []
    for _ in range(max(args.warmup, 0) and 1):
        cpu_reference(min(sample, 16), nth)
    for _ in range(args.steps):
        vals.append(cpu_reference(sample, nth))
    v = float(np.median([x["value"] for x in vals]))
    cb = dict(vals[-1])
    cb["value"] = round(v, 6)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(BATCH * 2 * K * 2 / (v * 1e9) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic (seeded counter-based generator, SURVEY §8d)",
            "config": {"workload": "cfg3+cfg4a: RS(2^16,2^15) encode 4096 cw + shared-pattern "
                                   "decode 4096 cw (2^15 erasures) per GPU; CPU arm times a "
                                   f"{sample}-codeword sample and extrapolates the rate",
                       "batch_per_gpu": BATCH, "n": N, "k": K},
            "cpu_baseline": cb,
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lch", choices=["lch", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--only", default="", help="encode|decode (profiling runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1404_3458_b200 as lch
    from paper_1404_3458_b200 import _lib
    from paper_1404_3458_b200.rs import decode_device, encode_device

    B = args.batch
    ft = lch.tables_for(16)
    bt = lch.build_basis_tables(ft, N)
    cp = lch.CodeParams(16, K)
    ctx = bt.ctx.handle
    stream = torch.cuda.current_stream()
    cw0 = rank * B

    # inputs resident in HBM (weak scaling: each rank owns its own codewords)
    msg = torch.empty((B, K), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_gen_symbols(ctx, SEED_MSG, cw0, B, K, msg.data_ptr(), K,
                                        stream.cuda_stream))
    cw = torch.empty((B, N), dtype=torch.int16, device="cuda")
    cw[:, :K].copy_(msg)
    parity = cw[:, K:]
    from paper_1404_3458_b200 import gen
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
    ok = bool(torch.equal(out, msg))
    if not ok:
        print(json.dumps({"error": "round trip failed", "rank": rank}), flush=True)
        return 1

    do_enc = args.only in ("", "encode")
    do_dec = args.only in ("", "decode")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for _ in range(args.warmup):
        if do_enc:
            step_encode()
        if do_dec:
            step_decode()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n0 = _lib.lib.lch_launch_count(ctx)
    enc_ms, dec_ms = [], []
    with ClockSampler(local) as clk:
        t_start = ev()
        t_start.record(stream)
        for _ in range(args.steps):
            e0, e1, e2 = ev(), ev(), ev()
            e0.record(stream)
            if do_enc:
                step_encode()
            e1.record(stream)
            if do_dec:
                step_decode()
            e2.record(stream)
            enc_ms.append((e0, e1))
            dec_ms.append((e1, e2))
        t_end = ev()
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = _lib.lib.lch_launch_count(ctx) - n0
    total_ms = t_start.elapsed_time(t_end)
    enc = float(np.mean([a.elapsed_time(b) for a, b in enc_ms]))
    dec = float(np.mean([a.elapsed_time(b) for a, b in dec_ms]))
    step_ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([step_ms, enc, dec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, enc, dec = (float(x) for x in t.tolist())

    msg_bytes = B * K * 2
    nphases = int(do_enc) + int(do_dec)
    value = world * nphases * msg_bytes / (step_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    # dominant kernel: the encode's pass_kernel launches (5 per encode)
    enc_launches = 5
    per_launch_ms = enc / enc_launches if do_enc else dec / 8
    per_launch_bytes = 4 * K * B  # 2 B read + 2 B write per symbol-position
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "pass_kernel_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    codec_alg = 2 * N * B  # encode: read k + write n-k symbols (2 B each) per codeword
    res = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
        "data": "synthetic (seeded counter-based generator, SURVEY §8d)",
        "config": {"workload": "cfg3+cfg4a: RS(2^16,2^15) encode 4096 cw + shared-pattern decode "
                               "4096 cw (2^15 erasures) per GPU",
                   "batch_per_gpu": B, "n": N, "k": K, "parallelism": f"codeword-shard x{world}",
                   "l2": "inputs larger than L2 (256 MiB message, 512 MiB received per GPU)"},
        "encode_ms": round(enc, 4), "decode_ms": round(dec, 4),
        "encode_gbs": round(world * msg_bytes / (enc * 1e-3) / 1e9, 3) if do_enc else None,
        "decode_gbs": round(world * msg_bytes / (dec * 1e-3) / 1e9, 3) if do_dec else None,
        "encode_hbm_frac": round(codec_alg / (enc * 1e-3) / 1e9 / peak, 4) if do_enc else None,
        "decode_hbm_frac": round((2 * (N - K) + 2 * K) * B / (dec * 1e-3) / 1e9 / peak, 4)
        if do_dec else None,
        "roofline": {"bound": "hbm", "kernel": "pass_kernel<16,0x1100B> (encode tile pass)",
                     "achieved": round(achieved, 2), "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "algorithmic_bytes_per_launch": per_launch_bytes,
                     "avg_launch_ms": round(per_launch_ms, 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    # e2e through the public API with pinned host buffers
    if not args.no_e2e:
        h_msg = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
        h_msg.copy_(msg.cpu())
        h_par = torch.empty((B, N - K), dtype=torch.int16, pin_memory=True)
        h_rx = torch.empty((B, N), dtype=torch.int16, pin_memory=True)
        h_rx.copy_(rx.cpu())
        h_out = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
        d_msg = torch.empty_like(msg)
        d_par = torch.empty((B, N - K), dtype=torch.int16, device="cuda")
        d_rx = torch.empty_like(cw)
        d_out = torch.empty_like(out)

        def e2e_step():
            d_msg.copy_(h_msg, non_blocking=True)
            encode_device(cp, bt, d_msg, d_par)
            h_par.copy_(d_par, non_blocking=True)
            d_rx.copy_(h_rx, non_blocking=True)
            decode_device(cp, bt, d_rx, bits, d_out, N - K)
            h_out.copy_(d_out, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        e2e_steps = max(1, min(args.steps, 5))
        for _ in range(e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        assert torch.equal(h_out, h_msg), "e2e round trip failed"
        res["e2e"] = {"value": round(world * 2 * msg_bytes / (e2e_ms * 1e-3) / 1e9, 3),
                      "unit": "GB/s", "h2d_bytes_per_step": B * K * 2 + B * N * 2,
                      "d2h_bytes_per_step": B * (N - K) * 2 + B * K * 2,
                      "ms_per_step": round(e2e_ms, 3)}

    if rank == 0 and not args.no_cpu:
        nth = cpu_threads()
        res["cpu_baseline"] = cpu_reference(max(8, min(nth, 64)), nth)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
