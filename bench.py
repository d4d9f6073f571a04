#!/usr/bin/env python3
"""Benchmark: ms per 2^32 x 2^32-bit GF(2)[x] multiply (BASELINE config 5) on B200.

Contract (one JSON line on rank 0):
  value        device-resident ms per multiply (inputs already in HBM), max over ranks, K steps
  e2e          the same through the C-ABI host entry point fpm_polymul with pinned HOST buffers:
               H2D of both operands + D2H of the product inside every timed step
  roofline     the dominant kernel class of the step, measured live with CUDA events
  cpu_baseline the reference CPU path (oracle/_ref, F4-patched build for >= 2^33-bit products)
               timed on this host's cores, rank 0 at N=1 only, on a bounded sample
  --impl reference   times the reference's own CPU implementation instead (rank 0 only)

Multi-GPU (torchrun, N>1): by default ONE product is sharded over the N GPUs
(paper_1803_11301_b200/dist.py: the top log2 N butterfly layers exchange halves -- over peer memory,
the partner's half read inside the butterfly kernel (--exchange peer, default), or NCCL send/recv
(--exchange nccl); "scaling": "strong"); --mode replicas runs N independent products ("weak").
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per 2^k-bit GF(2)[x] multiply (k=20..32); fraction of per-pass roofline"
CONFIGS = {  # BASELINE.json configs by index (1-based); operand bits
    1: 1 << 20, 2: 1 << 16, 3: 1 << 24, 4: 1 << 28, 5: 1 << 32,
}
BATCH = 4096  # config 2: independent 2^16 x 2^16 products per batch (split across ranks)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# Integer-issue peak: LOP3 microbenchmark on B200 (profiles/r01_ubench_gf128_mul.log):
# 63 ops/clk/SM x 148 SMs, scaled by the SM clock seen during the run.
LOP3_OPS_PER_CLK_SM = 63.0


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML (nvidia-ml-py) every 10 ms
    on a thread, plus one sample on entry and one on exit so short regions are covered; falls back
    to `nvidia-smi -lms 100` when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def _nvml_sample(self):
        n, h = self.nvml, self.handle
        sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
        try:
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:
            rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append((float(sm), float(mx), int(rs)))

    def _nvml_loop(self):
        while not self.stop.wait(0.01):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        names = list(self.REASONS)
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                mask = sum(self.REASONS[names[k]] for k in range(4) if parts[3 + k].lower() == "active")
                self.samples.append((float(parts[0]), float(parts[1]), mask))

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({k for _, _, m in self.samples for k, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml" if self.nvml else "nvidia-smi"}


SEEDS = (20261020, 20261021)  # tests/golden/make_golden.py: random_bitpoly(bits, mt19937_64(seed))


def golden_meta():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "reference_meta.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def blake(words) -> str:
    import hashlib

    import numpy as np
    return hashlib.blake2b(np.ascontiguousarray(words, np.uint64).tobytes(), digest_size=16).hexdigest()


def workload_config(cfg: int) -> dict:
    """The `config` object, identical in both arms (ours / --impl reference) for the same workload."""
    if cfg == 2:
        return {"workload": f"cfg2: batch of {BATCH} independent 2^16 x 2^16-bit products (one step = the batch)",
                "inputs": "product k = random_bitpoly(2^16, 30000+k) x random_bitpoly(2^16, 40000+k) (mt19937_64)",
                "field": "GF(2^128) transform (products are field-independent)",
                "l2": "batch operands 64 MiB (fit in L2)"}
    bits = CONFIGS[cfg]
    k = bits.bit_length() - 1
    return {"workload": f"cfg{cfg}: 2^{k} x 2^{k}-bit product, GF(2^128) Frobenius FFT (n=2^{k + 1}, l={k + 1 - 7})",
            "inputs": f"random_bitpoly(2^{k}, mt19937_64({SEEDS[0]})) x random_bitpoly(2^{k}, mt19937_64({SEEDS[1]}))",
            "field": "GF(2^128) (FieldChoice::kGF128)",
            "l2": "operands 512 MiB each (> L2): no flush needed" if bits >= 1 << 30 else
                  "operands fit in L2: L2 flushed (512 MiB written) before every timed step, steps timed individually"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))




def stage_pipes(stage: str, bits: int):
    """ncu pipe utilisation (percent of peak, duration-weighted over the stage's launches) from the
    committed --set full capture (profiles/pipes.json, tools/ncu_traffic.py), or None: SURVEY 8(d)
    asks for the ALU-pipe utilisation beside an int-bound roofline."""
    try:
        with open(os.path.join(ROOT, "profiles", "pipes.json")) as f:
            return json.load(f).get(f"{bits}:{stage}")
    except (OSError, ValueError):
        return None


def stage_traffic(stage: str, bits: int):
    """DRAM bytes (read + write) per launch of the stage's kernel from the committed ncu capture
    (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"{bits}:{stage}")
    except (OSError, ValueError):
        return None


def algorithmic(stage: str, bits: int, T: int, fused_ab: bool = False):
    """SURVEY.md 8(d) per-unit algorithmic work of one product with equal operands of `bits` bits,
    per pipeline stage (each stage is one kernel class).
    Returns (bytes, int32 ops): HBM bytes a perfect kernel moves, and 552 ops per GF(2^128)
    product (the schoolbook convention of 8(d)); the roofline time is the slower of the two."""
    n = 2 * bits
    n_p = n // 128                      # field elements per operand transform
    l = n_p.bit_length() - 1
    V = 16 * n_p                        # bytes of one evaluation vector
    if stage == "basiscvt":             # one read + write sweep per operand
        return 2 * 2 * (bits // 8), 0
    if stage == "ibasiscvt":
        return 2 * (n // 8), 0
    if stage == "encode":
        return 2 * (bits // 8 + V), 0
    if stage == "decode":
        return V + n // 8, 0
    if stage == "butterfly":            # radix-4 passes over layers [T, l) of both operands (+ tile pass of a)
        passes = (l - T + 1) // 2
        if fused_ab:
            return 2 * passes * 2 * V, 552 * (l - T) * n_p
        return 2 * passes * 2 * V + 2 * V, 552 * ((l - T) * n_p + T * n_p // 2)
    if stage == "pointwise":            # fused tile pass: b's (and a's) tile layers, a*b, inverse tile layers
        if fused_ab:
            return 3 * V, 552 * (3 * T * n_p // 2 + n_p)
        return 3 * V, 552 * (T * n_p + n_p)
    if stage == "ibutterfly":
        passes = (l - T + 1) // 2
        return passes * 2 * V, 552 * (l - T) * n_p // 2
    raise KeyError(stage)


GENERIC_CLK_PER_PRODUCT = 6.8  # gf_mul on the FMA/ALU pipes, register operands (tools/microbench/gfmul_rate.cu)
SMEM_BYTES_PER_CLK_SM = 128.0  # shared-memory bandwidth per SM (32 banks x 4 B)


def executed_work(stage: str, bits: int, T: int):
    """EXECUTED work of one stage of the tower-representation GF(2^128) pipeline (equal operands of
    `bits` bits), per binding unit:
      smem_bytes      M8-table products: 16 LDS.128 = 256 B of shared memory each
      generic         generic products (IMAD-hole Karatsuba, GENERIC_CLK_PER_PRODUCT each per SM)
      hbm_bytes       one algorithmic sweep of the stage's data
    butterfly/ibutterfly: radix-8 (+ one radix-4) passes over layers [T, l) of both operands / the
    product (one M8 product per butterfly); pointwise: the fused tower tile pass (per element position: (T-1) tile
    layers of both operands + (T-1) inverse, one M8 product per butterfly, 3 R<->poly conversions,
    2.5 generic products for layer 0 of both operands, the pointwise product and inverse layer 0)."""
    n = 2 * bits
    n_p = n // 128
    l = n_p.bit_length() - 1
    V = 16 * n_p
    # HBM passes of the top layers: radix-8 (three layers) in the tower pipeline, the remainder of one
    # radix-4 / radix-2 pass at the bottom
    passes = (l - T) // 3 + (1 if (l - T) % 3 else 0)
    w = {"smem_bytes": 0.0, "generic": 0.0, "hbm_bytes": 0.0}
    if stage == "basiscvt":
        w["hbm_bytes"] = 2 * 2 * (bits // 8)
    elif stage == "ibasiscvt":
        w["hbm_bytes"] = 2 * (n // 8)
    elif stage == "basiscvt+encode":    # fused (2^32-bit operands): read each operand, write its EvalVec
        w["hbm_bytes"] = 2 * (bits // 8 + V)
    elif stage == "decode+ibasiscvt":   # fused (2^33-bit product): read the EvalVec, write the product
        w["hbm_bytes"] = V + n // 8
    elif stage == "encode":
        w["hbm_bytes"] = 2 * (bits // 8 + V)
    elif stage == "decode":
        w["hbm_bytes"] = V + n // 8
    elif stage == "butterfly":
        w["smem_bytes"] = 256.0 * 2 * (l - T) * n_p / 2
        w["hbm_bytes"] = 2 * passes * 2 * V
    elif stage == "ibutterfly":
        w["smem_bytes"] = 256.0 * (l - T) * n_p / 2
        w["hbm_bytes"] = passes * 2 * V
    elif stage == "pointwise":
        w["smem_bytes"] = 256.0 * ((T - 1) * 1.5 + 3) * n_p
        w["generic"] = 2.5 * n_p
        w["hbm_bytes"] = 3 * V
    else:
        raise KeyError(stage)
    return w


def stage_roofline(stage: str, bits: int, T: int, seconds: float, mhz: float, hbm_gbs: float):
    """The stage's roofline time = the slowest of its units at peak; frac = that / measured."""
    w = executed_work(stage, bits, T)
    clk = mhz * 1e6
    smem_peak = SMEM_BYTES_PER_CLK_SM * 148 * clk  # B/s
    t = {"smem": w["smem_bytes"] / smem_peak, "hbm": w["hbm_bytes"] / (hbm_gbs * 1e9),
         "generic": w["generic"] * GENERIC_CLK_PER_PRODUCT / (148 * clk)}
    bound = max(t, key=t.get)
    if bound == "smem":
        out = {"bound": "smem", "achieved": round(w["smem_bytes"] / seconds / 1e9, 1), "peak": round(smem_peak / 1e9, 1),
               "unit": "GB/s"}
    elif bound == "hbm":
        out = {"bound": "hbm", "achieved": round(w["hbm_bytes"] / seconds / 1e9, 1), "peak": hbm_gbs, "unit": "GB/s"}
    else:
        out = {"bound": "generic", "achieved": round(w["generic"] / seconds / 1e9, 2),
               "peak": round(148 * clk / GENERIC_CLK_PER_PRODUCT / 1e9, 2), "unit": "Gproducts/s"}
    out["frac"] = round(t[bound] / seconds, 4)
    out["t_roof_ms"] = round(t[bound] * 1e3, 3)
    return out


def run_batch(args, ws, rank, local):
    """Config 2: a batch of 4096 independent 2^16 x 2^16 products (fpm_polymul_batch_dev: one CTA
    per product, everything in shared memory), split across ranks with no exchange
    (dist.polymul_batch_sharded; strong scaling over the fixed batch); one step = the whole batch.
    The inputs are the golden seeds, so the batch is checked against the reference's hash."""
    import numpy as np
    import torch

    import paper_1803_11301_b200 as pkg
    from paper_1803_11301_b200.dist import batch_shard

    dev = torch.device("cuda", local)
    bits = CONFIGS[2]
    wa = bits // 64
    wc = (2 * bits - 1 + 63) // 64
    start, per = batch_shard(BATCH, ws, rank)
    ha_np = np.concatenate([pkg.random_bitpoly(bits, 30000 + k) for k in range(start, start + per)])
    hb_np = np.concatenate([pkg.random_bitpoly(bits, 40000 + k) for k in range(start, start + per)])
    a = torch.from_numpy(ha_np.view(np.int64)).to(dev)
    b = torch.from_numpy(hb_np.view(np.int64)).to(dev)
    c = torch.empty(per * wc, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    def step(x, y):
        pkg.fp_polymul_batch_dev(x, bits, wa, y, bits, wa, c, wc, per)
        return c

    for _ in range(args.warmup):
        step(a, b)
    torch.cuda.synchronize()
    pkg.launch_count(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step(a, b)
        e1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
    launches = pkg.launch_count(reset=True)
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    dev_result = c.cpu().numpy().view(np.uint64).copy()
    # parity: the whole batch (gathered on rank 0) against the reference's hash
    parts = [dev_result]
    if ws > 1:
        parts = [None] * ws
        torch.distributed.all_gather_object(parts, dev_result)
    meta = golden_meta().get("cfg2_batch", {})
    got = blake(np.concatenate(parts)) if rank == 0 else None
    parity = {"blake2b128": got, "reference_blake2b128": meta.get("blake2b128_all"),
              "matches_reference": got is not None and got == meta.get("blake2b128_all"),
              "products": BATCH} if rank == 0 else None
    # e2e: pinned host operands in, products out, every step
    ha = torch.from_numpy(ha_np.view(np.int64)).pin_memory()
    hb = torch.from_numpy(hb_np.view(np.int64)).pin_memory()
    hc = torch.empty(per * wc, dtype=torch.int64, pin_memory=True)

    na, nb, nc = (x.numpy().view(np.uint64) for x in (ha, hb, hc))

    def e2e_step():  # the host-buffer batch entry fpm_polymul_batch (uploads / products / downloads overlapped)
        pkg.fp_polymul_batch(na, bits, wa, nb, bits, wa, nc, wc, per, device=local)
    e2e_step()
    k2 = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(k2):
        e2e_step()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / k2
    t = torch.tensor([e2e_ms], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(t.item())
    same = bool(np.array_equal(hc.numpy().view(np.uint64), dev_result))
    clocks = clk.summary()
    mhz = clocks.get("sm_mhz") or 1965.0
    peak_tops = LOP3_OPS_PER_CLK_SM * 148 * mhz * 1e6 / 1e12
    ops = 1.02e7 * BATCH  # ops per config-2 product (l = 10 transform + pointwise)
    achieved = ops / (ms * 1e-3) / 1e12
    smem_bytes = 256.0 * ((10 - 1) * 1.5 + 3) * 1024 * BATCH
    smem_peak = SMEM_BYTES_PER_CLK_SM * 148 * mhz * 1e6
    line = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (random_bitpoly, mt19937_64 seeded)",
        "config": workload_config(2),
        "parallelism": f"batch split over {ws} GPU(s) (dist.batch_shard), no exchange",
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "steps": k2, "h2d_bytes_per_step": 2 * BATCH * wa * 8,
                "d2h_bytes_per_step": BATCH * wc * 8, "matches_device_result": same},
        "parity": parity,
        "gpu_launches": int(launches),
        # executed work (as config 5's tower tile pass): per product 16.5 M8-table
        # products per element position (256 B of shared memory each) at T = l = 10 -- the batch's
        # tower pass is ~77 % of the step (ncu); the SURVEY 8(d) schoolbook figure is kept beside it
        "roofline": {"bound": "smem", "kernel": "fft_tile_tower_kernel<10> (one tile per product) + batch conversions / codec",
                     "achieved": round(smem_bytes / (ms * 1e-3) / 1e9, 1), "peak": round(smem_peak / 1e9, 1), "unit": "GB/s",
                     "frac": round(smem_bytes / smem_peak / (ms * 1e-3), 4), "traffic": None,
                     "peak_source": "128 B/clk/SM x 148 SMs at the sampled SM clock",
                     "schoolbook_equiv_tops": round(achieved, 2),
                     "schoolbook_convention": f"SURVEY 8(d): 1.02e7 int32 ops per 2^16 x 2^16 product; LOP3 peak {peak_tops:.2f} Tops/s"},
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            R = oracle.ref()
            x = ha_np[:wa].copy()
            y = hb_np[:wa].copy()
            R.polymul(x, bits, y, bits, field=0, parallel=False)
            nsample = 64
            t0 = time.perf_counter()
            for _ in range(nsample):
                R.polymul(x, bits, y, bits, field=0, parallel=False)
            per_prod = (time.perf_counter() - t0) / nsample
            line["cpu_baseline"] = {"value": round(per_prod * BATCH * 1e3, 1), "unit": "ms", "cores": 1,
                                    "kind": "reference",
                                    "sample": f"{nsample} serial products (ExecPolicy::kSerial, auto field) on 1 core, "
                                              f"scaled to the {BATCH}-product batch"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": "ms", "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU fp_polymul (oracle/_ref) on this host's cores."""
    if rank != 0:
        return
    import numpy as np

    import oracle

    bits = CONFIGS[args.config]
    f4 = 2 * bits >= (1 << 33)
    R = oracle.ref(f4=f4)
    threads = R.max_threads()
    if args.config == 2:  # batch: each step times a bounded sample of serial products, scaled
        P = oracle.port()
        x = P.random_bitpoly(bits, 30000)
        y = P.random_bitpoly(bits, 40000)
        R.polymul(x, bits, y, bits, field=args.ref_field, parallel=False)
        nsample, times = 256, []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for _ in range(nsample):
                R.polymul(x, bits, y, bits, field=args.ref_field, parallel=False)
            times.append((time.perf_counter() - t0) * 1e3 * BATCH / nsample)
        v = statistics.mean(times)
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": ws,
                "steps": len(times), "warmup": 1, "ms_per_step": round(v, 3), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (random_bitpoly, mt19937_64 seeded)",
                "config": workload_config(2), "library": os.path.basename(R.path),
                "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": 1, "kind": "reference",
                                 "sample": f"{nsample} serial products per step (ExecPolicy::kSerial, 1 core), "
                                           f"scaled to the {BATCH}-product batch"},
                "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    P = oracle.port()
    a = P.random_bitpoly(bits, SEEDS[0])
    b = P.random_bitpoly(bits, SEEDS[1])
    # Same field as our arm's config (GF(2^128), the north-star transform); --ref-field 0 times the
    # reference's default auto field (GF(2^64)) instead.
    field = args.ref_field
    for _ in range(min(args.warmup, 1)):  # cold call builds the twiddle plan (polymul.cpp:63-74)
        R.polymul(a, bits, b, bits, field=field)
    times = []
    budget = args.ref_budget_s
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        R.polymul(a, bits, b, bits, field=field)
        times.append((time.perf_counter() - t0) * 1e3)
        if time.perf_counter() - t_all > budget:
            break
    v = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": ws,
        "steps": len(times), "steps_requested": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": round(v, 3), "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (random_bitpoly, mt19937_64 seeded)",
        "config": workload_config(args.config) if field == 128 else
                  dict(workload_config(args.config), field={64: "GF(2^64)", 0: "auto (m=64, the reference default)"}[field]),
        "library": os.path.basename(R.path),
        "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": threads, "kind": "reference",
                         "sample": f"{len(times)} warm full products (ExecPolicy::kParallel, {threads} OpenMP "
                                   f"threads) after {min(args.warmup, 1)} cold call(s)"},
        "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(bits):
    import oracle

    f4 = 2 * bits >= (1 << 33)
    R = oracle.ref(f4=f4)
    P = oracle.port()
    a = P.random_bitpoly(bits, SEEDS[0])
    b = P.random_bitpoly(bits, SEEDS[1])
    t0 = time.perf_counter()
    R.polymul(a, bits, b, bits, field=128)  # cold: includes the l-layer twiddle plan build
    cold = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    R.polymul(a, bits, b, bits, field=128)
    warm = (time.perf_counter() - t0) * 1e3
    return {"value": round(warm, 1), "unit": "ms", "cores": R.max_threads(), "kind": "reference",
            "sample": f"1 warm GF(2^128) product of this config after 1 cold call ({cold:.0f} ms incl. plan "
                      f"build); {'F4-patched ' if f4 else ''}reference build, OpenMP kParallel"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS),
                    help="BASELINE config: 1, 3, 4, 5 = one product of 2^20/2^24/2^28/2^32 bits; 2 = the 4096-product batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--ref-field", type=int, default=128, choices=[0, 64, 128],
                    help="--impl reference: the reference's field (default GF(2^128), as our arm)")
    ap.add_argument("--mode", default="shard", choices=["shard", "replicas"],
                    help="N>1: shard one product over the GPUs (default) or run independent replicas")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="shard mode: exchanged FFT layers over peer memory (default) or NCCL send/recv")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_env()

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import numpy as np
    import torch

    import paper_1803_11301_b200 as pkg

    # FPM_BENCH_SHARE_GPU=1 (testing the N > 1 path on a one-GPU box only): every rank on cuda:0 with a
    # gloo control plane (NCCL cannot run two ranks on one GPU); the data plane is CUDA IPC as always.
    share = ws > 1 and os.environ.get("FPM_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    if args.config == 2:
        run_batch(args, ws, rank, local)
        return
    bits = CONFIGS[args.config]
    words = bits // 64
    out_words = (2 * bits - 1 + 63) // 64
    mode = "single" if ws == 1 else args.mode
    # the golden seeds (tests/golden/reference_meta.json holds the reference's product hash); every
    # rank holds the same operands (shard mode: one product; replicas: N copies of it)
    ha_np = pkg.random_bitpoly(bits, SEEDS[0])
    hb_np = pkg.random_bitpoly(bits, SEEDS[1])
    a = torch.from_numpy(ha_np.view(np.int64)).to(dev)
    b = torch.from_numpy(hb_np.view(np.int64)).to(dev)
    c = torch.empty(out_words, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    from paper_1803_11301_b200 import dist as pdist
    plan = pdist.make_plan(bits, bits, ws, rank) if mode == "shard" else None
    backend, exchange = None, None
    if mode == "shard":
        # exchanged layers over peer memory (NVLink loads fused into the pair kernel, dist.PeerBackend),
        # or NCCL send/recv + pair kernel; a peer setup failure on any rank falls back to NCCL on all
        ok = 0
        if args.exchange == "peer":
            try:
                backend = pdist.PeerBackend()
                backend.begin(plan)
                ok = 1
            except Exception as e:  # noqa: BLE001 - reported in the JSON line
                exchange = f"nccl (peer setup failed: {str(e)[:120]})"
        flag = torch.tensor([ok], device=dev)
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag.item()) == 1:
            exchange = "peer"
        else:
            backend = pdist.GpuBackend()
            exchange = exchange or "nccl"

    def step(x, y):
        if mode == "shard":
            return pdist.polymul_sharded(x, bits, y, bits, backend, plan)
        pkg.fp_polymul_dev(x, bits, y, bits, c, field=pkg.FIELD_GF128)
        return c

    for _ in range(args.warmup):
        step(a, b)
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs.  Operands that fit in L2 (configs 1, 3, 4): L2 is
    # flushed (a 512 MiB buffer written) before every step and each step is timed on its own.
    flush = bits < (1 << 30)
    scrub = torch.empty(1 << 27, dtype=torch.int32, device=dev) if flush else None
    pkg.launch_count(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for k in range(args.steps):
            if flush:
                scrub.fill_(k)
            step_ev[k][0].record(stream)
            res_dev = step(a, b)
            step_ev[k][1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = pkg.launch_count(reset=True)
    ms = sum(x.elapsed_time(y) for x, y in step_ev) / args.steps
    t = torch.tensor([ms], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    dev_result = res_dev.cpu().numpy().view(np.uint64).copy()
    want = golden_meta().get("configs", {}).get(f"{bits}x{bits}", {}).get("blake2b128")
    got = blake(dev_result)
    parity = {"blake2b128": got, "reference_blake2b128": want, "matches_reference": got == want,
              "product_bits": 2 * bits - 1}

    # ---- e2e: pinned HOST buffers; H2D of both operands and D2H of the product in every step
    ha = torch.from_numpy(ha_np.view(np.int64)).pin_memory()
    hb = torch.from_numpy(hb_np.view(np.int64)).pin_memory()
    hc = torch.empty(out_words, dtype=torch.int64, pin_memory=True)
    na, nb, nc = (x.numpy().view(np.uint64) for x in (ha, hb, hc))

    # sharded conversion (N >= 4, peer exchange): every rank uploads only its share of its operand and
    # downloads only its share of the product, over its own PCIe link (dist.polymul_sharded parts=True);
    # the job's host I/O is the operands and the product once, split over the N links
    parts = (mode == "shard" and exchange == "peer" and plan is not None and pdist.PeerBackend._sharded(plan))
    if parts:
        k_op, iw0, iper = pdist.operand_part_range(plan, rank)
        src = (ha, hb)[k_op]
        hpart = src[iw0:iw0 + max(0, min(iper, src.numel() - iw0))]
        ow0, oper = pdist.product_part_range(plan, rank)
        on = max(0, min(out_words, ow0 + oper) - ow0)
        hout = hc[ow0:ow0 + on]

    def e2e_step():
        if mode == "single":  # the C-ABI host entry point fpm_polymul (include/fpmul_b200.h)
            return pkg.fp_polymul(na, bits, nb, bits, field=pkg.FIELD_GF128, device=local, out=nc)
        if parts:
            xp = hpart.to(dev, non_blocking=True)
            r = pdist.polymul_sharded(xp, bits, xp, bits, backend, plan, parts=True)
            hout.copy_(r)
            torch.cuda.synchronize()
            return hout.numpy().view(np.uint64)
        xa = ha.to(dev, non_blocking=True)
        xb = hb.to(dev, non_blocking=True)
        r = step(xa, xb)
        hc.copy_(r)
        torch.cuda.synchronize()
        return nc

    for _ in range(2):  # (small products: the second call captures the pipeline's CUDA graph)
        e2e_step()
    e2e_steps = max(1, min(args.steps, 5))
    barrier()
    e2e_calls = []  # every call timed on its own: the value is the MEDIAN call (PCIe copies jitter on
    for _ in range(e2e_steps):  # shared hosts: one slow call in five moves a mean by a millisecond)
        t0 = time.perf_counter()
        res = e2e_step()
        e2e_calls.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = sorted(e2e_calls)[len(e2e_calls) // 2]
    e2e_mean = sum(e2e_calls) / len(e2e_calls)
    t = torch.tensor([e2e_ms], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(t.item())
    same = bool(np.array_equal(res, dev_result[ow0:ow0 + on] if parts else dev_result))
    if ws > 1:  # every rank's share must match
        t = torch.tensor([1 if same else 0], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
        same = bool(t.item())
    io_h2d, io_d2h = 2 * words * 8, out_words * 8  # per step, the whole job

    # ---- two concurrent callers of fpm_polymul (host threads, own pinned product buffers): the calls
    # lease separate stream sets, so one caller's PCIe copies overlap the other's kernels.  Reported
    # beside the single-call latency above (which stays the e2e value), never instead of it.
    two_callers = None
    if mode == "single" and bits >= (1 << 24):
        import threading
        hc2 = torch.empty(out_words, dtype=torch.int64, pin_memory=True)
        nouts = [nc, hc2.numpy().view(np.uint64)]
        per = max(2, e2e_steps)

        def caller(k, n):
            for _ in range(n):
                pkg.fp_polymul(na, bits, nb, bits, field=pkg.FIELD_GF128, device=local, out=nouts[k])

        caller(1, 1)
        # one untimed concurrent round: the second caller's scratch grows the library's memory pool
        # once (hundreds of ms for ~5 GiB of fresh device memory), then stays cached
        warm = [threading.Thread(target=caller, args=(k, 1)) for k in range(2)]
        for x in warm:
            x.start()
        for x in warm:
            x.join()
        th = [threading.Thread(target=caller, args=(k, per)) for k in range(2)]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        two_ms = (time.perf_counter() - t0) * 1e3 / (2 * per)
        two_callers = {"callers": 2, "products": 2 * per, "ms_per_product": round(two_ms, 3),
                       "all_match_device_result": bool(all(np.array_equal(o, dev_result) for o in nouts))}
    if ws > 1 and not parts and mode == "shard":  # every rank uploads both operands, downloads the product
        io_h2d, io_d2h = ws * io_h2d, ws * io_d2h

    # ---- roofline: per-stage CUDA-event times of one instrumented product (after one untimed
    # instrumented call: the host-buffer e2e calls above leave the library's memory pool holding
    # other blocks, and the first device call after them pays for fresh ones)
    for _ in range(2):
        st = [0.0] * pkg.NUM_STAGES
        pkg.fp_polymul_dev(a, bits, b, bits, c, field=pkg.FIELD_GF128, stage_seconds=st)
        torch.cuda.synchronize()
    stages = dict(zip(pkg.STAGE_NAMES, st))
    # At 2^33 bits the encode runs inside the forward conversion's last kernel and the decode inside
    # the inverse conversion's first one: their own stage marks then bracket no kernel, so the pairs
    # are timed (and get a roofline) as one stage.
    for conv, cod, name in (("basiscvt", "encode", "basiscvt+encode"), ("ibasiscvt", "decode", "decode+ibasiscvt")):
        if stages[cod] < 0.01 * stages[conv]:
            merged = {}
            for k, v in stages.items():
                if k == conv:
                    merged[name] = v + stages[cod]
                elif k != cod:
                    merged[k] = v
            stages = merged
    dom = max(stages, key=stages.get)
    l_fft = (2 * bits // 128).bit_length() - 1
    T = pkg.fft_tile_log2(l_fft)
    fab = pkg.pipeline_fuses_operands(l_fft)
    clocks = clk.summary()
    hbm, peak_kind = peaks()
    mhz = clocks.get("sm_mhz") or 1965.0
    # executed-work roofline per stage (the unit that binds: SMEM for table products, HBM for sweeps,
    # the FMA pipe for generic products); the dominant stage is the headline kernel
    per_stage = {k: stage_roofline(k, bits, T, v, mhz, hbm) for k, v in stages.items() if v > 0}
    roof = dict(per_stage[dom])
    roof["peak_source"] = {"smem": "128 B/clk/SM x 148 SMs at the sampled SM clock",
                           "hbm": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                           "generic": f"{GENERIC_CLK_PER_PRODUCT} clk/product/SM (tools/microbench/gfmul_rate.cu)"}[roof["bound"]]
    nbytes, ops = algorithmic(dom, bits, T, fab)
    peak_tops = LOP3_OPS_PER_CLK_SM * 148 * mhz * 1e6 / 1e12
    roof["schoolbook_equiv_tops"] = round(ops / stages[dom] / 1e12, 2) if ops else None
    roof["schoolbook_convention"] = "SURVEY 8(d): 552 int32 ops per GF(2^128) product; LOP3 peak " \
                                    f"{peak_tops:.2f} Tops/s -- a convention, not executed work"
    tower = fab and os.environ.get("FPM_TOWER", "1") != "0"  # tower-representation tile pass (k_fft.cu)
    roof["kernel"] = {"pointwise": ("fft_tile_tower_kernel" if tower else "fft_tile_fused2_kernel") if fab
                      else "fft_tile_fused_kernel",
                      "butterfly": "fft_top8_kernel + fft_top4_kernel" if fab else "fft_top4_kernel + fft_tile_kernel",
                      "ibutterfly": "fft_top8_kernel<inverse> + fft_top4_kernel<inverse>"}.get(dom, dom)
    roof["stage"] = dom
    roof["traffic"] = stage_traffic(dom, bits)
    roof["ncu_pipes"] = stage_pipes(dom, bits)
    roof["per_stage"] = {k: {kk: v[kk] for kk in ("bound", "frac", "t_roof_ms")} for k, v in per_stage.items()}
    # the DRAM bytes each stage's kernels actually move (committed ncu launch list, per product) against
    # the HBM peak: how close the sweeps run to HBM speed, beside the one-sweep algorithmic fraction
    for k, v in roof["per_stage"].items():
        tb = stage_traffic(k, bits)
        if tb:
            v["dram_bytes"] = tb
            v["dram_frac"] = round(tb / (hbm * 1e9) / stages[k], 4)
    roof["step_frac"] = round(sum(v["t_roof_ms"] for v in per_stage.values()) / (sum(stages.values()) * 1e3), 4)
    roof["stage_ms"] = {k: round(v * 1e3, 3) for k, v in stages.items()}

    # ---- the reference's default (auto) field, GF(2^64): same product, device-resident
    auto_field = None
    if mode == "single":
        for _ in range(2):
            pkg.fp_polymul_dev(a, bits, b, bits, c, field=pkg.FIELD_AUTO)
        k2 = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(k2):
            pkg.fp_polymul_dev(a, bits, b, bits, c, field=pkg.FIELD_AUTO)
        e1.record(stream)
        torch.cuda.synchronize()
        auto_ms = e0.elapsed_time(e1) / k2
        st = [0.0] * pkg.NUM_STAGES
        pkg.fp_polymul_dev(a, bits, b, bits, c, field=pkg.FIELD_AUTO, stage_seconds=st)
        torch.cuda.synchronize()
        auto_field = {"field": f"GF(2^{pkg.plan_mul(bits, bits)['field_degree']}) (plan_mul auto, the reference default)",
                      "value": round(auto_ms, 3), "unit": "ms", "steps": k2,
                      "same_product": bool(np.array_equal(c.cpu().numpy().view(np.uint64), dev_result)),
                      "stage_ms": {k: round(v * 1e3, 3) for k, v in zip(pkg.STAGE_NAMES, st)}}
        # the same through the host entry point (what a caller of the reference's fp_polymul with
        # default options gets): host buffers, both PCIe copies inside
        for _ in range(2):
            pkg.fp_polymul(na, bits, nb, bits, field=pkg.FIELD_AUTO, device=local, out=nc)
        calls = []
        for _ in range(k2):
            t0 = time.perf_counter()
            res = pkg.fp_polymul(na, bits, nb, bits, field=pkg.FIELD_AUTO, device=local, out=nc)
            calls.append((time.perf_counter() - t0) * 1e3)
        auto_field["e2e"] = {"value": round(sorted(calls)[len(calls) // 2], 3), "unit": "ms", "steps": k2,
                             "stat": "median of the timed calls", "mean_ms": round(sum(calls) / len(calls), 3),
                             "matches_device_result": bool(np.array_equal(res, dev_result))}

    line = {
        "metric": METRIC, "value": round(ms_max / ws if mode == "replicas" else ms_max, 3), "unit": "ms",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
        "higher_is_better": False, "scaling": "weak" if mode == "replicas" else "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (uniform random bits, seeded)",
        "config": workload_config(args.config),
        "parallelism": {"single": "single GPU", "replicas": f"{ws} independent products (replicas)",
                        "shard": f"one product sharded over {ws} GPUs: top {ws.bit_length() - 1} butterfly "
                                 f"layers exchanged ({exchange}), basis conversions "
                                 + (("sharded phase by phase, every 2^32-bit block on N/2 ranks (peer memory)"
                                     if exchange == "peer" and plan is not None and pdist.PeerBackend._sharded(plan)
                                     else "split over ranks 0/1 (peer memory)") if exchange == "peer" else "replicated")}[mode],
        "parity": parity,
        "e2e": {"value": round(e2e_ms / ws if mode == "replicas" else e2e_ms, 3), "unit": "ms", "steps": e2e_steps,
                "stat": "median of the timed calls", "mean_ms": round(e2e_mean / ws if mode == "replicas" else e2e_mean, 3),
                "calls_ms": [round(x, 3) for x in e2e_calls],
                "h2d_bytes_per_step": io_h2d, "d2h_bytes_per_step": io_d2h,
                "matches_device_result": same, **({"two_callers": two_callers} if two_callers else {})},
        "gpu_launches": int(launches),
        "roofline": roof,
        "clocks": clocks,
    }
    if auto_field:
        line["auto_field"] = auto_field
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(bits)
        except Exception as e:  # reference not built on this box
            line["cpu_baseline"] = {"value": None, "unit": "ms", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
