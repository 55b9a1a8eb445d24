#!/usr/bin/env python
"""Benchmark: wavelet-tree build throughput (symbol-levels/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Workload (BASELINE.json metric, north_star "n = 2^28"): config 4, n = 2^28
uint32 symbols uniform over sigma = 2^16 (16 levels), seed 4, synthetic.
A step is one full wt_build (every SURVEY §8(a) row: validation/histogram,
node table, all 16 levels of bitmaps with the fused splits, rank directory)
plus wt_free.  Inputs (1 GiB) are larger than the 126 MB L2, so no explicit
flush is needed between steps.

Multi-GPU (torchrun, N > 1): by default the sharded build
(paper_1407_8142_b200/dist.py): the config's S
split into N contiguous chunks, one per rank, one tree of S built
cooperatively -- digit counts all-gathered, the MSD radix exchange over NCCL
all-to-all, owners build the deep levels; the output stays distributed (each
rank keeps its level slices; --gather also all-gathers the complete tree onto
every rank); value = n*L / max-over-ranks time, scaling "strong".
--replicas: each rank builds its own independent tree of the configuration
(seed + rank), value = all ranks' symbol-levels / max-over-ranks time,
scaling "weak".

--impl reference times the CPU oracle (oracle/, single-threaded C, the
paper's serialWT analogue) on a bounded sample of the same workload.
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

import numpy as np  # noqa: E402

METRIC = "wavelet tree build: symbol-levels/sec and achieved HBM GB/s vs peak at 1 B200"
UNIT = "symbol-levels/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle-reason sampling during the timed region (NVML,
    every 5 ms plus one at the end; the nvidia-smi query of B200_PROFILING.md as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int, period_s: float = 0.005):
        self.idx = gpu_index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for name, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            self.sm.append(float(f[0]))
            self.mx.append(float(f[1]))
            for nm, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[2:6]):
                if v.lower() == "active":
                    self.reasons.add(nm)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        try:  # one more sample at the end of the timed region (short regions)
            self._sample_nvml() if self._nvml else self._sample_smi()
        except Exception:
            pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def aggregate(ms_local: float, units_per_rank: int, world: int, dist=None, device=None):
    """Max-over-ranks step time and whole-job throughput (units of all ranks)."""
    ms = ms_local
    if world > 1 and dist is not None:
        import torch
        t = torch.tensor([ms_local], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, units_per_rank * world / (ms / 1e3)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_oracle_sample(cfg, n_sample: int, repeats: int = 1, S=None):
    """Time the single-threaded C oracle (as it stands) on the first n_sample
    symbols of the config's stream; returns (symbol-levels/s, seconds, n)."""
    import gen
    import oracle
    if S is None:
        S = gen.config_input(cfg, n_sample)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        with oracle.OracleTree(S, cfg.sigma):
            pass
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return n_sample * cfg.levels / t, t, n_sample


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-log2", type=int, default=27,
                    help="cpu_baseline sample of the oracle (2^27 symbols of config 4: ~10 s)")
    ap.add_argument("--ref-sample-log2", type=int, default=25,
                    help="--impl reference: symbols per step (K + W steps must end within minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="cooperative sharded build (default when N > 1)")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent trees per rank (weak scaling)")
    ap.add_argument("--gather", action="store_true", help="sharded: all-gather the complete tree onto every rank")
    args = ap.parse_args()

    import gen
    cfg = gen.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    workload = {"workload": f"config {cfg.idx}: {cfg.name}", "n": cfg.n, "sigma": cfg.sigma,
                "levels": cfg.levels, "elem_bytes": cfg.elem_bytes, "seed": cfg.seed,
                "distribution": cfg.kind,
                "l2": "no flush: input %d MiB > 126 MB L2" % (cfg.n * cfg.elem_bytes >> 20),
                "parallelism": f"replicas{world}" if world > 1 else "single"}

    if args.impl == "reference":
        if rank != 0:
            return
        n_s = 1 << args.ref_sample_log2
        S_sample = gen.config_input(cfg, n_s)
        for _ in range(args.warmup):
            run_oracle_sample(cfg, 1 << 16, S=S_sample[:1 << 16])
        t0 = time.perf_counter()
        tot = 0.0
        for _ in range(args.steps):
            v, t, _n = run_oracle_sample(cfg, n_s, S=S_sample)
            tot += t
        ms = tot / args.steps * 1e3
        value = n_s * cfg.levels / (ms / 1e3)
        sample = f"first 2^{args.ref_sample_log2} symbols of the config-{cfg.idx} stream"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32" if cfg.elem_bytes == 4 else "u8",
            "data": "synthetic", "config": workload,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t0}))
        return

    import torch
    import torch.distributed as dist
    import paper_1407_8142_b200 as wt

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    if args.sharded or (world > 1 and not args.replicas):
        return bench_sharded(args, cfg, workload, rank, world, local_rank, dist, wt)

    # input: the config stream (rank r of a replica run uses seed + r)
    if world > 1 and rank > 0:
        S_host = gen.uniform_bits(cfg.n, cfg.levels, cfg.seed + rank, dtype=cfg.dtype) \
            if cfg.kind == "uniform" else gen.zipf_permuted(cfg.n, cfg.seed + rank, dtype=cfg.dtype)
    else:
        S_host = gen.config_input(cfg)
    S_pinned = torch.from_numpy(S_host).pin_memory()
    S_dev = S_pinned.cuda()
    stream = torch.cuda.current_stream()
    units = cfg.n * cfg.levels

    for _ in range(args.warmup):
        wt.build(S_dev, cfg.sigma).free()
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM) ----
    # pass 1 times the builds as a user runs them (no per-kernel events: the
    # library's ~25 event pairs per build cost ~0.14 ms on config 4); pass 2
    # repeats the same K steps with the library's per-kernel CUDA events (on the
    # build stream) for the kernel shares and the roofline's launch durations
    kern_ms, kern_bytes, kern_launch = {}, {}, {}
    launches = 0
    sampler = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            wt.build(S_dev, cfg.sigma, stream).free()
        e1.record(stream)
        torch.cuda.synchronize()
        wt.profile_enable(True)
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(args.steps):
            wt.build(S_dev, cfg.sigma, stream).free()
        p1.record(stream)
        torch.cuda.synchronize()
    prof = wt.last_profile(total=True)  # per-kernel events of the K instrumented builds, summed
    launches = prof["total_launches"]
    for k in prof["kernels"]:
        kern_ms[k["name"]] = k["ms"]
        kern_bytes[k["name"]] = k["algo_bytes"]
        kern_launch[k["name"]] = k["launches"]
    barrier()
    wt.profile_enable(False)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms_instrumented = p0.elapsed_time(p1) / args.steps
    ms, value = aggregate(ms_local, units, world, dist if world > 1 else None, torch.device("cuda"))

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        wt.build_host(S_pinned, cfg.sigma, stream).free()
        torch.cuda.synchronize()
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            wt.build_host(S_pinned, cfg.sigma, stream).free()
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms, e2e_val = aggregate(t0.elapsed_time(t1) / args.steps, units, world,
                                    dist if world > 1 else None, torch.device("cuda"))
        e2e = {"value": e2e_val, "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": cfg.n * cfg.elem_bytes,
               "d2h_bytes_per_step": 12}  # error flag (u32) + total node count (u64)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    peak, peak_kind = peaks()
    dom = max(kern_ms, key=lambda k: kern_ms[k]) if kern_ms else None
    roof = None
    if dom:
        per_launch_ms = kern_ms[dom] / kern_launch[dom]
        per_launch_bytes = kern_bytes[dom] / kern_launch[dom]
        achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                traffic = tj.get(f"config{cfg.idx}", {}).get(dom)
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                "algo_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                "timing": "library CUDA events on the build stream, second pass of the same K steps"}
    L, n, w = cfg.levels, cfg.n, cfg.elem_bytes
    bmin = n * w + L * (((n + 511) // 512) * 8) * 8 + L * (2 * ((n + 511) // 512) + 8 * ((n + 65535) // 65536 + 1))
    kernels = {k: {"ms_per_step": kern_ms[k] / args.steps, "share": kern_ms[k] / max(1e-9, sum(kern_ms.values())),
                   "launches_per_step": kern_launch[k] / args.steps} for k in sorted(kern_ms, key=lambda x: -kern_ms[x])}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        v, t, ns = run_oracle_sample(cfg, 1 << args.cpu_sample_log2)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first 2^{args.cpu_sample_log2} symbols of the config-{cfg.idx} stream "
                         f"({t:.1f} s single-threaded)", "cpu": cpu_model(), "host_cores": os.cpu_count()}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32" if w == 4 else ("u16" if w == 2 else "u8"),
        "data": "synthetic", "config": workload,
        "elements_per_s": n * world / (ms / 1e3),
        "build_hbm": {"b_min_bytes": bmin, "b_min_gbs": bmin / (ms / 1e3) / 1e9,
                      "frac_of_peak": bmin / (ms / 1e3) / 1e9 / peak},
        "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": sampler.summary(), "gpu_launches": launches,
        "ms_per_step_instrumented": ms_instrumented,
        "paper_context": {"levelWT_T40_rand2^16_symbol_levels_per_s": 2.44e9,
                          "hardware": "4x Xeon E7-8870, 40 cores (PAPER.md:626-633, 682)"},
        "gpu": torch.cuda.get_device_name(local_rank),
    }
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def bench_sharded(args, cfg, workload, rank, world, local_rank, dist, wt):
    """One tree of the config's S built by all ranks together."""
    import torch
    from paper_1407_8142_b200 import dist as wdist
    S_host = gen_config(cfg)
    lo, hi = cfg.n * rank // world, cfg.n * (rank + 1) // world
    S_pin = torch.from_numpy(S_host[lo:hi].copy()).pin_memory()
    S_dev = S_pin.cuda()
    del S_host
    comm = wdist.TorchComm() if world > 1 else _SoloComm()

    def step(S):
        t = wdist.build_sharded(S, cfg.sigma, comm, gather=args.gather)
        t.free()

    for _ in range(args.warmup):
        step(S_dev)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(local_rank)
    wt.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(S_dev)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = wt.last_profile(total=True)["total_launches"]
    wt.profile_enable(False)
    if world > 1:
        dist.barrier()
    units = cfg.n * cfg.levels  # one tree of the whole S (strong scaling)
    ms, value = aggregate(e0.elapsed_time(e1) / args.steps, units // world, world,
                          dist if world > 1 else None, torch.device("cuda"))
    # end to end: this rank's chunk copied from pinned host memory every step
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(S_pin.cuda(non_blocking=True))
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms, e2e_val = aggregate(t0.elapsed_time(t1) / args.steps, units // world, world,
                                dist if world > 1 else None, torch.device("cuda"))
    if rank == 0:
        workload = dict(workload, parallelism=f"shard{world}", output="complete tree on every rank" if args.gather
                        else "distributed (level slices per rank)")
        tau = min(8, cfg.levels)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32" if cfg.elem_bytes == 4 else "u8", "data": "synthetic",
            "config": workload, "mode": "sharded", "clocks": sampler.summary(), "gpu_launches": launches,
            "e2e": {"value": e2e_val, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": (hi - lo) * cfg.elem_bytes,
                    "d2h_bytes_per_step": world * ((1 << tau) + 1) * 8},  # the all-gathered digit counts
            "gpu": torch.cuda.get_device_name(local_rank)}))
    if world > 1:
        dist.destroy_process_group()


def gen_config(cfg):
    import gen
    return gen.config_input(cfg)


class _SoloComm:
    """World size 1 without a process group (the collectives are identities)."""
    rank, world = 0, 1

    def all_gather(self, t):
        return [t.clone()]

    def all_gather_v(self, t):
        return [t.clone()]

    def all_to_all_v(self, t, send_counts):
        return t.clone()


if __name__ == "__main__":
    main()
