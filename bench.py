#!/usr/bin/env python
"""Benchmark of the DIS flow hot path (BASELINE.json metric: flow
frame-pairs/sec at 1024x436 & 1080p on 1/2/4/8 B200) — see DESIGN.md §5.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1]
    python bench.py --impl reference ...      # the host-CPU reference arm

A step = one pass of the whole coarse-to-fine DIS pipeline over one batch of
the config's synthetic pairs.  The headline workload is BASELINE configs[1]
(c1: 64 pairs of 1024x436 per GPU, θps 8 / θov 0.5 / θsf 1 / θit 32,
refinement 1 outer / 5 inner); the same JSON line carries a ``c3`` block
(BASELINE configs[3]: 256 pairs of 1920x1080, sharded across the GPUs), so
both resolutions of the metric are timed in every run.

Multi-GPU: one process per GPU.  Under torchrun the ranks come from the
environment; ``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks (127.0.0.1 rendezvous).  Pairs are
independent: c0/c1/c2 give every rank its own batch (weak scaling), c3's 256
pairs and c4's 31 stream pairs are split across the ranks (strong scaling).
No collective touches the data path; NCCL carries the barrier and the
max-over-ranks of the step time only.

One JSON line on rank 0.  `value` = device-resident throughput (inputs in HBM
before the timed region); `e2e` = the same metric through the C ABI's
host-buffer entry point (pinned host frames in, host float64 flow out, copies
inside the timed region); `roofline` = the dominant kernel class against
what bounds it, with the measured DRAM traffic beside the algorithmic bytes;
`cpu_baseline` = the reference path on this host's cores (tools/refcpu.py).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import multiprocessing as mp
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from tools import synth  # noqa: E402

METRIC = "flow frame-pairs/sec"
UNIT = "pairs/s"

# how each config's pairs are spread over the ranks
SCALING = {"c0": "weak", "c1": "weak", "c2": "weak", "c3": "strong", "c4": "strong"}


# --------------------------------------------------------------------------
# algorithmic bytes (e = 8: float64 derived rasters)
# --------------------------------------------------------------------------

def level_dims(cfg, s):
    return cfg.height >> s, cfg.width >> s


def grid_n(dim, ps, ov):
    op = int(math.floor(ov * ps + 1e-9))
    sp = max(1, ps - op)
    last = dim - ps
    nreg = last // sp + 1
    return nreg + (1 if (nreg - 1) * sp != last else 0)


def algorithmic_bytes(cfg, params, e=8):
    """Per-pair bytes of each kernel class, SURVEY §8(d) accounting."""
    ss, sf, ps = params.coarsest_scale, params.finest_scale, params.patch_size
    N = {s: level_dims(cfg, s)[0] * level_dims(cfg, s)[1] for s in range(ss + 2)}
    P = {s: grid_n(level_dims(cfg, s)[1], ps, params.overlap)
         * grid_n(level_dims(cfg, s)[0], ps, params.overlap) for s in range(sf, ss + 1)}
    vi = params.variational.inner_sor_iters
    outer = {s: params.variational.outer_iters(s) for s in range(sf, ss + 1)}
    b = {}
    b["pyramid"] = 2 * (4 * N[0] + sum(e * N[s] for s in range(1, ss + 1))
                        + sum(2 * e * N[s] for s in range(sf, ss + 1)))
    b["patch_search"] = sum(4 * e * N[s] + (2 * e * N[s + 1] if s < ss else 0) + 3 * e * P[s]
                            for s in range(sf, ss + 1))
    b["densify"] = sum(2 * e * N[s] + 3 * e * P[s] + 2 * e * N[s] for s in range(sf, ss + 1))
    b["tensor_assemble"] = sum(14 * e * N[s] * outer[s] for s in range(sf, ss + 1))
    b["sor"] = sum(12 * e * N[s] * vi * outer[s] for s in range(sf, ss + 1))
    b["upsample"] = sum(2 * e * N[s] + 2 * e * N[s - 1] for s in range(1, sf + 1))
    if sf == 0:
        b["upsample"] = 2 * e * N[0] + 2 * e * N[0]  # interleave pass
    return b


# Algorithmic FP64 flops, counted on the reference's formulation (one flop
# per + - * / of inverse_search.py / variational.py; abs, compares, clamps
# and floors not counted):
#   patch search: precompute 7 per template sample (tsum, h00, h01, h11;
#     inverse_search.py:89-96) per patch; one window evaluation 23 per sample
#     (_bilin 11 incl. the two fractions + bx+ox, by+oy + the wsum add = 14;
#     the residual pass e, mar, ssd, b0, b1 = 9; inverse_search.py:130-150);
#   SOR: 62 per pixel update at an interior pixel (4 neighbours x 11 +
#     den_u, val_u (4), du (4), den_v, val_v (4), dv (4);
#     variational.py:133-165).
SEARCH_PRE_FLOPS = 7
SEARCH_EVAL_FLOPS = 23
SOR_UPDATE_FLOPS = 62
MAX_SWEEPS_PER_PASS = 8  # variational.cu kMaxSweepsPerPass


def algorithmic_flops(cfg, params, B, evals_total):
    ss, sf, ps = params.coarsest_scale, params.finest_scale, params.patch_size
    P = sum(grid_n(level_dims(cfg, s)[1], ps, params.overlap)
            * grid_n(level_dims(cfg, s)[0], ps, params.overlap) for s in range(sf, ss + 1))
    vi = params.variational.inner_sor_iters
    sor = sum(level_dims(cfg, s)[0] * level_dims(cfg, s)[1] * vi * params.variational.outer_iters(s)
              for s in range(sf, ss + 1))
    return {"patch_search": B * P * SEARCH_PRE_FLOPS * ps * ps
            + evals_total * SEARCH_EVAL_FLOPS * ps * ps,
            "sor": B * sor * SOR_UPDATE_FLOPS}


def sor_diag_steps(h, w, sweeps):
    """Anti-diagonal steps of one wavefront pass of `sweeps` lexicographic
    sweeps over an h x w level: pixel (x, y) of sweep t runs at step
    x + y + 2t."""
    return w + h - 1 + 2 * (sweeps - 1)


def sor_passes(sweeps):
    out = []
    while sweeps > 0:
        s = min(sweeps, MAX_SWEEPS_PER_PASS)
        out.append(s)
        sweeps -= s
    return out


def measured_peak_gbs():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name, kernel_class, launches_per_step):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    a kernel class, from the committed `ncu --set full` capture of one
    pipeline step (profiles/ncu_traffic.json holds the class's per-step
    total), or None."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(config_name, {}).get(kernel_class)
        src = d.get("_source", {}).get(config_name)
        return (None, None) if v is None else (v / max(1.0, launches_per_step), src)
    except Exception:
        return None, None


# --------------------------------------------------------------------------
# inputs and sharding
# --------------------------------------------------------------------------

def _gen_chunk(args):
    name, seed, first, count = args
    return synth.make_batch(synth.CONFIGS[name], seed=seed, count=count, first=first)


def make_inputs(cfg, seed, count, workers, first=0):
    """Synthetic pairs [first, first + count) (pair i from seed + i),
    generated in parallel."""
    if count <= 0:
        z = np.zeros((0, cfg.height, cfg.width), dtype=np.float32)
        return z, z.copy()
    if cfg.stream or workers <= 1 or count <= 2:
        return synth.make_batch(cfg, seed=seed, count=count, first=first)
    chunks = []
    step = max(1, math.ceil(count / workers))
    for a in range(first, first + count, step):
        chunks.append((cfg.name, seed, a, min(step, first + count - a)))
    with mp.get_context("fork").Pool(min(workers, len(chunks))) as pool:
        parts = pool.map(_gen_chunk, chunks)
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def rank_pairs(cfg, rank, world, batch=0):
    """(first, count, total) pairs of a config this rank computes.  Weak: the
    config's batch per rank (pair seeds continue across ranks); strong: the
    config's batch split into contiguous blocks (sharding.shard_range; for
    c4's stream this is also the sequence split, sharding.shard_sequence)."""
    from paper_1603_03590_b200 import sharding

    B = batch or cfg.batch
    if SCALING[cfg.name] == "weak":
        return rank * B, B, B * world
    a, b = sharding.shard_range(B, rank, world)
    return a, b - a, B


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def config_block(cfg, params, world, pairs_rank, total, extra=None):
    d = {"workload": cfg.name, "pairs_total": total, "pairs_per_gpu": pairs_rank,
         "height": cfg.height, "width": cfg.width, "patch_size": cfg.patch_size,
         "overlap": cfg.overlap, "iterations": cfg.iterations,
         "finest_scale": cfg.finest_scale, "coarsest_scale": params.coarsest_scale,
         "refinement": f"{params.variational.outer_iters(0)} outer / "
                       f"{params.variational.inner_sor_iters} inner",
         "parallelism": (f"pair-sharded x{world}, no collective ("
                         f"{'each GPU its own batch' if SCALING[cfg.name] == 'weak' else 'batch split across GPUs'})")}
    if extra:
        d.update(extra)
    return d


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------

class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    (nvidia-ml-py) polled every 5 ms from a thread; nvidia-smi -lms 100 as
    the fallback."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            bus = None
            try:
                import torch

                bus = torch.cuda.get_device_properties(self.dev).pci_bus_id
            except Exception:
                pass
            h = None
            if bus:
                try:
                    h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
                except Exception:
                    h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.nvml = (pynvml, h)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_ev.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((mhz, int(bits)))
            except Exception:
                pass
            self.stop_ev.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.nvml is not None:
            self.stop_ev.set()
            self.thread.join(timeout=2)
            sm = [r[0] for r in self.rows]
            reasons = sorted({name for _, bits in self.rows
                              for bit, name in self.REASONS.items() if bits & bit})
            if not sm:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                        "samples": 0, "source": "nvml"}
            return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": min(sm),
                    "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(sm),
                    "source": "nvml 5 ms"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 100 ms"}


# --------------------------------------------------------------------------
# the host-CPU reference arm (--impl reference)
# --------------------------------------------------------------------------

def run_reference(args, cfg, params):
    """--impl reference: the reference path on the host CPU (the reference
    package itself from baseline/_ref when installed, else the C port), one
    process per physical core, same metric/config; each step is the config's
    per-GPU batch, or a bounded sample of it (``--ref-pairs``)."""
    from tools import refcpu

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    first, count, total = rank_pairs(cfg, 0, 1, args.batch)
    info = refcpu.host_info()
    sample = args.ref_pairs or (count if count <= 4 * info["physical"] else 2 * info["physical"])
    sample = max(1, min(sample, count))
    f1, f2 = make_inputs(cfg, seed=0, count=sample, workers=host_cores())
    pool = refcpu.CpuPool(f1, f2, params, kind=args.ref_kind)
    for _ in range(min(args.warmup, 3)):
        pool.run(sample)
    walls = []
    per_pair = []
    used = 0
    for _ in range(args.steps):
        wall, n, used, pp = pool.run(sample)
        walls.append(wall)
        per_pair.append(pp)
    pool.close()
    value = sample * len(walls) / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": SCALING[cfg.name], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, params, 1, count, total),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": pool.kind,
                         "sample": pool.describe(sample, used),
                         "cpu_model": info["model"], "physical_cores": info["physical"],
                         "logical_cpus": info["logical"],
                         "single_process_s_per_pair": float(np.median(per_pair))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, params, f1, f2, n, kind="auto"):
    """The reference path on this host (one process per physical core) over
    n of the pairs — a bounded sample, reported beside the GPU numbers."""
    from tools import refcpu

    n = max(1, min(n, f1.shape[0]))
    pool = refcpu.CpuPool(f1[:n], f2[:n], params, kind=kind)
    wall, n, used, pp = pool.run(n)
    pool.close()
    info = pool.info
    return {"value": n / wall, "unit": UNIT, "cores": used, "kind": pool.kind,
            "sample": pool.describe(n, used) + f"; {wall:.1f} s",
            "cpu_model": info["model"], "physical_cores": info["physical"],
            "logical_cpus": info["logical"], "single_process_s_per_pair": pp}


# --------------------------------------------------------------------------
# the GPU arm
# --------------------------------------------------------------------------

def measure(cfg, params, args, dev, rank, world, steps, e2e_steps, tag):
    """Time one workload on this rank: graph-replayed device-resident steps
    (`value`), an eager pass with per-launch CUDA events (kernel breakdown,
    rooflines, SOR diagonal-step rates) and the host-buffer e2e path."""
    import torch

    from paper_1603_03590_b200 import FlowEngine, _lib, sharding

    first, B, total = rank_pairs(cfg, rank, world, args.batch if tag == "main" else 0)
    gen_workers = max(1, host_cores() // max(1, world))
    t_gen = time.perf_counter()
    f1_np, f2_np = make_inputs(cfg, seed=0, count=B, workers=gen_workers, first=first)
    t_gen = time.perf_counter() - t_gen
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    if B == 0:  # more ranks than pairs: this rank idles but joins every barrier
        eng = None
    else:
        eng = FlowEngine(B, cfg.height, cfg.width, params, device=dev)
        f1 = torch.from_numpy(f1_np).to(dev)
        f2 = torch.from_numpy(f2_np).to(dev)
        out = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64, device=dev)
        for i in range(max(3, args.warmup)):  # first call checks the status word
            eng.run(f1, f2, out=out, stream=stream, check=(i == 0))
        torch.cuda.synchronize(dev)
    launches_per_step = int(L.dis_last_launch_count()) if eng else 0

    # untimed census step: window evaluations of the patch search (FP64
    # roofline numerator), and the FP64 peak of this device
    evals_step = 0
    if eng:
        _lib.check(L.dis_census_enable(1))
        eng.run(f1, f2, out=out, stream=stream, check=False)
        torch.cuda.synchronize(dev)
        ev_n, ev_p = ctypes.c_longlong(0), ctypes.c_longlong(0)
        _lib.check(L.dis_census_read(ctypes.byref(ev_n), ctypes.byref(ev_p)))
        _lib.check(L.dis_census_enable(0))
        evals_step = int(ev_n.value)
    dadd, dmul = ctypes.c_double(0), ctypes.c_double(0)
    _lib.check(L.dis_selftest_fp64_peak(ctypes.byref(dadd), ctypes.byref(dmul),
                                        _lib.stream_handle(torch.cuda.current_stream(dev))))
    fp64_peak_tflops = min(dadd.value, dmul.value) / 1e3

    # ---- timed region: device-resident inputs (> L2: 2 x B x H x W x 4 B) ----
    # `value`: each step replayed as one CUDA graph (FlowEngine.run(graph=True):
    # the same kernels and arguments, without the per-launch gaps), captured
    # and replayed once before timing.  Then a second timed pass of the same
    # steps with eager launches and a CUDA event pair around every launch
    # gives the kernel breakdown (events between launches add a little time,
    # so that pass's step time is reported beside `value`).
    gstream = torch.cuda.Stream(device=dev)
    gstream.wait_stream(torch.cuda.current_stream(dev))
    use_graph = not args.no_graph
    if eng and use_graph:
        eng.run(f1, f2, out=out, stream=gstream, check=True, graph=True)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev.index).start()
    sharding.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(gstream)
    if eng:
        for _ in range(steps):
            eng.run(f1, f2, out=out, stream=gstream, check=False, graph=use_graph)
    ev1.record(gstream)
    torch.cuda.synchronize(dev)
    sharding.barrier()
    ms_total = sharding.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    if eng:
        eng.check_status(gstream)  # any non-finite / coverage failure raises here
    # kernel-breakdown pass (eager, an event pair per launch)
    L.dis_profile_reset()
    L.dis_profile_enable(1)
    sharding.barrier()
    torch.cuda.synchronize(dev)
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    if eng:
        for _ in range(steps):
            eng.run(f1, f2, out=out, stream=stream, check=False)
    ev3.record(stream)
    torch.cuda.synchronize(dev)
    sharding.barrier()
    clk = clocks.stop()
    L.dis_profile_enable(0)
    ms_eager = sharding.max_over_ranks(ev2.elapsed_time(ev3), device=dev) / steps
    if eng:
        eng.check_status(stream)
    nk = len(_lib.KERNEL_CLASSES)
    kms = (ctypes.c_double * nk)()
    kcnt = (ctypes.c_int64 * nk)()
    _lib.check(L.dis_profile_read(kms, kcnt, nk))
    nlog = max(0, int(L.dis_profile_log(None, None, None, 0)))
    lcls = (ctypes.c_int32 * max(1, nlog))()
    llev = (ctypes.c_int32 * max(1, nlog))()
    lms = (ctypes.c_double * max(1, nlog))()
    L.dis_profile_log(lcls, llev, lms, nlog)
    kernels = {name: {"ms_per_step": kms[i] / steps, "launches_per_step": kcnt[i] / steps}
               for i, name in enumerate(_lib.KERNEL_CLASSES)}
    ms_step = ms_total / steps
    value = total / (ms_step / 1e3)

    # ---- rooflines (each kernel class against what bounds it) ----
    per_pair = algorithmic_bytes(cfg, params)
    peak, peak_kind = measured_peak_gbs()
    flops = algorithmic_flops(cfg, params, B, evals_step)
    total_ms = sum(x["ms_per_step"] for x in kernels.values())
    for name, k in kernels.items():
        if k["ms_per_step"] <= 0:
            continue
        sec = k["ms_per_step"] / 1e3
        k["share"] = k["ms_per_step"] / max(1e-12, total_ms)
        k["algorithmic_GBps"] = per_pair[name] * B / sec / 1e9
        k["hbm_frac"] = k["algorithmic_GBps"] / peak
        tr, _ = ncu_traffic(cfg.name, name, 1.0)
        if tr is not None and B == cfg.batch:
            # measured DRAM bytes of one step of this class (ncu, same config)
            k["dram_GBps"] = tr / sec / 1e9
            k["dram_frac"] = k["dram_GBps"] / peak
        if name in flops:
            k["algorithmic_TFLOPs"] = flops[name] / sec / 1e12
            k["fp64_frac"] = k["algorithmic_TFLOPs"] / fp64_peak_tflops

    # SOR: anti-diagonal steps per second, per level (the wavefront's own rate)
    sor_cls = _lib.KERNEL_CLASSES.index("sor")
    per_level = {}
    for i in range(nlog):
        if lcls[i] != sor_cls:
            continue
        per_level.setdefault(int(llev[i]), []).append(float(lms[i]))
    sor_levels = []
    steps_sum = ms_sum = 0.0
    vi = params.variational.inner_sor_iters
    for s in sorted(per_level, reverse=True):
        h, w = level_dims(cfg, s)
        passes = sor_passes(vi)
        outer = params.variational.outer_iters(s)
        launches = len(per_level[s]) / steps
        diag = outer * sum(sor_diag_steps(h, w, S) for S in passes)  # per step
        ms = sum(per_level[s]) / steps
        steps_sum += diag
        ms_sum += ms
        sor_levels.append({"level": s, "width": w, "height": h, "launches": launches,
                           "ms": ms, "diag_steps": diag, "diag_steps_per_s": diag / (ms / 1e3),
                           "us_per_diag_step": 1e3 * ms / diag,
                           "pixel_updates_per_s": B * h * w * vi * outer / (ms / 1e3)})
    if "sor" in kernels and ms_sum > 0:
        kernels["sor"]["diag_steps_per_s"] = steps_sum / (ms_sum / 1e3)
        kernels["sor"]["levels"] = sor_levels

    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    d = kernels[dom]
    launches = max(1.0, d["launches_per_step"])
    ms_per_launch = d["ms_per_step"] / launches
    traffic, tsrc = ncu_traffic(cfg.name, dom, launches)
    if B != cfg.batch:
        traffic = None  # the committed capture is of the per-GPU batch of this config
    if dom == "patch_search":
        per_launch = flops[dom] / launches
        achieved = per_launch / (ms_per_launch / 1e3) / 1e12
        roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved,
                    "peak": fp64_peak_tflops, "unit": "TFLOP/s",
                    "frac": achieved / fp64_peak_tflops, "traffic": traffic,
                    "peak_source": "measured live: DADD independent chains, no FMA "
                                   "(dis_selftest_fp64_peak)",
                    "algorithmic_flops_per_launch": per_launch,
                    "evaluations_per_step": evals_step, "hbm_frac": d["hbm_frac"]}
    else:
        bytes_per_launch = per_pair[dom] * B / launches
        achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                    "peak_source": peak_kind, "algorithmic_bytes_per_launch": bytes_per_launch}
        if "fp64_frac" in d:
            roofline["fp64_frac"] = d["fp64_frac"]
    if traffic is not None:
        # what the kernel actually moves (ncu DRAM bytes, cold-cache capture of
        # the same config) over the same measured launch time
        roofline["dram_GBps"] = traffic / (ms_per_launch / 1e3) / 1e9
        roofline["dram_frac"] = roofline["dram_GBps"] / peak
        roofline["traffic_source"] = f"profiles/{tsrc}" if tsrc else "profiles/ncu_traffic.json"
    if dom == "sor" and "diag_steps_per_s" in d:
        roofline["diag_steps_per_s"] = d["diag_steps_per_s"]

    # ---- e2e: host buffers through the C ABI (copies in the timed region) ----
    e2e = None
    if not args.no_e2e:
        e_s = 0.0
        h1 = h2 = ho = None
        if eng:
            pin1 = torch.from_numpy(f1_np).pin_memory()
            pin2 = torch.from_numpy(f2_np).pin_memory()
            pout = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64).pin_memory()
            h1, h2, ho = pin1.numpy(), pin2.numpy(), pout.numpy()
            eng.run_host(h1, h2, out=ho, stream=stream)
            eng.run_host(h1, h2, out=ho, stream=stream)  # captured as a graph on this call
            torch.cuda.synchronize(dev)
        sharding.barrier()
        t0 = time.perf_counter()
        if eng:
            for _ in range(e2e_steps):
                eng.run_host(h1, h2, out=ho, stream=stream)
        t1 = time.perf_counter()
        e_s = sharding.max_over_ranks(t1 - t0, device=dev) / e2e_steps
        if eng:
            assert np.array_equal(ho[-1], out[-1].cpu().numpy()), "host path != device path"
        h2d = sharding.sum_over_ranks(float(2 * f1_np.nbytes), device=dev)
        d2h = sharding.sum_over_ranks(float(B * cfg.height * cfg.width * 16), device=dev)
        blocking = {"value": total / e_s, "unit": UNIT, "ms_per_step": 1e3 * e_s,
                    "steps": e2e_steps,
                    "api": "FlowEngine.run_host -> dis_flow_batch_host: one blocking call per "
                           "step (pinned host frames in, float64 host flow out)"}
        e2e = dict(blocking, h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h))
        # ---- the same calls, two in flight (the streaming use of the path) ----
        # Two engines (own workspace, output buffer and stream each) alternate:
        # submit_host enqueues a call, finish_host waits for it, so one call's
        # flow copy-out (the PCIe-bound part) overlaps the next call's copy-in
        # and kernels.  Every call still copies its frames in and its flow out
        # inside the timed region, which starts before the first submit and ends
        # after the last finish.
        if not args.no_pipelined:
            pipe = None
            try:
                pipe = e2e_pipelined(cfg, params, dev, eng, B, h1, h2, ho,
                                     out if eng else None, max(2 * e2e_steps, 6))
            except Exception as exc:  # (memory: the blocking number stands)
                pipe = {"error": f"{type(exc).__name__}: {exc}"}
            p_s = sharding.max_over_ranks(pipe.get("s_per_step", 0.0) if pipe else 0.0,
                                          device=dev)
            ok = sharding.max_over_ranks(0.0 if (pipe and "s_per_step" in pipe) or not eng
                                         else 1.0, device=dev) == 0.0
            if ok and p_s > 0:
                e2e = {"value": total / p_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * p_s,
                       "steps": pipe["steps"] if pipe else 0,
                       "api": "FlowEngine.submit_host / finish_host -> dis_flow_batch_host_async "
                              "+ dis_host_batch_finish: two calls in flight (double-buffered; "
                              "pinned host frames in, float64 host flow out, every call's "
                              "copies inside the timed region)",
                       "calls_per_step": pipe["calls_per_step"] if pipe else 0,
                       "pairs_per_call": pipe["pairs_per_call"] if pipe else 0,
                       "blocking": blocking}
            elif pipe and "error" in pipe:
                e2e["pipelined_error"] = pipe["error"]
            # side number, NOT the headline: the same float64 computation with the
            # flow rounded to float32 on the device before the copy-out (opt-in
            # DIS_HOST_FLOW_F32; the copy-out bounds this path, this halves it)
            if ok and p_s > 0 and not args.no_f32_out:
                try:
                    p32 = e2e_pipelined(cfg, params, dev, eng, B, h1, h2, ho,
                                        out if eng else None, max(2 * e2e_steps, 6), f32=True)
                except Exception as exc:
                    p32 = {"error": f"{type(exc).__name__}: {exc}"}
                s32 = sharding.max_over_ranks(p32.get("s_per_step", 0.0), device=dev)
                ok32 = sharding.max_over_ranks(0.0 if "s_per_step" in p32 else 1.0,
                                               device=dev) == 0.0
                if ok32 and s32 > 0:
                    e2e["float32_flow_out"] = {
                        "value": total / s32, "unit": UNIT, "ms_per_step": 1e3 * s32,
                        "d2h_bytes_per_step": int(d2h) // 2,
                        "note": "not the headline: same float64 pipeline, flow rounded to "
                                "float32 on the device before the copy-out "
                                "(out=float32, DIS_HOST_FLOW_F32; == flow.astype(float32)); "
                                "two calls in flight"}
    res = {"value": value, "ms_per_step": ms_step, "pairs_rank": B, "pairs_total": total,
           "e2e": e2e, "roofline": roofline, "kernels": kernels, "clocks": clk,
           "gpu_launches": launches_per_step * steps,
           "timing": {"value": ("CUDA-graph replay of each step (FlowEngine.run(graph=True))"
                                if use_graph else "eager launches"),
                      "kernels": "second timed pass: eager launches, a CUDA event pair around "
                                 "every launch on the launch stream",
                      "eager_ms_per_step": ms_eager, "input_generation_s": t_gen},
           "fp64_peak": {"dadd_TFLOPs": dadd.value / 1e3, "dmul_TFLOPs": dmul.value / 1e3},
           "workspace_bytes": eng.workspace_bytes if eng else 0,
           "frames_bytes": 2 * f1_np.nbytes, "_np": (f1_np, f2_np)}
    del eng
    torch.cuda.empty_cache()
    return res


def e2e_pipelined(cfg, params, dev, eng, B, h1, h2, ho, dev_out, steps, f32=False):
    """Host-buffer calls with two in flight (FlowEngine.submit_host /
    finish_host).  Engines of the config's batch when two of their workspaces
    fit comfortably beside what is resident, else of half the batch (two
    calls per step, e.g. c3's 256 pairs of 1080p).  Returns seconds per step
    (a step = the rank's B pairs), checked against the device-path flow."""
    import torch

    from paper_1603_03590_b200 import FlowEngine, _lib

    if eng is None:
        return {"s_per_step": 0.0, "steps": steps, "calls_per_step": 0, "pairs_per_call": 0}
    L = _lib.lib()
    eng._host_ws = None  # the blocking path's workspace is not needed any more
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(dev)
    code = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.uint8): 2}[h1.dtype]

    def ws_bytes(b):
        return int(L.dis_host_workspace_bytes(b, cfg.height, cfg.width, code,
                                              ctypes.byref(eng.cparams)))
    Be = B
    if 2 * ws_bytes(Be) > 0.6 * free:
        if B % 2 or 2 * ws_bytes(B // 2) > 0.6 * free:
            raise MemoryError(f"two host workspaces do not fit ({free / 2**30:.0f} GiB free)")
        Be = B // 2
    calls_per_step = B // Be
    engs = [FlowEngine(Be, cfg.height, cfg.width, params, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    if f32:  # the opt-in float32 flow (DIS_HOST_FLOW_F32): its own pinned outputs
        ho = torch.empty(ho.shape, dtype=torch.float32).pin_memory().numpy()
    odt = torch.float32 if f32 else torch.float64
    if Be == B:  # each slot its own pinned output; the (read-only) frames are shared
        outs = [ho, torch.empty(ho.shape, dtype=odt).pin_memory().numpy()]
        ins = [(h1, h2), (h1, h2)]
    else:        # each slot one half of the pinned buffers
        outs = [ho[:Be], ho[Be:]]
        ins = [(h1[:Be], h2[:Be]), (h1[Be:], h2[Be:])]
    for o in outs:
        o[...] = 0.0

    def run(n_calls):
        busy = [False, False]
        for i in range(n_calls):
            k = i & 1
            if busy[k]:
                engs[k].finish_host()
            engs[k].submit_host(ins[k][0], ins[k][1], outs[k], stream=streams[k])
            busy[k] = True
        for k in range(2):
            if busy[k]:
                engs[k].finish_host()

    for _ in range(3):  # eager, captured as graphs, replayed
        run(2)
    torch.cuda.synchronize(dev)
    n_calls = steps * calls_per_step
    n_calls += n_calls & 1  # both slots used equally
    t0 = time.perf_counter()
    run(n_calls)
    t1 = time.perf_counter()
    same = True
    for k in range(2):  # first and last pair of each slot against the device-path flow
        base = 0 if Be == B else k * Be
        for i in (0, Be - 1):
            want = dev_out[base + i].cpu().numpy()
            same = same and np.array_equal(outs[k][i], want.astype(np.float32) if f32 else want)
    assert same, "pipelined host path != device path"
    del engs
    torch.cuda.empty_cache()
    return {"s_per_step": (t1 - t0) / (n_calls / calls_per_step), "steps": n_calls // calls_per_step,
            "calls_per_step": calls_per_step, "pairs_per_call": Be}


def run_ours(args, cfg, params):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if torch.cuda.device_count() <= local:
            raise RuntimeError(f"rank {rank}: LOCAL_RANK {local} but only "
                               f"{torch.cuda.device_count()} CUDA devices are visible")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else torch.cuda.current_device())

    main = measure(cfg, params, args, dev, rank, world, args.steps, args.e2e_steps, "main")
    c3 = None
    if cfg.name == "c1" and not args.no_c3:
        c3cfg = synth.CONFIGS["c3"]
        c3p = synth.dis_params(c3cfg)
        c3 = measure(c3cfg, c3p, args, dev, rank, world, args.steps,
                     max(1, min(args.e2e_steps, 3)), "c3")

    # ---- CPU baseline (rank 0, N = 1 only): the reference path on the host ----
    cpu = None
    c3_cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        f1_np, f2_np = main["_np"]
        cpu = cpu_baseline(cfg, params, f1_np, f2_np, args.cpu_pairs, args.ref_kind)
        if c3 is not None:
            a, b = c3["_np"]
            c3_cpu = cpu_baseline(synth.CONFIGS["c3"], synth.dis_params(synth.CONFIGS["c3"]),
                                  a, b, max(8, min(32, cpu["physical_cores"])), args.ref_kind)

    if rank == 0:
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": SCALING[cfg.name], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (tools/synth.py, BASELINE configs' shapes and "
                                    "distributions)",
            "config": config_block(cfg, params, world, main["pairs_rank"], main["pairs_total"], {
                "l2": "inputs larger than L2 (frames "
                      f"{main['frames_bytes'] / 2**20:.0f} MiB + workspace "
                      f"{main['workspace_bytes'] / 2**20:.0f} MiB per GPU per step)"}),
            "roofline": main["roofline"], "cpu_baseline": cpu, "e2e": main["e2e"],
            "gpu_launches": main["gpu_launches"], "clocks": main["clocks"],
            "kernels": main["kernels"], "timing": main["timing"],
            "fp64_peak": main["fp64_peak"],
        }
        if c3 is not None:
            c3cfg = synth.CONFIGS["c3"]
            line["c3"] = {
                "metric": METRIC, "value": c3["value"], "unit": UNIT, "n_gpus": world,
                "ms_per_step": c3["ms_per_step"], "scaling": SCALING["c3"],
                "config": config_block(c3cfg, synth.dis_params(c3cfg), world, c3["pairs_rank"],
                                       c3["pairs_total"], {
                                           "l2": "inputs larger than L2 (frames "
                                                 f"{c3['frames_bytes'] / 2**20:.0f} MiB per GPU)"}),
                "e2e": c3["e2e"], "roofline": c3["roofline"], "kernels": c3["kernels"],
                "clocks": c3["clocks"], "gpu_launches": c3["gpu_launches"],
                "timing": c3["timing"], "cpu_baseline": c3_cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------
# launcher: --gpus N without torchrun -> N ranks under torch.distributed.run
# --------------------------------------------------------------------------

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(n, argv):
    """Re-run this script as N ranks (one per GPU) under torch.distributed.run
    with a 127.0.0.1 rendezvous; returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def launch_selftest(args, cfg):
    """--launch-selftest: each rank joins a gloo group (no GPU), computes its
    share of the config's pairs and reports; rank 0 prints the plan and the
    reductions the bench relies on (barrier, sum and max over ranks)."""
    import torch.distributed as dist

    from paper_1603_03590_b200 import sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    first, count, total = rank_pairs(cfg, rank, world)
    sharding.barrier()
    n_sum = sharding.sum_over_ranks(count)
    t_max = sharding.max_over_ranks(1.0 + rank)
    if rank == 0:
        print(json.dumps({"launch_selftest": True, "world": world, "config": cfg.name,
                          "scaling": SCALING[cfg.name], "pairs_total": total,
                          "pairs_sum_over_ranks": n_sum, "max_over_ranks": t_max,
                          "rank0": [first, count]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(synth.CONFIGS))
    ap.add_argument("--batch", type=int, default=0,
                    help="pairs per GPU (weak configs) / in total (strong); default: config")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f32-out", action="store_true",
                    help="e2e: skip the float32-flow-out side measurement")
    ap.add_argument("--no-pipelined", action="store_true",
                    help="e2e: blocking calls only (skip the two-in-flight measurement)")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of the CUDA-graph replay")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the 1080p block of the c1 line")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-pairs", type=int, default=64)
    ap.add_argument("--ref-pairs", type=int, default=0)
    ap.add_argument("--ref-kind", default="auto", choices=["auto", "reference", "port"],
                    help="host-CPU baseline: the reference package (baseline/_ref), the C "
                         "port, or the package when installed (auto)")
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    cfg = synth.CONFIGS[args.config]
    params = synth.dis_params(cfg)
    in_torchrun = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not in_torchrun:
        if args.impl == "ours" and not args.launch_selftest:
            import torch

            n_dev = torch.cuda.device_count()
            if n_dev < args.gpus:
                raise SystemExit(f"bench.py --gpus {args.gpus}: only {n_dev} CUDA devices are "
                                 "visible (one rank per GPU)")
        if args.impl == "ours" or args.launch_selftest:
            return launch_ranks(args.gpus, argv)
    if in_torchrun and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"[bench] WORLD_SIZE={os.environ['WORLD_SIZE']} overrides --gpus {args.gpus}",
              file=sys.stderr)
    if args.launch_selftest:
        return launch_selftest(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg, params)
    return run_ours(args, cfg, params)


if __name__ == "__main__":
    sys.exit(main())
