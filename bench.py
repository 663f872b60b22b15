#!/usr/bin/env python
"""Benchmark of the DIS flow hot path (BASELINE.json metric: flow
frame-pairs/sec) — see DESIGN.md "Measurement".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1]
    python bench.py --impl reference ...      # the CPU reference arm

A step = one pass of the whole coarse-to-fine DIS pipeline over one batch of
the config's synthetic pairs (c1: 64 pairs of 1024x436, DIS medium operating
point, refinement 1 outer / 5 inner).  Multi-GPU: one process per GPU
(torchrun), each rank runs its own batch of independent pairs (no
collective on the data path; weak scaling); the step time is the max over
ranks.

One JSON line on rank 0.  `value` = device-resident throughput (inputs in HBM
before the timed region); `e2e` = the same metric through the C ABI's
host-buffer entry point (pinned host frames in, host flow out, copies inside
the timed region); `roofline` = the dominant kernel class against the
measured HBM copy peak; `cpu_baseline` = the CPU oracle (a port of the
reference path, oracle/dis_oracle.c) on a bounded sample on this host.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import multiprocessing as mp
import os
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


def measured_peak_gbs():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config_name, kernel_class, launches_per_step):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    a kernel class, from the committed `ncu --set full` capture of one
    pipeline step (profiles/ncu_traffic.json holds the class's per-step
    total), or None."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            v = json.load(f).get(config_name, {}).get(kernel_class)
        return None if v is None else v / max(1.0, launches_per_step)
    except Exception:
        return None


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------

def _gen_chunk(args):
    name, seed, first, count = args
    return synth.make_batch(synth.CONFIGS[name], seed=seed, count=count, first=first)


def make_inputs(cfg, seed, count, workers):
    """Synthetic pairs (pair i from seed + i), generated in parallel."""
    if cfg.stream or workers <= 1 or count <= 2:
        return synth.make_batch(cfg, seed=seed, count=count)
    chunks = []
    step = max(1, math.ceil(count / workers))
    for first in range(0, count, step):
        chunks.append((cfg.name, seed, first, min(step, count - first)))
    with mp.get_context("fork").Pool(min(workers, len(chunks))) as pool:
        parts = pool.map(_gen_chunk, chunks)
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# CPU oracle (reference path port) — bounded sample on all host cores
# --------------------------------------------------------------------------

def _oracle_worker(args):
    f1, f2, params = args
    from oracle import oracle

    t = time.perf_counter()
    oracle.dis_flow_batch_f32(f1, f2, params)
    return time.perf_counter() - t, f1.shape[0]


def cpu_oracle_rate(cfg, params, f1, f2, cores, pairs):
    """pairs/s of the oracle over `pairs` pairs spread over `cores` processes
    (one process per core, each a scalar C port of the reference path)."""
    pairs = min(pairs, f1.shape[0])
    idx = [list(range(i, pairs, cores)) for i in range(cores)]
    idx = [i for i in idx if i]
    jobs = [(f1[i], f2[i], params) for i in idx]
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        pool.map(_oracle_worker, [(f1[:1], f2[:1], params)] * len(jobs))  # warm
        t = time.perf_counter()
        res = pool.map(_oracle_worker, jobs)
        wall = time.perf_counter() - t
    return pairs / wall, len(jobs), pairs, wall


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
# arms
# --------------------------------------------------------------------------

def run_reference(args, cfg, params):
    """--impl reference: the reference path on the host CPU (oracle port,
    all host cores), same metric/config; each step = a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = host_cores()
    sample = max(cores, args.ref_pairs or cores)
    f1, f2 = make_inputs(cfg, seed=0, count=sample, workers=cores)
    rates = []
    walls = []
    for _ in range(args.steps):
        r, used, n, wall = cpu_oracle_rate(cfg, params, f1, f2, cores, sample)
        rates.append(r)
        walls.append(wall)
    value = sample * len(rates) / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "pairs_per_step": sample, "height": cfg.height,
                   "width": cfg.width},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port",
                         "sample": f"{sample} {cfg.name} pairs per step over {used} processes "
                                   "(oracle/dis_oracle.c, one scalar process per core)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg, params):
    import torch
    import torch.distributed as dist

    from paper_1603_03590_b200 import FlowEngine, _lib, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    B = args.batch or cfg.batch
    cores = host_cores()
    gen_workers = max(1, cores // max(1, world))
    f1_np, f2_np = make_inputs(cfg, seed=1000 * rank, count=B, workers=gen_workers)
    eng = FlowEngine(B, cfg.height, cfg.width, params, device=dev)
    stream = torch.cuda.current_stream(dev)
    f1 = torch.from_numpy(f1_np).to(dev)
    f2 = torch.from_numpy(f2_np).to(dev)
    out = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64, device=dev)
    L = _lib.lib()

    barrier = sharding.barrier

    # warm-up (first call checks the status word: errors surface here)
    for i in range(max(1, args.warmup)):
        eng.run(f1, f2, out=out, stream=stream, check=(i == 0))
    torch.cuda.synchronize(dev)
    launches_per_step = int(L.dis_last_launch_count())

    # untimed census step: window evaluations of the patch search (FP64
    # roofline numerator), and the FP64 peak of this device
    _lib.check(L.dis_census_enable(1))
    eng.run(f1, f2, out=out, stream=stream, check=False)
    torch.cuda.synchronize(dev)
    ev_n, ev_p = ctypes.c_longlong(0), ctypes.c_longlong(0)
    _lib.check(L.dis_census_read(ctypes.byref(ev_n), ctypes.byref(ev_p)))
    _lib.check(L.dis_census_enable(0))
    evals_step = int(ev_n.value)
    dadd, dmul = ctypes.c_double(0), ctypes.c_double(0)
    _lib.check(L.dis_selftest_fp64_peak(ctypes.byref(dadd), ctypes.byref(dmul),
                                        _lib.stream_handle(stream)))
    fp64_peak_tflops = min(dadd.value, dmul.value) / 1e3

    # ---- timed region: device-resident inputs (> L2: 2 x B x H x W x 4 B) ----
    # `value`: the step replayed as one CUDA graph (FlowEngine.run(graph=True):
    # the same kernels and arguments, without the per-launch gaps); captured
    # and replayed once before timing.  Then a second timed pass of the same
    # steps with eager launches and per-kernel-class CUDA events gives the
    # kernel breakdown and the rooflines (events between launches add a
    # little time, so that pass's step time is reported beside `value`).
    gstream = torch.cuda.Stream(device=dev)
    gstream.wait_stream(stream)
    use_graph = not args.no_graph
    if use_graph:
        eng.run(f1, f2, out=out, stream=gstream, check=True, graph=True)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev.index).start()
    barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(gstream)
    for _ in range(args.steps):
        eng.run(f1, f2, out=out, stream=gstream, check=False, graph=use_graph)
    ev1.record(gstream)
    torch.cuda.synchronize(dev)
    barrier()
    ms_total = sharding.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    eng.check_status(gstream)  # any non-finite / coverage failure raises here
    # kernel-breakdown pass (eager, per-class events)
    L.dis_profile_reset()
    L.dis_profile_enable(1)
    barrier()
    torch.cuda.synchronize(dev)
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(args.steps):
        eng.run(f1, f2, out=out, stream=stream, check=False)
    ev3.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    L.dis_profile_enable(0)
    ms_eager = sharding.max_over_ranks(ev2.elapsed_time(ev3), device=dev) / args.steps
    eng.check_status(stream)
    nk = len(_lib.KERNEL_CLASSES)
    kms = (ctypes.c_double * nk)()
    kcnt = (ctypes.c_int64 * nk)()
    _lib.check(L.dis_profile_read(kms, kcnt, nk))
    kernels = {name: {"ms_per_step": kms[i] / args.steps,
                      "launches_per_step": kcnt[i] / args.steps}
               for i, name in enumerate(_lib.KERNEL_CLASSES)}
    ms_step = ms_total / args.steps
    value = world * B / (ms_step / 1e3)

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
        if name in flops:
            k["algorithmic_TFLOPs"] = flops[name] / sec / 1e12
            k["fp64_frac"] = k["algorithmic_TFLOPs"] / fp64_peak_tflops
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    d = kernels[dom]
    launches = max(1.0, d["launches_per_step"])
    ms_per_launch = d["ms_per_step"] / launches
    if dom == "patch_search":
        # FP64-bound: no stage of the patch search streams HBM (windows hit L1)
        per_launch = flops[dom] / launches
        achieved = per_launch / (ms_per_launch / 1e3) / 1e12
        roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved,
                    "peak": fp64_peak_tflops, "unit": "TFLOP/s",
                    "frac": achieved / fp64_peak_tflops,
                    "traffic": ncu_traffic(cfg.name, dom, launches),
                    "peak_source": "measured live: DADD independent chains, no FMA "
                                   "(dis_selftest_fp64_peak)",
                    "algorithmic_flops_per_launch": per_launch,
                    "evaluations_per_step": evals_step,
                    "hbm_frac": d["hbm_frac"]}
    else:
        bytes_per_launch = per_pair[dom] * B / launches
        achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak,
                    "traffic": ncu_traffic(cfg.name, dom, launches), "peak_source": peak_kind,
                    "algorithmic_bytes_per_launch": bytes_per_launch}
        if "fp64_frac" in d:
            roofline["fp64_frac"] = d["fp64_frac"]

    # ---- e2e: host buffers through the C ABI (copies in the timed region) ----
    e2e = None
    if not args.no_e2e:
        pin1 = torch.from_numpy(f1_np).pin_memory()
        pin2 = torch.from_numpy(f2_np).pin_memory()
        pout = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64).pin_memory()
        h1, h2, ho = pin1.numpy(), pin2.numpy(), pout.numpy()
        eng.run_host(h1, h2, out=ho, stream=stream)
        torch.cuda.synchronize(dev)
        e_steps = max(1, min(args.steps, args.e2e_steps))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            eng.run_host(h1, h2, out=ho, stream=stream)
        t1 = time.perf_counter()
        e_s = sharding.max_over_ranks(t1 - t0, device=dev) / e_steps
        assert np.array_equal(ho[0], out[0].cpu().numpy()), "host path != device path"
        e2e = {"value": world * B / e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h1.nbytes + h2.nbytes),
               "d2h_bytes_per_step": int(ho.nbytes), "ms_per_step": 1e3 * e_s,
               "steps": e_steps}

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n = min(B, max(cores, args.cpu_pairs))
        rate, used, npairs, wall = cpu_oracle_rate(cfg, params, f1_np, f2_np, cores, n)
        cpu = {"value": rate, "unit": UNIT, "cores": used, "kind": "port",
               "sample": f"{npairs} {cfg.name} pairs over {used} processes in {wall:.1f} s "
                         "(oracle/dis_oracle.c, one scalar process per core)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "pairs_per_gpu": B, "height": cfg.height,
                       "width": cfg.width, "patch_size": cfg.patch_size,
                       "overlap": cfg.overlap, "iterations": cfg.iterations,
                       "finest_scale": cfg.finest_scale,
                       "coarsest_scale": params.coarsest_scale,
                       "refinement": f"{params.variational.outer_iters(0)} outer / "
                                     f"{params.variational.inner_sor_iters} inner",
                       "parallelism": f"pair-sharded x{world}, no collective",
                       "l2": "inputs larger than L2 (frames "
                             f"{2 * f1_np.nbytes / 2**20:.0f} MiB + workspace "
                             f"{eng.workspace_bytes / 2**20:.0f} MiB per step)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk, "kernels": kernels,
            "timing": {"value": ("CUDA-graph replay of each step (FlowEngine.run(graph=True))"
                                 if use_graph else "eager launches"),
                       "kernels": "second timed pass: eager launches, per-class CUDA events "
                                  "on the launch stream",
                       "eager_ms_per_step": ms_eager},
            "fp64_peak": {"dadd_TFLOPs": dadd.value / 1e3, "dmul_TFLOPs": dmul.value / 1e3},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(synth.CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="pairs per GPU (default: config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of the CUDA-graph replay")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-pairs", type=int, default=64)
    ap.add_argument("--ref-pairs", type=int, default=0)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    cfg = synth.CONFIGS[args.config]
    params = synth.dis_params(cfg)
    if args.impl == "reference":
        return run_reference(args, cfg, params)
    return run_ours(args, cfg, params)


if __name__ == "__main__":
    sys.exit(main())
