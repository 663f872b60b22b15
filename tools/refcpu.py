"""The host-CPU baselines that bench.py times beside the GPU.

* ``reference``: the UNMODIFIED reference package (``disflow``, numba,
  float64) installed into ``baseline/_ref`` by
  ``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of
  /root/reference/pkg>``, called through its public entry point
  ``disflow.dis_flow(frame1, frame2, params)`` (pipeline.py:150-163).  The only
  non-default object is the parameter set: BASELINE's "1 outer" refinement is
  a ``VarParams`` subclass whose ``outer_iters`` returns 1 — the hook the
  reference's ``refine`` calls (variational.py:252).
* ``port``: the C restatement of the same path (``oracle/dis_oracle.c``),
  used when the reference package is not installed.

Both run one single-threaded worker process per PHYSICAL host core (pinned to
one logical CPU of that core), as BASELINE.md §3 plans: numba's own threading
only covers the patch loop and is slower than processes.  Workers
are forked after the parent has JIT-compiled every reference kernel, so no
compilation happens inside a timed region.
"""

from __future__ import annotations

import dataclasses
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(REPO, "baseline", "_ref")


# --------------------------------------------------------------------------
# host description
# --------------------------------------------------------------------------

def _affinity():
    try:
        return sorted(os.sched_getaffinity(0))
    except Exception:
        return list(range(os.cpu_count() or 1))


def host_info() -> dict:
    """CPU model, logical CPUs usable by this process, and one logical CPU per
    physical core among them (``/proc/cpuinfo`` physical id + core id)."""
    cpus = _affinity()
    model = "unknown"
    core_of = {}
    try:
        with open("/proc/cpuinfo") as f:
            blocks = f.read().strip().split("\n\n")
        for b in blocks:
            kv = {}
            for line in b.splitlines():
                if ":" in line:
                    k, v = line.split(":", 1)
                    kv[k.strip()] = v.strip()
            if "processor" not in kv:
                continue
            cpu = int(kv["processor"])
            model = kv.get("model name", model)
            core_of[cpu] = (kv.get("physical id", "0"), kv.get("core id", str(cpu)))
    except Exception:
        pass
    seen = {}
    for c in cpus:
        key = core_of.get(c, ("0", str(c)))
        seen.setdefault(key, c)
    phys = sorted(seen.values())
    return {"model": model, "logical": len(cpus), "physical": len(phys), "physical_cpus": phys,
            "sockets": len({k[0] for k in seen})}


# --------------------------------------------------------------------------
# the reference package
# --------------------------------------------------------------------------

_REF = None


def load_reference():
    """Import the installed reference (baseline/_ref) or return None."""
    global _REF
    if _REF is not None:
        return _REF
    if not os.path.isdir(os.path.join(REF_DIR, "disflow")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    os.environ["NUMBA_NUM_THREADS"] = "1"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import disflow  # noqa: F401
        from disflow import core, inverse_search, pipeline
    except Exception as e:  # numba missing / broken install
        print(f"[refcpu] reference import failed: {e!r}", file=sys.stderr)
        return None

    @dataclasses.dataclass(frozen=True)
    class VarParamsFixed(core.VarParams):
        """VarParams with a fixed number of outer iterations (BASELINE's
        "1 outer"); the reference's own hook, variational.py:252."""

        fixed_outer: int = 1

        def outer_iters(self, scale_index: int) -> int:
            return self.fixed_outer

    _REF = {"disflow": disflow, "core": core, "pipeline": pipeline, "inv": inverse_search,
            "VarParamsFixed": VarParamsFixed}
    return _REF


def reference_params(ref, params):
    """The reference's DisParams for one of our DisParams (same fields)."""
    core = ref["core"]
    vp = params.variational
    var = None
    if vp is not None:
        kw = dict(intensity_weight=vp.intensity_weight, gradient_weight=vp.gradient_weight,
                  smoothness_weight=vp.smoothness_weight, inner_sor_iters=vp.inner_sor_iters,
                  penalizer_eps=vp.penalizer_eps, sor_omega=vp.sor_omega)
        var = (ref["VarParamsFixed"](fixed_outer=vp.outer_iters_fixed, **kw)
               if vp.outer_iters_fixed else core.VarParams(**kw))
    return core.DisParams(
        patch_size=params.patch_size, overlap=params.overlap, iterations=params.iterations,
        finest_scale=params.finest_scale, coarsest_scale=params.coarsest_scale,
        downscale=params.downscale, use_mean_normalization=params.use_mean_normalization,
        use_densification=params.use_densification, residual_norm=params.residual_norm,
        huber_b=params.huber_b, variational=var, mode=params.mode,
        bidirectional=params.bidirectional)


def warm_reference(ref):
    """JIT-compile every reference kernel in this (parent) process: the
    package's own warmup() plus _window_stats, which warmup never reaches
    (SURVEY §6b)."""
    ref["pipeline"].warmup()
    inv = ref["inv"]
    q = np.random.default_rng(0).uniform(0, 255, (12, 16))
    xs = np.array([2.0])
    ys = np.array([2.0])
    inv._window_stats(q, xs, ys, 4, np.zeros((1, 16)), np.zeros(1), np.ones(1, dtype=np.bool_),
                      np.zeros((1, 2)), True, np.zeros(1), np.zeros(1))


# --------------------------------------------------------------------------
# process pool over pairs
# --------------------------------------------------------------------------

_JOB = {}


def _pin(cpu_list):
    if cpu_list is None:
        return
    try:
        ident = mp.current_process()._identity
        k = (ident[0] - 1) if ident else 0
        os.sched_setaffinity(0, {cpu_list[k % len(cpu_list)]})
    except Exception:
        pass


def _run_indices(idx):
    kind = _JOB["kind"]
    f1, f2 = _JOB["f1"], _JOB["f2"]
    t = time.perf_counter()
    if kind == "reference":
        dis_flow = _JOB["ref"]["pipeline"].dis_flow
        p = _JOB["rparams"]
        for i in idx:
            dis_flow(f1[i], f2[i], p)
    else:
        from oracle import oracle

        for i in idx:
            oracle.dis_flow_batch_f32(f1[i:i + 1], f2[i:i + 1], _JOB["params"])
    return time.perf_counter() - t, len(idx)


def _init_worker(cpu_list):
    _pin(cpu_list)


class CpuPool:
    """One forked single-threaded worker per physical core (pinned), over the
    pairs of ``f1``/``f2``; ``kind`` "reference" (numba package) or "port"."""

    def __init__(self, f1, f2, params, kind="auto", workers=None):
        self.info = host_info()
        ref = load_reference() if kind in ("auto", "reference") else None
        if kind == "reference" and ref is None:
            raise RuntimeError("reference package not installed in baseline/_ref")
        self.kind = "reference" if ref is not None else "port"
        _JOB.clear()
        _JOB.update(kind=self.kind, f1=f1, f2=f2, params=params, ref=ref)
        if ref is not None:
            _JOB["rparams"] = reference_params(ref, params)
            warm_reference(ref)
            ref["pipeline"].dis_flow(f1[0], f2[0], _JOB["rparams"])  # one untimed pair
        else:
            from oracle import oracle

            oracle.lib()
        cpus = self.info["physical_cpus"]
        self.workers = workers or len(cpus)
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_init_worker,
                                                initargs=(cpus,))
        # wake every worker (fork + first touch) outside the timed region
        self.pool.map(_run_indices, [[0]] * self.workers, chunksize=1)

    def run(self, n_pairs):
        """Wall time to process pairs 0..n_pairs-1 (round-robin over workers)."""
        n = min(n_pairs, self._len())
        parts = [list(range(w, n, self.workers)) for w in range(self.workers)]
        parts = [p for p in parts if p]
        t = time.perf_counter()
        res = self.pool.map(_run_indices, parts, chunksize=1)
        wall = time.perf_counter() - t
        per_pair = sum(r[0] for r in res) / max(1, sum(r[1] for r in res))
        return wall, n, len(parts), per_pair

    def _len(self):
        return _JOB["f1"].shape[0]

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, n, used):
        src = ("reference package disflow (numba, float64) from baseline/_ref via "
               "disflow.dis_flow" if self.kind == "reference"
               else "oracle/dis_oracle.c (C port of the reference path)")
        return (f"{n} pairs per step over {used} single-threaded processes, one per physical "
                f"core ({self.info['model']}; {self.info['physical']} physical / "
                f"{self.info['logical']} logical CPUs available); {src}")
