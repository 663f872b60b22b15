"""Summarise a bench.py JSON line: python tools/bench_summary.py gpurun_out/bench_X.log"""
import json
import sys


def summ(d, name):
    e = d.get("e2e") or {}
    print(f"{name}: value {d['value']:.0f} pairs/s, {d['ms_per_step']:.3f} ms/step; "
          f"e2e {e.get('value', 0):.0f} ({e.get('ms_per_step', 0):.2f} ms)")
    r = d.get("roofline", {})
    print("  roofline", r.get("kernel"), r.get("bound"), round(r.get("frac", 0), 3),
          "dram_frac", round(r.get("dram_frac", 0) or 0, 3))
    for k, v in d["kernels"].items():
        print(f"  {k:16s} {v['ms_per_step']:7.3f} ms  hbm {v.get('hbm_frac', 0):.3f}  "
              f"fp64 {v.get('fp64_frac', 0):.3f}  launches {v['launches_per_step']:.0f}")
    if d.get("cpu_baseline"):
        print("  cpu", round(d["cpu_baseline"]["value"], 1), d["cpu_baseline"].get("kind"))


for path in sys.argv[1:]:
    line = [ln for ln in open(path).read().splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    summ(d, d["config"]["workload"])
    if "c3" in d:
        summ(d["c3"], "c3")
    print("  clocks", d.get("clocks"))
