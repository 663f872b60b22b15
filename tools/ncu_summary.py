#!/usr/bin/env python
"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py --tag r1a --launches gpurun_out/launches_r1a.csv \
        [--rep gpurun_out/full_r1a.ncu-rep] [--config c1] [--steps 4]

* launch list (``ncu --metrics gpu__time_duration.sum --csv``): per-kernel
  launch count, total and mean duration, share of the GPU time;
* full capture (``ncu --set full`` .ncu-rep, read with ``ncu -i --page raw``):
  per launch duration, DRAM bytes read/written, achieved DRAM GB/s, FP64 pipe
  utilisation, issue-slot utilisation, achieved occupancy, top stall reasons.

Writes profiles/<tag>_launches.csv (trimmed), profiles/<tag>_summary.md and
merges each kernel class's DRAM traffic over the captured step into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic, per launch).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

# kernel name -> bench.py kernel class
CLASS_OF = [
    (r"k_sor", "sor"),
    (r"k_tensor_assemble", "tensor_assemble"),
    (r"k_patch|k_bidir_prep|k_pad_query", "patch_search"),
    (r"k_densify", "densify"),
    (r"k_upsample|k_interleave|k_flow_to_f32", "upsample"),
    (r"k_level1|k_downsample|k_gradients|k_convert|k_level0|k_pyr_", "pyramid"),
]


def kclass(name):
    for pat, c in CLASS_OF:
        if re.search(pat, name):
            return c
    return "other"


def short(name):
    return re.sub(r"\(.*", "", name).replace("void ", "").strip()


def read_csv_skip(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.reader(io.StringIO("".join(lines))))


def launches(path):
    rows = read_csv_skip(path)
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in rows[1:]:
        if len(r) <= vi or re.search(r"fp64_peak|selftest", r[ki]):
            continue  # bench's peak microbenchmark, not the flow path
        out.append((short(r[ki]), float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0),
                    r[gi], r[bi]))
    return out


RAW_KEYS = {
    "dur_us": ("gpu__time_duration.sum", {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                           "msecond": 1e3, "nsecond": 1e-3}),
    "dram_rd": ("dram__bytes_read.sum", None),
    "dram_wr": ("dram__bytes_write.sum", None),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", None),
    "issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "occ_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "l1_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "inst": ("smsp__inst_executed.sum", None),
}
BYTE_UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
              "GB": 1e9}


def full_capture(rep):
    if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
        with open(rep) as f:
            txt = f.read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = [r for r in csv.reader(io.StringIO(txt)) if r]
    while rows and "Kernel Name" not in rows[0]:
        rows.pop(0)
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[idx["Kernel Name"]]), "grid": r[idx["Grid Size"]],
             "block": r[idx["Block Size"]]}
        for k, (col, sc) in RAW_KEYS.items():
            if col not in idx:
                continue
            v = r[idx[col]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[idx[col]]
            if sc is not None:
                x *= sc.get(u, 1.0)
            elif k.startswith("dram_r") or k.startswith("dram_w"):
                x *= BYTE_UNITS.get(u, 1.0)
            d[k] = x
        st = []
        for c in stall_cols:
            try:
                st.append((float(r[idx[c]]), c[len("smsp__average_warps_issue_stalled_"):
                                               -len("_per_issue_active.ratio")]))
            except ValueError:
                pass
        d["stalls"] = [f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:4]]
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--rep", default=None)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--steps", type=int, default=1, help="pipeline steps in the launch list")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)

    L = launches(args.launches)
    agg = collections.OrderedDict()
    for name, us, grid, block in L:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    md = [f"# ncu summary {args.tag} ({args.config})", ""]
    if args.note:
        md += [args.note, ""]
    md += [f"Launch list: {len(L)} launches over {args.steps} pipeline step(s), "
           f"GPU time {tot / 1e3:.3f} ms ({tot / 1e3 / args.steps:.3f} ms per step). "
           "ncu per-launch times are serialised and cold-cache (`--clock-control none`).", "",
           "| kernel | class | launches | total ms | mean us | share |", "|---|---|---|---|---|---|"]
    cls_tot = collections.Counter()
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        cls_tot[kclass(name)] += us
        md.append(f"| `{name}` | {kclass(name)} | {n} | {us / 1e3:.3f} | {us / n:.1f} | "
                  f"{100 * us / tot:.1f}% |")
    md += ["", "| class | share of GPU time |", "|---|---|"]
    for c, us in cls_tot.most_common():
        md.append(f"| {c} | {100 * us / tot:.1f}% |")
    with open(os.path.join(PROF, f"{args.tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "class", "grid", "block", "us"])
        for name, us, grid, block in L:
            w.writerow([name, kclass(name), grid, block, f"{us:.3f}"])

    if args.rep:
        F = full_capture(args.rep)
        md += ["", f"## Full captures (`ncu --set full`, {os.path.basename(args.rep)})", "",
               "| kernel | grid x block | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | FP64 pipe % "
               "| issue % | warps active % | L1 % | top stalls (per issue) |",
               "|---|---|---|---|---|---|---|---|---|---|---|"]
        traffic = {}
        for d in F:
            rd, wr, us = d.get("dram_rd", 0.0), d.get("dram_wr", 0.0), d.get("dur_us", 0.0)
            gbs = (rd + wr) / (us * 1e-6) / 1e9 if us else 0.0
            md.append(f"| `{d['kernel']}` | {d['grid']} x {d['block']} | {us:.1f} | "
                      f"{rd / 1e6:.2f} | {wr / 1e6:.2f} | {gbs:.0f} | "
                      f"{d.get('fp64_pct', 0):.1f} | {d.get('issue_pct', 0):.1f} | "
                      f"{d.get('occ_pct', 0):.1f} | {d.get('l1_pct', 0):.1f} | "
                      f"{'; '.join(d['stalls'])} |")
            c = kclass(d["kernel"])
            traffic.setdefault(c, []).append(rd + wr)
        path = os.path.join(PROF, "ncu_traffic.json")
        try:
            with open(path) as f:
                tj = json.load(f)
        except Exception:
            tj = {}
        # DRAM bytes of a class over the captured pipeline step (bench.py
        # divides by its per-step launch count of the class)
        tj[args.config] = {c: sum(v) for c, v in traffic.items()}
        tj.setdefault("_source", {})[args.config] = f"{args.tag}: {os.path.basename(args.rep)}"
        with open(path, "w") as f:
            json.dump(tj, f, indent=1, sort_keys=True)
    with open(os.path.join(PROF, f"{args.tag}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
