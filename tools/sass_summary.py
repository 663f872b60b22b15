#!/usr/bin/env python
"""Instruction mix and stall hot spots from `ncu --page source --print-source
sass --csv` pages (tools/gpu_round.sh's sass_<kernel>_<tag>.csv):

    python tools/sass_summary.py --tag r1g gpurun_out/sass_k_*_r1g.csv

Writes profiles/<tag>_sass_summary.md."""

import argparse
import collections
import csv
import os


def summarise(path, top=12):
    rows = list(csv.reader(open(path)))
    name = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else path
    hdr = rows[1]
    i_src = hdr.index("Source")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    mix = collections.Counter()
    stalls = []
    tot_ex = tot_st = 0
    for r in rows[2:]:
        if len(r) <= i_ex or not r[0].startswith("0x"):
            continue
        op = r[i_src].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        opc = op.split()[0] if op else "?"
        ex = int(r[i_ex] or 0)
        st = int(r[i_st] or 0)
        mix[opc] += ex
        tot_ex += ex
        tot_st += st
        stalls.append((st, op))
    stalls.sort(reverse=True)
    out = [f"### `{name.split('(')[0]}`", "",
           f"{tot_ex:,} warp instructions, {tot_st:,} stall samples.", "",
           "| opcode | share of instructions |", "|---|---|"]
    out += [f"| `{o}` | {100 * n / max(1, tot_ex):.1f} % |" for o, n in mix.most_common(top)]
    out += ["", "| stall samples | instruction |", "|---|---|"]
    out += [f"| {100 * s / max(1, tot_st):.1f} % | `{o[:70]}` |" for s, o in stalls[:8]]
    return out + [""]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("pages", nargs="+")
    args = ap.parse_args()
    md = [f"# SASS instruction mix and stall hot spots ({args.tag})", "",
          "Source pages of single launches (the finest level's launch of a warm-up "
          "step of `bench.py --config c1`), `ncu --set full --import-source on`.", ""]
    for p in args.pages:
        md += summarise(p)
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       f"{args.tag}_sass_summary.md")
    open(dst, "w").write("\n".join(md))
    print(dst)


if __name__ == "__main__":
    main()
