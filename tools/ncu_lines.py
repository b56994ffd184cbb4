#!/usr/bin/env python
"""Per-source-line instructions and warp-stall samples of one kernel of an
ncu report (``--set full --import-source on``):

    python tools/ncu_lines.py gpurun_out/x.ncu-rep KERNEL_REGEX [N] [--by inst|samples]
"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def lines(rep, kern):
    """[(file, line, source, instructions, samples)] over every source file
    the kernel's code maps to."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          "regex:" + kern, "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    res, fname, h = [], "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            fname, h = r[1].split("/")[-1], None
        elif r[0] == "Line No":
            h = r
        elif h is not None and "Instructions Executed" in h and len(r) == len(h) and r[0]:
            res.append((fname, r[0], r[1], num(r[h.index("Instructions Executed")]),
                        num(r[h.index("Warp Stall Sampling (All Samples)")])))
    return res


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    by = "inst"
    if "--by" in sys.argv:
        by = sys.argv[sys.argv.index("--by") + 1]
        args.remove(by)
    rep, kern = args[0], args[1]
    n = int(args[2]) if len(args) > 2 else 30
    L = lines(rep, kern)
    ti = sum(x[3] for x in L) or 1.0
    ts = sum(x[4] for x in L) or 1.0
    print("warp instructions %d, stall samples %d" % (ti, ts))
    key = 3 if by == "inst" else 4
    for f, ln, src, i, s in sorted(L, key=lambda x: -x[key])[:n]:
        print("%-16s %5s %5.1f%% inst %5.1f%% samp  %s" % (f, ln, 100 * i / ti, 100 * s / ts,
                                                           src.strip()[:90]))


if __name__ == "__main__":
    main()
