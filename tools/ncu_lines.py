"""Per-source-line view of an ncu capture: joins the SASS page of an `.ncu-rep` (instructions
executed, stall samples per SASS address) with the `-lineinfo` line table of the same build
(`nvdisasm -g`), and prints the hottest source lines.

Usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTRING [top] [FILE:LO-HI]
The object must be the one the profiled run loaded (same build).  With FILE:LO-HI, also prints
the stall-reason breakdown of the samples on those source lines.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                       capture_output=True)
        cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], check=True,
                             capture_output=True, text=True).stdout
    table, cur, infn, line = [], None, False, None
    for raw in dis.splitlines():
        if raw.startswith(".text.") and raw.rstrip(":").endswith(tuple([""])):
            infn = kernel in raw
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', raw)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", raw)
        if m:
            table.append((int(m.group(1), 16), line, m.group(2).strip()))
    return table


def main():
    rep, obj, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][ia], 16)
    table = {off: (ln, s) for off, ln, s in line_table(obj, kernel)}
    agg = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    stall_cols = [(k, h) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    rng = None
    if len(sys.argv) > 5:
        f, lh = sys.argv[5].split(":")
        rng = (f, *map(int, lh.split("-")))
    stalls = collections.Counter()
    for r in data:
        off = int(r[ia], 16) - base
        ln = table.get(off, (None, ""))[0]
        if rng and ln and ln[0] == rng[0] and rng[1] <= ln[1] <= rng[2]:
            for k, h in stall_cols:
                stalls[h] += int(float(r[k] or 0))
        i, s = int(float(r[ie] or 0)), int(float(r[isamp] or 0))
        agg[ln][0] += i
        agg[ln][1] += s
        tot_i += i
        tot_s += s
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    for ln, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{str(ln):32s} inst {i:>12,} ({100*i/max(tot_i,1):5.1f}%)  samples {s:>8,} ({100*s/max(tot_s,1):5.1f}%)")
    if rng:
        tot = sum(stalls.values()) or 1
        print(f"stall reasons on {sys.argv[5]} ({tot:,} samples):")
        for h, v in stalls.most_common(8):
            print(f"  {h:28s} {v:>8,} ({100 * v / tot:5.1f}%)")


if __name__ == "__main__":
    main()
