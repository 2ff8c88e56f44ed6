"""Aggregate tools/ncu_lines.py output by source-line ranges ("phases").

  python tools/ncu_phases.py REPORT OBJ KERNEL FILE name:lo-hi name:lo-hi ...
Lines of FILE outside every range, and lines of other files (inlined helpers), are grouped
as 'other:<file>' / 'helpers'.
"""
import re
import subprocess
import sys


def main():
    rep, obj, kern, fname = sys.argv[1:5]
    ranges = []
    for spec in sys.argv[5:]:
        n, r = spec.split(":")
        lo, hi = r.split("-")
        ranges.append((int(lo), int(hi), n))
    out = subprocess.run([sys.executable, __file__.replace("ncu_phases", "ncu_lines"), rep, obj, kern, "100000"],
                         capture_output=True, text=True).stdout
    agg = {}
    for l in out.splitlines()[1:]:
        m = re.match(r"\('(\S+)', (\d+)\)\s+inst\s+([\d,]+).*samples\s+([\d,]+)", l)
        if m:
            f, ln = m.group(1), int(m.group(2))
            i, s = int(m.group(3).replace(",", "")), int(m.group(4).replace(",", ""))
            name = "helpers:" + f
            if f == fname:
                name = next((n for lo, hi, n in ranges if lo <= ln <= hi), f"{fname}:other")
        else:
            m = re.match(r"(\S+)\s+inst\s+([\d,]+).*samples\s+([\d,]+)", l)
            if not m:
                continue
            name, i, s = "unmapped", int(m.group(2).replace(",", "")), int(m.group(3).replace(",", ""))
        a = agg.setdefault(name, [0, 0])
        a[0] += i
        a[1] += s
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} inst {100 * v[0] / ti:5.1f}%  samples {100 * v[1] / ts:5.1f}%")


if __name__ == "__main__":
    main()
