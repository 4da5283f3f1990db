#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: opcode mix, stall reasons, hot instructions.

usage: python tools/ncu_sass_hotspots.py REPORT.ncu-rep [--top N]
"""
import collections
import csv
import io
import subprocess
import sys


def pages(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    cur, name = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            if name:
                yield name, cur
            name, cur = line.split('","')[1].rstrip('",'), []
        else:
            cur.append(line)
    if name:
        yield name, cur


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    for name, lines in pages(rep):
        rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
        if not rows:
            continue
        stall_keys = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
        ops = collections.Counter()
        stalls = collections.Counter()
        samples = 0
        for r in rows:
            src = r["Source"].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            ex = int(float(r["Instructions Executed"] or 0))
            ops[op.split(".")[0]] += ex
            for k in stall_keys:
                stalls[k] += int(float(r[k] or 0))
            samples += int(float(r["Warp Stall Sampling (All Samples)"] or 0))
        tot = sum(ops.values())
        print(f"== {name}\n   warp instructions executed {tot:,}; stall samples {samples:,}")
        print("   opcode mix (warp-level, % of executed):")
        for op, c in ops.most_common(24):
            print(f"     {op:10s} {100 * c / tot:6.2f}%")
        print("   stall reasons (% of samples):")
        for k, c in stalls.most_common(10):
            print(f"     {k:24s} {100 * c / max(samples, 1):6.2f}%")
        hot = sorted(rows, key=lambda r: -int(float(r["Warp Stall Sampling (All Samples)"] or 0)))[:top]
        print("   hottest instructions:")
        for r in hot:
            print(f"     {r['Address'][-5:]} {int(float(r['Warp Stall Sampling (All Samples)'])):6d}  {r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
