"""Per-source-line instruction counts from `ncu --page source --csv --print-source cuda,sass` (diagnostic).
  python tools/ncu_lines.py <csv> <pairs> [top]"""
import csv
import sys


def main(path, pairs, top=40):
    cur = None
    agg = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0] and r[0].isdigit() and len(r) > 7:
            try:
                ie = float(r[7])
                smp = float(r[4])
            except ValueError:
                continue
            if ie or smp:
                a = agg.setdefault((cur, int(r[0]), r[1].strip()[:80]), [0.0, 0.0])
                a[0] += ie
                a[1] += smp
    ti = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total thread-inst/eval {32 * ti / pairs:.1f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{32 * v[0] / pairs:7.1f} inst/eval {100 * v[1] / ts:5.1f}% smp  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
