"""Aggregate `ncu --page source --csv --print-source=cuda,sass` output per CUDA source line."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=28):
    rows = list(csv.reader(open(path)))
    cur_file = cur_fn = hdr = None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            cur_fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0]:
            try:
                ln = int(r[0])
            except ValueError:
                continue
            ie = f(r[hdr.index("Instructions Executed")])
            smp = f(r[hdr.index("Warp Stall Sampling (All Samples)")])
            key = ((cur_fn or "")[:60], cur_file, ln, r[1][:90])
            a = agg.setdefault(key, [0.0, 0.0])
            a[0] += ie
            a[1] += smp
    for fn in sorted(set(k[0] for k in agg)):
        items = [(k, v) for k, v in agg.items() if k[0] == fn]
        ti = sum(v[0] for _, v in items) or 1
        ts = sum(v[1] for _, v in items) or 1
        print("=====", fn, "total warp-inst %.4g samples %d" % (ti, ts))
        for k, v in sorted(items, key=lambda kv: -kv[1][1])[:top]:
            print("%5.1f%% inst %5.1f%% smp  %s:%d  %s" % (100 * v[0] / ti, 100 * v[1] / ts, k[1], k[2], k[3]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 28)
