"""Per-pair opcode mix and stall totals from an ncu SASS source-page CSV (diagnostic).

  ncu -i REP --page source --csv --print-source sass --launch-skip S --launch-count 1 > src.csv
  python tools/ncu_mix.py src.csv PAIRS
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    pairs = float(sys.argv[2])
    which = int(sys.argv[3]) if len(sys.argv) > 3 else 0      # k-th kernel block of the CSV
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append((r[1], cur))
        elif cur is not None:
            cur.append(r)
    name, blk = blocks[which]
    print(name)
    hdr = blk[0]
    data = [r for r in blk[1:] if len(r) == len(hdr) and r[0] != "Address"]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[iex] or 0) for r in data)
    print(f"warp instructions {tot:.0f}  thread instructions per pair {32 * tot / pairs:.1f}")
    c = collections.Counter()
    for r in data:
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += float(r[iex] or 0)
    for o, v in c.most_common(25):
        print(f"  {o:10s} {32 * v / pairs:7.1f} per pair  {100 * v / tot:5.1f}%")
    st = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in stall}
    s = sum(st.values())
    print("stalls:", ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]))


if __name__ == "__main__":
    main()
