"""Instruction counts and stall samples per device function (diagnostic).

  ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:bessel_eval_kernel \
      --launch-count 1 > src.csv
  python tools/ncu_funcs.py src.csv <pairs>
Each source line is charged to the nearest preceding __device__ function of its
file; lines of the __global__ kernel body land on the last helper above it
(printed as "kernel body").
"""
import csv, re, sys
src = {}
for f in ("bessel_math.cuh", "fastmath.cuh", "bessel_kernels.cu"):
    lines = open("paper_2409_08729_b200/csrc/" + f).read().split("\n")
    cur = "?"
    m = []
    for i, l in enumerate(lines, 1):
        mm = re.search(r"__device__[^(]*?\b(\w+)\s*\(", l) or re.search(r"^(\w[\w<>:, ]*?)\s+(\w+)\(.*\)\s*\{\s*$", l)
        if mm and "__device__" in l:
            cur = mm.group(1)
        if "__global__" in l:
            cur = "kernel body"
        m.append(cur)
    src[f] = m
agg = {}
cur = None
for r in csv.reader(open(sys.argv[1])):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0].isdigit() and len(r) > 7 and cur in src:
        try: smp = float(r[4]); ie = float(r[7])
        except ValueError: continue
        fn = src[cur][int(r[0]) - 1]
        a = agg.setdefault(cur + ":" + fn, [0, 0]); a[0] += ie; a[1] += smp
ts = sum(a[1] for a in agg.values()); pairs = float(sys.argv[2])
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{32*a[0]/pairs:7.1f} inst/pair {100*a[1]/ts:5.1f}% smp  {k}")
