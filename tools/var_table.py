"""Compact table of a variant_bench.py result (fused ms per set, bench-grid sum)."""
import json
import sys

d = json.load(open(sys.argv[1]))
names = list(d["bench_grid_ms"])
print("set".ljust(8) + "".join(n.rjust(9) for n in names))
for k, v in d["sets"].items():
    print(k.ljust(8) + "".join(f"{v[n].get('ivkv', {}).get('ms', float('nan')):9.4f}" for n in names))
print("grid".ljust(8) + "".join(f"{d['bench_grid_ms'][n].get('ivkv', float('nan')):9.3f}" for n in names))
print("grid_iv".ljust(8) + "".join(f"{d['bench_grid_ms'][n]['log_iv']:9.3f}" for n in names))
print("grid_kv".ljust(8) + "".join(f"{d['bench_grid_ms'][n]['log_kv']:9.3f}" for n in names))
print("grid_f32".ljust(8) + "".join(f"{d['bench_grid_ms'][n].get('ivkv32', float('nan')):9.3f}" for n in names))
md = max(v[n].get("ivkv", {}).get("maxdiff", 0) for v in d["sets"].values() for n in names)
print("max output diff vs first variant:", md)
