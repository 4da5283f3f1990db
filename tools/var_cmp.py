"""Compact table of a tools/variant_bench.py JSON (diagnostic)."""
import json
import sys

d = json.load(open(sys.argv[1]))
names = list(d["bench_grid_ms"])
print("grid ms", {n: d["bench_grid_ms"][n] for n in names})
for s, r in d["sets"].items():
    print(f"{s:7s}", " ".join(f"{n}:{r[n]['ivkv']['ms']:.4f}/{r[n]['log_iv']['ms']:.4f}/{r[n]['log_kv']['ms']:.4f}/{r[n].get('ivkv32', {}).get('ms', 0):.4f}" for n in names),
          " maxdiff", " ".join(f"{max(r[n][f]['maxdiff'] for f in ('ivkv', 'log_iv', 'log_kv')):.1e}" for n in names[1:]))
