import json, sys
d = json.load(open(sys.argv[1]))
print(d["bench_grid_ms"])
for s, row in d["sets"].items():
    print(f"{s:8s}", "  ".join(f"{nm}: I {r['log_iv']['ms']:.3f} K {r['log_kv']['ms']:.3f}" + (f" IK {r['ivkv']['ms']:.3f}" if 'ivkv' in r else "") + f" d{max(r['log_iv']['maxdiff'], r['log_kv']['maxdiff'], r.get('ivkv', {}).get('maxdiff', 0)):.0e}" for nm, r in row.items()))
