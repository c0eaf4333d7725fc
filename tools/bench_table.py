"""Markdown table from bench.py JSON lines: python tools/bench_table.py f1.json f2.json ..."""
import json, sys
print("| config | DOF-updates/s | per time step | achieved (design bytes) | frac | frac @ 32 B/DOF | e2e | CPU arm |")
print("|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    line = None
    for l in open(f):
        l = l.strip()
        if l.startswith("{"):
            line = json.loads(l)
    if not line:
        continue
    r = line.get("roofline", {})
    cb = line.get("cpu_baseline", {})
    e2e = line.get("e2e", {}).get("value")
    print(f"| {line['config']['workload'].split(':')[0]} | {line['value']:.3e} | {r.get('launch_us', 0):.1f} us | "
          f"{r.get('achieved', 0):.0f} GB/s | {r.get('frac', 0):.2f} | {r.get('frac_at_nominal_bytes', float('nan')):.2f} | "
          f"{(e2e or 0):.3e} | {cb.get('value', 0):.3e} ({cb.get('kind', '')}, {cb.get('cores', '')} thr) |")
