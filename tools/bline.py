"""Print the headline fields of a bench.py JSON line (value, ms/step, breakdown, sub-records)."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print(f"value {d.get('value', 0) / 1e6:.1f} M {d.get('unit')}  ms/step {d.get('ms_per_step', 0):.3f}  "
          f"e2e {(d.get('e2e') or {}).get('value', 0) / 1e6:.1f} M  roofline {(d.get('roofline') or {}).get('frac')}")
    if "latency_ms" in d:
        print("latency", d["latency_ms"], "warm", d.get("warm_start", {}).get("latency_ms"))
    for k, v in d.get("breakdown", {}).items():
        print(f"  {k:16s} {v['ms_per_step']:8.3f} ms  x{v['launches_per_step']}")
    for k, v in (d.get("sub") or {}).items():
        print(f"sub {k}: value {v.get('value', 0) / 1e6:.2f} M ms/step {v.get('ms_per_step')}",
              "latency", v.get("latency_ms"), "warm", v.get("warm_start", {}).get("latency_ms"))
