"""Print a one-line summary of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "unavailable" in d:
        print(d)
        continue
    ph = {k: round(v, 3) for k, v in d.get("phases_ms", {}).items()}
    rf = d.get("roofline") or {}
    print(d["config"]["workload"].split(":")[0], f"{d['value']:.3e} mult/s", f"{d['ms_per_step']:.3f} ms",
          f"frac={rf.get('frac', 0):.3f}({rf.get('kernel')})", d["config"].get("partition", ""), ph)
