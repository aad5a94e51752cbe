"""Print the key fields of the last bench.py JSON line in a log file."""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
c = d.get("config", {})
print(f"value {d.get('value'):.1f} k3_ms {c.get('k3_ms')} frac {d.get('roofline', {}).get('frac')} "
      f"e2e {d.get('e2e', {}).get('value')} ms/step {d.get('ms_per_step')}")
