"""Summarise ab_env.sh output lines '[tag] {json}' -> tag, ms_per_step (us), value."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("["):
        continue
    tag, _, rest = line.partition("] ")
    try:
        d = json.loads(rest)
    except ValueError:
        print(line.strip()[:200])
        continue
    print(f"{tag}] {d.get('config', {}).get('workload', '')[:50]:50s} {d['ms_per_step'] * 1e3:9.1f} us  {d['value']:9.1f}")
