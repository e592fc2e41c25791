"""Summarise ab_libs.py / ab_env.sh lines '[tag] {bench json}' of the vector
workload: literal and dense step times (probe, not product)."""
import sys, json
for line in sys.stdin:
    if not line.startswith("["): continue
    tag, _, rest = line.partition("] ")
    try: d = json.loads(rest)
    except Exception: continue
    print(f"{tag}] literal {d['ms_per_step']*1e3:8.1f} us  dense {d['dense_index']['ms_per_step']*1e3:8.1f} us")
