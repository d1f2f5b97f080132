"""Prints one summary line of a bench JSON log (used by tools/gpu_sweep.sh)."""
import json
import sys

tag, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    cls = {k: v for k, v in d["roofline"]["class_ms_per_step"].items() if v > 0.5}
    print(f"[{tag}] {d['ms_per_step']} ms {d['value']} GF {cls}")
except Exception:
    print(f"[{tag}] failed: {open(path).read()[-800:]}")
