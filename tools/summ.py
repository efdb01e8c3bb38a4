"""Summarise bench JSON lines (used while iterating)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e)
        continue
    bd = d.pop("breakdown_ms", {})
    print(f, d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["kernel"], d["roofline"]["achieved"],
          d["roofline"]["frac"], d["gemm_summary"])
    print(list(bd.items())[:18])
