#!/bin/bash
# Same-box A/B over environment settings: each argument is an env assignment list (e.g. "WLR_ITC_CPS=1").
for envs in "$@"; do
  env $envs python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
l=json.loads([x for x in sys.stdin if x.startswith('{')][-1])
print('[$envs]', round(l['value'],1), {k:round(v*1e3,2) for k,v in l['roofline']['kernel_ms'].items()})"
done
