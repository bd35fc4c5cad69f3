#!/bin/bash
# A/B on one box: bench + cold timeline for the default and an env variant.  Usage:
#   scripts/gpu_ab.sh "WLR_X=1" [tag]
V="$1"; T="${2:-ab}"
for rep in 1 2; do
  python bench.py --steps 200 --warmup 5 > gpurun_out/${T}_base_$rep.log 2>&1
  env $V python bench.py --steps 200 --warmup 5 > gpurun_out/${T}_var_$rep.log 2>&1
done
python scripts/diag_timeline.py 3 > gpurun_out/${T}_tl_base.log 2>&1
env $V python scripts/diag_timeline.py 3 > gpurun_out/${T}_tl_var.log 2>&1
for f in gpurun_out/${T}_base_*.log gpurun_out/${T}_var_*.log; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']))"
done
