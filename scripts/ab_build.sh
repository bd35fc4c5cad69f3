#!/bin/bash
# A/B over compile-time variants: for each "flags" argument, rebuild libwlr.so with
# WLR_NVCC_EXTRA=flags and run a short bench (config 3), printing value and kernel times.
# usage: scripts/ab_build.sh "" "-DWLR_IT_NR=4" ...
for fl in "$@"; do
  WLR_NVCC_EXTRA="$fl" python paper_1703_06303_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $fl"; continue; }
  python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
l=json.loads([x for x in sys.stdin if x.startswith('{')][-1])
print('[$fl]', round(l['value'],1), {k:round(v*1e3,2) for k,v in l['roofline']['kernel_ms'].items()})"
done
python paper_1703_06303_b200/build.py --force > /dev/null 2>&1
