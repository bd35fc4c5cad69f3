#!/bin/bash
# A/B of row-solver builds on one box: usage scripts/ab_rowsolve.sh TAG "v1 v2 ..." (libwlr_<v>.so in the package)
O=gpurun_out/$1; mkdir -p $O
L=paper_1703_06303_b200
sum() { python -c "
import json,sys
l=json.loads([x for x in open('$1') if x.startswith('{')][-1])
print('$2', round(l['value'],2), {k:round(v*1e3,3) for k,v in l['roofline']['kernel_ms'].items()})"; }
cp $L/libwlr.so /tmp/libwlr_keep.so
for rep in 1 2; do
 for v in $2; do
  cp $L/libwlr_$v.so $L/libwlr.so
  for c in 5 4; do
   s=20; [ $c = 4 ] && s=100
   timeout 300 python bench.py --config $c --steps $s --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${v}_c${c}_$rep.log 2>&1
   sum $O/b_${v}_c${c}_$rep.log "[$v cfg$c]" >> $O/summary.txt 2>&1
  done
 done
done
cp /tmp/libwlr_keep.so $L/libwlr.so
cat $O/summary.txt
