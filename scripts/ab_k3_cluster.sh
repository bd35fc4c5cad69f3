for cl in 16 12 10 8 16; do WLR_K3_CL=$cl python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
l=json.loads([x for x in sys.stdin if x.startswith('{')][-1])
print('CL', $cl, round(l['value'],1), {k:round(v*1e3,2) for k,v in l['roofline']['kernel_ms'].items()})"; done
