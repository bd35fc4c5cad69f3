"""Aggregate an ncu '--page source --print-source cuda,sass --csv' dump by CUDA source line:
top lines by warp-stall samples with their dominant stall reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None; agg = []
reasons = ['stall_barrier', 'stall_long_sb', 'stall_no_inst', 'stall_wait', 'stall_short_sb', 'stall_selected',
           'stall_math', 'stall_branch_resolving', 'stall_lg', 'stall_membar', 'stall_not_selected', 'stall_dispatch']
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] == '' or r[2] != '-':
        continue
    d = dict(zip(hdr, r))
    try:
        smp = float(r[4])
    except ValueError:
        continue
    if smp > 0:
        rs = sorted(((float(d.get(k, 0) or 0), k[6:]) for k in reasons), reverse=True)[:3]
        agg.append((smp, fname, int(r[0]), r[1].strip()[:80], d.get('Instructions Executed'), rs))
agg.sort(reverse=True)
tot = sum(a[0] for a in agg)
print("total samples", tot)
for a in agg[:top]:
    print(f"{int(a[0]):5d} {a[1]}:{a[2]:<5d} inst={a[4]:>8s} " + ",".join(f"{k}={int(v)}" for v, k in a[5] if v) + f"  | {a[3]}")
