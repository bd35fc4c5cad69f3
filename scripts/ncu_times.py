"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name, the
launch durations in microseconds."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    hdr = None
    d = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            if x["Metric Name"] == "gpu__time_duration.sum":
                scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(x["Metric Unit"], 1.0)
                d.setdefault(x["Kernel Name"][:70], []).append(float(x["Metric Value"].replace(",", "")) * scale)
    for k, v in d.items():
        print(f"{path}: {k:70s} n={len(v):4d} mean={sum(v)/len(v):10.1f} us  [{', '.join(f'{t:.1f}' for t in v[:6])}]")
