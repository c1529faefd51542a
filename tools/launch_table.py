"""Mean duration per kernel from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, collections, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, tot = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                tot[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
    print(f)
    for k, v in tot.items():
        print(f"  {k:60s} {len(v):3d} launches  mean {sum(v) / len(v) / 1e3:9.1f} us")
