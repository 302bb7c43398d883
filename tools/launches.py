"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per kernel count,
total and mean device time (optionally only the last `--last` launches)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
            data.append((d["Kernel Name"], v))
    return data


if __name__ == "__main__":
    data = load(sys.argv[1])
    if len(sys.argv) > 2:
        data = data[-int(sys.argv[2]):]
    agg = collections.OrderedDict()
    for k, v in data:
        agg.setdefault(k.split("(")[0][:70], []).append(v)
    tot = sum(v for _, v in data)
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} {sum(v):11.1f} us {100*sum(v)/tot:5.1f}%  avg {sum(v)/len(v):9.1f}  {k}")
    print(f"total {tot:.1f} us over {len(data)} launches")
