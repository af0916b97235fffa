"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


if __name__ == "__main__":
    data = load(sys.argv[1])
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        k = d["Kernel Name"].split("(")[0][:48] + " grid=" + d["Grid Size"].split(",")[0].strip("( ")
        t = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
        tot[k] += t
        cnt[k] += 1
    print(f"{len(data)} launches, {sum(tot.values()):.1f} us")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.1f} us {cnt[k]:4d}  avg {v / cnt[k]:7.2f}  {k}")
