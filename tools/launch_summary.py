"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys


def summarise(path):
    hdr, agg = None, collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        if "grouped_gemm_pair_kernel" in name:
            name = "K4 grouped_gemm_pair " + name[name.index("<"):name.index(">") + 1]
        else:
            name = name.split("(")[0].replace("void ", "").split("<")[0]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        agg[name].append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -sum(kv[1]))
    print(f"{'kernel':60s} {'launches':>8s} {'avg us':>10s} {'share':>7s}")
    for k, v in rows:
        print(f"{k:60s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v) / tot:7.1%}")


if __name__ == "__main__":
    summarise(sys.argv[1])
