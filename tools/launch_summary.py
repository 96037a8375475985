"""Per-kernel share of GPU time and DRAM bytes from an ncu launch list
(--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv)."""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    hdr, recs = None, collections.defaultdict(dict)
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        recs[(int(d["ID"]), d["Kernel Name"])][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in recs.items():
        if "grouped_gemm_pair_kernel" in name or "grouped_gemm_single_kernel" in name:
            fam = "pair" if "pair_kernel" in name else "cta1"
            key = f"K4 grouped_gemm_{fam} " + name[name.index("<"):name.index(">") + 1]
        else:
            key = name.split("(")[0].replace("void ", "").split("<")[0]
        a = agg[key]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    return agg


def main(path, json_out=None):
    agg = load(path)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':50s} {'launches':>8s} {'avg us':>9s} {'share':>7s} {'MB read':>9s} {'MB write':>9s} {'GB/s':>7s}")
    rows = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        n, t, rd, wr = a
        gbs = (rd + wr) / t / 1e9 if t else 0.0
        print(f"{k:50s} {n:8d} {t / n * 1e6:9.1f} {t / tot:7.1%} {rd / n / 1e6:9.1f} {wr / n / 1e6:9.1f} {gbs:7.0f}")
        rows[k] = {"launches": n, "avg_us": t / n * 1e6, "share": t / tot, "dram_read_per_launch": rd / n,
                   "dram_write_per_launch": wr / n}
    k4 = {k: r for k, r in rows.items() if k.startswith("K4")}
    totals = {"k4_dram_bytes": sum((r["dram_read_per_launch"] + r["dram_write_per_launch"]) * r["launches"]
                                   for r in k4.values()),
              "k4_launches": sum(r["launches"] for r in k4.values()),
              "k4_share": sum(r["share"] for r in k4.values()), "kernels": sum(a[0] for a in agg.values())}
    print(json.dumps(totals))
    if json_out:
        json.dump({"per_kernel": rows, "totals": totals}, open(json_out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
