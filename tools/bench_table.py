"""One row per bench JSON line: throughput, balance ratios, skews, roofline and comm figures."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable", e)
        continue
    if d.get("impl") == "reference":
        print(f"{path}: reference arm {d['value']:.0f} {d['unit']} ({d['cpu_baseline']['sample']})")
        continue
    b = d["balance"]
    c = d["config"]
    pol = {k: (round(v["ms_per_step"], 2), round(v["skew"], 3)) for k, v in b.items() if isinstance(v, dict)}
    comm = {k: v["gb_per_s"] for k, v in d.get("comm", {}).items()}
    print(f"{path}: N={d['n_gpus']} {c['workload'].split(' ')[0]} z={c.get('zipf_s', '-')} group={c['gpu_group']} "
          f"{d['value'] / 1e6:.2f}M tok/s {d['ms_per_step']:.2f} ms e2e {d['e2e']['value'] / 1e6:.2f}M "
          f"frac={d['roofline']['frac']} x_static={b.get('speedup_vs_static', 0):.3f} "
          f"of_balanced={b.get('frac_of_balanced', 0):.3f} clk={d['clocks']['sm_mhz']}")
    print(f"    policies (ms, skew): {pol}")
    print(f"    comm GB/s: {comm}")
