"""Generate wire-format golden files with the REFERENCE package (test infrastructure only).

Writes tests/golden/io/: a small routing trace directory produced by the reference's own
`generate_synthetic_trace` + `save_trace` (routing.py:240-256, 385-440), and the plan files its
`solve` command writes (cli.py:124-185 -> planio.py:25-52, replicate.py:539-560), plus
meta.json with the trace_id.  tests/test_io_golden.py checks that this package reads them back
identically, re-writes them byte for byte, and that its own planners produce byte-identical plan
files from the same trace.

Run in the build container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_io.py
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_io.py --acceptance   (criteria 6/7 study, ~5 min)
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_io.py --qwen3        (production-shape trace + plans)
"""

import json
import shutil
import sys
from pathlib import Path

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "io"

CASES = {
    # name: (nodes, gpus_per_node, experts, layers, micro_batches, top_k, tokens, domains, alpha, focus,
    #        samples_per_gpu, seed, solve seeds, replica slots)
    "small": (2, 2, 16, 2, 3, 2, 256, 3, 0.5, 0.0, 0, 5, 4, 2),
    "samples": (2, 2, 8, 1, 2, 2, 64, 2, 0.3, 0.4, 4, 11, 2, 1),
    "samples2": (2, 2, 16, 2, 3, 2, 128, 3, 0.5, 0.3, 6, 21, 3, 2),
}


def main():
    sys.path.insert(0, REF)
    from moebalance import cli  # noqa: E402
    from moebalance import routing as rt  # noqa: E402

    OUT.mkdir(parents=True, exist_ok=True)
    for name in CASES:  # the acceptance/ study is regenerated separately (--acceptance)
        if (OUT / name).exists():
            shutil.rmtree(OUT / name)
    meta = {}
    for name, (nodes, gpn, e, layers, mb, k, tok, dom, alpha, focus, spg, seed, seeds, slots) in CASES.items():
        tdir, pdir = OUT / name / "trace", OUT / name / "plans"
        rc = cli.main(["gen", "--out", str(tdir), "--nodes", str(nodes), "--gpus-per-node", str(gpn),
                       "--experts", str(e), "--layers", str(layers), "--micro-batches", str(mb), "--top-k", str(k),
                       "--tokens-per-gpu", str(tok), "--domains", str(dom), "--alpha", str(alpha),
                       "--focus", str(focus), "--samples-per-gpu", str(spg), "--seed", str(seed)])
        assert rc == 0
        rc = cli.main(["solve", "--trace", str(tdir), "--out", str(pdir), "--seeds", str(seeds),
                       "--replica-slots", str(slots), "--threads", "1"])
        assert rc == 0
        if spg > 0:  # data-locality sample placement (reorder.py:365-568) as well
            rc = cli.main(["solve", "--trace", str(tdir), "--out", str(OUT / name / "plans_sl"), "--seeds",
                           str(seeds), "--replica-slots", str(slots), "--threads", "1", "--sample-locality"])
            assert rc == 0
        trace = rt.load_trace(tdir)
        meta[name] = {"trace_id": trace.trace_id(), "seeds": seeds, "replica_slots": slots,
                      "shape": list(trace.matrices.shape)}
    (OUT / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__" and "--acceptance" not in sys.argv and "--qwen3" not in sys.argv:
    main()


def acceptance_study():
    """Criteria 6/7 of the reference's acceptance suite (test_acceptance.py:289-368) at EP 8..64:
    the reference generates the traces and runs run_baseline for every policy; the traces and the
    exact per-policy results (total time as float.hex, per-micro-batch skew) are written to
    tests/golden/io/acceptance/ so tests/test_acceptance_golden.py can replay them with this
    package's planners."""
    sys.path.insert(0, REF)
    import numpy as np
    from moebalance import replicate as rep
    from moebalance import reorder as ro
    from moebalance import routing as rt
    from moebalance import sim
    from moebalance.topology import HardwareProfile, build_topology

    out = OUT / "acceptance"
    out.mkdir(parents=True, exist_ok=True)
    cfgs = sim.SimConfigs(anneal=ro.AnnealConfig(seeds=tuple(range(8)), cooling_rate=0.9995),
                          replica=rep.ReplicaConfig(1), threads=2)
    results = {}
    for ep in (8, 16, 32, 64):
        hw = HardwareProfile(2.577e10, 4.5e5, 2.5e4, 1.0)
        topo = build_topology(max(ep // 8, 1), min(ep, 8), hw)
        model = rt.ModelProfile(num_layers=1, num_experts=128, top_k=8)
        spec = rt.TraceGenSpec(num_domains=3, dirichlet_alpha=4096.0, tokens_per_gpu=1024, rng_seed=11,
                               domain_focus=0.82, redraw_concentration=64.0)
        trace = rt.generate_synthetic_trace(spec, model, topo, 32)
        rt.save_trace(trace, out / f"ep{ep}")
        policies = ("static", "relibra") + (("lpt_only", "eplb_like", "lplb_like", "balanced_oracle")
                                             if ep == 32 else ())
        res = {}
        for pol in policies:
            r = sim.run_baseline(trace, pol, topo, model, hw, cfgs)
            res[pol] = {"total_time": float(r.total_time).hex(), "skew": [float(v).hex() for v in r.skew.ravel()]}
        results[f"ep{ep}"] = res
        print(f"acceptance ep{ep} done", flush=True)
    (out / "results.json").write_text(json.dumps(results, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__" and "--acceptance" in sys.argv:
    acceptance_study()


QWEN3_CASES = {  # name: (nodes, gpus per node) -- EP=4 one group; EP=8 two groups of 4 (north-star config)
    "qwen3_ep4": (1, 4),
    "qwen3_ep8": (2, 4),
}


def qwen3():
    """A Qwen3-30B-A3B-shaped trace (E=128, k=8, h=2048, h'=768; one group of 4 GPUs, 8
    micro-batches of 8192 tokens per GPU, domain-focused skew) written by the reference's `gen`
    with B200-like cost-model units, and the plan files its `solve` writes for it.  The GPU bench
    replays both through the kernels (bench.py --trace ... --plans ...)."""
    sys.path.insert(0, REF)
    from moebalance import cli  # noqa: E402
    for name, (nodes, gpn) in QWEN3_CASES.items():
        out = OUT / name
        if out.exists():
            shutil.rmtree(out)
        rc = cli.main(["gen", "--out", str(out / "trace"), "--nodes", str(nodes), "--gpus-per-node", str(gpn),
                       "--experts", "128", "--layers", "1", "--micro-batches", "8", "--top-k", "8",
                       "--tokens-per-gpu", "8192", "--domains", "4", "--alpha", "0.3", "--focus", "0.5", "--seed", "7",
                       "--hidden", "2048", "--intermediate", "768", "--flops", "1.0e15", "--bw-nvlink", "6.5e11",
                       "--bw-rdma", "6.5e11", "--bytes-per-token", "4096"])
        assert rc == 0
        rc = cli.main(["solve", "--trace", str(out / "trace"), "--out", str(out / "plans"), "--seeds", "8",
                       "--replica-slots", "2", "--threads", "8"])
        assert rc == 0
        print(f"wrote {out}")


if __name__ == "__main__" and "--qwen3" in sys.argv:
    qwen3()
