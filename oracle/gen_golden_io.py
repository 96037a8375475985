"""Generate wire-format golden files with the REFERENCE package (test infrastructure only).

Writes tests/golden/io/: a small routing trace directory produced by the reference's own
`generate_synthetic_trace` + `save_trace` (routing.py:240-256, 385-440), and the plan files its
`solve` command writes (cli.py:124-185 -> planio.py:25-52, replicate.py:539-560), plus
meta.json with the trace_id.  tests/test_io_golden.py checks that this package reads them back
identically, re-writes them byte for byte, and that its own planners produce byte-identical plan
files from the same trace.

Run in the build container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_io.py
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
}


def main():
    sys.path.insert(0, REF)
    from moebalance import cli  # noqa: E402
    from moebalance import routing as rt  # noqa: E402

    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
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
        trace = rt.load_trace(tdir)
        meta[name] = {"trace_id": trace.trace_id(), "seeds": seeds, "replica_slots": slots,
                      "shape": list(trace.matrices.shape)}
    (OUT / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
