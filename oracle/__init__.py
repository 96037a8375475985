"""TEST INFRASTRUCTURE ONLY -- the CPU oracle of the ReLibra MoE-layer hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this package, and only as the checker (or the timed CPU reference arm); the product
path (paper_2605_08639_b200) never imports it and has no CPU fallback.

Contents:
  moe_ref.py     numpy/torch-fp32 restatement of the data plane: expert histogram
                 (RoutingTrace.matrices, routing.py:151-168), integer flow / executed loads
                 (costmodel.flow_matrix, costmodel.py:91-108 with replicate.round_split,
                 replicate.py:501-525), the canonical permutation, and the SwiGLU expert FFN
                 forward/backward with gate-weighted combine.
  gen_golden.py  regenerates tests/golden/planners.json (planner golden vectors and KATs) by
                 importing the reference package from /root/reference (this container only;
                 the fixtures travel, the reference does not).
  gen_golden_io.py  regenerates tests/golden/io/: trace directories and plan files written by the
                 reference's own `gen` / `solve`, and its acceptance study (criteria 6/7).

Parity pinning: the planners are pinned against golden vectors produced by the reference
itself (tests/golden/planners.json, tests/golden/io/) plus the reference's own KATs; the
oracle's executed flow is checked against the reference's flow_matrix semantics; the histogram
and the permutation are integer work checked bit-exactly; the layer math has no reference
implementation (the reference models it analytically), so its parity is against this fp32
restatement at the north_star tolerance rel 2e-2 ("parity unpinned" for the layer math in
the sense of the task statement: no reference numbers exist for it).
"""
