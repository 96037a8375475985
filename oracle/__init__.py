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
  planners_np.py numpy restatement of the reference planners (reorder.py, replicate.py,
                 lp.py, sim.py) used as the CPU reference arm of bench.py.
  gen_golden.py  regenerates tests/golden/ by importing the reference package from
                 /root/reference (this container only; the fixtures travel, the reference
                 does not).

Parity pinning: the planners are pinned against golden vectors produced by the reference
itself (tests/golden/planners_*.npz) plus the reference's own KATs; the histogram and the
permutation are integer work checked bit-exactly; the layer math has no reference
implementation (the reference models it analytically), so its parity is against this fp32
restatement at the north_star tolerance rel 2e-2 ("parity unpinned" for the layer math in
the sense of the task statement: no reference numbers exist for it).
"""
