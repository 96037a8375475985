"""bench.py contract pieces that run without a GPU: the CPU reference arm's JSON line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    ref_built = os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "moebalance"))
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_built else "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["layer_port_tokens_per_s"] > 0
    assert d["config"]["workload"].startswith("qwen3-30b-a3b MoE layer fwd+bwd")


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=2" in (out.stderr + out.stdout)


def test_relabel_for_overlap_keeps_most_experts():
    """The group-wise GPU relabeling used at batch boundaries: a plan that is the old one with its
    GPUs permuted (inside and across groups) relabels back to it exactly; any relabeling keeps
    group membership (replicas stay inside a group)."""
    import numpy as np
    from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile
    from paper_2605_08639_b200.moe_layer import relabel_for_overlap
    topo = b200_box_topology(8, 4, b200_profile(2048))
    rng = np.random.default_rng(1)
    old = rng.permutation(np.repeat(np.arange(8), 16))
    perm = np.array([5, 7, 4, 6, 1, 0, 3, 2])       # swaps the two groups and shuffles inside each
    new = perm[old]
    assert np.array_equal(relabel_for_overlap(new, old, topo), old)
    other = rng.permutation(np.repeat(np.arange(8), 16))
    rel = relabel_for_overlap(other, old, topo)
    # a bijection on GPUs that maps groups onto groups, never worse than the identity
    assert sorted(np.bincount(rel, minlength=8)) == [16] * 8
    same_group = [(rel[other == g] // 4 == rel[other == g][0] // 4).all() for g in range(8)]
    assert all(same_group)
    assert (rel == old).sum() >= (other == old).sum()
