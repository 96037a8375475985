"""Step schedule of the data plane (moe_layer.schedule): every phase of every micro-batch issued
once, and the two in-order streams linked by their events cannot deadlock."""

import pytest

from paper_2605_08639_b200.moe_layer import schedule


def _needs(mode):
    """(comm needs, compute needs): op -> (op it waits for, micro-batch offset), as
    MoEDataPlane.forward_backward links the two streams."""
    if mode == "micro_batch":
        return {"C": ("F", 0), "X": ("W", 0)}, {"F": ("D", 0), "B": ("C", 0), "W": ("X", -1)}
    return {"C": ("F", 0), "X": ("B", 0)}, {"F": ("D", 0), "B": ("C", 0)}


def _simulate(comm, comp, mode="step"):
    """Run both in-order queues to completion; an op starts once its dependency finished."""
    comm_needs, comp_needs = _needs(mode)
    done, ci, pi, order = set(), 0, 0, []

    def ready(needs, op, m):
        if op not in needs:
            return True
        dop, off = needs[op]
        return m + off < 0 or (dop, m + off) in done

    while ci < len(comm) or pi < len(comp):
        progressed = False
        if ci < len(comm):
            op, m = comm[ci]
            if ready(comm_needs, op, m):
                done.add((op, m)); order.append((op, m)); ci += 1; progressed = True
        if pi < len(comp):
            op, m = comp[pi]
            if ready(comp_needs, op, m):
                done.add((op, m)); order.append((op, m)); pi += 1; progressed = True
        if not progressed:
            raise AssertionError(f"deadlock at comm {comm[ci:ci+1]} compute {comp[pi:pi+1]}")
    return order


@pytest.mark.parametrize("mb", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("mode", ["step", "micro_batch"])
def test_schedule_complete_and_deadlock_free(mb, mode):
    comm, comp = schedule(mb, mode)
    assert sorted(comm) == sorted((p, m) for m in range(mb) for p in "DCX")
    ops = "FB" if mode == "step" else "FBW"
    assert sorted(comp) == sorted((p, m) for m in range(mb) for p in ops)
    order = _simulate(comm, comp, mode)
    pos = {o: i for i, o in enumerate(order)}
    for m in range(mb):
        assert pos[("D", m)] < pos[("F", m)] < pos[("C", m)] < pos[("B", m)] < pos[("X", m)]
        if mode == "micro_batch":
            # per expert gradient: W(m) then X(m) (push-back) then W(m + 1): never concurrent
            assert pos[("B", m)] < pos[("W", m)] < pos[("X", m)]
            if m + 1 < mb:
                assert pos[("X", m)] < pos[("W", m + 1)]


@pytest.mark.parametrize("mb", [3, 4, 8, 16])
def test_ring_sets_reuse_after_all_ranks_finished(mb):
    """wgrad_mode micro_batch keeps RING_SETS buffer sets: on every rank's comm stream, D(m + 3)
    (the first writer of micro-batch m's set) comes after X(m) (whose barrier means every rank
    finished B(m) / W(m)), and C(m + 2) -- the barrier before B(m + 2) overwrites replica-gradient
    ring set m % 2 -- comes after X(m)'s push-back reads it."""
    from paper_2605_08639_b200.moe_layer import GRAD_RING, RING_SETS
    comm, _ = schedule(mb, "micro_batch")
    pos = {o: i for i, o in enumerate(comm)}
    for m in range(mb):
        if m + RING_SETS < mb:
            assert pos[("X", m)] < pos[("D", m + RING_SETS)]
        if m + GRAD_RING < mb:
            assert pos[("X", m)] < pos[("C", m + GRAD_RING)]


@pytest.mark.parametrize("mb", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("early", [True, False])
def test_replica_ring_guards(mb, early):
    """Step mode: B(m) overwrites replica-gradient ring set m % 2, which the owners read in
    X(m - 2).  Either C(m) (whose barrier B(m) waits for) follows X(m - 2) on the comm stream, or
    B(m) carries a guard on the start barrier of a later un-permute, which every rank reaches only
    after its X(m - 2); with the guard as an extra dependency the two streams still cannot deadlock."""
    from paper_2605_08639_b200.moe_layer import GRAD_RING, replica_ring_guards
    comm, comp = schedule(mb, "step", early_last=early)
    guards = replica_ring_guards(comm, mb)
    pos = {o: i for i, o in enumerate(comm)}
    for m in range(GRAD_RING, mb):
        if m in guards:
            assert pos[("X", m - GRAD_RING)] < pos[("X", guards[m])] and pos[("C", m)] < pos[("X", m - GRAD_RING)]
        else:
            assert pos[("X", m - GRAD_RING)] < pos[("C", m)]
    if early and mb >= 3:   # the last combine is ahead of the third-to-last un-permute
        assert pos[("C", mb - 1)] < pos[("X", mb - 3)] and guards == {mb - 1: mb - 2}
    else:
        assert guards == {}
    # B(m) also waits for X(guards[m]): simulate with that dependency added
    done, ci, pi = set(), 0, 0
    while ci < len(comm) or pi < len(comp):
        progressed = False
        if ci < len(comm):
            op, m = comm[ci]
            need = {"C": ("F", m), "X": ("B", m)}.get(op)
            if need is None or need in done:
                done.add((op, m)); ci += 1; progressed = True
        if pi < len(comp):
            op, m = comp[pi]
            needs = [("D", m)] if op == "F" else [("C", m)] + ([("X", guards[m])] if m in guards else [])
            if all(n in done for n in needs):
                done.add((op, m)); pi += 1; progressed = True
        assert progressed, f"deadlock at comm {comm[ci:ci + 1]} compute {comp[pi:pi + 1]}"


def test_at_most_two_micro_batches_ahead():
    # the dispatch of micro-batch m is queued behind the combine of m-2: a rank can never start
    # the GEMMs of a micro-batch while two earlier ones have not been combined everywhere
    comm, _ = schedule(8)
    pos = {o: i for i, o in enumerate(comm)}
    for m in range(2, 8):
        assert pos[("C", m - 2)] < pos[("D", m)]


def test_migration_moves_cover_every_expert_once():
    import numpy as np
    from paper_2605_08639_b200.moe_layer import migration_moves
    rng = np.random.default_rng(0)
    world, E = 4, 32
    old = np.repeat(np.arange(world), E // world)
    new = rng.permutation(old)
    moves = migration_moves(old, new, world)
    seen = []
    for d, mv in enumerate(moves):
        assert [s for s, _, _ in mv] == list(range(E // world))
        for s, src, ss in mv:
            e = int(np.flatnonzero(new == d)[s])
            assert old[e] == src and int(np.flatnonzero(old == src)[ss]) == e
            seen.append(e)
    assert sorted(seen) == list(range(E))


@pytest.mark.parametrize("T,parts", [(8192, 1), (8192, 2), (7, 2), (5, 3), (1, 2), (0, 2)])
def test_token_parts_cover_every_token_once(T, parts):
    from paper_2605_08639_b200.moe_layer import _token_parts
    ranges = _token_parts(T, parts)
    covered = [t for a, b in ranges for t in range(a, b)]
    assert covered == list(range(T))
    assert all(b > a for a, b in ranges) and len(ranges) <= parts


def test_comm_sm_defaults(monkeypatch):
    """Row movers: none reserved at N=1 (register engine between GEMM launches), 28 at N=2/4, 32 at N>=8 and for the 4096-wide
    rows of Qwen3-235B (measured with 32), 8 for wide-FFN experts."""
    from paper_2605_08639_b200 import moe_layer as ml
    from paper_2605_08639_b200.workload import SHAPES
    monkeypatch.delenv("MB_COMM_SMS", raising=False)
    assert ml.default_comm_sms(1, SHAPES["qwen3-30b-a3b"]["shape"]) == 0
    assert ml.default_comm_sms(8, SHAPES["qwen3-30b-a3b"]["shape"]) == 32
    assert ml.default_comm_sms(4, SHAPES["qwen3-30b-a3b"]["shape"]) == 28
    assert ml.default_comm_sms(4, SHAPES["qwen3-235b-a22b"]["shape"]) == 32
    assert ml.default_comm_sms(4, SHAPES["mixtral-8x7b"]["shape"]) == 8
    assert ml.ROW_MOVERS[1] == "regs" and ml.ROW_MOVERS_MULTI == "tma"


def test_replica_set_defaults(monkeypatch):
    """One layer-shared replica set (exactly replica_memory "layer-shared") unless an expert is big
    enough that pulling it again for the backward costs more than a second set (Mixtral-8x7B)."""
    from paper_2605_08639_b200 import moe_layer as ml
    from paper_2605_08639_b200.workload import SHAPES
    monkeypatch.delenv("MB_REPLICA_SETS", raising=False)
    assert ml.default_replica_sets(SHAPES["qwen3-30b-a3b"]["shape"]) == 1
    assert ml.default_replica_sets(SHAPES["qwen3-235b-a22b"]["shape"]) == 1
    assert ml.default_replica_sets(SHAPES["mixtral-8x7b"]["shape"]) == 2
