"""Plan compiler parity (proj/tests/test_plan.cpp) through the C ABI, CPU only.
The per-device timestep/step-assignment schedule is a bit-exact contract:
every plan is compared integer-for-integer with the oracle's restatement."""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O


def uniform_partition(N, cost=100):  # test_plan.cpp:14-22
    return adx.Partition.create([[n + 1] for n in range(N)], list(range(N)), [cost] * N)


def test_plan_bit_exact_vs_oracle_many_tuples():
    rng = O.Rng(31)
    for _ in range(300):
        T = 1 + rng.below(200)
        w = 1 + rng.below(T)
        S = 1 + rng.below(2)
        N = (2 if S == 2 else 1) + rng.below(6)
        shift = bool(rng.below(2))
        ours = adx.plan_async(T, w, N, S, shift).to_flat()
        ref = O.plan_async_flat(T, w, N, S, shift)
        assert np.array_equal(ours, ref), (T, w, N, S, shift)


def test_t50_w1_n2_s1():  # test_plan.cpp:26-34
    plan = adx.plan_async(50, 1, 2, 1)
    assert len(plan.rounds) == 49
    assert adx.validate_plan(plan) == []
    c = adx.plan_counts(plan, uniform_partition(2))
    assert c.broadcasts_paper_convention == 49
    assert c.broadcasts_strictly_needed == 48
    assert c.device_count == 2


def test_t50_w1_n3_s2():  # test_plan.cpp:36-47
    plan = adx.plan_async(50, 1, 3, 2)
    assert adx.validate_plan(plan) == []
    c = adx.plan_counts(plan, uniform_partition(3))
    assert c.broadcasts_paper_convention == 25
    assert c.device_count == 4 and plan.D == 4
    assert len(plan.rounds) == 25
    assert len(plan.rounds[-1].sampler_steps) == 1
    assert len(plan.rounds[0].sampler_steps) == 2


def test_w_equals_T_is_pure_warmup():  # test_plan.cpp:49-58
    plan = adx.plan_async(50, 50, 4, 1)
    assert plan.rounds == [] and len(plan.warmup_steps) == 50
    assert adx.validate_plan(plan) == []
    c = adx.plan_counts(plan, uniform_partition(4))
    assert c.broadcasts_paper_convention == 0
    assert all(v == 50 * 100 for v in c.per_device_macs)


@pytest.mark.parametrize("args", [(50, 0, 2, 1), (50, 51, 2, 1), (50, 1, 1, 2), (50, 1, 0, 1), (50, 1, 2, 3)])
def test_infeasible_tuples(args):  # test_plan.cpp:60-66
    with pytest.raises(adx.InvalidArgument):
        adx.plan_async(*args)


def test_broadcast_count_formulas():  # test_plan.cpp:68-84
    rng = O.Rng(31)
    for _ in range(120):
        T = 2 + rng.below(199)
        w = 1 + rng.below(T)
        S = 1 + rng.below(2)
        N = (2 if S == 2 else 1) + rng.below(3)
        plan = adx.plan_async(T, w, N, S)
        assert adx.validate_plan(plan) == []
        rounds = len(plan.rounds)
        assert rounds == (T - w if S == 1 else (T - w + 1) // 2)
        assert plan.D == N + S - 1


@pytest.mark.parametrize("T,w,N,S", [(50, 1, 3, 2), (50, 3, 4, 1), (17, 5, 2, 2), (9, 9, 2, 1), (8, 2, 3, 2)])
def test_every_timestep_once_in_order(T, w, N, S):  # test_plan.cpp:86-105
    plan = adx.plan_async(T, w, N, S)
    order = list(plan.warmup_steps)
    for r in plan.rounds:
        emitted = set()
        for e in r.evals:
            assert (e.emits_eps_for is not None) == (e.segment == N)
            if e.emits_eps_for is not None:
                emitted.add(e.emits_eps_for)
        for st in r.sampler_steps:
            assert st in emitted
            order.append(st)
    assert order == list(range(T, 0, -1))


@pytest.mark.parametrize("T,w,N,S", [(40, 2, 4, 1), (40, 2, 4, 2), (12, 1, 2, 2)])
def test_staleness_exactly_one_round(T, w, N, S):  # test_plan.cpp:107-121
    plan = adx.plan_async(T, w, N, S)
    for r in plan.rounds:
        for e in r.evals:
            if e.input.kind == "cached":
                assert e.input.producer_segment == e.segment - 1
                assert e.input.producer_round == (adx.kWarmupRound if r.index == 0 else r.index - 1)


def test_stride_round_structure():  # test_plan.cpp:123-151
    plan = adx.plan_async(20, 2, 3, 2)
    r0 = plan.rounds[0]
    assert r0.sampler_steps == [18, 17]
    lead = [e for e in r0.evals if e.embed_t == 18]
    tail = [e for e in r0.evals if e.embed_t == 17]
    assert len(lead) == 1 and lead[0].segment == 3
    assert len(tail) == 3
    assert {e.device for e in r0.evals} == {0, 1, 2, 3}
    finals = [e for e in r0.evals if e.segment == 3]
    assert len(finals) == 2
    assert finals[0].input.producer_segment == finals[1].input.producer_segment == 2
    assert finals[0].input.producer_round == finals[1].input.producer_round


def test_time_shift():  # test_plan.cpp:153-166
    plain = adx.plan_async(50, 2, 2, 1, False)
    shifted = adx.plan_async(50, 2, 2, 1, True)
    for a, b in zip(plain.rounds, shifted.rounds):
        for ea, eb in zip(a.evals, b.evals):
            assert eb.embed_t == min(ea.embed_t + 1, 50)
        assert a.sampler_steps == b.sampler_steps
    assert adx.validate_plan(shifted) == []


def test_shift_embeddings_examples():  # test_plan.cpp:168-184
    full = list(range(50, 0, -1))
    sh = adx.shift_embeddings(full, 2)
    assert sh[:4] == [50, 49, 49, 48] and sh[-1] == 2
    assert all(sh[i] == full[i - 1] for i in range(2, 50))
    assert adx.shift_embeddings([3, 2, 1], 1) == [3, 3, 2]
    assert adx.shift_embeddings([3, 2, 1], 3) == [3, 2, 1]
    with pytest.raises(adx.InvalidArgument):
        adx.shift_embeddings([1, 2], 1)


def test_validate_flags_dangling_ref():  # test_plan.cpp:186-196
    plan = adx.plan_async(10, 1, 3, 1)
    plan.rounds[3].evals[1].input.producer_round = 0
    v = adx.validate_plan(plan)
    assert v and "round 3" in v[0] and "segment 2" in v[0]


def test_validate_flags_duplicate_sampler_step():
    plan = adx.plan_async(10, 1, 2, 1)
    plan.rounds[1].sampler_steps = list(plan.rounds[0].sampler_steps)
    assert adx.validate_plan(plan)


def test_validate_flags_device_twice():
    plan = adx.plan_async(10, 1, 3, 1)
    plan.rounds[0].evals[2].device = 0
    v = adx.validate_plan(plan)
    assert any("device 0" in s for s in v)


def test_validate_flags_eps_from_non_final():
    plan = adx.plan_async(10, 1, 3, 1)
    plan.rounds[0].evals[0].emits_eps_for = 9
    assert adx.validate_plan(plan)


def test_validate_flags_ref_into_non_broadcast_round():
    plan = adx.plan_async(10, 8, 2, 1)
    plan.rounds[0].broadcast = False
    v = adx.validate_plan(plan)
    assert v and "non-broadcast" in v[0]


def test_plan_counts_load_ratios():  # test_plan.cpp:225-243
    for N in (2, 3, 4):
        plan = adx.plan_async(50, 1, N, 1)
        c = adx.plan_counts(plan, uniform_partition(N))
        assert c.max_device_macs / c.sequential_total_macs == pytest.approx(1.0 / N, rel=0.02)
    plan = adx.plan_async(50, 3, 3, 2)
    c = adx.plan_counts(plan, uniform_partition(3))
    assert c.max_device_macs / c.sequential_total_macs == pytest.approx(1.0 / 6.0, rel=0.15)


def test_plan_counts_n_mismatch():
    with pytest.raises(adx.InvalidArgument):
        adx.plan_counts(adx.plan_async(10, 1, 3, 1), uniform_partition(2))


def test_render_plan_grid():  # test_plan.cpp:250-255
    g = adx.render_plan(adx.plan_async(10, 2, 3, 2))
    assert "dev0" in g and "dev3" in g and "warm-up steps: 10 9" in g


def test_flat_roundtrip():
    for args in [(20, 1, 2, 1), (20, 3, 3, 2), (7, 7, 1, 1)]:
        p = adx.plan_async(*args)
        assert adx.ExecutionPlan.from_flat(p.to_flat()) == p
