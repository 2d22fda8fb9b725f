"""Partition DP and model construction parity (proj/tests/test_partition.cpp,
test_denoiser.cpp host parts) through the C ABI, CPU only."""
import itertools

import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O


def model_with_costs(costs):  # test_partition.cpp:16-23
    L = len(costs)
    widths = [2] + [4] * (L - 1) + [2]
    m = adx.make_denoiser_shell(L, widths, [], 2)
    for i, c in enumerate(costs):
        m.stages[i].cost_macs = c
    return m


def brute_force_min_max(costs, N):
    L = len(costs)
    best = None
    for cuts in itertools.combinations(range(1, L), N - 1):
        b = [0, *cuts, L]
        mx = max(sum(costs[b[k]:b[k + 1]]) for k in range(N))
        best = mx if best is None else min(best, mx)
    return best


def test_uniform_costs_split_evenly():
    p = adx.partition_balanced(model_with_costs([5] * 8), 4)
    assert p.num_segments() == 4
    assert all(len(s) == 2 for s in p.segments)
    assert p.max_segment_macs() == p.total_macs() // 4
    assert p.contiguous()


def test_4114_max5():
    p = adx.partition_balanced(model_with_costs([4, 1, 1, 4]), 2)
    assert p.max_segment_macs() == 5
    assert p.segments == [[1, 2], [3, 4]]


def test_first_last_grouped():
    m = model_with_costs([3] * 6)
    p = adx.partition_balanced(m, 3, "first-last-grouped")
    assert p.segments[0] == [1, 6]
    assert not p.contiguous()
    assert p.segment_of_stage(1) == p.segment_of_stage(6)
    assert len(p.segments[1]) == 2 and len(p.segments[2]) == 2
    assert p.segment_macs[0] == 6
    p.validate(m)
    p1 = adx.partition_balanced(model_with_costs([1, 2, 3]), 1, "first-last-grouped")
    assert p1.segments == [[1, 2, 3]] and p1.contiguous()


def test_infeasible_n():
    m = model_with_costs([1, 1, 1, 1])
    with pytest.raises(adx.InvalidArgument):
        adx.partition_balanced(m, 5)
    with pytest.raises(adx.InvalidArgument):
        adx.partition_balanced(m, 0)
    with pytest.raises(adx.InvalidArgument):
        adx.partition_balanced(m, 4, "first-last-grouped")
    adx.partition_balanced(m, 3, "first-last-grouped")


def test_optimality_vs_brute_force_and_oracle():
    rng = O.Rng(404)
    for _ in range(60):
        L = 2 + rng.below(11)
        costs = [1 + rng.below(50) for _ in range(L)]
        N = 1 + rng.below(L)
        p = adx.partition_balanced(model_with_costs(costs), N)
        assert p.max_segment_macs() == brute_force_min_max(costs, N)
        assert p.num_segments() == N and p.contiguous()
        # tie-breaking bit-exact with the oracle's restatement of min_max_split
        ss, sm = O.partition_balanced(costs, N)
        ours = [0] * L
        for n, seg in enumerate(p.segments):
            for s in seg:
                ours[s - 1] = n + 1
        assert ours == ss.tolist() and p.segment_macs == sm.tolist()


def test_first_last_grouped_optimality():
    rng = O.Rng(405)
    for _ in range(40):
        L = 3 + rng.below(9)
        costs = [1 + rng.below(50) for _ in range(L)]
        N = 2 + rng.below(L - 2)
        p = adx.partition_balanced(model_with_costs(costs), N, "first-last-grouped")
        expected = max(costs[0] + costs[-1], brute_force_min_max(costs[1:-1], N - 1))
        assert p.max_segment_macs() == expected


def test_crossing_links():
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 5)
    p = adx.partition_balanced(m, 2)
    assert len(adx.crossing_links(m, p)) == 3
    assert adx.crossing_links(m, adx.partition_balanced(m, 1)) == []


def test_skip_specs():
    assert adx.build_toy_denoiser(4, [2, 8, 8, 8, 2], "none", 1).skip_links == []
    assert adx.build_toy_denoiser(6, [2] + [8] * 5 + [2], "unet-mirror", 1).skip_links == [(1, 6), (2, 5), (3, 4)]
    assert adx.build_toy_denoiser(5, [2, 8, 8, 8, 8, 2], "unet-mirror", 1).skip_links == [(1, 5), (2, 4)]


def test_determinism_and_errors():
    a = adx.build_toy_denoiser(4, [2, 8, 6, 8, 2], "unet-mirror", 42)
    b = adx.build_toy_denoiser(4, [2, 8, 6, 8, 2], "unet-mirror", 42)
    c = adx.build_toy_denoiser(4, [2, 8, 6, 8, 2], "unet-mirror", 43)
    assert np.array_equal(a.stages[0].w1, b.stages[0].w1)
    assert not np.array_equal(a.stages[0].w1, c.stages[0].w1)
    with pytest.raises(adx.InvalidArgument):
        adx.build_toy_denoiser(1, [2, 2], "none", 1)
    with pytest.raises(adx.InvalidArgument):
        adx.build_toy_denoiser(4, [2, 8, 8, 2], "none", 1)
    with pytest.raises(adx.InvalidArgument):
        adx.build_toy_denoiser(4, [2, 8, 8, 8, 3], "none", 1)


def test_stage_widths_account_for_concat():
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 1, 8)
    assert m.stages[0].in_width() == 10
    assert m.stages[3].in_width() == 16
    assert m.stages[5].in_width() == 16
    assert all(s.cost_macs > 0 for s in m.stages)


def test_weights_bit_identical_to_oracle_init():
    """xavier init from Rng(seed) (denoiser.cpp:21-27, 124-142): the product's
    std::mt19937_64 path and the oracle's C MT19937-64 agree bit for bit."""
    widths = [2, 8, 6, 10, 6, 8, 2]
    m = adx.build_toy_denoiser(6, widths, "unet-mirror", 1234, 8)
    om = O.Model.build_toy(6, widths, "unet-mirror", 1234, 8)
    assert np.array_equal(m.proj, om.tensor(1, O.PROJ))
    for i in range(1, 7):
        st = m.stages[i - 1]
        for name, tid in (("w1", O.W1), ("time_in", O.TIN), ("w2", O.W2)):
            assert np.array_equal(getattr(st, name), om.tensor(i, tid)), (i, name)
        assert st.cost_macs == om.stage_macs(i)


def test_schedule_bit_identical_to_oracle():
    for T, a, b, k in [(20, 0.01, 0.15, "linear"), (50, 1e-4, 0.02, "scaled-linear"), (1, 0.5, 0.5, "linear")]:
        s = adx.build_schedule(T, a, b, k)
        o = O.build_schedule(T, a, b, k)
        assert np.array_equal(s.alpha_bars, o.alpha_bars) and np.array_equal(s.betas, o.betas)
    s = adx.build_schedule(3, 0.1, 0.3)
    assert s.alpha_bar(3) == pytest.approx(0.504)
    with pytest.raises(adx.OutOfRange):
        s.alpha_bar(4)
    with pytest.raises(adx.InvalidArgument):
        adx.build_schedule(5, 0.3, 0.2)


def test_sinusoid_matches_oracle():
    for t in (1, 7, 50):
        assert np.array_equal(adx.sinusoid(t, 8), O.sinusoid(t, 8))
    assert np.abs(adx.sinusoid(7, 8)).max() <= 1.0


def test_partition_by_cost_is_minmax_optimal():
    """partition_by_cost (extension): the partition.cpp min-max DP over arbitrary stage
    costs -- optimal against brute force, ties to the smallest cut, MACs still reported."""
    import itertools
    rng = np.random.default_rng(3)
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2])
    for _ in range(40):
        costs = rng.integers(1, 6, size=6).astype(float) * 0.25
        for N in (1, 2, 3, 4):
            p = adx.partition_by_cost(m, N, costs)
            segs = p.segments
            got = max(sum(costs[s - 1] for s in sg) for sg in segs)
            best = None
            for cuts in itertools.combinations(range(1, 6), N - 1):
                b = (0,) + cuts + (6,)
                v = max(sum(costs[b[k]:b[k + 1]]) for k in range(N))
                if best is None or v < best[0] - 1e-12:
                    best = (v, cuts)
            assert abs(got - best[0]) < 1e-12
            assert sum(p.segment_macs) == m.total_macs()
    with pytest.raises(adx.InvalidArgument):
        adx.partition_by_cost(m, 2, [1.0, 2.0])
