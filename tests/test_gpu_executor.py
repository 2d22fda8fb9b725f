"""Executor contract on the GPU engine (proj/tests/test_executor.cpp).
Multi-device runs use several virtual devices mapped onto the one GPU (one
stream pair each, event-ordered exchange): no kernel ever waits on another."""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O

pytestmark = pytest.mark.gpu


class Fixture:  # test_executor.cpp:14-29
    def __init__(self, T=20, seed=11):
        self.model = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", seed)
        self.schedule = adx.build_schedule(T, 0.01, 0.15)
        self.x_T = adx.Latent(O.random_normals(seed + 1, 2), T)


def random_toy_case(seed, max_T=24):  # test_util.hpp:56-73
    rng = O.Rng(seed)
    d = 2 + 2 * rng.below(2)
    L = 2 + rng.below(5)
    widths = [d] + [4 + 2 * rng.below(4) for _ in range(L - 1)] + [d]
    spec = "unet-mirror" if rng.below(2) else "none"
    model = adx.build_toy_denoiser(L, widths, spec, rng.next_u64(), 8)
    T = 4 + rng.below(max_T - 4)
    sched = adx.build_schedule(T, 1e-3, 0.05)
    x = adx.Latent(np.array([rng.normal() for _ in range(d)]), T)
    return model, sched, x


def test_async_trajectory_finite_and_complete():
    f = Fixture()
    for N, S, w in [(2, 1, 1), (3, 1, 2), (2, 2, 3), (3, 2, 1), (4, 1, 5)]:
        plan = adx.plan_async(20, w, N, S)
        p = adx.partition_balanced(f.model, N)
        traj, stats = adx.run_serial(plan, f.model, p, f.x_T, f.schedule, precision="f64")
        assert len(traj.latents) == 21 and len(traj.eps_used) == 20
        assert np.all(np.isfinite(traj.latent_matrix()))
        assert stats.broadcast_count == len(plan.rounds)


def test_parallel_matches_serial_bit_exactly_random_cases():  # test_executor.cpp:83-106
    rng = O.Rng(2025)
    for rep in range(12):
        model, sched, x = random_toy_case(5000 + rep)
        T = sched.T
        S = 1 + rng.below(2)
        N = (2 if S == 2 else 1) + rng.below(3)
        N = min(N, model.num_stages())
        if S == 2 and N < 2:
            N = 2
        w = 1 + rng.below(T)
        plan = adx.plan_async(T, w, N, S)
        p = adx.partition_balanced(model, N)
        opts = adx.RunOptions(jitter_seed=rng.next_u64(), max_jitter_s=0.002)
        serial, ss = adx.run_serial(plan, model, p, x, sched, opts, precision="f64")
        par, ps = adx.run_parallel(plan, model, p, x, sched, plan.D, opts, precision="f64")
        assert np.array_equal(serial.latent_matrix(), par.latent_matrix())
        assert np.array_equal(np.stack(serial.eps_used), np.stack(par.eps_used))
        assert ps.broadcast_count == ss.broadcast_count
        # eager (non-graph, instrumented) enqueue gives the same bits
        eager, _ = adx.run_parallel(plan, model, p, x, sched, plan.D, adx.RunOptions(use_graph=False, instrument=True),
                                    precision="f64")
        assert np.array_equal(eager.latent_matrix(), par.latent_matrix())


def test_parallel_on_two_ordinal_slots_same_gpu():
    """virtual devices mapped via an explicit ordinal list (all on GPU 0)."""
    f = Fixture()
    plan = adx.plan_async(20, 2, 3, 2)
    p = adx.partition_balanced(f.model, 3)
    ref, _ = adx.run_serial(plan, f.model, p, f.x_T, f.schedule, precision="f32")
    par, _ = adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, plan.D, precision="f32", devices=(0, 0, 0, 0))
    assert np.array_equal(ref.latent_matrix(), par.latent_matrix())


def test_worker_count_must_match():  # test_executor.cpp:108-114
    f = Fixture()
    plan = adx.plan_async(20, 1, 3, 2)
    p = adx.partition_balanced(f.model, 3)
    with pytest.raises(adx.InvalidArgument):
        adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, 3)


def test_rejects_invalid_plans_and_partitions():  # test_executor.cpp:116-133
    f = Fixture()
    plan = adx.plan_async(20, 1, 3, 1)
    p3 = adx.partition_balanced(f.model, 3)
    p2 = adx.partition_balanced(f.model, 2)
    with pytest.raises(adx.InvalidArgument):
        adx.run_serial(plan, f.model, p2, f.x_T, f.schedule)
    bad = adx.ExecutionPlan.from_flat(plan.to_flat())
    bad.rounds[2].evals[1].input.producer_round = 0
    with pytest.raises(adx.InvalidArgument):
        adx.run_serial(bad, f.model, p3, f.x_T, f.schedule)
    fl = adx.partition_balanced(f.model, 3, "first-last-grouped")
    with pytest.raises(adx.InvalidArgument):
        adx.run_serial(plan, f.model, fl, f.x_T, f.schedule)


def test_store_retention_flat():  # test_executor.cpp:135-160
    """the engine's BundleStore ledger (replayed from the bundles its enqueue commits) equals
    the oracle's BundleStore occupancy round by round, flat at 3 (N - 1) after round 0"""
    f = Fixture()
    om = O.Model.build_toy(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 8)
    for N, S, w in [(3, 1, 2), (2, 2, 1), (4, 1, 1), (3, 2, 3), (1, 1, 2)]:
        plan = adx.plan_async(20, w, N, S)
        p = adx.partition_balanced(f.model, N)
        _, stats = adx.run_serial(plan, f.model, p, f.x_T, f.schedule)
        _, pst = adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, plan.D)
        ss, _ = O.partition_balanced(om.costs(), N)
        _, _, entries, _ = O.run_serial(om, ss, N, O.plan_async_flat(20, w, N, S), f.schedule.alpha_bars,
                                        f.x_T.values)
        assert stats.store_entries_per_round == entries == pst.store_entries_per_round, (N, S, w)
        assert set(entries[1:]) <= {3 * (N - 1)}


def test_start_jitter_delays_devices_not_results():  # executor.cpp:445-449
    """max_jitter_s delays each device's first work by Rng(mix_seed(seed, d)).uniform() * max;
    the trajectory is unchanged and the instrumented wall time grows by the largest draw"""
    f = Fixture()
    plan = adx.plan_async(20, 1, 3, 1)
    p = adx.partition_balanced(f.model, 3)
    base, bst = adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, 3,
                                 adx.RunOptions(use_graph=False, instrument=True))
    seed, mx = 99, 0.05
    jit, jst = adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, 3,
                                adx.RunOptions(jitter_seed=seed, max_jitter_s=mx, use_graph=False, instrument=True))
    assert np.array_equal(base.latent_matrix(), jit.latent_matrix())
    draws = [O.Rng(O.mix_seed(seed, d)).uniform() * mx for d in range(3)]
    assert jst.total_wall_s >= bst.total_wall_s + 0.8 * max(draws)
    with pytest.raises(adx.InvalidArgument):
        adx.run_parallel(plan, f.model, p, f.x_T, f.schedule, 3, adx.RunOptions(max_jitter_s=-1.0))


def test_zero_delays_identical():  # test_executor.cpp:162-173
    f = Fixture()
    plan = adx.plan_async(20, 1, 2, 1)
    p = adx.partition_balanced(f.model, 2)
    plain, _ = adx.run_serial(plan, f.model, p, f.x_T, f.schedule)
    delayed, _ = adx.run_serial(plan, adx.inject_delay(f.model, [0.0, 0.0]), p, f.x_T, f.schedule)
    assert np.array_equal(plain.latent_matrix(), delayed.latent_matrix())
    with pytest.raises(adx.InvalidArgument):
        adx.inject_delay(f.model, [-0.1, 0.0])


def test_busy_time_tracks_injected_sleeps():  # test_executor.cpp:175-193
    f = Fixture()
    plan = adx.plan_async(20, 1, 4, 1)
    p = adx.partition_balanced(f.model, 4)
    _, stats = adx.run_parallel(plan, adx.inject_delay(f.model, [0.005] * 4), p, f.x_T, f.schedule, 4)
    for d in range(4):
        assert stats.device_evals[d] == 20
        assert 0.100 <= stats.device_busy_s[d] <= 0.200
    assert sum(stats.device_busy_s) <= stats.total_wall_s * 4.0 * 1.05


def test_round_wall_tracks_slowest_device():  # test_executor.cpp:195-204
    f = Fixture(12)
    plan = adx.plan_async(12, 1, 4, 1)
    p = adx.partition_balanced(f.model, 4)
    _, stats = adx.run_parallel(plan, adx.inject_delay(f.model, [0.040, 0.010, 0.010, 0.010]), p, f.x_T,
                                f.schedule, 4)
    for wall in stats.round_wall_s:
        assert 0.040 * 0.95 <= wall <= 0.040 * 1.5


def test_round_timeout_names_the_laggard():  # test_executor.cpp:206-215
    f = Fixture()
    plan = adx.plan_async(20, 1, 2, 1)
    p = adx.partition_balanced(f.model, 2)
    with pytest.raises(adx.AdxRuntimeError, match="timeout"):
        adx.run_parallel(plan, adx.inject_delay(f.model, [0.0, 0.5]), p, f.x_T, f.schedule, 2,
                         adx.RunOptions(round_timeout_s=0.02))


def test_sequential_error_wraps_timestep():
    m = adx.build_toy_denoiser(3, [2, 4, 4, 2], "none", 9)
    m.stages[2].w2[0, 0] = np.inf
    s = adx.build_schedule(5, 0.01, 0.1)
    with pytest.raises(adx.AdxRuntimeError, match=r"t=5: eval: non-finite activation at stage 3"):
        adx.sequential_denoise(m, adx.Latent(np.ones(2), 5), s)


def test_rank_session_single_rank_matches_sequential():
    """NCCL rank path (rank.cu) with one rank: N=1 plan == sequential_denoise bit-exactly."""
    f = Fixture()
    plan = adx.plan_async(20, 1, 1, 1)
    part = adx.partition_balanced(f.model, 1)
    sess = adx.RankSession(f.model, f.schedule, plan, part, 0, adx.nccl_unique_id(), 0, "f64")
    lat, eps = np.zeros((21, 2)), np.zeros((20, 2))
    sess.run_into(np.ascontiguousarray(f.x_T.values), lat, eps)
    seq = adx.sequential_denoise(f.model, f.x_T, f.schedule, precision="f64")
    assert np.array_equal(lat, seq.latent_matrix())
    assert sess.time(2) > 0
