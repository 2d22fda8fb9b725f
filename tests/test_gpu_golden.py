"""Reference goldens reproduced by the sm_100a path (fp64 mode), through the C ABI.

G1 proj/tests/test_executor.cpp:66-81, G2 proj/tests/test_metrics.cpp:42-55,
G3 proj/tests/test_diffusion.cpp:119-132, equivalences test_executor.cpp:33-50,
parallel == serial test_executor.cpp:83-106.
"""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O

pytestmark = pytest.mark.gpu

G1 = 0.0011860077151787584
G2 = 0.00027252781017261107


def fixture(T=20, seed=11):
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", seed)
    s = adx.build_schedule(T, 0.01, 0.15, "linear")
    x_T = adx.Latent(O.random_normals(seed + 1, 2), T)
    return m, s, x_T


def test_g1_async_divergence_w1():
    m, s, x_T = fixture()
    seq = adx.sequential_denoise(m, x_T, s, precision="f64")
    plan = adx.plan_async(20, 1, 2, 1)
    part = adx.partition_balanced(m, 2)
    traj, stats = adx.run_serial(plan, m, part, x_T, s, precision="f64")
    mse = ((traj.final_latent().values - seq.final_latent().values) ** 2).sum() / 2.0
    assert mse == pytest.approx(G1, rel=1e-9)
    assert stats.broadcast_count == len(plan.rounds)


def test_g2_compare_trajectories_w3():
    m, s, x_T = fixture()
    seq = adx.sequential_denoise(m, x_T, s, precision="f64")
    plan = adx.plan_async(20, 3, 2, 1)
    part = adx.partition_balanced(m, 2)
    traj, _ = adx.run_serial(plan, m, part, x_T, s, precision="f64")
    rep = adx.compare_trajectories(seq, traj)
    assert rep.final_mse == pytest.approx(G2, rel=1e-9)


def test_g3_scalar_ddim_on_gpu():
    sched = adx.NoiseSchedule(2, np.zeros(2), np.zeros(2), np.array([1.0, 0.81, 0.25]))
    out = adx.ddim_step(adx.Latent(np.array([1.0]), 2), np.array([0.5]), 2, sched, precision="f64")
    assert out.values[0] == pytest.approx(1.23852208377104, rel=1e-12)
    assert out.timestep == 1
    # bit-identical to the oracle's IEEE expression
    ref = O.ddim_step(np.array([1.0]), np.array([0.5]), 2, sched.alpha_bars)
    assert out.values[0] == ref[0]


def test_w_equals_T_is_sequential_bit_exact():
    m, s, x_T = fixture()
    seq = adx.sequential_denoise(m, x_T, s, precision="f64")
    plan = adx.plan_async(20, 20, 3, 1)
    part = adx.partition_balanced(m, 3)
    traj, stats = adx.run_serial(plan, m, part, x_T, s, precision="f64")
    assert np.array_equal(traj.latent_matrix(), seq.latent_matrix())
    assert stats.broadcast_count == 0


def test_n1_equals_sequential_any_w():
    m, s, x_T = fixture()
    seq = adx.sequential_denoise(m, x_T, s, precision="f64")
    part = adx.partition_balanced(m, 1)
    for w in (1, 5, 19, 20):
        traj, _ = adx.run_serial(adx.plan_async(20, w, 1, 1), m, part, x_T, s, precision="f64")
        assert np.array_equal(traj.latent_matrix(), seq.latent_matrix())


@pytest.mark.parametrize("N,S,w", [(2, 1, 1), (3, 1, 2), (2, 2, 3), (3, 2, 1), (4, 1, 5)])
def test_gpu_matches_oracle_trajectory(N, S, w):
    m, s, x_T = fixture()
    plan = adx.plan_async(20, w, N, S)
    part = adx.partition_balanced(m, N)
    traj, _ = adx.run_serial(plan, m, part, x_T, s, precision="f64")
    par, _ = adx.run_parallel(plan, m, part, x_T, s, plan.D, precision="f64")
    assert np.array_equal(traj.latent_matrix(), par.latent_matrix())
    om = O.Model.build_toy(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 8)
    ss, _ = O.partition_balanced(om.costs(), N)
    olat, oeps, _, _ = O.run_serial(om, ss, N, O.plan_async_flat(20, w, N, S), s.alpha_bars, x_T.values)
    assert np.abs(traj.latent_matrix() - olat).max() < 1e-12
    assert np.abs(np.stack(traj.eps_used) - oeps).max() < 1e-12
