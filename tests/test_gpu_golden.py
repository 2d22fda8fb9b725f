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


def test_c1b_f32_async_trajectory_matches_oracle():
    """SURVEY §7 minimum slice: C1b (the reference's MLP-stage model at d=4096, square widths,
    seed 11, T=20, N=2 w=1 S=1) in fp32 within rel-L2 1e-3 of the fp64 C oracle (final latent
    and every step), and async-vs-sequential divergence equal to the oracle's"""
    widths = [4096] * 7
    m = adx.build_toy_denoiser(6, widths, "unet-mirror", 11)
    s = adx.build_schedule(20, 0.01, 0.15)
    x = adx.Latent(O.random_normals(12, 4096), 20)
    part = adx.partition_balanced(m, 2)
    plan = adx.plan_async(20, 1, 2, 1)
    par, _ = adx.run_parallel(plan, m, part, x, s, plan.D, precision="f32")
    seq = adx.sequential_denoise(m, x, s, precision="f32")
    O.set_threads(16)
    om = O.Model.build_toy(6, widths, "unet-mirror", 11, 8)
    ss, _ = O.partition_balanced(om.costs(), 2)
    olat, _, _, _ = O.run_serial(om, ss, 2, O.plan_async_flat(20, 1, 2, 1), s.alpha_bars, x.values)
    oseq, _ = O.sequential_denoise(om, s.alpha_bars, x.values)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert max(rel(par.latent_matrix()[k], olat[k]) for k in range(21)) < 1e-3
    assert rel(seq.latent_matrix()[-1], oseq[-1]) < 1e-3
    _, g, _ = O.compare_trajectories(seq.latent_matrix(), par.latent_matrix())
    _, o, _ = O.compare_trajectories(oseq, olat)
    assert abs(g - o) <= 1e-2 * o, (g, o)
