"""Pin the CPU oracle (oracle/adx_oracle.c) to the reference's own golden and
known-answer vectors.  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O

G1 = 0.0011860077151787584  # proj/tests/test_executor.cpp:80
G2 = 0.00027252781017261107  # proj/tests/test_metrics.cpp:54


def fixture():
    m = O.Model.build_toy(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 8)
    s = O.build_schedule(20, 0.01, 0.15)
    x = O.random_normals(12, 2)
    return m, s, x


def test_mt19937_64_known_answer():
    # std::mt19937_64 default seed 5489: the 10000th output is 9981545732273789042
    r = O.Rng(5489)
    v = None
    for _ in range(10000):
        v = r.next_u64()
    assert v == 9981545732273789042


def test_rng_uniform_and_normal_are_deterministic():
    a, b = O.Rng(7), O.Rng(7)
    assert [a.uniform() for _ in range(5)] == [b.uniform() for _ in range(5)]
    assert [a.normal() for _ in range(5)] == [b.normal() for _ in range(5)]
    u = [O.Rng(3).uniform() for _ in range(1)]
    assert 0.0 <= u[0] < 1.0


def test_g1_async_divergence_w1():
    m, s, x = fixture()
    seq, _ = O.sequential_denoise(m, s.alpha_bars, x)
    ss, sm = O.partition_balanced(m.costs(), 2)
    assert ss.tolist() == [1, 1, 1, 2, 2, 2] and sm.tolist() == [592, 564]
    lat, _, _, bc = O.run_serial(m, ss, 2, O.plan_async_flat(20, 1, 2, 1), s.alpha_bars, x)
    mse = ((lat[-1] - seq[-1]) ** 2).sum() / 2.0
    assert mse == pytest.approx(G1, rel=1e-9)
    assert bc == 19


def test_g2_compare_trajectories_w3():
    m, s, x = fixture()
    seq, _ = O.sequential_denoise(m, s.alpha_bars, x)
    ss, _ = O.partition_balanced(m.costs(), 2)
    lat, _, _, _ = O.run_serial(m, ss, 2, O.plan_async_flat(20, 3, 2, 1), s.alpha_bars, x)
    _, fm, _ = O.compare_trajectories(seq, lat)
    assert fm == pytest.approx(G2, rel=1e-9)


def test_g3_scalar_ddim():  # test_diffusion.cpp:119-132
    ab = np.array([1.0, 0.81, 0.25])
    out = O.ddim_step(np.array([1.0]), np.array([0.5]), 2, ab)
    assert out[0] == pytest.approx(1.23852208377104, rel=1e-12)


def test_schedule_known_answers():  # test_diffusion.cpp:36-48
    s = O.build_schedule(3, 0.1, 0.3)
    assert s.alpha_bars[3] == pytest.approx(0.504, rel=1e-12)
    sl = O.build_schedule(3, 0.01, 0.09, "scaled-linear")
    assert sl.betas[1] == pytest.approx(0.04, rel=1e-12)
    one = O.build_schedule(1, 0.5, 0.5)
    assert one.alpha_bars[1] == pytest.approx(0.5)
    with pytest.raises(ValueError):
        O.build_schedule(0, 0.1, 0.2)
    with pytest.raises(ValueError):
        O.build_schedule(5, 0.3, 0.2)


def test_forward_diffuse_known_answer():  # test_diffusion.cpp:80-85
    ab = np.array([1.0, 0.64])
    out = O.forward_diffuse(np.array([1.0, 0.0]), np.array([0.0, 1.0]), 1, ab)
    assert out == pytest.approx([0.8, 0.6], rel=1e-12)


def test_exact_noise_ddim_lands_on_forward_marginal():  # test_diffusion.cpp:103-117
    s = O.build_schedule(10, 0.01, 0.2)
    rng = np.random.default_rng(0)
    x0, noise = rng.normal(size=3), rng.normal(size=3)
    for t in range(2, 11):
        xt = O.forward_diffuse(x0, noise, t, s.alpha_bars)
        prev = O.ddim_step(xt, noise, t, s.alpha_bars)
        want = O.forward_diffuse(x0, noise, t - 1, s.alpha_bars)
        assert np.abs(prev - want).max() < 1e-12


def test_g4_hand_model_two_by_two():  # test_denoiser.cpp:71-88
    m = O.Model.shell(2, [2, 2, 2], [], 2)
    m.tensor(1, O.W1)[:] = np.array([[1, 0, 0, 0], [0, 1, 0, 0]], float)
    m.tensor(1, O.W2)[:] = np.array([[2, 0], [0, 3]], float)
    m.tensor(2, O.W1)[:] = np.array([[1, 1], [0, 1]], float)
    m.tensor(2, O.W2)[:] = np.array([[0.5, 0], [0, 0.5]], float)
    out = m.eval_full(np.array([1.0, 2.0]), 1)
    assert out == pytest.approx([4.0, 3.0], rel=1e-15)


def test_g5_plan_shapes():  # test_plan.cpp:26-47
    f = O.plan_async_flat(50, 1, 2, 1)
    assert f[6] == 49 and f[4] == 2
    f = O.plan_async_flat(50, 1, 3, 2)
    assert f[6] == 25 and f[4] == 4


def test_g6_partition_4114():  # test_partition.cpp:56-63
    ss, sm = O.partition_balanced([4, 1, 1, 4], 2)
    assert ss.tolist() == [1, 1, 2, 2]
    assert max(sm) == 5


def test_zero_eps_telescoping():  # test_diffusion.cpp:157-170 (zero model -> eps = 0)
    m = O.Model.shell(2, [2, 3, 2], [], 2)
    s = O.build_schedule(10, 0.01, 0.1)
    x = np.array([0.3, -1.2])
    lat, eps = O.sequential_denoise(m, s.alpha_bars, x)
    assert np.all(eps == 0)
    # with eps = 0 every step rescales by sqrt(abar_{t-1}/abar_t): x_0 = x_T / sqrt(abar_T)
    assert lat[-1] == pytest.approx(x / np.sqrt(s.alpha_bars[10]), rel=1e-12)


def test_parallel_equals_serial_random_cases():  # test_executor.cpp:83-106
    rng = O.Rng(2025)
    for rep in range(6):
        trng = O.Rng(5000 + rep)
        d = 2 + 2 * trng.below(2)
        L = 2 + trng.below(5)
        widths = [d] + [4 + 2 * trng.below(4) for _ in range(L - 1)] + [d]
        spec = "unet-mirror" if trng.below(2) else "none"
        m = O.Model.build_toy(L, widths, spec, trng.next_u64(), 8)
        T = 4 + trng.below(20)
        s = O.build_schedule(T, 1e-3, 0.05)
        x = np.array([trng.normal() for _ in range(d)])
        S = 1 + rng.below(2)
        N = (2 if S == 2 else 1) + rng.below(3)
        N = min(N, L)
        if S == 2 and N < 2:
            N = 2
        w = 1 + rng.below(T)
        ss, _ = O.partition_balanced(m.costs(), N)
        pf = O.plan_async_flat(T, w, N, S)
        a, ae, _, _ = O.run_serial(m, ss, N, pf, s.alpha_bars, x)
        b, be, _ = O.run_parallel(m, ss, N, pf, s.alpha_bars, x)
        assert np.array_equal(a, b) and np.array_equal(ae, be)
