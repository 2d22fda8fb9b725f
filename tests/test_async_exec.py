"""Pins the model-agnostic executor restatement (oracle/async_exec.py) against the
C oracle's run_serial and the reference goldens on the reference's own fixture
(proj/tests/test_executor.cpp:14-29, 66-81; test_metrics.cpp:42-55) before it is
used as the async oracle of the UNet family (tests/test_gpu_unet_async.py).
CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle.async_exec import AsyncOracle, mlp_stage_fn


def fixture():
    m = O.Model.build_toy(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 8)
    s = O.build_schedule(20, 0.01, 0.15)
    return m, s, O.random_normals(12, 2)


@pytest.mark.parametrize("w,golden", [(1, 0.0011860077151787584), (3, 0.00027252781017261107)])
def test_async_exec_reproduces_goldens(w, golden):
    m, s, x = fixture()
    ss, _ = O.partition_balanced(m.costs(), 2)
    plan = O.plan_async_flat(20, w, 2, 1)
    ex = AsyncOracle(m.L, m.links, mlp_stage_fn(m))
    lat, eps, entries, bc = ex.run_serial(ss, plan, s.alpha_bars, x)
    clat, ceps, centries, cbc = O.run_serial(m, ss, 2, plan, s.alpha_bars, x)
    assert np.array_equal(lat, clat) and np.array_equal(eps, ceps)
    assert entries == centries and bc == cbc
    seq, _ = O.sequential_denoise(m, s.alpha_bars, x)
    _, fm, _ = O.compare_trajectories(seq, lat)
    assert abs(fm - golden) <= 1e-9 * golden


@pytest.mark.parametrize("N,S,w", [(1, 1, 1), (2, 1, 2), (3, 1, 1), (2, 2, 1), (3, 2, 2), (6, 1, 1)])
def test_async_exec_equals_c_oracle(N, S, w):
    rng = np.random.default_rng(N * 10 + S)
    m = O.Model.build_toy(6, [3, 7, 5, 9, 6, 4, 3], "unet-mirror", 21 + N, 8)
    s = O.build_schedule(9, 0.01, 0.2)
    x = rng.standard_normal(3)
    ss, _ = O.partition_balanced(m.costs(), N)
    plan = O.plan_async_flat(9, w, N, S)
    lat, eps, entries, bc = AsyncOracle(m.L, m.links, mlp_stage_fn(m)).run_serial(ss, plan, s.alpha_bars, x)
    clat, ceps, centries, cbc = O.run_serial(m, ss, N, plan, s.alpha_bars, x)
    assert np.array_equal(lat, clat) and np.array_equal(eps, ceps)
    assert entries == centries and bc == cbc
