"""Denoiser evaluation on the sm_100a path (proj/tests/test_denoiser.cpp), fp64 mode."""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_hand_computed_2x2():  # test_denoiser.cpp:71-88 (G4)
    m = adx.make_denoiser_shell(2, [2, 2, 2], [], 2)
    m.stages[0].w1[:] = [[1, 0, 0, 0], [0, 1, 0, 0]]
    m.stages[0].w2[:] = [[2, 0], [0, 3]]
    m.stages[1].w1[:] = [[1, 1], [0, 1]]
    m.stages[1].w2[:] = [[0.5, 0], [0, 0.5]]
    out = adx.eval_full(m, adx.Latent(np.array([1.0, 2.0]), 1), 1, precision="f64")
    assert out == pytest.approx([4.0, 3.0], rel=1e-15)


def test_zero_weights_zero_output():
    m = adx.make_denoiser_shell(3, [2, 4, 4, 2], [(1, 3)], 2)
    out = adx.eval_full(m, adx.Latent(np.array([-3.0, 7.0]), 5), 5, precision="f64")
    assert np.linalg.norm(out) == 0.0


def test_non_finite_names_the_stage():
    m = adx.build_toy_denoiser(3, [2, 4, 4, 2], "none", 9)
    m.stages[1].w2[0, 0] = np.inf
    with pytest.raises(adx.DomainError, match="stage 2"):
        adx.eval_full(m, adx.Latent(np.ones(2), 1), 1, precision="f64")


def test_segment_chaining_equals_eval_full_bit_exact():  # test_denoiser.cpp:106-129
    rng = O.Rng(77)
    for rep in range(10):
        m = adx.build_toy_denoiser(6, [2, 8, 6, 10, 6, 8, 2], "unet-mirror", 1000 + rep)
        p = adx.partition_balanced(m, 3)
        x = adx.Latent(np.array([rng.normal(), rng.normal()]), 7)
        t = 1 + rng.below(20)
        whole = adx.eval_full(m, x, t, precision="f64")
        skips = {}
        so = adx.eval_segment(m, p, 1, x, skips, t, precision="f64")
        for seg in (2, 3):
            assert so.produced_by == seg - 1 and so.produced_at == t
            skips.update(so.skips)
            so = adx.eval_segment(m, p, seg, so, skips, t, precision="f64")
        assert np.array_equal(whole, so)
        # and matches the oracle
        om = O.Model.build_toy(6, [2, 8, 6, 10, 6, 8, 2], "unet-mirror", 1000 + rep, 8)
        assert np.abs(om.eval_full(x.values, t) - whole).max() < 1e-13


def test_n1_segment_equals_eval_full():
    m = adx.build_toy_denoiser(4, [2, 6, 6, 6, 2], "unet-mirror", 3)
    p = adx.partition_balanced(m, 1)
    x = adx.Latent(np.array([0.3, -0.7]), 4)
    assert np.array_equal(adx.eval_segment(m, p, 1, x, {}, 4, precision="f64"),
                          adx.eval_full(m, x, 4, precision="f64"))


def test_stale_bundles_are_legal():
    m = adx.build_toy_denoiser(4, [2, 6, 6, 6, 2], "none", 3)
    p = adx.partition_balanced(m, 2)
    x = adx.Latent(np.array([0.1, 0.9]), 9)
    b9 = adx.eval_segment(m, p, 1, x, {}, 9, precision="f64")
    assert b9.produced_at == 9
    eps = adx.eval_segment(m, p, 2, b9, {}, 8, precision="f64")
    assert np.all(np.isfinite(eps))


def test_input_contract_errors():
    m = adx.build_toy_denoiser(4, [2, 6, 6, 6, 2], "none", 3)
    p = adx.partition_balanced(m, 2)
    x = adx.Latent(np.ones(2), 4)
    with pytest.raises(adx.InvalidArgument):
        adx.eval_segment(m, p, 2, x, {}, 4, precision="f64")
    b = adx.eval_segment(m, p, 1, x, {}, 4, precision="f64")
    with pytest.raises(adx.InvalidArgument):
        adx.eval_segment(m, p, 1, b, {}, 4, precision="f64")
    wrong = adx.HiddenBundle(b.boundary, b.skips, produced_by=2, produced_at=4)
    with pytest.raises(adx.InvalidArgument, match="segment"):
        adx.eval_segment(m, p, 2, wrong, {}, 4, precision="f64")


def test_missing_crossing_skip_names_the_link():
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 5)
    p = adx.partition_balanced(m, 3)
    assert p.segments[0] == [1, 2]
    x = adx.Latent(np.ones(2), 3)
    b1 = adx.eval_segment(m, p, 1, x, {}, 3, precision="f64")
    assert len(b1.skips) == 2
    b2 = adx.eval_segment(m, p, 2, b1, {}, 3, precision="f64")
    assert b2.skips == {}
    with pytest.raises(adx.AdxRuntimeError, match="->"):
        adx.eval_segment(m, p, 3, b2, {}, 3, precision="f64")


def test_skip_completeness():
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 5)
    for N in (2, 3, 4, 5):
        p = adx.partition_balanced(m, N)
        x = adx.Latent(np.ones(2), 3)
        seen, skips = [], {}
        so = adx.eval_segment(m, p, 1, x, skips, 3, precision="f64")
        for seg in range(2, N + 1):
            for l, f in so.skips.items():
                seen.append(l)
                skips[l] = f
            so = adx.eval_segment(m, p, seg, so, skips, 3, precision="f64")
        assert sorted(seen) == sorted(adx.crossing_links(m, p))


@pytest.mark.parametrize("prec,tol", [("f32", 1e-5), ("bf16", 2e-2)])
def test_reduced_precision_eval_within_tolerance(prec, tol):
    m = adx.build_toy_denoiser(6, [64] * 7, "unet-mirror", 21)
    x = adx.Latent(O.random_normals(3, 64), 10)
    ref = adx.eval_full(m, x, 10, precision="f64")
    out = adx.eval_full(m, x, 10, precision=prec)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < tol


def test_ddim_errors():
    s = adx.build_schedule(5, 0.01, 0.1)
    x = adx.Latent(np.zeros(3), 5)
    with pytest.raises(adx.OutOfRange):
        adx.ddim_step(x, np.zeros(3), 6, s)
    with pytest.raises(adx.DomainError, match="t=3"):
        adx.ddim_step(x, np.array([0.0, np.nan, 1.0]), 3, s)
