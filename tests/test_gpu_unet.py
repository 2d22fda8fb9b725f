"""UNet-shaped family on the sm_100a path (tcgen05 conv/GEMM/attention stages):
numerics vs the builder-written numpy oracle (oracle/unet_oracle.py over the
independent model restatement oracle/unet_model.py -- parity unpinned by
reference vectors), and the reference's executor invariants,
which are model-agnostic and exact.
  precision "bf16": bf16 activations, fp32 latent     -> TOL 3e-2 vs the bf16-rounding oracle
  precision "f32":  fp32 activations, split-bf16 MMAs -> TOL_F32 1e-3 vs the fp64 oracle
                    (the north_star's rel-L2 <= 1e-3 bar)"""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O
from oracle.unet_oracle import UNetOracle

pytestmark = pytest.mark.gpu

SMALL = dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128, seed=5)
TOL = 3e-2  # bf16 activations: relative L2 of eps / latents vs the fp32-math oracle
TOL_F32 = 1e-3  # fp32 mode: relative L2 of eps and of the final latent vs the fp64 oracle


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))


@pytest.fixture(scope="module")
def small():
    m = adx.build_unet_denoiser(**SMALL)
    s = adx.build_schedule(4, 0.01, 0.15)
    x = adx.Latent(O.random_normals(12, m.data_dim()).astype(np.float64), 4)
    return m, s, x


def test_unet_sequential_matches_oracle(small):
    m, s, x = small
    traj = adx.sequential_denoise(m, x, s, precision="bf16")
    orc = UNetOracle(SMALL)
    xv = x.values.astype(np.float32)
    lat = [xv]
    for k, t in enumerate(range(4, 0, -1)):
        eps = orc.eval_full(lat[-1], t)
        assert rel(traj.eps_used[k], eps) < TOL, (t, rel(traj.eps_used[k], eps))
        # continue the oracle from the GPU latent so errors do not compound across steps
        lat.append(O.ddim_step(traj.latents[k].values, eps, t, s.alpha_bars).astype(np.float32))
        assert rel(traj.latents[k + 1].values, lat[-1]) < TOL
    assert np.all(np.isfinite(traj.latent_matrix()))


def test_unet_async_invariants_bit_exact(small):
    m, s, x = small
    seq = adx.sequential_denoise(m, x, s, precision="bf16")
    for N in (2, 3):
        part = adx.partition_balanced(m, N)
        full, _ = adx.run_serial(adx.plan_async(4, 4, N, 1), m, part, x, s, precision="bf16")
        assert np.array_equal(full.latent_matrix(), seq.latent_matrix())  # w = T == sequential
        plan = adx.plan_async(4, 1, N, 1)
        ser, _ = adx.run_serial(plan, m, part, x, s, precision="bf16")
        par, _ = adx.run_parallel(plan, m, part, x, s, plan.D, precision="bf16")
        assert np.array_equal(ser.latent_matrix(), par.latent_matrix())  # parallel == serial
    one = adx.partition_balanced(m, 1)
    for w in (1, 3):
        t1, _ = adx.run_serial(adx.plan_async(4, w, 1, 1), m, one, x, s, precision="bf16")
        assert np.array_equal(t1.latent_matrix(), seq.latent_matrix())  # N = 1 == sequential


def test_unet_stride_async_runs(small):
    m, s, x = small
    part = adx.partition_balanced(m, 2)
    plan = adx.plan_async(4, 1, 2, 2)
    ser, _ = adx.run_serial(plan, m, part, x, s, precision="bf16")
    par, _ = adx.run_parallel(plan, m, part, x, s, plan.D, precision="bf16")
    assert np.array_equal(ser.latent_matrix(), par.latent_matrix())
    assert np.all(np.isfinite(ser.latent_matrix()))


def test_unet_rank_session_single_rank_matches_sequential(small):
    """NCCL one-process-per-GPU path (rank.cu) on the UNet family with one rank:
    N=1 plan == sequential_denoise bit-exactly (bf16 stage buffers through the
    rank program, fp32 trajectory)."""
    m, s, x = small
    T = 4
    plan = adx.plan_async(T, 1, 1, 1)
    part = adx.partition_balanced(m, 1)
    sess = adx.RankSession(m, s, plan, part, 0, adx.nccl_unique_id(), 0, "bf16")
    d = m.data_dim()
    lat, eps = np.zeros((T + 1, d)), np.zeros((T, d))
    sess.run_into(np.ascontiguousarray(x.values, np.float64), lat, eps)
    seq = adx.sequential_denoise(m, x, s, precision="bf16")
    assert np.array_equal(lat, seq.latent_matrix())
    assert sess.time(1) > 0


def test_unet_f32_mode_matches_fp64_oracle(small):
    """ADX_F32 mode: per-step eps and the whole 4-step trajectory within rel-L2 1e-3 of
    the fp64 oracle (no bf16 rounding anywhere on either side)."""
    m, s, x = small
    traj = adx.sequential_denoise(m, x, s, precision="f32")
    orc = UNetOracle(SMALL, exact=True)
    lat = x.values.astype(np.float64)
    for k, t in enumerate(range(4, 0, -1)):
        eps = orc.eval_full(lat, t)
        assert rel(traj.eps_used[k], eps) < TOL_F32, (t, rel(traj.eps_used[k], eps))
        lat = O.ddim_step(lat, eps, t, s.alpha_bars)  # the oracle's own trajectory (errors may compound)
    assert rel(traj.latents[-1].values, lat) < TOL_F32, rel(traj.latents[-1].values, lat)


def test_unet_f32_async_invariants_bit_exact(small):
    m, s, x = small
    seq = adx.sequential_denoise(m, x, s, precision="f32")
    part = adx.partition_balanced(m, 2)
    full, _ = adx.run_serial(adx.plan_async(4, 4, 2, 1), m, part, x, s, precision="f32")
    assert np.array_equal(full.latent_matrix(), seq.latent_matrix())  # w = T == sequential
    plan = adx.plan_async(4, 1, 2, 1)
    ser, _ = adx.run_serial(plan, m, part, x, s, precision="f32")
    par, _ = adx.run_parallel(plan, m, part, x, s, plan.D, precision="f32")
    assert np.array_equal(ser.latent_matrix(), par.latent_matrix())  # parallel == serial


# SDXL-shaped (BASELINE config 4) in miniature: 3 levels, transformer depths 0 / 2 / 3, mid
# depth 2, classifier-free guidance (batch-2 stages, eps_u + s (eps_c - eps_u))
SMALL_XL = dict(H=16, W=16, ch=(64, 128, 128), attn=(0, 2, 3), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128,
                mid_attn=2, cfg=True, cfg_scale=4.0, seed=7)


@pytest.fixture(scope="module")
def small_xl():
    m = adx.build_unet_denoiser(**SMALL_XL)
    s = adx.build_schedule(3, 0.01, 0.15)
    x = adx.Latent(O.random_normals(13, m.data_dim()).astype(np.float64), 3)
    return m, s, x


# guidance combines two evaluations with weights (1 - s, s): the bf16 error of the guided eps
# grows with s (stated bf16-CFG tolerance TOL * s / 2); the f32 mode keeps the 1e-3 bar
@pytest.mark.parametrize("prec,exact,tol", [("bf16", False, TOL * SMALL_XL["cfg_scale"] / 2), ("f32", True, TOL_F32)])
def test_unet_xl_cfg_matches_oracle(small_xl, prec, exact, tol):
    m, s, x = small_xl
    traj = adx.sequential_denoise(m, x, s, precision=prec)
    orc = UNetOracle(SMALL_XL, exact=exact)
    lat = x.values.astype(np.float64)
    for k, t in enumerate(range(3, 0, -1)):
        eps = orc.eval_full(lat if exact else traj.latents[k].values.astype(np.float32), t)
        assert rel(traj.eps_used[k], eps) < tol, (prec, t, rel(traj.eps_used[k], eps))
        lat = O.ddim_step(lat, np.asarray(eps, np.float64), t, s.alpha_bars)
    if exact:
        assert rel(traj.latents[-1].values, lat) < tol


def test_unet_xl_cfg_async_invariants_bit_exact(small_xl):
    m, s, x = small_xl
    seq = adx.sequential_denoise(m, x, s)
    part = adx.partition_balanced(m, 2)
    full, _ = adx.run_serial(adx.plan_async(3, 3, 2, 1), m, part, x, s)
    assert np.array_equal(full.latent_matrix(), seq.latent_matrix())
    plan = adx.plan_async(3, 1, 2, 1)
    ser, _ = adx.run_serial(plan, m, part, x, s)
    par, _ = adx.run_parallel(plan, m, part, x, s, plan.D)
    assert np.array_equal(ser.latent_matrix(), par.latent_matrix())


# AnimateDiff-shaped (BASELINE config 5) in miniature: the latent holds every frame, a
# temporal-attention motion module follows every resnet; frames 3 exercises a partly
# filled frame capacity of the temporal kernel, 16 the C5 frame count
def video_spec(frames):
    return dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128,
                frames=frames, motion=True, seed=9)


def small_video(frames):
    m = adx.build_unet_denoiser(**video_spec(frames))
    s = adx.build_schedule(3, 0.01, 0.15)
    x = adx.Latent(O.random_normals(14, m.data_dim()).astype(np.float64), 3)
    return m, s, x


@pytest.mark.parametrize("frames", [3, 16])
@pytest.mark.parametrize("prec,exact,tol", [("bf16", False, TOL), ("f32", True, TOL_F32)])
def test_unet_video_motion_matches_oracle(frames, prec, exact, tol):
    m, s, x = small_video(frames)
    assert m.data_dim() == frames * 16 * 16 * 4
    traj = adx.sequential_denoise(m, x, s, precision=prec)
    orc = UNetOracle(video_spec(frames), exact=exact)
    lat = x.values.astype(np.float64)
    for k, t in enumerate(range(3, 0, -1)):
        eps = orc.eval_full(lat if exact else traj.latents[k].values.astype(np.float32), t)
        assert rel(traj.eps_used[k], eps) < tol, (prec, frames, t, rel(traj.eps_used[k], eps))
        lat = O.ddim_step(lat, np.asarray(eps, np.float64), t, s.alpha_bars)
    if exact:
        assert rel(traj.latents[-1].values, lat) < tol


def test_unet_video_frames_are_mixed():
    """the motion modules couple the frames: perturbing frame 0 of the input latent changes
    every frame's eps (without them each frame would be denoised independently)"""
    m, s, x = small_video(3)
    e0 = adx.sequential_denoise(m, x, s).eps_used[0].reshape(3, -1)
    v = x.values.copy().reshape(3, -1)
    v[0] += 0.5
    e1 = adx.sequential_denoise(m, adx.Latent(v.reshape(-1), 3), s).eps_used[0].reshape(3, -1)
    for f in range(3):
        assert rel(e1[f], e0[f]) > 1e-4, f


def test_unet_video_async_invariants_bit_exact():
    m, s, x = small_video(4)
    seq = adx.sequential_denoise(m, x, s)
    part = adx.partition_balanced(m, 2)
    full, _ = adx.run_serial(adx.plan_async(3, 3, 2, 1), m, part, x, s)
    assert np.array_equal(full.latent_matrix(), seq.latent_matrix())
    plan = adx.plan_async(3, 1, 2, 1)
    ser, _ = adx.run_serial(plan, m, part, x, s)
    par, _ = adx.run_parallel(plan, m, part, x, s, plan.D)
    assert np.array_equal(ser.latent_matrix(), par.latent_matrix())


@pytest.mark.parametrize("family", ["video", "xl_cfg"])
def test_unet_batched_families_rank_session_matches_sequential(family):
    """the one-process-per-GPU program (rank.cu) with one rank on the batched families
    (16-frame video stages, CFG batch-2 stages): bit-exact with sequential_denoise"""
    if family == "video":
        m, s, x = small_video(16)
    else:
        m = adx.build_unet_denoiser(**SMALL_XL)
        s = adx.build_schedule(3, 0.01, 0.15)
        x = adx.Latent(O.random_normals(13, m.data_dim()).astype(np.float64), 3)
    T = 3
    plan = adx.plan_async(T, 1, 1, 1)
    part = adx.partition_balanced(m, 1)
    sess = adx.RankSession(m, s, plan, part, 0, adx.nccl_unique_id(), 0, "bf16")
    d = m.data_dim()
    lat, eps = np.zeros((T + 1, d)), np.zeros((T, d))
    sess.run_into(np.ascontiguousarray(x.values, np.float64), lat, eps)
    seq = adx.sequential_denoise(m, x, s, precision="bf16")
    assert np.array_equal(lat, seq.latent_matrix())


@pytest.mark.parametrize("prec,tol", [("bf16", TOL), ("f32", TOL_F32)])
@pytest.mark.parametrize("spec", [SMALL, SMALL_XL, dict(video_spec(3))], ids=["sd", "xl_cfg", "video"])
def test_every_stage_through_eval_segment_matches_oracle(spec, prec, tol):
    """every stage of the miniatures on its own one-stage segment (eval_segment with a host
    HiddenBundle in and out: the bundle wire format in both precisions) vs the oracle stage
    on the same inputs"""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_unet_full import stage_parity
    from oracle.unet_model import build_unet_model
    L = build_unet_model(**spec).L
    for st in range(1, L + 1):
        e, info, _ = stage_parity(repr(spec), spec, st, prec)
        assert e < tol, (st, info, e)
