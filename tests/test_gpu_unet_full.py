"""UNet parity at the sizes the bench times (VERDICT r1 "parity at the
configurations the bench times"): the GPU path against the builder's numpy
oracle over the INDEPENDENT model restatement (oracle/unet_model.py: its own
topology and MT19937-64 parameter streams -- no product call on the oracle
side; tests/test_unet_model.py pins the two models bit-for-bit).

  c2 (SD-2.1-shaped, 96x96x4, the bench default), full model:
    f32 mode:  eps of the first two steps of the T=50 trajectory and the latent
               after them within rel-L2 1e-3 of the fp64 oracle's own trajectory
               (the north_star tolerance);
    bf16 mode: eps at the first two steps within 3e-2 of the bf16-rounding
               oracle (fed the GPU latent); the whole 50-step bf16 trajectory
               within TOL_TRAJ_BF16 of the 50-step f32-mode trajectory;
    async run: N=2 w=9 (BASELINE configs[1]) run_parallel == run_serial
               bit-exactly and the broadcast count == plan_counts (run_one's
               invariants, experiment.cpp:263-274).
  c4 (SDXL-shaped + CFG) and c5 (16-frame AnimateDiff-shaped) full models: one
    stage of every kind evaluated through eval_segment on a one-stage segment,
    against the oracle's stage on the same (bf16-representable) inputs.

Each oracle c2 evaluation takes ~40-50 s of host CPU, so this module runs for a
few minutes."""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O
from oracle.unet_model import build_unet_model
from oracle.unet_oracle import UNetOracle, bf

pytestmark = pytest.mark.gpu

C2 = dict(H=96, W=96, seed=0)
C4 = dict(H=128, W=128, ch=(320, 640, 1280), attn=(0, 2, 10), mid_attn=10, ctx_dim=2048, cfg=True, cfg_scale=5.0,
          seed=0)
C5 = dict(H=64, W=64, ctx_dim=768, frames=16, motion=True, seed=0)
TOL_BF16 = 3e-2      # bf16 activations, per evaluation / per stage
TOL_F32 = 1e-3       # f32 mode vs fp64 oracle (north_star)
TOL_TRAJ_BF16 = 5e-2  # bf16 50-step final latent vs the f32-mode 50-step final latent


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / (np.linalg.norm(b) + 1e-30))


@pytest.fixture(scope="module")
def c2():
    m = adx.build_unet_denoiser(**C2)
    s = adx.build_schedule(50, 0.01, 0.19)
    x = adx.Latent(O.random_normals(12, m.data_dim()), 50)
    return m, s, x, build_unet_model(**C2)


@pytest.fixture(scope="module")
def c2_f32_traj(c2):
    m, s, x, _ = c2
    return adx.sequential_denoise(m, x, s, precision="f32")


def test_c2_f32_trajectory_matches_fp64_oracle(c2, c2_f32_traj):
    m, s, x, om = c2
    traj = c2_f32_traj
    orc = UNetOracle(om, exact=True)
    lat = x.values.astype(np.float64)
    errs = []
    for k, t in enumerate((50, 49)):
        eps = orc.eval_full(lat, t)
        errs.append(rel(traj.eps_used[k], eps))
        assert errs[-1] < TOL_F32, (t, errs)
        lat = O.ddim_step(lat, eps, t, s.alpha_bars)  # the oracle's own trajectory
    e_lat = rel(traj.latents[2].values, lat)
    print(f"c2 f32: eps rel-L2 {errs}, latent after 2 steps {e_lat:.2e}")
    assert e_lat < TOL_F32


def test_c2_bf16_eval_matches_oracle(c2):
    m, s, x, om = c2
    traj = adx.sequential_denoise(m, x, s, precision="bf16")
    orc = UNetOracle(om)
    errs = []
    for k, t in enumerate((50, 49)):
        eps = orc.eval_full(traj.latents[k].values.astype(np.float32), t)
        errs.append(rel(traj.eps_used[k], eps))
    print(f"c2 bf16: eps rel-L2 {errs}")
    assert max(errs) < TOL_BF16, errs


def test_c2_bf16_trajectory_within_stated_tolerance_of_f32_mode(c2, c2_f32_traj):
    m, s, x, _ = c2
    b = adx.sequential_denoise(m, x, s, precision="bf16")
    e = rel(b.latents[-1].values, c2_f32_traj.latents[-1].values)
    print(f"c2 50-step final latent, bf16 vs f32 mode: rel-L2 {e:.3e}")
    assert e < TOL_TRAJ_BF16


def test_c2_async_run_one_invariants(c2):
    """experiment.cpp:263-274 at BASELINE configs[1] (N=2, S=1, w=9, T=50)"""
    m, s, x, _ = c2
    part = adx.partition_balanced(m, 2)
    plan = adx.plan_async(50, 9, 2, 1)
    ser, sst = adx.run_serial(plan, m, part, x, s)
    par, pst = adx.run_parallel(plan, m, part, x, s, plan.D)
    assert np.array_equal(ser.latent_matrix(), par.latent_matrix())
    assert pst.broadcast_count == adx.plan_counts(plan, part).broadcasts_paper_convention == len(plan.rounds)
    assert np.all(np.isfinite(par.latent_matrix()))


# ------------------------------------------------------------- per-stage, c4 / c5
def pick_stages(om):
    """one stage of every kind: conv_in, the first resnet with a transformer (or the first
    resnet), the first down, the mid resnet with a transformer, the first decoder resnet
    (skip concat), the first up, out"""
    kinds = [om.info(s)["kind"] for s in range(1, om.L + 1)]
    first = lambda pred: next(s for s in range(1, om.L + 1) if pred(s))
    sel = {1, om.L,
           first(lambda s: kinds[s - 1] == "down"),
           first(lambda s: kinds[s - 1] == "up"),
           first(lambda s: kinds[s - 1] == "mid_res"),
           first(lambda s: kinds[s - 1] == "res" and om.info(s)["cskip"] > 0)}
    attn_res = [s for s in range(1, om.L + 1) if kinds[s - 1] == "res" and om.info(s)["attn"] > 0
                and om.info(s)["cskip"] == 0]
    sel.add(attn_res[0] if attn_res else first(lambda s: kinds[s - 1] == "res"))
    return sorted(sel)


_MODELS = {}


def models(name, spec):
    """one product model (its engines -- uploaded weights -- are cached per precision) and one
    oracle model (parameters generated on first use) per config"""
    if name not in _MODELS:
        _MODELS.clear()  # free the previous config's device weights
        _MODELS[name] = (adx.build_unet_denoiser(**spec), build_unet_model(**spec))
    return _MODELS[name]


def stage_parity(name, spec, stage, prec, t=37):
    m, om = models(name, spec)
    L = om.L
    rng = np.random.default_rng(stage)
    info = om.info(stage)
    sp = om.spec
    B = sp.batch()
    lat_shape = (sp.frames, sp.H, sp.W, sp.c_lat) if sp.frames > 1 else (sp.H, sp.W, sp.c_lat)

    def act(width, C):  # bf16-representable activations, (batch, H, W, C) flat
        return bf(rng.standard_normal(width).astype(np.float32)).astype(np.float64)

    if stage == 1:
        segs = [[1], list(range(2, L + 1))]
        seg = 1
    elif stage == L:
        segs = [list(range(1, L)), [L]]
        seg = 2
    else:
        segs = [list(range(1, stage)), [stage], list(range(stage + 1, L + 1))]
        seg = 2
    part = adx.Partition.create(segs)
    skips = {(p, c): act(om.widths[p], None) for (p, c) in om.links if c == stage}
    if stage == 1:
        main = rng.standard_normal(om.widths[0])
        out = adx.eval_segment(m, part, 1, adx.Latent(main, t), skips, t, precision=prec)
    else:
        main = act(om.widths[stage - 1], None)
        b = adx.HiddenBundle(boundary=main, produced_by=1, produced_at=t)
        out = adx.eval_segment(m, part, seg, b, skips, t, precision=prec)
    y = out if stage == L else out.boundary

    orc = UNetOracle(om, exact=(prec == "f32"))
    dt = orc.dt
    cin = info["cin"]

    def shaped(v, p_stage):  # producer stage output -> oracle layout
        s_ = om.stages[p_stage - 1]
        shp = (s_.Ho, s_.Wo, s_.cout)
        v = np.asarray(v, dt)
        return v.reshape((B,) + shp) if B > 1 else v.reshape(shp)

    ins = [np.asarray(main, dt) if stage == 1 else shaped(main, stage - 1)]
    ins += [shaped(skips[(p, c)], p) for (p, c) in om.links if c == stage]
    if sp.cfg:  # two cascades per stage, guidance combine at the out stage
        ys = []
        for ci in (0, 1):
            orc.ci = ci
            ys.append(orc.stage(stage, [ins[0]] if stage == 1 else [x[ci] for x in ins], t))
        if stage == L:
            eu, ec = ys
            ref = eu + sp.cfg_scale * (ec - eu)
        else:
            ref = np.stack(ys)
    else:
        ref = orc.stage(stage, ins, t)
    ref = np.asarray(ref, np.float64).reshape(-1)
    return rel(y, ref), info, cin


@pytest.mark.parametrize("name,spec", [("c4", C4), ("c5", C5)])
def test_full_size_stage_parity_bf16(name, spec):
    _, om = models(name, spec)
    res = {}
    for st in pick_stages(om):
        e, info, _ = stage_parity(name, spec, st, "bf16")
        res[st] = (info["kind"], info["attn"], round(e, 5))
        assert e < TOL_BF16, (name, st, info, e)
    print(name, "bf16 per-stage rel-L2:", res)


@pytest.mark.parametrize("name,spec", [("c4", C4), ("c5", C5)])
def test_full_size_stage_parity_f32(name, spec):
    """the f32 mode at the c4 / c5 shapes on the two heaviest stage kinds (the mid resnet with
    its transformer, the first decoder resnet) against the fp64 oracle"""
    _, om = models(name, spec)
    kinds = [om.info(s)["kind"] for s in range(1, om.L + 1)]
    sel = [kinds.index("mid_res") + 1,
           next(s for s in range(1, om.L + 1) if kinds[s - 1] == "res" and om.info(s)["cskip"] > 0)]
    for st in sel:
        e, info, _ = stage_parity(name, spec, st, "f32")
        print(name, "f32 stage", st, info["kind"], e)
        assert e < TOL_F32, (name, st, info, e)
