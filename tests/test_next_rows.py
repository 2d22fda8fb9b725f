"""§8(f) next rows: checkpoint and plan JSON formats (serialize.cpp), cost model
(costsim.cpp, proj/tests/test_costsim.cpp), exchange bytes.  CPU only except
the last two GPU tests."""
import json
import os

import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O


def reference_checkpoint_json(m):
    """serialize.cpp:226-250 restated: nlohmann dump(2) == sorted keys, indent 2."""
    L = m.num_stages()
    tensors, off = [], 0
    shapes = [("time_embed.proj", m.time_embed_dim, m.time_embed_dim)]
    for i, st in enumerate(m.stages, 1):
        h, inn, out, E = st.hidden_width(), st.in_width(), st.out_width(), m.time_embed_dim
        shapes += [(f"stage{i}.w1", h, inn), (f"stage{i}.b1", h, 1), (f"stage{i}.time_in", h, E),
                   (f"stage{i}.w2", out, h), (f"stage{i}.b2", out, 1)]
    for name, r, c in shapes:
        tensors.append({"name": name, "rows": r, "cols": c, "offset_doubles": off})
        off += r * c
    meta = {"format": "asyncdiff-checkpoint-v1", "L": L, "widths": m.widths, "time_embed_dim": m.time_embed_dim,
            "skip_links": [list(l) for l in m.skip_links], "tensors": tensors, "total_doubles": off,
            "endianness": "little"}
    return json.dumps(meta, indent=2, sort_keys=True) + "\n"


def reference_blob(m):
    parts = [m.proj]
    for st in m.stages:
        parts += [st.w1, st.b1, st.time_in, st.w2, st.b2]
    return b"".join(np.ascontiguousarray(p, "<f8").tobytes() for p in parts)


def test_checkpoint_bytes_match_reference_format(tmp_path):
    m = adx.build_toy_denoiser(6, [2, 8, 6, 10, 6, 8, 2], "unet-mirror", 17)
    base = str(tmp_path / "model")
    adx.save_checkpoint(base, m)
    assert open(base + ".json").read() == reference_checkpoint_json(m)
    assert open(base + ".bin", "rb").read() == reference_blob(m)


def test_checkpoint_roundtrip_and_foreign_writer(tmp_path):
    m = adx.build_toy_denoiser(5, [4, 8, 8, 8, 8, 4], "unet-mirror", 3)
    m.stages[1].b1[:] = np.linspace(-1, 1, 8)  # non-zero biases survive the trip
    base = str(tmp_path / "a")
    adx.save_checkpoint(base, m)
    m2 = adx.load_checkpoint(base)
    assert m2.widths == m.widths and m2.skip_links == m.skip_links
    for a, b in zip(m.stages, m2.stages):
        for name in ("w1", "b1", "time_in", "w2", "b2"):
            assert np.array_equal(getattr(a, name), getattr(b, name))
    # a checkpoint written by an independent restatement of the writer loads too
    base2 = str(tmp_path / "b")
    open(base2 + ".json", "w").write(reference_checkpoint_json(m))
    open(base2 + ".bin", "wb").write(reference_blob(m))
    m3 = adx.load_checkpoint(base2)
    assert np.array_equal(m3.stages[1].b1, m.stages[1].b1)
    open(base2 + ".bin", "wb").write(reference_blob(m)[:-8])
    with pytest.raises(adx.AdxRuntimeError, match="truncated"):
        adx.load_checkpoint(base2)
    with pytest.raises(adx.AdxRuntimeError, match="cannot read"):
        adx.load_checkpoint(str(tmp_path / "missing"))


def reference_plan_json(plan):
    """serialize.cpp:109-133 restated."""
    rounds = []
    for r in plan.rounds:
        evals = []
        for e in r.evals:
            inp = ({"kind": "current-latent"} if e.input.kind == "latent" else
                   {"kind": "cached", "segment": e.input.producer_segment, "round": e.input.producer_round})
            je = {"segment": e.segment, "device": e.device, "embed_t": e.embed_t, "input": inp}
            if e.emits_eps_for is not None:
                je["emits_eps_for"] = e.emits_eps_for
            evals.append(je)
        rounds.append({"index": r.index, "evals": evals, "sampler_steps": r.sampler_steps, "broadcast": r.broadcast})
    return json.dumps({"T": plan.T, "w": plan.w, "N": plan.N, "S": plan.S, "D": plan.D,
                       "time_shift": plan.time_shift, "warmup_steps": plan.warmup_steps, "rounds": rounds},
                      indent=2, sort_keys=True)


@pytest.mark.parametrize("args", [(20, 1, 2, 1, False), (10, 2, 3, 2, True), (5, 5, 1, 1, False)])
def test_plan_json_matches_reference_and_roundtrips(args):
    plan = adx.plan_async(*args)
    text = adx.plan_to_json(plan)
    assert text == reference_plan_json(plan)
    assert adx.plan_from_json(text) == plan


def test_cost_model_worked_example():  # test_costsim.cpp:29-42 (G8)
    plan = adx.plan_async(50, 1, 4, 1)
    rep = adx.predict_async(plan, adx.CostModel([0.010] * 4, 0.001, 0.0))
    assert rep.sequential_total_s == pytest.approx(2.0, rel=1e-12)
    assert rep.async_total_s == pytest.approx(0.040 + 0.49 + 0.048, rel=1e-12)
    assert rep.speedup == pytest.approx(2.0 / 0.578, rel=1e-9)
    assert rep.approx_total_s == pytest.approx(0.040 + 49 * 0.011, rel=1e-12)


def test_cost_model_properties():  # test_costsim.cpp:14-27, 44-70
    for N in (2, 3, 4):
        rep = adx.predict_async(adx.plan_async(1000, 1, N, 1), adx.CostModel([0.01] * N))
        assert rep.speedup == pytest.approx(N, rel=0.01)
    cm = adx.CostModel([0.010] * 3, 0.002)
    r1 = adx.predict_async(adx.plan_async(50, 1, 3, 1), cm)
    r2 = adx.predict_async(adx.plan_async(50, 1, 3, 2), cm)
    assert r2.comm_total_s < 0.55 * r1.comm_total_s + 0.002 and r2.async_total_s < r1.async_total_s
    for w in (1, 5, 20):
        rep = adx.predict_async(adx.plan_async(20, w, 1, 1), adx.CostModel([0.013]))
        assert rep.async_total_s == pytest.approx(adx.predict_sequential(20, adx.CostModel([0.013])), rel=1e-12)
    with pytest.raises(adx.InvalidArgument):
        adx.predict_async(adx.plan_async(20, 1, 3, 1), adx.CostModel([0.01] * 2))


def test_calibrate_and_compare():  # costsim.cpp:52-79
    plan = adx.plan_async(20, 1, 2, 1)
    stats = adx.RunStats(round_comm_s=[0.001] * 19, broadcast_count=19, total_wall_s=0.01 * 2 + 19 * 0.011)
    c = adx.calibrate_and_compare(plan, [0.01, 0.01], stats)
    assert c.calibrated_comm_cost_s == pytest.approx(0.001)
    assert c.predicted_total_s == pytest.approx(0.02 + 19 * 0.01 + 18 * 0.001)
    assert c.rel_error_total < 0.01


def test_round_exchange_bytes_and_bytes_aware_model():
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    plan, part = adx.plan_async(20, 1, 2, 1), adx.partition_balanced(m, 2)
    b = adx.round_exchange_bytes(plan, part, m, "f64")
    # stages 1, 2, 3 (skips (1,6), (2,5) and the boundary; (3,4) is the boundary itself) + eps
    assert b[:-1] == [(3 * 8 + 2) * 8] * 18 and b[-1] == 2 * 8
    cm = adx.CostModel([1e-4, 1e-4], comm_latency_s=5e-6, link_gbs=770.0)
    rep = adx.predict_async(plan, cm, b)
    assert rep.round_comm_s[0] == pytest.approx(5e-6 + 208 / 770e9)


@pytest.mark.gpu
def test_similarity_profile_on_gpu():  # metrics.cpp:73-101
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    s = adx.build_schedule(20, 0.01, 0.15)
    seq = adx.sequential_denoise(m, adx.Latent(O.random_normals(12, 2), 20), s, precision="f64")
    prof = adx.similarity_profile(m, adx.partition_balanced(m, 3), seq, s, precision="f64")
    assert len(prof.cosine) == 2 and len(prof.pair_t) == 19
    # against the oracle restatement of metrics.cpp:73-101 on the oracle's own model
    from oracle.async_exec import AsyncOracle, mlp_stage_fn, similarity_profile
    om = O.Model.build_toy(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 8)
    ss, _ = O.partition_balanced(om.costs(), 3)
    pt, cos, rl = similarity_profile(AsyncOracle(om.L, om.links, mlp_stage_fn(om)), ss,
                                     [x.values for x in seq.latents], [x.timestep for x in seq.latents])
    assert prof.pair_t == pt
    assert np.allclose(prof.cosine, cos, rtol=0, atol=1e-12) and np.allclose(prof.rel_l2, rl, rtol=1e-9, atol=1e-14)
    assert prof.median_cosine() > 0.9


@pytest.mark.gpu
def test_similarity_profile_unet_matches_oracle():  # metrics.cpp:73-101 on the UNet family (bf16)
    from oracle.async_exec import AsyncOracle, similarity_profile, unet_stage_fn
    from oracle.unet_model import build_unet_model
    from oracle.unet_oracle import UNetOracle
    spec = dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128, seed=5)
    m = adx.build_unet_denoiser(**spec)
    s = adx.build_schedule(4, 0.01, 0.15)
    seq = adx.sequential_denoise(m, adx.Latent(O.random_normals(12, m.data_dim()), 4), s, precision="f32")
    prof = adx.similarity_profile(m, adx.partition_balanced(m, 3), seq, s, precision="f32")
    om = build_unet_model(**spec)
    ss, _ = O.partition_balanced(om.costs(), 3)
    orc = UNetOracle(om, exact=True)
    pt, cos, rl = similarity_profile(AsyncOracle(om.L, om.links, unet_stage_fn(orc)), ss,
                                     [x.values for x in seq.latents], [x.timestep for x in seq.latents])
    assert prof.pair_t == pt
    assert np.allclose(prof.cosine, cos, rtol=0, atol=1e-5)
    assert np.allclose(prof.rel_l2, rl, rtol=1e-2, atol=1e-5)


@pytest.mark.gpu
def test_cmd_bench_style_calibration_on_gpu():  # experiment.cpp:391-455 with GPU sleeps
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    s = adx.build_schedule(12, 0.01, 0.15)
    plan, part = adx.plan_async(12, 1, 2, 1), adx.partition_balanced(m, 2)
    delays = [0.004, 0.004]
    _, stats = adx.run_parallel(plan, adx.inject_delay(m, delays), part, adx.Latent(O.random_normals(12, 2), 12), s, 2)
    c = adx.calibrate_and_compare(plan, delays, stats)
    assert c.rel_error_total < 0.25


def test_round_exchange_bytes_unet_stage_element_sizes():
    """UNet stage outputs travel as bf16 in the bf16 mode and fp32 in the f32 mode;
    eps (the last segment's output) at the fp32 trajectory size in both (host-only)."""
    m = adx.build_unet_denoiser(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64,
                                temb_dim=128, seed=5)
    part = adx.partition_balanced(m, 2)
    plan = adx.plan_async(4, 1, 2, 1)
    b16 = adx.round_exchange_bytes(plan, part, m, "bf16")
    b32 = adx.round_exchange_bytes(plan, part, m, "f32")
    eps = m.data_dim() * 4
    assert len(b16) == len(plan.rounds) and all(b > eps for b in b16[:-1])
    for x, y in zip(b16, b32):
        assert y - eps == 2 * (x - eps)  # stage payload doubles, the eps send does not
    assert adx.round_exchange_bytes(plan, part, m) == b16  # the UNet default precision is bf16


def test_unet_sdxl_shape_and_cfg_build():
    """SDXL-shaped builder (host only): transformer depth per level, CFG doubles the stage
    widths (batch 2) and MACs but not the latent / eps, two contexts, per-block parameters."""
    kw = dict(H=16, W=16, ch=(64, 128, 128), attn=(0, 2, 3), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128,
              mid_attn=2, seed=7)
    a = adx.build_unet_denoiser(**kw)
    b = adx.build_unet_denoiser(cfg=True, **kw)
    assert a.num_stages() == b.num_stages()
    assert a.data_dim() == b.data_dim() == 16 * 16 * 4
    assert b.total_macs() == 2 * a.total_macs()
    assert adx.unet_context(a).shape == (1, 8, 64) and adx.unet_context(b).shape == (2, 8, 64)
    assert np.array_equal(adx.unet_context(a)[0], adx.unet_context(b)[1])  # the conditional context
    depths = {adx.unet_stage_info(a, i)["attn"] for i in range(1, a.num_stages() + 1)}
    assert depths == {0, 2, 3}
    st = next(i for i in range(1, a.num_stages() + 1) if adx.unet_stage_info(a, i)["attn"] == 3)
    names = set(adx.unet_stage_params(a, st))
    assert {"tf.qkv.w", "tf.b1.qkv.w", "tf.b2.ff2.w"} <= names and "tf.b3.qkv.w" not in names
    with pytest.raises(adx.InvalidArgument):
        adx.build_unet_denoiser(**dict(kw, ctx_dim=100))


def test_unet_video_motion_build():
    """AnimateDiff-shaped builder (host only): the latent / eps and every stage carry all
    frames, motion modules add parameters to every resnet stage (not to conv / down / up /
    out), frames share one context, invalid combinations are rejected."""
    kw = dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128, seed=9)
    a = adx.build_unet_denoiser(**kw)
    v = adx.build_unet_denoiser(frames=4, motion=True, **kw)
    assert v.num_stages() == a.num_stages() and v.skip_links == a.skip_links
    assert v.data_dim() == 4 * a.data_dim()
    assert adx.unet_context(v).shape == (1, 8, 64)
    assert v.total_macs() > 4 * a.total_macs()  # + the motion modules
    for i in range(1, v.num_stages() + 1):
        kind = adx.unet_stage_info(v, i)["kind"]
        names = set(adx.unet_stage_params(v, i))
        has = {"mm.gn.gamma", "mm.a1.qkv.w", "mm.a2.o.w", "mm.ff1.w", "mm.proj_out.w"} <= names
        assert has == (kind in ("res", "mid_res")), (i, kind)
        assert names >= set(adx.unet_stage_params(a, i))  # the spatial parameters are unchanged
    for i in range(1, a.num_stages() + 1):
        for k, w in adx.unet_stage_params(a, i).items():
            assert np.array_equal(w, adx.unet_stage_params(v, i)[k])
    with pytest.raises(adx.InvalidArgument):
        adx.build_unet_denoiser(frames=4, cfg=True, **kw)
    with pytest.raises(adx.InvalidArgument):
        adx.build_unet_denoiser(frames=1, motion=True, **kw)
    with pytest.raises(adx.InvalidArgument):
        adx.build_unet_denoiser(frames=33, motion=True, **kw)


@pytest.mark.gpu
def test_warmup_sweep_on_gpu():  # experiment.cpp:312-389 (cmd_sweep), scored against the sequential run
    m = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    s = adx.build_schedule(20, 0.01, 0.15)
    x = adx.Latent(O.random_normals(12, 2), 20)
    rows = adx.warmup_sweep(m, x, s, [(2, 20, 1), (2, 1, 1), (3, 3, 1), (3, 1, 2)], precision="f64")
    assert [r["config"] for r in rows] == ["N2_w20_S1", "N2_w1_S1", "N3_w3_S1", "N3_w1_S2"]
    assert rows[0]["final_mse"] == 0.0 and rows[0]["final_rel_l2"] == 0.0  # w = T: sequential
    # the (N=2, w=1) row is the reference's golden G1 (test_executor.cpp:66-81): its final MSE
    # is compare_trajectories' mean over d=2 -- the golden's |delta|^2 / 2
    gold = 0.0011860077151787584
    assert abs(rows[1]["final_mse"] - gold) <= 1e-9 * gold, rows[1]["final_mse"]
    for r in rows[1:]:
        assert np.isfinite(r["final_mse"]) and r["final_rel_l2"] > 0.0
    plan = adx.plan_async(20, 1, 3, 2)
    assert rows[3]["device_count"] == plan.D == 4
    assert rows[3]["per_device_macs"] == adx.plan_counts(plan, adx.partition_balanced(m, 3)).max_device_macs
