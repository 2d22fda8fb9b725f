"""The UNet family's model builder (product: csrc/unet.cpp via adx_unet_stage_info /
adx_unet_stage_params / adx_unet_context, host code, no GPU needed) against the
oracle's independent restatement (oracle/unet_model.py): same stage list, skip
links, widths, MAC costs, and every parameter and context value bit-for-bit.  This
is what makes the UNet parity tests two-sided: the oracle never reads the
product's model."""
import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle.unet_model import build_unet_model, contexts, stage_params

MINIS = {
    "sd": dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128, seed=5),
    "xl_cfg": dict(H=16, W=16, ch=(64, 128, 128), attn=(0, 2, 3), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128,
                   mid_attn=2, cfg=True, cfg_scale=4.0, seed=7),
    "video": dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64, temb_dim=128, frames=3,
                  motion=True, seed=9),
}
FULL = {
    "c2": dict(H=96, W=96, seed=0),
    "c4": dict(H=128, W=128, ch=(320, 640, 1280), attn=(0, 2, 10), mid_attn=10, ctx_dim=2048, cfg=True,
               cfg_scale=5.0, seed=0),
    "c5": dict(H=64, W=64, ctx_dim=768, frames=16, motion=True, seed=0),
}


def same_topology(spec):
    m = adx.build_unet_denoiser(**spec)
    om = build_unet_model(**spec)
    assert om.L == m.num_stages()
    assert om.links == m.skip_links
    assert om.widths == m.widths
    assert om.costs() == [st.cost_macs for st in m.stages]
    for s in range(1, om.L + 1):
        assert om.info(s) == adx.unet_stage_info(m, s), s
    return m, om


def same_params(m, om, stage):
    a, b = adx.unet_stage_params(m, stage), stage_params(om, stage)
    assert list(a) == list(b), stage
    for k in a:
        assert a[k].shape == b[k].shape and a[k].tobytes() == b[k].tobytes(), (stage, k)


@pytest.mark.parametrize("name", sorted(MINIS))
def test_miniature_models_bit_identical(name):
    m, om = same_topology(MINIS[name])
    for s in range(0, om.L + 1):
        same_params(m, om, s)
    assert adx.unet_context(m).tobytes() == contexts(om.spec).tobytes()


@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size_topology_and_sampled_params_bit_identical(name):
    """c2 / c4 / c5 at full size: the whole topology, and the parameters of the time-embedding
    MLP, conv_in, the first down conv, the first decoder resnet and the out stage"""
    m, om = same_topology(FULL[name])
    kinds = [om.info(s)["kind"] for s in range(1, om.L + 1)]
    sel = {0, 1, om.L, kinds.index("down") + 1,
           next(s for s in range(1, om.L + 1) if om.info(s)["cskip"] > 0)}
    for s in sorted(sel):
        same_params(m, om, s)
    assert adx.unet_context(m).tobytes() == contexts(om.spec).tobytes()


def test_c2_parameter_count():
    """SD-2.1-shaped UNet: ~0.87 G parameters in this stage list (the attention K/V context
    projections included)"""
    om = build_unet_model(**FULL["c2"])
    n = sum(v.size for s in range(0, om.L + 1) for v in stage_params(om, s).values())
    assert 0.8e9 < n < 0.95e9, n
