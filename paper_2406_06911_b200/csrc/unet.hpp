// unet.hpp -- UNet-shaped denoiser family behind the reference's stage
// contract: a stage is a UNet block, the reference's
// mirror skip links are channel-concat skips, the per-stage time projection is
// a per-channel add of the timestep embedding (precomputed per t, like the MLP
// family's c_t table).  Activations are bf16 NHWC; the latent / eps are fp32
// H x W x c_lat (HWC) vectors so the sampler, plan and exchange are unchanged.
#pragma once

#include "host.hpp"

#include <memory>
#include <vector>

namespace adx {

struct UNetSpec {
    int H = 96, W = 96;                       // latent spatial size
    int c_lat = 4;                            // latent channels
    std::vector<int> ch = {320, 640, 1280, 1280};
    int n_res = 2;                            // resnets per down level (up levels use n_res+1)
    std::vector<int> attn = {1, 1, 1, 0};     // SpatialTransformer depth after the level's resnets
                                              // (0: none; SD-2.1: 1, SDXL: 0 / 2 / 10 blocks)
    int head_dim = 64;
    int ctx_len = 77, ctx_dim = 1024;         // cross-attention context (synthetic, seeded)
    int temb_dim = 1280;
    int groups = 32;
    int mid_attn = 1;                         // mid-block transformer depth
    uint64_t seed = 0;
    // classifier-free guidance: the stages run a batch of 2 (image 0 with the unconditional
    // context, image 1 with the conditional one) and the out stage returns
    // eps_u + cfg_scale * (eps_c - eps_u); the latent / eps stay one image
    int cfg = 0;
    float cfg_scale = 5.0f;
    // video (AnimateDiff-shaped): `frames` latents per sample (the latent / eps are
    // frames x H x W x c_lat) and, with motion = 1, a temporal-attention motion module after
    // every resnet (attention across the frames of each pixel); CFG and frames exclusive
    int frames = 1;
    int motion = 0;
    int batch() const { return cfg ? 2 : frames; }     // images every stage processes
    int contexts() const { return cfg ? 2 : 1; }        // text contexts (video frames share one)
};

enum UKind { kConvIn = 0, kRes = 1, kDown = 2, kUp = 3, kOut = 4, kMidRes = 5 };

struct UStage {
    int kind = 0;
    int cin = 0;      // main input channels (previous stage output / padded latent)
    int cskip = 0;    // concatenated skip channels (0: none)
    int cout = 0;
    int H = 0, W = 0; // input spatial size (DOWN halves it, UP doubles it)
    int attn = 0;     // depth of the following SpatialTransformer (RES / MidRes; 0: none)
    int motion = 0;   // followed by a temporal motion module (RES / MidRes, video models)
    long long macs = 0;
    int Ho() const { return kind == kDown ? H / 2 : kind == kUp ? 2 * H : H; }
    int Wo() const { return kind == kDown ? W / 2 : kind == kUp ? 2 * W : W; }
};

struct UNetDesc {
    UNetSpec spec;
    std::vector<UStage> st;  // index 0 = stage 1
    std::vector<float> ctx;  // batch x ctx_len x ctx_dim contexts (CFG: [uncond, cond])
};

// Model (topology + costs, no MLP weights) for the engine / partitioner / plan
Model build_unet_model(const UNetSpec& spec);

// Deterministic fp32 parameters of one stage, generated from (seed, stage):
// names + flat arrays in a fixed order (the numpy oracle reads the same list).
struct UParam {
    std::string name;
    std::vector<int> shape;
    std::vector<float> data;
};
std::vector<UParam> unet_stage_params(const UNetDesc& d, int stage);
// timestep-embedding MLP (shared, stage 0) and the per-RES time projection
std::vector<float> unet_temb(const UNetDesc& d, int t);                        // temb_dim
std::vector<float> unet_chan_add(const std::vector<UParam>& stage_params, const std::vector<float>& temb);  // cout

}  // namespace adx
