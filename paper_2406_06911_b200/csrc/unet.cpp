// unet.cpp -- host side of the UNet-shaped family: stage list (SD-2.1-like
// topology), MAC costs for the FLOP-balanced partition, deterministic
// parameters and the per-t time-embedding tables (see unet.hpp).
#include "unet.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace adx {

namespace {

long long conv_macs(int H, int W, int cout, int cin) { return static_cast<long long>(H) * W * cout * 9 * cin; }

// a SpatialTransformer of `depth` blocks: proj_in / proj_out once, per block QKV, self and
// cross attention, o1 / q2 / o2, GEGLU FF (the context K / V projection is precomputed)
long long attn_macs(int L, int C, int Lc, int depth) {
    const long long l = L, c = C;
    return l * c * c * 2 + depth * (l * c * c * (3 + 1 + 1 + 1 + 8 + 4) + 2 * l * l * c + 2 * l * Lc * c);
}

}  // namespace

Model build_unet_model(const UNetSpec& sp) {
    if (sp.ch.empty() || sp.attn.size() != sp.ch.size()) throw std::invalid_argument("unet: ch / attn mismatch");
    for (int c : sp.ch)
        if (c % 64 || c % sp.groups) throw std::invalid_argument("unet: channels must be multiples of 64 and groups");
    if (sp.head_dim != 64) throw std::invalid_argument("unet: head_dim must be 64");
    if (sp.ctx_dim % 64) throw std::invalid_argument("unet: ctx_dim must be a multiple of 64");
    if (sp.frames < 1 || sp.frames > 32) throw std::invalid_argument("unet: frames must be in 1..32");
    if (sp.cfg && sp.frames > 1) throw std::invalid_argument("unet: CFG and video frames are exclusive");
    if (sp.motion && sp.frames < 2) throw std::invalid_argument("unet: motion modules need frames >= 2");
    for (int a : sp.attn)
        if (a < 0) throw std::invalid_argument("unet: transformer depth must be >= 0");
    if (sp.mid_attn < 0) throw std::invalid_argument("unet: mid transformer depth must be >= 0");
    const int levels = static_cast<int>(sp.ch.size());
    if (sp.H % (1 << (levels - 1)) || sp.W % (1 << (levels - 1)))
        throw std::invalid_argument("unet: H, W must be divisible by 2^(levels-1)");
    auto d = std::make_shared<UNetDesc>();
    d->spec = sp;
    std::vector<UStage>& st = d->st;
    std::vector<std::pair<int, int>> links;
    std::vector<std::pair<int, int>> skips;  // (stage, channels) stack
    int H = sp.H, W = sp.W, c = sp.ch[0];
    UStage s0;
    s0.kind = kConvIn;
    s0.cin = 64;
    s0.cout = sp.ch[0];
    s0.H = H;
    s0.W = W;
    st.push_back(s0);
    skips.emplace_back(1, c);
    for (int l = 0; l < levels; ++l) {
        for (int r = 0; r < sp.n_res; ++r) {
            UStage s;
            s.kind = kRes;
            s.cin = c;
            s.cout = sp.ch[l];
            s.H = H;
            s.W = W;
            s.attn = sp.attn[l];
            st.push_back(s);
            c = s.cout;
            skips.emplace_back(static_cast<int>(st.size()), c);
        }
        if (l + 1 < levels) {
            UStage s;
            s.kind = kDown;
            s.cin = s.cout = c;
            s.H = H;
            s.W = W;
            st.push_back(s);
            H /= 2;
            W /= 2;
            skips.emplace_back(static_cast<int>(st.size()), c);
        }
    }
    for (int m = 0; m < 2; ++m) {
        UStage s;
        s.kind = kMidRes;
        s.cin = s.cout = c;
        s.H = H;
        s.W = W;
        s.attn = m == 0 ? sp.mid_attn : 0;
        st.push_back(s);
    }
    for (int l = levels - 1; l >= 0; --l) {
        for (int r = 0; r < sp.n_res + 1; ++r) {
            const auto sk = skips.back();
            skips.pop_back();
            UStage s;
            s.kind = kRes;
            s.cin = c;
            s.cskip = sk.second;
            s.cout = sp.ch[l];
            s.H = H;
            s.W = W;
            s.attn = sp.attn[l];
            st.push_back(s);
            links.emplace_back(sk.first, static_cast<int>(st.size()));
            c = s.cout;
        }
        if (l > 0) {
            UStage s;
            s.kind = kUp;
            s.cin = s.cout = c;
            s.H = H;
            s.W = W;
            st.push_back(s);
            H *= 2;
            W *= 2;
        }
    }
    UStage so;
    so.kind = kOut;
    so.cin = c;
    so.cout = sp.c_lat;
    so.H = H;
    so.W = W;
    st.push_back(so);
    if (!skips.empty()) throw std::logic_error("unet: unbalanced skip stack");

    for (UStage& s : st)
        if (s.kind == kRes || s.kind == kMidRes) s.motion = sp.motion;
    // costs (implemented MACs: stride-2 convs run at full resolution)
    for (UStage& s : st) {
        const int cin = s.cin + s.cskip;
        switch (s.kind) {
            case kConvIn: s.macs = conv_macs(s.H, s.W, s.cout, 64); break;
            case kDown: s.macs = conv_macs(s.H, s.W, s.cout, cin); break;
            case kUp: s.macs = conv_macs(2 * s.H, 2 * s.W, s.cout, cin); break;
            case kOut: s.macs = conv_macs(s.H, s.W, 32, cin); break;
            default:
                s.macs = conv_macs(s.H, s.W, s.cout, cin) + conv_macs(s.H, s.W, s.cout, s.cout) +
                         (cin != s.cout ? static_cast<long long>(s.H) * s.W * s.cout * cin : 0);
                if (s.attn) s.macs += attn_macs(s.H * s.W, s.cout, sp.ctx_len, s.attn);
                if (s.motion)  // proj_in / out, 2 x (QKV + out proj + F x F attention), GEGLU FF
                    s.macs += static_cast<long long>(s.H) * s.W * s.cout *
                              (2LL * s.cout + 2 * (4LL * s.cout + 2LL * sp.frames) + 12LL * s.cout);
        }
        s.macs *= sp.batch();
    }
    // synthetic cross-attention contexts ~ N(0, 1): the conditional one (seed 1000003) and,
    // with CFG, an unconditional one (seed 1000004) placed first (image 0)
    const size_t csz = static_cast<size_t>(sp.ctx_len) * sp.ctx_dim;
    d->ctx.resize(csz * sp.contexts());
    {
        Rng rng(mix_seed(sp.seed, 1000003));
        for (size_t i = 0; i < csz; ++i) d->ctx[(sp.contexts() - 1) * csz + i] = static_cast<float>(rng.normal());
    }
    if (sp.cfg) {
        Rng rng(mix_seed(sp.seed, 1000004));
        for (size_t i = 0; i < csz; ++i) d->ctx[i] = static_cast<float>(rng.normal());
    }

    Model m;
    m.kind = 1;
    m.unet = d;
    m.L = static_cast<int>(st.size());
    m.E = 8;  // unused by the UNet stages; keeps the shared etab path trivial
    m.proj.assign(64, 0.0);
    const int lat = sp.frames * sp.H * sp.W * sp.c_lat;  // latent / eps: every frame
    m.widths.push_back(lat);
    for (size_t i = 0; i < st.size(); ++i) {
        const UStage& s = st[i];
        m.widths.push_back(i + 1 == st.size() ? lat : sp.batch() * s.cout * s.Ho() * s.Wo());
    }
    m.links = links;
    std::sort(m.links.begin(), m.links.end());
    m.stages.resize(st.size());
    for (size_t i = 0; i < st.size(); ++i) {
        Stage& g = m.stages[i];
        g.index = static_cast<int>(i) + 1;
        int in = i == 0 ? m.widths[0] + m.E : m.widths[i];
        for (auto& l : m.links_into(static_cast<int>(i) + 1)) in += m.widths[l.first];
        g.in = in;
        g.hidden = 0;
        g.out = m.widths[i + 1];
        g.cost_macs = st[i].macs;
    }
    return m;
}

namespace {

struct Gen {
    Rng rng;
    explicit Gen(uint64_t s) : rng(s) {}
    std::vector<float> xavier(int rows, int cols, double fan_in, double fan_out) {
        const double a = std::sqrt(6.0 / (fan_in + fan_out));
        std::vector<float> v(static_cast<size_t>(rows) * cols);
        for (auto& x : v) x = static_cast<float>(rng.uniform(-a, a));
        return v;
    }
    std::vector<float> uni(int n, double lo, double hi) {
        std::vector<float> v(n);
        for (auto& x : v) x = static_cast<float>(rng.uniform(lo, hi));
        return v;
    }
};

void add(std::vector<UParam>& ps, const std::string& n, std::vector<int> shape, std::vector<float> v) {
    ps.push_back({n, std::move(shape), std::move(v)});
}

void norm_params(Gen& g, std::vector<UParam>& ps, const std::string& n, int C) {
    auto gm = g.uni(C, -0.1, 0.1);
    for (auto& x : gm) x += 1.0f;
    add(ps, n + ".gamma", {C}, gm);
    add(ps, n + ".beta", {C}, g.uni(C, -0.1, 0.1));
}

void conv_params(Gen& g, std::vector<UParam>& ps, const std::string& n, int cout, int cin) {
    add(ps, n + ".w", {cout, 9 * cin}, g.xavier(cout, 9 * cin, 9.0 * cin, 9.0 * cout));
    add(ps, n + ".b", {cout}, g.uni(cout, -0.05, 0.05));
}

void lin_params(Gen& g, std::vector<UParam>& ps, const std::string& n, int out, int in, bool bias) {
    add(ps, n + ".w", {out, in}, g.xavier(out, in, in, out));
    if (bias) add(ps, n + ".b", {out}, g.uni(out, -0.05, 0.05));
}

}  // namespace

// Parameter list of one stage in a fixed order (stage 0 = shared temb MLP).
std::vector<UParam> unet_stage_params(const UNetDesc& d, int stage) {
    const UNetSpec& sp = d.spec;
    Gen g(mix_seed(sp.seed, static_cast<uint64_t>(stage)));
    std::vector<UParam> ps;
    if (stage == 0) {
        lin_params(g, ps, "temb.lin1", sp.temb_dim, sp.ch[0], true);
        lin_params(g, ps, "temb.lin2", sp.temb_dim, sp.temb_dim, true);
        return ps;
    }
    const UStage& s = d.st.at(stage - 1);
    const int cin = s.cin + s.cskip;
    switch (s.kind) {
        case kConvIn: {
            conv_params(g, ps, "conv", s.cout, 64);
            auto& w = ps[0].data;  // zero the padded input channels
            for (int o = 0; o < s.cout; ++o)
                for (int k = 0; k < 9; ++k)
                    for (int ci = sp.c_lat; ci < 64; ++ci) w[static_cast<size_t>(o) * 576 + k * 64 + ci] = 0.f;
            break;
        }
        case kDown:
        case kUp: conv_params(g, ps, "conv", s.cout, cin); break;
        case kOut: {
            norm_params(g, ps, "gn", cin);
            conv_params(g, ps, "conv", 32, cin);
            for (size_t o = static_cast<size_t>(sp.c_lat); o < 32; ++o) {
                for (int k = 0; k < 9 * cin; ++k) ps[2].data[o * 9 * cin + k] = 0.f;
                ps[3].data[o] = 0.f;
            }
            break;
        }
        default: {
            const int C = s.cout;
            norm_params(g, ps, "gn1", cin);
            conv_params(g, ps, "conv1", C, cin);
            lin_params(g, ps, "temb", C, sp.temb_dim, true);
            norm_params(g, ps, "gn2", C);
            conv_params(g, ps, "conv2", C, C);
            if (cin != C) lin_params(g, ps, "short", C, cin, true);
            if (s.attn) {
                norm_params(g, ps, "tf.gn", C);
                lin_params(g, ps, "tf.proj_in", C, C, true);
                norm_params(g, ps, "tf.ln1", C);
                lin_params(g, ps, "tf.qkv", 3 * C, C, false);
                lin_params(g, ps, "tf.o1", C, C, true);
                norm_params(g, ps, "tf.ln2", C);
                lin_params(g, ps, "tf.q2", C, C, false);
                lin_params(g, ps, "tf.k2", C, sp.ctx_dim, false);
                lin_params(g, ps, "tf.v2", C, sp.ctx_dim, false);
                lin_params(g, ps, "tf.o2", C, C, true);
                norm_params(g, ps, "tf.ln3", C);
                lin_params(g, ps, "tf.ff1", 8 * C, C, true);
                lin_params(g, ps, "tf.ff2", C, 4 * C, true);
                lin_params(g, ps, "tf.proj_out", C, C, true);
                // further transformer blocks (depth > 1), appended so depth-1 stages keep
                // exactly the parameters above
                for (int b = 1; b < s.attn; ++b) {  // (motion-module parameters follow below)
                    const std::string pre = "tf.b" + std::to_string(b) + ".";
                    norm_params(g, ps, pre + "ln1", C);
                    lin_params(g, ps, pre + "qkv", 3 * C, C, false);
                    lin_params(g, ps, pre + "o1", C, C, true);
                    norm_params(g, ps, pre + "ln2", C);
                    lin_params(g, ps, pre + "q2", C, C, false);
                    lin_params(g, ps, pre + "k2", C, sp.ctx_dim, false);
                    lin_params(g, ps, pre + "v2", C, sp.ctx_dim, false);
                    lin_params(g, ps, pre + "o2", C, C, true);
                    norm_params(g, ps, pre + "ln3", C);
                    lin_params(g, ps, pre + "ff1", 8 * C, C, true);
                    lin_params(g, ps, pre + "ff2", C, 4 * C, true);
                }
            }
            if (s.motion) {  // temporal motion module: attention across the frames of each pixel
                norm_params(g, ps, "mm.gn", C);
                lin_params(g, ps, "mm.proj_in", C, C, true);
                for (int a = 1; a <= 2; ++a) {
                    const std::string pre = "mm.a" + std::to_string(a) + ".";
                    norm_params(g, ps, pre + "ln", C);
                    lin_params(g, ps, pre + "qkv", 3 * C, C, false);
                    lin_params(g, ps, pre + "o", C, C, true);
                }
                norm_params(g, ps, "mm.ln3", C);
                lin_params(g, ps, "mm.ff1", 8 * C, C, true);
                lin_params(g, ps, "mm.ff2", C, 4 * C, true);
                lin_params(g, ps, "mm.proj_out", C, C, true);
            }
        }
    }
    return ps;
}

namespace {
float siluf(float x) { return x / (1.0f + std::exp(-x)); }
}

// temb(t) = lin2(silu(lin1(sinusoid(t, ch0))))  (fp32, host)
std::vector<float> unet_temb(const UNetDesc& d, int t) {
    const UNetSpec& sp = d.spec;
    const auto ps = unet_stage_params(d, 0);
    const auto s = sinusoid(t, sp.ch[0]);
    std::vector<float> h(sp.temb_dim), o(sp.temb_dim);
    for (int i = 0; i < sp.temb_dim; ++i) {
        float a = ps[1].data[i];
        for (int k = 0; k < sp.ch[0]; ++k) a += ps[0].data[static_cast<size_t>(i) * sp.ch[0] + k] * static_cast<float>(s[k]);
        h[i] = siluf(a);
    }
    for (int i = 0; i < sp.temb_dim; ++i) {
        float a = ps[3].data[i];
        for (int k = 0; k < sp.temb_dim; ++k) a += ps[2].data[static_cast<size_t>(i) * sp.temb_dim + k] * h[k];
        o[i] = a;
    }
    return o;
}

// per-channel add of a RES stage: temb.w . silu(temb) + temb.b
std::vector<float> unet_chan_add(const std::vector<UParam>& ps, const std::vector<float>& temb) {
    const UParam* w = nullptr;
    const UParam* b = nullptr;
    for (auto& p : ps) {
        if (p.name == "temb.w") w = &p;
        if (p.name == "temb.b") b = &p;
    }
    if (!w) return {};
    const int C = w->shape[0], K = w->shape[1];
    std::vector<float> out(C);
    for (int i = 0; i < C; ++i) {
        float a = b->data[i];
        for (int k = 0; k < K; ++k) a += w->data[static_cast<size_t>(i) * K + k] * siluf(temb[k]);
        out[i] = a;
    }
    return out;
}

}  // namespace adx
