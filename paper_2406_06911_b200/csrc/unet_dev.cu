// unet_dev.cu -- device side of the UNet-shaped family: per-GPU parameters,
// per-t channel-add tables, cross-attention K/V precomputed from the fixed
// context, scratch per stream, and the per-stage enqueue (resnet / spatial
// transformer / down / up / in / out) on the tcgen05 GEMM + conv kernels.
#include "unet_dev.hpp"

#include "tc_attn.cuh"
#include "tc_gemm.cuh"
#include "unet_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace adx {

#define CKD(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

namespace {

using bf16 = __nv_bfloat16;

uint16_t to_bf16_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

void* upload_bf16(const std::vector<float>& v) {
    std::vector<uint16_t> h(v.size());
    for (size_t i = 0; i < v.size(); ++i) h[i] = to_bf16_bits(v[i]);
    void* d = nullptr;
    CKD(cudaMalloc(&d, std::max<size_t>(h.size(), 8) * 2));
    CKD(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    return d;
}

void* upload_f32(const std::vector<float>& v) {
    void* d = nullptr;
    CKD(cudaMalloc(&d, std::max<size_t>(v.size(), 8) * 4));
    CKD(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    return d;
}

int pad64(int n) { return (n + 63) / 64 * 64; }

// host split of an fp32 matrix [rows][K] into the ADX_F32 mode's B operand: every group of
// g columns -> [hi | lo | hi] (bf16 bits), hi = bf16(w), lo = bf16(w - hi)
std::vector<uint16_t> split_b(const std::vector<float>& w, long long rows, int K, int g) {
    std::vector<uint16_t> out(static_cast<size_t>(rows) * 3 * K);
    for (long long r = 0; r < rows; ++r)
        for (int c = 0; c < K; ++c) {
            const float x = w[static_cast<size_t>(r) * K + c];
            const uint16_t hb = to_bf16_bits(x);
            float hf;
            const uint32_t hu = static_cast<uint32_t>(hb) << 16;
            std::memcpy(&hf, &hu, 4);
            const uint16_t lb = to_bf16_bits(x - hf);
            const int grp = c / g, cg = c % g;
            uint16_t* o = out.data() + static_cast<size_t>(r) * 3 * K + 3LL * grp * g + cg;
            o[0] = hb;
            o[g] = lb;
            o[2 * g] = hb;
        }
    return out;
}

float bf16_to_float(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

bool ends_with(const std::string& s, const char* suf) {
    const size_t n = std::strlen(suf);
    return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

// bf16 mode, ADX_LN_FOLD=1 on a -DADX_TC_STATW=2 build: LayerNorm folded into the GEMM that
// consumes it (statistics warps in the GEMM, gain in the weights).  Off by default: measured
// slower at c2 / c4 than the standalone layernorm_k pass -- the statistics of a
// tile finish after its MMAs.
bool ln_fold() {
    static const bool on = [] {
        const char* e = getenv("ADX_LN_FOLD");
        return e && *e == '1' && tc_ln_fold_supported();
    }();
    return on;
}

// LN(h) W^T + b = rstd (h W'^T - mean colsum(W')) + (b + W beta) with W' = W diag(gamma):
// rewrites the consumer weight `w` [rows][K] into W', its bias into b + W beta (created when the
// layer has none) and returns colsum(W') over the bf16-rounded W' the tensor cores multiply by
std::vector<float> fold_layer_norm(std::vector<float>& w, int rows, int K, const std::vector<float>& gamma,
                                   const std::vector<float>& beta, std::vector<float>& bias) {
    if (bias.empty()) bias.assign(rows, 0.f);
    std::vector<float> colsum(rows);
    for (int n = 0; n < rows; ++n) {
        double b = 0.0, cs = 0.0;
        float* r = w.data() + static_cast<size_t>(n) * K;
        for (int k = 0; k < K; ++k) {
            b += static_cast<double>(r[k]) * beta[k];
            r[k] *= gamma[k];
            cs += bf16_to_float(to_bf16_bits(r[k]));
        }
        bias[n] = static_cast<float>(bias[n] + b);
        colsum[n] = static_cast<float>(cs);
    }
    return colsum;
}

void* device_zeros(size_t bytes) {
    void* d = nullptr;
    CKD(cudaMalloc(&d, std::max<size_t>(bytes, 16)));
    CKD(cudaMemset(d, 0, std::max<size_t>(bytes, 16)));
    return d;
}

void* upload_bf16(const std::vector<float>& v);

// K2 [Lp][C] = ctx . Wk^T and V2 [Lp][C] = ctx . Wv^T on the tensor cores (private stream,
// synchronous: runs at stage preparation, outside any capture); rows >= Lc stay zero
void ctx_projection(const float* ctx, int Lc, int Dc, const std::vector<float>& wk, const std::vector<float>& wv,
                    int C, __nv_bfloat16* k2, __nv_bfloat16* v2) {
    std::vector<float> c(ctx, ctx + static_cast<size_t>(Lc) * Dc);
    void* dctx = upload_bf16(c);
    void* dwk = upload_bf16(wk);
    void* dwv = upload_bf16(wv);
    cudaStream_t st;
    CKD(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    TcArgs a;
    a.out_bf16 = k2;
    a.ldo = C;
    tc_gemm(dctx, dwk, Lc, C, Dc, a, st);
    TcArgs b;
    b.out_bf16 = v2;
    b.ldo = C;
    tc_gemm(dctx, dwv, Lc, C, Dc, b, st);
    CKD(cudaStreamSynchronize(st));
    CKD(cudaStreamDestroy(st));
    cudaFree(dctx);
    cudaFree(dwk);
    cudaFree(dwv);
}

void* upload_u16(const std::vector<uint16_t>& h) {
    void* d = nullptr;
    CKD(cudaMalloc(&d, std::max<size_t>(h.size(), 8) * 2));
    CKD(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    return d;
}

}  // namespace

UNetDevice::UNetDevice(const Model& m, int ordinal, bool exact)
    : m_(m), d_(*m.unet), ordinal_(ordinal), exact_(exact) {
    st_.resize(m.L + 1);
}

UNetDevice::~UNetDevice() {
    cudaSetDevice(ordinal_);
    for (auto& s : st_) {
        for (auto& kv : s.p) cudaFree(kv.second);
        cudaFree(s.chan_add);
        for (auto* q : s.k2) cudaFree(q);
        for (auto* q : s.vt2) cudaFree(q);
        for (auto* q : s.kv2x) cudaFree(q);
        for (auto* q : s.pe_proj) cudaFree(q);
    }
    for (auto& kv : scratch_) {
        UScratch& s = kv.second;
        for (void* p : {static_cast<void*>(s.a), static_cast<void*>(s.b), static_cast<void*>(s.c),
                        static_cast<void*>(s.r), static_cast<void*>(s.qkv), static_cast<void*>(s.att),
                        static_cast<void*>(s.ff), static_cast<void*>(s.ff2), static_cast<void*>(s.P),
                        static_cast<void*>(s.VT), static_cast<void*>(s.S), static_cast<void*>(s.gn),
                        static_cast<void*>(s.fa), static_cast<void*>(s.fb), static_cast<void*>(s.fc),
                        static_cast<void*>(s.fr), static_cast<void*>(s.fqkv), static_cast<void*>(s.fatt),
                        static_cast<void*>(s.fff), static_cast<void*>(s.fvt), static_cast<void*>(s.sa),
                        static_cast<void*>(s.sq), static_cast<void*>(s.sk), static_cast<void*>(s.sv), s.attn_ws,
                        static_cast<void*>(s.eps2)})
            cudaFree(p);
    }
}

long long UNetDevice::param_bytes(int stage) const {
    long long b = 0;
    for (auto& kv : st_[stage].bytes) b += kv.second;
    return b;
}

void UNetDevice::ensure_stage(int stage) {
    UDevStage& ds = st_[stage];
    if (ds.ready) return;
    CKD(cudaSetDevice(ordinal_));
    const UNetSpec& sp = d_.spec;
    auto ps = unet_stage_params(d_, stage);
    if (!exact_ && ln_fold()) {
        // LayerNorm fold of the transformer blocks: qkv <- ln1, q2 <- ln2, ff1 <- ln3 (weights,
        // bias and colsum; ff1's GEGLU row interleave below then applies to all three alike)
        std::map<std::string, UParam*> by;
        for (auto& p : ps) by[p.name] = &p;
        std::vector<UParam> extra;
        for (auto& p : ps) {
            if (p.name.rfind("tf.", 0) != 0) continue;
            const char* sufs[3][2] = {{"qkv.w", "ln1"}, {"q2.w", "ln2"}, {"ff1.w", "ln3"}};
            for (auto& sf : sufs) {
                if (!ends_with(p.name, sf[0])) continue;
                const std::string pre = p.name.substr(0, p.name.size() - std::strlen(sf[0]));
                const std::string layer = p.name.substr(0, p.name.size() - 2);  // drop ".w"
                auto g = by.find(pre + sf[1] + ".gamma"), b = by.find(pre + sf[1] + ".beta");
                if (g == by.end() || b == by.end()) throw std::logic_error("unet: missing LayerNorm of " + p.name);
                const int rows = p.shape[0], K = p.shape[1];
                auto bi = by.find(layer + ".b");
                std::vector<float> bias = bi != by.end() ? bi->second->data : std::vector<float>();
                std::vector<float> cs = fold_layer_norm(p.data, rows, K, g->second->data, b->second->data, bias);
                if (bi != by.end())
                    bi->second->data = bias;
                else
                    extra.push_back(UParam{layer + ".b", {rows}, bias});
                extra.push_back(UParam{layer + ".lncs", {rows}, cs});
            }
        }
        for (auto& e : extra) {
            if (ends_with(e.name, "ff1.lncs")) {  // GEGLU interleave, as for ff1's weight rows and bias
                const int H = static_cast<int>(e.data.size()) / 2, G = tc_geglu_group();
                std::vector<float> perm(e.data.size());
                for (int t = 0; t < H / G; ++t)
                    for (int i = 0; i < 2 * G; ++i) perm[2 * G * t + i] = e.data[i < G ? G * t + i : H + G * t + i - G];
                e.data = perm;
            }
            ps.push_back(std::move(e));
        }
    }
    for (auto& p : ps) {
        const bool matrix = p.shape.size() == 2;
        const bool ctx_proj = ends_with(p.name, ".k2.w") || ends_with(p.name, ".v2.w");  // precomputed below
        const bool ff1 = ends_with(p.name, ".ff1.w") || ends_with(p.name, ".ff1.b");
        if (exact_ && matrix && !ctx_proj && p.name != "temb.w") {
            // ADX_F32: split-bf16 weights, [hi | lo | hi] per conv tap (g = Cin) or per row (g = K);
            // the GEGLU ff1 rows are tile-interleaved first, exactly as in the bf16 mode
            const int rows = p.shape[0], K = p.shape[1];
            std::vector<float> w = p.data;
            if (ff1) {
                const int H = rows / 2, G = tc_geglu_group();
                if (H % G) throw std::invalid_argument("unet: GEGLU width must be a multiple of the tile group");
                for (int t = 0; t < H / G; ++t)
                    for (int i = 0; i < 2 * G; ++i) {
                        const int src = i < G ? G * t + i : H + G * t + (i - G);
                        std::copy_n(p.data.begin() + static_cast<size_t>(src) * K, K,
                                    w.begin() + static_cast<size_t>(2 * G * t + i) * K);
                    }
            }
            const bool conv = p.name.rfind("conv", 0) == 0;
            ds.p[p.name] = upload_u16(split_b(w, rows, K, conv ? K / 9 : K));
            ds.bytes[p.name] = static_cast<long long>(w.size()) * 6;
            continue;
        }
        if (ff1) {
            // GEGLU fused into the ff1 GEMM epilogue: rows [hidden | gate] interleaved per
            // N tile of 2G: tile t = hidden rows [Gt, Gt+G) then gate rows 4C + same (G = tc_geglu_group())
            const int rows = p.shape[0], cols = matrix ? p.shape[1] : 1, H = rows / 2, G = tc_geglu_group();
            if (H % G) throw std::invalid_argument("unet: GEGLU width must be a multiple of the tile group");
            std::vector<float> perm(p.data.size());
            for (int t = 0; t < H / G; ++t)
                for (int i = 0; i < 2 * G; ++i) {
                    const int src = i < G ? G * t + i : H + G * t + (i - G);
                    std::copy_n(p.data.begin() + static_cast<size_t>(src) * cols, cols,
                                perm.begin() + static_cast<size_t>(2 * G * t + i) * cols);
                }
            ds.p[p.name] = matrix ? upload_bf16(perm) : upload_f32(perm);
            ds.bytes[p.name] = static_cast<long long>(p.data.size()) * (matrix ? 2 : 4);
            continue;
        }
        if (ctx_proj || p.name == "temb.w" || p.name == "temb.b") continue;
        ds.p[p.name] = matrix ? upload_bf16(p.data) : upload_f32(p.data);
        ds.bytes[p.name] = static_cast<long long>(p.data.size()) * (matrix ? 2 : 4);
    }
    const UStage& s = d_.st[stage - 1];
    if (s.attn) {
        // cross-attention K2 = ctx . Wk2^T and V2^T = Wv2 . ctx^T are constant per run: computed
        // once per (block, context), context length padded to a multiple of 64 (zeros)
        const int C = s.cout, Lc = sp.ctx_len, Lp = pad64(Lc), Dc = sp.ctx_dim, B = sp.contexts();
        const size_t csz = static_cast<size_t>(Lc) * Dc;
        for (int b = 0; b < s.attn; ++b) {
            const std::string pre = b == 0 ? "tf." : "tf.b" + std::to_string(b) + ".";
            const std::vector<float>* wk = nullptr;
            const std::vector<float>* wv = nullptr;
            for (auto& p : ps) {
                if (p.name == pre + "k2.w") wk = &p.data;
                if (p.name == pre + "v2.w") wv = &p.data;
            }
            if (!wk || !wv) throw std::logic_error("unet: missing cross-attention projection of " + pre);
            for (int img = 0; img < B; ++img) {
                const float* ctx = d_.ctx.data() + img * csz;
                if (exact_) {  // fp32 on the host, then split operands (K2' per head, V2'^T along keys)
                    std::vector<float> k2(static_cast<size_t>(Lp) * C, 0.f), vt2(static_cast<size_t>(C) * Lp, 0.f);
                    for (int l = 0; l < Lc; ++l)
                        for (int c = 0; c < C; ++c) {
                            float ak = 0.f, av = 0.f;
                            for (int k = 0; k < Dc; ++k) {
                                const float x = ctx[static_cast<size_t>(l) * Dc + k];
                                ak += (*wk)[static_cast<size_t>(c) * Dc + k] * x;
                                av += (*wv)[static_cast<size_t>(c) * Dc + k] * x;
                            }
                            k2[static_cast<size_t>(l) * C + c] = ak;
                            vt2[static_cast<size_t>(c) * Lp + l] = av;
                        }
                    ds.k2.push_back(static_cast<bf16*>(upload_u16(split_b(k2, Lp, C, 64))));
                    ds.vt2.push_back(static_cast<bf16*>(upload_u16(split_b(vt2, C, Lp, Lp))));
                    const size_t pl = static_cast<size_t>(Lp) * C;
                    std::vector<uint16_t> x4(4 * pl);
                    for (int l = 0; l < Lp; ++l)
                        for (int c = 0; c < C; ++c) {
                            const size_t i = static_cast<size_t>(l) * C + c;
                            const float kv[2] = {k2[i], vt2[static_cast<size_t>(c) * Lp + l]};
                            for (int w = 0; w < 2; ++w) {
                                const uint16_t hb = to_bf16_bits(kv[w]);
                                x4[2 * w * pl + i] = hb;
                                x4[(2 * w + 1) * pl + i] = to_bf16_bits(kv[w] - bf16_to_float(hb));
                            }
                        }
                    ds.kv2x.push_back(static_cast<bf16*>(upload_u16(x4)));
                } else {  // bf16 on the tensor cores: two GEMMs (SDXL: 10 blocks x 2 contexts per stage)
                    ds.k2.push_back(static_cast<bf16*>(device_zeros(static_cast<size_t>(Lp) * C * 2)));
                    ds.vt2.push_back(static_cast<bf16*>(device_zeros(static_cast<size_t>(Lp) * C * 2)));
                    ctx_projection(ctx, Lc, Dc, *wk, *wv, C, ds.k2.back(), ds.vt2.back());  // V2 row-major
                }
            }
        }
    }
    if (s.motion) {
        // frame positions (sinusoidal, AnimateDiff's PositionalEncoding layout: sin on even,
        // cos on odd channels) are added to the normed tokens before the QKV projection:
        // (a + pe) W^T = a W^T + pe W^T, the second term precomputed here with the weights the
        // device multiplies by (bf16-rounded, or fp32 in the ADX_F32 mode)
        const int C = s.cout, F = sp.frames;
        std::vector<double> pe(static_cast<size_t>(F) * C);
        for (int f = 0; f < F; ++f)
            for (int i = 0; i < C / 2; ++i) {
                const double w = std::exp(-(2.0 * i) * std::log(10000.0) / C);
                pe[static_cast<size_t>(f) * C + 2 * i] = std::sin(f * w);
                pe[static_cast<size_t>(f) * C + 2 * i + 1] = std::cos(f * w);
            }
        for (int a = 1; a <= 2; ++a) {
            const std::string nm = "mm.a" + std::to_string(a) + ".qkv.w";
            const std::vector<float>* w = nullptr;
            for (auto& p : ps)
                if (p.name == nm) w = &p.data;
            if (!w) throw std::logic_error("unet: missing " + nm);
            std::vector<float> proj(static_cast<size_t>(F) * 3 * C);
            for (int f = 0; f < F; ++f)
                for (int n = 0; n < 3 * C; ++n) {
                    double acc = 0.0;
                    for (int c = 0; c < C; ++c) {
                        float wv = (*w)[static_cast<size_t>(n) * C + c];
                        if (!exact_) wv = bf16_to_float(to_bf16_bits(wv));
                        acc += pe[static_cast<size_t>(f) * C + c] * wv;
                    }
                    proj[static_cast<size_t>(f) * 3 * C + n] = static_cast<float>(acc);
                }
            ds.pe_proj.push_back(static_cast<float*>(upload_f32(proj)));
        }
    }
    ds.ready = true;
}

void UNetDevice::ensure_tables(int T) {
    CKD(cudaSetDevice(ordinal_));
    std::vector<std::vector<float>> temb;
    for (int stage = 1; stage <= m_.L; ++stage) {
        UDevStage& ds = st_[stage];
        const UStage& s = d_.st[stage - 1];
        if (!ds.ready || ds.chan_T >= T || (s.kind != kRes && s.kind != kMidRes)) continue;
        if (temb.empty())
            for (int t = 0; t <= T; ++t) temb.push_back(unet_temb(d_, t));
        const auto ps = unet_stage_params(d_, stage);
        std::vector<float> flat;
        for (int t = 0; t <= T; ++t) {
            const auto ca = unet_chan_add(ps, temb[t]);
            flat.insert(flat.end(), ca.begin(), ca.end());
        }
        cudaFree(ds.chan_add);
        ds.chan_add = static_cast<float*>(upload_f32(flat));
        ds.chan_T = T;
    }
}

UScratch& UNetDevice::scratch(cudaStream_t st) {
    auto it = scratch_.find(st);
    if (it != scratch_.end()) return it->second;
    CKD(cudaSetDevice(ordinal_));
    const UNetSpec& sp = d_.spec;
    size_t act = 0, qkv = 0, ff = 0, S = 0, vt = 0, gn = 0;
    for (const UStage& s : d_.st) {
        const size_t hw = static_cast<size_t>(s.H) * s.W;
        act = std::max({act, hw * (s.cin + s.cskip), static_cast<size_t>(s.Ho()) * s.Wo() * s.cout, hw * 64,
                        4 * hw * s.cin});
        gn = std::max({gn, group_norm_scratch_bytes(sp.batch(), static_cast<int>(4 * hw), sp.groups,
                                                    s.cin + s.cskip + s.cout)});
        if (s.attn || s.motion) {
            qkv = std::max(qkv, hw * 3 * s.cout);
            ff = std::max(ff, hw * 8 * s.cout);
        }
        if (s.attn) {
            const size_t L = hw, Lp = pad64(static_cast<int>(L));
            S = std::max(S, L * std::max(Lp, static_cast<size_t>(pad64(sp.ctx_len))));
            vt = std::max(vt, static_cast<size_t>(s.cout) * Lp * sp.batch());  // every image's V^T
        }
    }
    // activations / GEMM operands hold the whole CFG batch; S, V^T and the attention work
    // space are per image (attention runs image by image)
    act *= sp.batch();
    qkv *= sp.batch();
    ff *= sp.batch();
    UScratch s;
    auto al = [](size_t bytes) {
        void* p = nullptr;
        CKD(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        return p;
    };
    s.a = static_cast<bf16*>(al(act * 2));
    s.b = static_cast<bf16*>(al(act * 2));
    s.c = static_cast<bf16*>(al(act * 2));
    s.r = static_cast<bf16*>(al(act * 2));
    s.qkv = static_cast<bf16*>(al(qkv * 2));
    s.att = static_cast<bf16*>(al(act * 2));
    s.ff = static_cast<bf16*>(al(ff * 2));
    s.ff2 = static_cast<bf16*>(al(ff * 2));
    s.P = static_cast<bf16*>(al(S * 2));
    s.S = static_cast<float*>(al(S * 4));
    s.VT = static_cast<bf16*>(al(vt * 2));
    s.gn = static_cast<float2*>(al(gn));
    s.eps2 = static_cast<float*>(al(static_cast<size_t>(sp.batch()) * sp.H * sp.W * sp.c_lat * 4));
    for (const UStage& stg : d_.st)
        if (stg.attn) {
            const int L = stg.H * stg.W;
            s.attn_ws_bytes = std::max({s.attn_ws_bytes, tc_attention_ws_bytes(L, L, stg.cout, sp.batch()),
                                        tc_attention_ws_bytes(sp.batch() * L, sp.ctx_len, stg.cout)});
        }
    if (s.attn_ws_bytes) {
        s.attn_ws = al(s.attn_ws_bytes);
        CKD(cudaMemsetAsync(s.attn_ws, 0, s.attn_ws_bytes, st));
    }
    if (exact_) {
        size_t spl = 0, ffx = 0, vtx = 0;
        for (const UStage& st : d_.st) {
            const size_t hw = static_cast<size_t>(st.H) * st.W;
            spl = std::max({spl, 3 * 4 * hw * st.cin, 3 * hw * (st.cin + st.cskip), 3 * hw * st.cout});
            if (st.attn || st.motion) {
                spl = std::max(spl, 3 * hw * 4 * st.cout);
                ffx = std::max(ffx, hw * 4 * st.cout);
            }
            if (st.attn) {
                const size_t L = hw, Lp = pad64(static_cast<int>(L));
                spl = std::max(spl, 3 * L * Lp);
                vtx = std::max(vtx, 64 * Lp);
            }
        }
        spl *= sp.batch();  // split operands of whole-batch GEMMs (attention ones are per image)
        ffx *= sp.batch();
        s.fa = static_cast<float*>(al(act * 4));
        s.fb = static_cast<float*>(al(act * 4));
        s.fc = static_cast<float*>(al(act * 4));
        s.fr = static_cast<float*>(al(act * 4));
        s.fatt = static_cast<float*>(al(act * 4));
        s.fqkv = static_cast<float*>(al(qkv * 4));
        s.fff = static_cast<float*>(al(ffx * 4));
        s.fvt = static_cast<float*>(al(vtx * 4));
        s.sa = static_cast<bf16*>(al(spl * 2));
        s.sq = static_cast<bf16*>(al(3 * act * 2));
        s.sk = static_cast<bf16*>(al(3 * act * 2));
        s.sv = static_cast<bf16*>(al(3 * vtx * 2));
    }
    CKD(cudaMemsetAsync(s.gn, 0, gn, st));  // group_norm's ticket counter starts at zero (stream-ordered:
                                             // also valid when first reached inside a graph capture)
    return scratch_.emplace(st, s).first->second;
}

const void* UNetDevice::P(int stage, const char* name) const {
    auto it = st_[stage].p.find(name);
    if (it == st_[stage].p.end()) throw std::logic_error(std::string("unet: missing parameter ") + name);
    return it->second;
}
const float* UNetDevice::F(int stage, const char* name) const { return static_cast<const float*>(P(stage, name)); }

// multi-head attention out[L x C] = softmax(q k^T / 8) v (64-wide heads), q / k / v row-major
void UNetDevice::attention(UScratch& s, const bf16* q, long long ldq, const bf16* k, long long ldk, const bf16* v,
                           long long ldv, int L, int Lk, int C, bf16* out, cudaStream_t st, int batch) {
    const int Lkp = pad64(Lk);
    static const bool unfused = [] {
        const char* e = getenv("ADX_ATTN");
        return e && std::string(e) == "unfused";
    }();
    if (!unfused) {  // fused tcgen05 flash attention (tc_attn.cu): S and P stay in TMEM
        tc_attention(q, ldq, k, ldk, v, ldv, L, Lk, C, out, C, st, s.attn_ws, s.attn_ws_bytes, batch);
        return;
    }
    if (batch > 1) {  // the unfused debugging path runs image by image
        for (int b = 0; b < batch; ++b)
            attention(s, q + b * L * ldq, ldq, k + b * Lk * ldk, ldk, v + b * Lk * ldv, ldv, L, Lk, C,
                      out + static_cast<long long>(b) * L * C, st, 1);
        return;
    }
    for (int h = 0; h < C / 64; ++h) {
        TcArgs a;
        a.out_f32 = s.S;
        a.ldo = Lkp;
        a.out_scale = 0.125f;  // 1/sqrt(64)
        tc_gemm_strided(q + h * 64, ldq, k + h * 64, ldk, L, Lk, 64, a, st);
        softmax_rows(s.S, Lkp, L, Lk, s.P, Lkp, Lkp, st);
        transpose_head(v + h * 64, ldv, Lk, Lkp, 64, s.VT, st);
        TcArgs o;
        o.out_bf16 = out + h * 64;
        o.ldo = C;
        tc_gemm(s.P, s.VT, L, 64, Lkp, o, st);
    }
}

template <typename T>
void UNetDevice::gn_images(const Cat2T<T>& x, int HW, const float* gamma, const float* beta, float eps, int act,
                           T* out, UScratch& s, cudaStream_t st) {
    const int B = d_.spec.batch();
    static const int batched_from = [] {  // ADX_GN_BATCH_MIN: smallest batch using the batched pair
        const char* e = getenv("ADX_GN_BATCH_MIN");
        return e ? atoi(e) : 2;
    }();
    // CFG pairs and video frames: one batched stats + apply pair instead of B fused launches
    // (c4 pass 21.37 -> 20.96 ms); a single image keeps the one-launch cooperative kernel
    if (B >= batched_from) {
        group_norm(x, B, HW, d_.spec.groups, gamma, beta, eps, act, out, s.gn, st);
        return;
    }
    const long long i0 = static_cast<long long>(HW) * x.c0, i1 = static_cast<long long>(HW) * x.c1;
    for (int b = 0; b < B; ++b)
        group_norm(Cat2T<T>{x.p0 + b * i0, x.c0, x.p1 ? x.p1 + b * i1 : nullptr, x.c1}, 1, HW, d_.spec.groups, gamma,
                   beta, eps, act, out + b * (i0 + i1), s.gn, st);
}

// Temporal motion module (video UNets, AnimateDiff-shaped): GN (per frame) -> proj_in ->
// 2 x [LN -> +frame positions -> self-attention across the frames of each pixel -> out
// proj + residual] -> LN -> GEGLU FF + residual -> proj_out + x.  Tokens are frame-major
// [F][HW][C]; the QKV GEMMs add PE . W^T per frame in the epilogue (chan_add_rows = HW).
void UNetDevice::motion(int stage, const bf16* x, int H, int W, int C, bf16* y, cudaStream_t st) {
    UScratch& s = scratch(st);
    const UNetSpec& sp = d_.spec;
    const int L = H * W, NF = sp.frames, FL = NF * L;
    gn_images(Cat2{x, C, nullptr, 0}, L, F(stage, "mm.gn.gamma"), F(stage, "mm.gn.beta"), 1e-6f, 0, s.a, s, st);
    TcArgs pi;
    pi.bias = F(stage, "mm.proj_in.b");
    pi.out_bf16 = s.b;
    pi.ldo = C;
    tc_gemm(s.a, P(stage, "mm.proj_in.w"), FL, C, C, pi, st);  // h = s.b
    for (int a = 1; a <= 2; ++a) {
        const std::string pre = "mm.a" + std::to_string(a) + ".";
        layer_norm(s.b, FL, C, F(stage, (pre + "ln.gamma").c_str()), F(stage, (pre + "ln.beta").c_str()), 1e-5f, s.a,
                   st);
        TcArgs qk;
        qk.chan_add = st_[stage].pe_proj[a - 1];
        qk.chan_add_rows = L;  // row f * HW + p adds frame f's projected position
        qk.out_bf16 = s.qkv;
        qk.ldo = 3 * C;
        tc_gemm(s.a, P(stage, (pre + "qkv.w").c_str()), FL, 3 * C, C, qk, st);
        temporal_attention(s.qkv, NF, L, C, s.att, st);
        TcArgs o;
        o.bias = F(stage, (pre + "o.b").c_str());
        o.residual = s.b;
        o.ldr = C;
        o.out_bf16 = s.b;
        o.ldo = C;
        tc_gemm(s.att, P(stage, (pre + "o.w").c_str()), FL, C, C, o, st);
    }
    layer_norm(s.b, FL, C, F(stage, "mm.ln3.gamma"), F(stage, "mm.ln3.beta"), 1e-5f, s.a, st);
    TcArgs f1;
    f1.bias = F(stage, "mm.ff1.b");
    f1.act = 2;
    f1.out_bf16 = s.ff2;
    f1.ldo = 4 * C;
    tc_gemm(s.a, P(stage, "mm.ff1.w"), FL, 8 * C, C, f1, st);
    TcArgs f2;
    f2.bias = F(stage, "mm.ff2.b");
    f2.residual = s.b;
    f2.ldr = C;
    f2.out_bf16 = s.b;
    f2.ldo = C;
    tc_gemm(s.ff2, P(stage, "mm.ff2.w"), FL, C, 4 * C, f2, st);
    TcArgs po;
    po.bias = F(stage, "mm.proj_out.b");
    po.residual = x;
    po.ldr = C;
    po.out_bf16 = y;
    po.ldo = C;
    tc_gemm(s.b, P(stage, "mm.proj_out.w"), FL, C, C, po, st);
}

void UNetDevice::motion_exact(int stage, const float* x, int H, int W, int C, float* y, cudaStream_t st) {
    UScratch& s = scratch(st);
    const UNetSpec& sp = d_.spec;
    const int L = H * W, NF = sp.frames, FL = NF * L;
    gn_images(Cat2F{x, C, nullptr, 0}, L, F(stage, "mm.gn.gamma"), F(stage, "mm.gn.beta"), 1e-6f, 0, s.fa, s, st);
    TcArgs pi;
    pi.bias = F(stage, "mm.proj_in.b");
    pi.out_f32 = s.fb;
    pi.ldo = C;
    gemm_x(s, s.fa, FL, C, "mm.proj_in.w", stage, C, pi, st);
    for (int a = 1; a <= 2; ++a) {
        const std::string pre = "mm.a" + std::to_string(a) + ".", n_qkv = pre + "qkv.w", n_o = pre + "o.w";
        layer_norm(s.fb, FL, C, F(stage, (pre + "ln.gamma").c_str()), F(stage, (pre + "ln.beta").c_str()), 1e-5f,
                   s.fa, st);
        TcArgs qk;
        qk.chan_add = st_[stage].pe_proj[a - 1];
        qk.chan_add_rows = L;
        qk.out_f32 = s.fqkv;
        qk.ldo = 3 * C;
        gemm_x(s, s.fa, FL, C, n_qkv.c_str(), stage, 3 * C, qk, st);
        temporal_attention(s.fqkv, NF, L, C, s.fatt, st);
        TcArgs o;
        o.bias = F(stage, (pre + "o.b").c_str());
        o.residual_f32 = s.fb;
        o.ldr = C;
        o.out_f32 = s.fb;
        o.ldo = C;
        gemm_x(s, s.fatt, FL, C, n_o.c_str(), stage, C, o, st);
    }
    layer_norm(s.fb, FL, C, F(stage, "mm.ln3.gamma"), F(stage, "mm.ln3.beta"), 1e-5f, s.fa, st);
    TcArgs f1;
    f1.bias = F(stage, "mm.ff1.b");
    f1.act = 2;
    f1.out_f32 = s.fff;
    f1.ldo = 4 * C;
    gemm_x(s, s.fa, FL, C, "mm.ff1.w", stage, 8 * C, f1, st);
    TcArgs f2;
    f2.bias = F(stage, "mm.ff2.b");
    f2.residual_f32 = s.fb;
    f2.ldr = C;
    f2.out_f32 = s.fb;
    f2.ldo = C;
    gemm_x(s, s.fff, FL, 4 * C, "mm.ff2.w", stage, C, f2, st);
    TcArgs po;
    po.bias = F(stage, "mm.proj_out.b");
    po.residual_f32 = x;
    po.ldr = C;
    po.out_f32 = y;
    po.ldo = C;
    gemm_x(s, s.fb, FL, C, "mm.proj_out.w", stage, C, po, st);
}

// SpatialTransformer: GN -> proj_in -> [LN self-attn] -> [LN cross-attn] -> [LN GEGLU FF] -> proj_out + x
// SpatialTransformer: GN -> proj_in -> depth x ([LN self-attn] [LN cross-attn] [LN GEGLU FF])
// -> proj_out + x.  With CFG the batch holds 2 images: GEMMs / LN run over both, GN and
// attention per image (image i cross-attends to context i).
void UNetDevice::transformer(int stage, const bf16* x, int H, int W, int C, bf16* y, cudaStream_t st) {
    UScratch& s = scratch(st);
    const UNetSpec& sp = d_.spec;
    const int L = H * W, B = sp.batch(), BL = B * L, depth = d_.st[stage - 1].attn;
    const long long img = static_cast<long long>(L) * C;
    gn_images(Cat2{x, C, nullptr, 0}, L, F(stage, "tf.gn.gamma"), F(stage, "tf.gn.beta"), 1e-6f, 0, s.a, s, st);
    // LayerNorm fold: the GEMM reading LN(h) (qkv, q2, ff1) takes h itself, reduces each token's
    // statistics from its A tiles and has the gain folded into its weights: no standalone
    // LayerNorm pass, no normalised copy of h
    const bool fold = ln_fold();
    TcArgs pi;
    pi.bias = F(stage, "tf.proj_in.b");
    pi.out_bf16 = s.b;
    pi.ldo = C;
    tc_gemm(s.a, P(stage, "tf.proj_in.w"), BL, C, C, pi, st);  // h = s.b
    for (int blk = 0; blk < depth; ++blk) {
        const std::string pre = blk == 0 ? "tf." : "tf.b" + std::to_string(blk) + ".";
        auto Pn = [&](const char* n) { return P(stage, (pre + n).c_str()); };
        auto Fn = [&](const char* n) { return F(stage, (pre + n).c_str()); };
        // the consumer side: A = h (raw) with the fold, else the normalised copy in s.a
        auto consume = [&](TcArgs& a, const char* layer, const char* ln) -> const bf16* {
            if (!fold) {
                layer_norm(s.b, BL, C, Fn((std::string(ln) + ".gamma").c_str()),
                           Fn((std::string(ln) + ".beta").c_str()), 1e-5f, s.a, st);
                return s.a;
            }
            a.ln_eps = 1e-5f;
            a.ln_colsum = Fn((std::string(layer) + ".lncs").c_str());
            a.bias = Fn((std::string(layer) + ".b").c_str());
            return s.b;
        };
        // self attention
        TcArgs qk;
        qk.out_bf16 = s.qkv;
        qk.ldo = 3 * C;
        const bf16* a1 = consume(qk, "qkv", "ln1");
        tc_gemm(a1, Pn("qkv.w"), BL, 3 * C, C, qk, st);
        // self attention of every image in one launch (stacked rows)
        attention(s, s.qkv, 3 * C, s.qkv + C, 3 * C, s.qkv + 2 * C, 3 * C, L, L, C, s.att, st, B);
        TcArgs o1;
        o1.bias = Fn("o1.b");
        o1.residual = s.b;
        o1.ldr = C;
        o1.out_bf16 = s.b;  // in place: each element is read and written by one epilogue thread
        o1.ldo = C;
        tc_gemm(s.att, Pn("o1.w"), BL, C, C, o1, st);
        // cross attention against the fixed context(s)
        TcArgs q2;
        q2.out_bf16 = s.qkv;
        q2.ldo = C;
        const bf16* a2 = consume(q2, "q2", "ln2");
        tc_gemm(a2, Pn("q2.w"), BL, C, C, q2, st);
        if (sp.contexts() == 1)  // one shared context: every image's queries in one launch
            attention(s, s.qkv, C, st_[stage].k2[blk], C, st_[stage].vt2[blk], C, BL, sp.ctx_len, C, s.att, st);
        else
            for (int b = 0; b < B; ++b)
                attention(s, s.qkv + b * img, C, st_[stage].k2[blk * B + b], C, st_[stage].vt2[blk * B + b], C, L,
                          sp.ctx_len, C, s.att + b * img, st);
        TcArgs o2;
        o2.bias = Fn("o2.b");
        o2.residual = s.b;
        o2.ldr = C;
        o2.out_bf16 = s.b;
        o2.ldo = C;
        tc_gemm(s.att, Pn("o2.w"), BL, C, C, o2, st);
        // GEGLU feed-forward
        TcArgs f1;
        f1.bias = Fn("ff1.b");
        f1.act = 2;  // GEGLU in the epilogue: s.ff2 = hidden * gelu(gate), 4C wide
        f1.out_bf16 = s.ff2;
        f1.ldo = 4 * C;
        const bf16* a3 = consume(f1, "ff1", "ln3");
        tc_gemm(a3, Pn("ff1.w"), BL, 8 * C, C, f1, st);
        TcArgs f2;
        f2.bias = Fn("ff2.b");
        f2.residual = s.b;
        f2.ldr = C;
        f2.out_bf16 = s.b;
        f2.ldo = C;
        tc_gemm(s.ff2, Pn("ff2.w"), BL, C, 4 * C, f2, st);
    }
    TcArgs po;
    po.bias = F(stage, "tf.proj_out.b");
    po.residual = x;
    po.ldr = C;
    po.out_bf16 = y;
    po.ldo = C;
    tc_gemm(s.b, P(stage, "tf.proj_out.w"), BL, C, C, po, st);
}

void UNetDevice::enqueue(int stage, const std::vector<Seg>& in, int t, void* y, bool latent_f64, cudaStream_t st) {
    ensure_stage(stage);
    if (exact_) return enqueue_exact(stage, in, t, y, latent_f64, st);
    const UNetSpec& sp = d_.spec;
    const UStage& s = d_.st[stage - 1];
    UScratch& sc = scratch(st);
    const int HW = s.H * s.W, B = sp.batch();
    switch (s.kind) {
        case kConvIn: {
            pack_latent(in[0].p, latent_f64, static_cast<long long>(sp.frames) * HW, sp.c_lat, 64, sc.a, st);
            if (sp.cfg)  // both CFG images start from the same latent (video: one latent per frame)
                CKD(cudaMemcpyAsync(sc.a + static_cast<long long>(HW) * 64, sc.a, static_cast<size_t>(HW) * 64 * 2,
                                    cudaMemcpyDeviceToDevice, st));
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_bf16 = static_cast<bf16*>(y);
            a.ldo = s.cout;
            tc_conv3x3(sc.a, P(stage, "conv.w"), B, s.H, s.W, 64, s.cout, a, st);
            break;
        }
        case kDown: {
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_bf16 = static_cast<bf16*>(y);
            a.ldo = s.cout;
            a.sub2 = 1;
            tc_conv3x3(in[0].p, P(stage, "conv.w"), B, s.H, s.W, s.cin, s.cout, a, st);
            break;
        }
        case kUp: {
            upsample2x(static_cast<const bf16*>(in[0].p), B, s.H, s.W, s.cin, sc.a, st);
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_bf16 = static_cast<bf16*>(y);
            a.ldo = s.cout;
            tc_conv3x3(sc.a, P(stage, "conv.w"), B, 2 * s.H, 2 * s.W, s.cin, s.cout, a, st);
            break;
        }
        case kOut: {
            if (latent_f64) throw std::invalid_argument("unet: the UNet family runs in f32 trajectory precision");
            const bf16* x = static_cast<const bf16*>(in[0].p);
            gn_images(Cat2{x, s.cin, nullptr, 0}, HW, F(stage, "gn.gamma"), F(stage, "gn.beta"), 1e-5f, 1, sc.a, sc, st);
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_f32 = sp.cfg ? sc.eps2 : static_cast<float*>(y);  // video: every frame's eps
            a.ldo = sp.c_lat;
            a.n_store = sp.c_lat;
            tc_conv3x3(sc.a, P(stage, "conv.w"), B, s.H, s.W, s.cin, 32, a, st);
            if (sp.cfg)
                cfg_combine(sc.eps2, static_cast<long long>(HW) * sp.c_lat, sp.cfg_scale, static_cast<float*>(y), st);
            break;
        }
        default: {  // resnet (+ transformer)
            const int C = s.cout, cin = s.cin + s.cskip;
            const bf16* x0 = static_cast<const bf16*>(in[0].p);
            const bf16* x1 = s.cskip ? static_cast<const bf16*>(in[1].p) : nullptr;
            gn_images(Cat2{x0, s.cin, x1, s.cskip}, HW, F(stage, "gn1.gamma"), F(stage, "gn1.beta"), 1e-5f, 1, sc.a, sc,
                      st);
            TcArgs c1;
            c1.bias = F(stage, "conv1.b");
            c1.chan_add = st_[stage].chan_add + static_cast<long long>(t) * C;
            c1.chan_add_shared = 1;  // one timestep for every image of the batch
            c1.out_bf16 = sc.b;
            c1.ldo = C;
            tc_conv3x3(sc.a, P(stage, "conv1.w"), B, s.H, s.W, cin, C, c1, st);
            gn_images(Cat2{sc.b, C, nullptr, 0}, HW, F(stage, "gn2.gamma"), F(stage, "gn2.beta"), 1e-5f, 1, sc.a, sc, st);
            const bf16* res = x0;
            if (cin != C) {
                TcArgs sh;
                sh.bias = F(stage, "short.b");
                sh.out_bf16 = sc.r;
                sh.ldo = C;
                static const bool cat_gemm = [] {  // ADX_CAT_GEMM=0: materialise the concat (A/B)
                    const char* e = getenv("ADX_CAT_GEMM");
                    return !(e && *e == '0');
                }();
                if (cat_gemm && s.cskip && s.cin % 64 == 0 && s.cskip % 64 == 0)  // [x | skip] in place along K
                    tc_gemm_cat(x0, s.cin, x1, s.cskip, P(stage, "short.w"), B * HW, C, sh, st);
                else if (s.cskip) {
                    concat_channels(Cat2{x0, s.cin, x1, s.cskip}, static_cast<long long>(B) * HW, sc.c, st);
                    tc_gemm(sc.c, P(stage, "short.w"), B * HW, C, cin, sh, st);
                } else {
                    tc_gemm(x0, P(stage, "short.w"), B * HW, C, cin, sh, st);
                }
                res = sc.r;
            }
            TcArgs c2;
            c2.bias = F(stage, "conv2.b");
            c2.residual = res;
            c2.ldr = C;
            bf16* out = s.attn || s.motion ? sc.c : static_cast<bf16*>(y);
            c2.out_bf16 = out;
            c2.ldo = C;
            tc_conv3x3(sc.a, P(stage, "conv2.w"), B, s.H, s.W, C, C, c2, st);
            // resnet -> [spatial transformer] -> [temporal motion module]
            if (s.attn) transformer(stage, sc.c, s.H, s.W, C, s.motion ? sc.r : static_cast<bf16*>(y), st);
            if (s.motion) motion(stage, s.attn ? sc.r : sc.c, s.H, s.W, C, static_cast<bf16*>(y), st);
        }
    }
}

// ------------------------------------------------------------------ ADX_F32 mode
// Every contraction runs on the bf16 tcgen05 kernels as A'.W'^T with A' = [hi|hi|lo] and
// W' = [hi|lo|hi] concatenated along K (= hi.hi + hi.lo + lo.hi, fp32 accumulation in
// TMEM); activations, norms, softmax and residuals stay fp32.

void UNetDevice::gemm_x(UScratch& s, const float* x, int M, int K, const char* wname, int stage, int N, TcArgs a,
                        cudaStream_t st) {
    split3(x, M, K, K, K, 0, s.sa, st);
    tc_gemm(s.sa, P(stage, wname), M, N, 3 * K, a, st);
}

void UNetDevice::conv_x(UScratch& s, const float* x, int H, int W, int Cin, const char* wname, int stage, int Cout,
                        TcArgs a, cudaStream_t st) {
    const int B = d_.spec.batch();
    split3(x, static_cast<long long>(B) * H * W, Cin, Cin, Cin, 0, s.sa, st);
    tc_conv3x3(s.sa, P(stage, wname), B, H, W, 3 * Cin, Cout, a, st);
}

// unfused attention, one 64-wide head at a time: S = Q'_h K'_h^T (K = 192), fp32 softmax in
// place, P' = split(P) along keys, O_h = P' V'_h^T (K = 3 * Lkp); ks = K' [Lk][3C] split per
// head (B pattern); V from fp32 v (transposed + split here) or pre-split vts [C][3 * Lkp]
void UNetDevice::attention_exact(UScratch& s, const float* q, long long ldq, const bf16* ks, const float* v,
                                 long long ldv, const bf16* vts, int L, int Lk, int C, float* out, cudaStream_t st) {
    const int Lkp = pad64(Lk);
    split3(q, L, C, ldq, 64, 0, s.sq, st);
    for (int h = 0; h < C / 64; ++h) {
        TcArgs a;
        a.out_f32 = s.S;
        a.ldo = Lkp;
        a.out_scale = 0.125f;
        tc_gemm_strided(s.sq + h * 192, 3LL * C, ks + h * 192, 3LL * C, L, Lk, 192, a, st);
        softmax_split_rows(s.S, Lkp, L, Lk, Lkp, s.sa, st);  // P' = split(softmax(S)), S read once
        const bf16* vt = vts ? vts + static_cast<long long>(h) * 64 * 3 * Lkp : s.sv;
        if (!vts) {
            transpose_f32(v + h * 64, ldv, Lk, Lkp, 64, s.fvt, st);
            split3(s.fvt, 64, Lkp, Lkp, Lkp, 1, s.sv, st);
        }
        TcArgs o;
        o.out_f32 = out + h * 64;
        o.ldo = C;
        tc_gemm(s.sa, vt, L, 64, 3 * Lkp, o, st);
    }
}

void UNetDevice::transformer_exact(int stage, const float* x, int H, int W, int C, float* y, cudaStream_t st) {
    UScratch& s = scratch(st);
    const UNetSpec& sp = d_.spec;
    const int L = H * W, B = sp.batch(), BL = B * L, depth = d_.st[stage - 1].attn;
    const long long img = static_cast<long long>(L) * C;
    static const bool fused = [] {  // ADX_F32_ATTN=unfused: S through HBM, one head at a time (A/B)
        const char* e = getenv("ADX_F32_ATTN");
        return !(e && std::string(e) == "unfused");
    }();
    gn_images(Cat2F{x, C, nullptr, 0}, L, F(stage, "tf.gn.gamma"), F(stage, "tf.gn.beta"), 1e-6f, 0, s.fa, s, st);
    TcArgs pi;
    pi.bias = F(stage, "tf.proj_in.b");
    pi.out_f32 = s.fb;
    pi.ldo = C;
    gemm_x(s, s.fa, BL, C, "tf.proj_in.w", stage, C, pi, st);  // h = fb
    for (int blk = 0; blk < depth; ++blk) {
        const std::string pre = blk == 0 ? "tf." : "tf.b" + std::to_string(blk) + ".";
        const std::string n_qkv = pre + "qkv.w", n_o1 = pre + "o1.w", n_q2 = pre + "q2.w", n_o2 = pre + "o2.w",
                          n_ff1 = pre + "ff1.w", n_ff2 = pre + "ff2.w";
        auto Fn = [&](const char* n) { return F(stage, (pre + n).c_str()); };
        layer_norm(s.fb, BL, C, Fn("ln1.gamma"), Fn("ln1.beta"), 1e-5f, s.fa, st);
        TcArgs qk;
        qk.out_f32 = s.fqkv;
        qk.ldo = 3 * C;
        gemm_x(s, s.fa, BL, C, n_qkv.c_str(), stage, 3 * C, qk, st);
        if (fused) {  // hi / lo planes of q | k | v, then every image and head in one launch
            bf16 *hi = s.sa, *lo = s.sa + 3 * BL * static_cast<long long>(C);
            split2(s.fqkv, 3LL * BL * C, hi, lo, st);
            tc_attention_x(hi, lo, 3LL * C, hi + C, lo + C, 3LL * C, hi + 2 * C, lo + 2 * C, 3LL * C, L, L, C, s.fatt,
                           C, st, s.attn_ws, s.attn_ws_bytes, B);
        } else {
            for (int b = 0; b < B; ++b) {
                const float* q = s.fqkv + b * 3 * img;
                split3(q + C, L, C, 3LL * C, 64, 1, s.sk, st);
                attention_exact(s, q, 3LL * C, s.sk, q + 2 * C, 3LL * C, nullptr, L, L, C, s.fatt + b * img, st);
            }
        }
        TcArgs o1;
        o1.bias = Fn("o1.b");
        o1.residual_f32 = s.fb;
        o1.ldr = C;
        o1.out_f32 = s.fb;
        o1.ldo = C;
        gemm_x(s, s.fatt, BL, C, n_o1.c_str(), stage, C, o1, st);
        layer_norm(s.fb, BL, C, Fn("ln2.gamma"), Fn("ln2.beta"), 1e-5f, s.fa, st);
        TcArgs q2;
        q2.out_f32 = s.fqkv;
        q2.ldo = C;
        gemm_x(s, s.fa, BL, C, n_q2.c_str(), stage, C, q2, st);
        if (fused) {
            bf16 *hi = s.sa, *lo = s.sa + BL * static_cast<long long>(C);
            split2(s.fqkv, static_cast<long long>(BL) * C, hi, lo, st);
            const long long pl = static_cast<long long>(pad64(sp.ctx_len)) * C;
            const int nimg = sp.contexts() == 1 ? 1 : B;  // one shared context: all B * L queries at once
            for (int b = 0; b < nimg; ++b) {
                const bf16* kv = st_[stage].kv2x[sp.contexts() == 1 ? blk : blk * B + b];
                tc_attention_x(hi + b * img, lo + b * img, C, kv, kv + pl, C, kv + 2 * pl, kv + 3 * pl, C,
                               nimg == 1 ? BL : L, sp.ctx_len, C, s.fatt + b * img, C, st, s.attn_ws,
                               s.attn_ws_bytes, 1);
            }
        } else {
            for (int b = 0; b < B; ++b) {
                const int ci = sp.contexts() == 1 ? blk : blk * B + b;  // video frames share one context
                attention_exact(s, s.fqkv + b * img, C, st_[stage].k2[ci], nullptr, 0, st_[stage].vt2[ci], L,
                                sp.ctx_len, C, s.fatt + b * img, st);
            }
        }
        TcArgs o2;
        o2.bias = Fn("o2.b");
        o2.residual_f32 = s.fb;
        o2.ldr = C;
        o2.out_f32 = s.fb;
        o2.ldo = C;
        gemm_x(s, s.fatt, BL, C, n_o2.c_str(), stage, C, o2, st);
        layer_norm(s.fb, BL, C, Fn("ln3.gamma"), Fn("ln3.beta"), 1e-5f, s.fa, st);
        TcArgs f1;
        f1.bias = Fn("ff1.b");
        f1.act = 2;  // GEGLU in the epilogue, fp32 out, 4C wide
        f1.out_f32 = s.fff;
        f1.ldo = 4 * C;
        gemm_x(s, s.fa, BL, C, n_ff1.c_str(), stage, 8 * C, f1, st);
        TcArgs f2;
        f2.bias = Fn("ff2.b");
        f2.residual_f32 = s.fb;
        f2.ldr = C;
        f2.out_f32 = s.fb;
        f2.ldo = C;
        gemm_x(s, s.fff, BL, 4 * C, n_ff2.c_str(), stage, C, f2, st);
    }
    TcArgs po;
    po.bias = F(stage, "tf.proj_out.b");
    po.residual_f32 = x;
    po.ldr = C;
    po.out_f32 = y;
    po.ldo = C;
    gemm_x(s, s.fb, BL, C, "tf.proj_out.w", stage, C, po, st);
}

void UNetDevice::enqueue_exact(int stage, const std::vector<Seg>& in, int t, void* y, bool latent_f64,
                               cudaStream_t st) {
    const UNetSpec& sp = d_.spec;
    const UStage& s = d_.st[stage - 1];
    UScratch& sc = scratch(st);
    const int HW = s.H * s.W, B = sp.batch();
    float* yf = static_cast<float*>(y);
    switch (s.kind) {
        case kConvIn: {
            pack_latent_f32(in[0].p, latent_f64, static_cast<long long>(sp.frames) * HW, sp.c_lat, 64, sc.fa, st);
            if (sp.cfg)
                CKD(cudaMemcpyAsync(sc.fa + static_cast<long long>(HW) * 64, sc.fa, static_cast<size_t>(HW) * 64 * 4,
                                    cudaMemcpyDeviceToDevice, st));
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_f32 = yf;
            a.ldo = s.cout;
            conv_x(sc, sc.fa, s.H, s.W, 64, "conv.w", stage, s.cout, a, st);
            break;
        }
        case kDown: {
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_f32 = yf;
            a.ldo = s.cout;
            a.sub2 = 1;
            conv_x(sc, static_cast<const float*>(in[0].p), s.H, s.W, s.cin, "conv.w", stage, s.cout, a, st);
            break;
        }
        case kUp: {
            // nearest 2x of fp32 = the bf16 copy kernel over twice the channel count
            upsample2x(static_cast<const bf16*>(in[0].p), B, s.H, s.W, 2 * s.cin, reinterpret_cast<bf16*>(sc.fa), st);
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_f32 = yf;
            a.ldo = s.cout;
            conv_x(sc, sc.fa, 2 * s.H, 2 * s.W, s.cin, "conv.w", stage, s.cout, a, st);
            break;
        }
        case kOut: {
            if (latent_f64) throw std::invalid_argument("unet: the UNet family runs in f32 trajectory precision");
            const float* x = static_cast<const float*>(in[0].p);
            gn_images(Cat2F{x, s.cin, nullptr, 0}, HW, F(stage, "gn.gamma"), F(stage, "gn.beta"), 1e-5f, 1, sc.fa, sc,
                      st);
            TcArgs a;
            a.bias = F(stage, "conv.b");
            a.out_f32 = sp.cfg ? sc.eps2 : yf;
            a.ldo = sp.c_lat;
            a.n_store = sp.c_lat;
            conv_x(sc, sc.fa, s.H, s.W, s.cin, "conv.w", stage, 32, a, st);
            if (sp.cfg) cfg_combine(sc.eps2, static_cast<long long>(HW) * sp.c_lat, sp.cfg_scale, yf, st);
            break;
        }
        default: {  // resnet (+ transformer)
            const int C = s.cout, cin = s.cin + s.cskip;
            const float* x0 = static_cast<const float*>(in[0].p);
            const float* x1 = s.cskip ? static_cast<const float*>(in[1].p) : nullptr;
            gn_images(Cat2F{x0, s.cin, x1, s.cskip}, HW, F(stage, "gn1.gamma"), F(stage, "gn1.beta"), 1e-5f, 1, sc.fa,
                      sc, st);
            TcArgs c1;
            c1.bias = F(stage, "conv1.b");
            c1.chan_add = st_[stage].chan_add + static_cast<long long>(t) * C;
            c1.chan_add_shared = 1;
            c1.out_f32 = sc.fb;
            c1.ldo = C;
            conv_x(sc, sc.fa, s.H, s.W, cin, "conv1.w", stage, C, c1, st);
            gn_images(Cat2F{sc.fb, C, nullptr, 0}, HW, F(stage, "gn2.gamma"), F(stage, "gn2.beta"), 1e-5f, 1, sc.fa, sc,
                      st);
            const float* res = x0;
            if (cin != C) {
                const float* xin = x0;
                if (s.cskip) {  // fp32 channel concat = the bf16 copy kernel over twice the channels
                    concat_channels(Cat2{reinterpret_cast<const bf16*>(x0), 2 * s.cin, reinterpret_cast<const bf16*>(x1),
                                         2 * s.cskip},
                                    static_cast<long long>(B) * HW, reinterpret_cast<bf16*>(sc.fc), st);
                    xin = sc.fc;
                }
                TcArgs sh;
                sh.bias = F(stage, "short.b");
                sh.out_f32 = sc.fr;
                sh.ldo = C;
                gemm_x(sc, xin, B * HW, cin, "short.w", stage, C, sh, st);
                res = sc.fr;
            }
            TcArgs c2;
            c2.bias = F(stage, "conv2.b");
            c2.residual_f32 = res;
            c2.ldr = C;
            float* out = s.attn || s.motion ? sc.fc : yf;
            c2.out_f32 = out;
            c2.ldo = C;
            conv_x(sc, sc.fa, s.H, s.W, C, "conv2.w", stage, C, c2, st);
            if (s.attn) transformer_exact(stage, sc.fc, s.H, s.W, C, s.motion ? sc.fr : yf, st);
            if (s.motion) motion_exact(stage, s.attn ? sc.fr : sc.fc, s.H, s.W, C, yf, st);
        }
    }
}

}  // namespace adx
