// capi.cpp -- extern "C" boundary of libasyncdiff_b200.so (include/asyncdiff_b200.h).
// Exceptions are mapped onto status codes per the reference's exception
// classes; the message text is kept for adx_last_error().
#include "../../include/asyncdiff_b200.h"

#include "engine.hpp"
#include "extras.hpp"
#include "host.hpp"
#include "schedule.hpp"
#include "tc_attn.cuh"
#include "tc_gemm.cuh"
#include "unet.hpp"
#include "unet_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>

struct adx_model {
    adx::Model m;
};
struct adx_partition {
    adx::Partition p;
};
struct adx_plan {
    adx::Plan p;
};
struct adx_engine {
    std::unique_ptr<adx::Engine> e;
};
struct adx_session {
    std::unique_ptr<adx::Session> s;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return ADX_OK;
    } catch (const adx::cuda_error& e) {
        g_err = e.what();
        return ADX_ERR_CUDA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return ADX_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return ADX_ERR_OUT_OF_RANGE;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return ADX_ERR_DOMAIN;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return ADX_ERR_LOGIC;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return ADX_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ADX_ERR_RUNTIME;
    } catch (...) {
        g_err = "unknown error";
        return ADX_ERR_RUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

#define CKC(x)                                                                                         \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess)                                                                         \
            throw adx::cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

// device scratch freed on scope exit
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { CKC(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
};

// fp64 host values <-> device elements of `eb` bytes (8: fp64, 4: fp32, 2: bf16 RNE)
void to_dev(int eb, const double* src, size_t n, std::vector<unsigned char>& out) {
    out.resize(n * eb);
    for (size_t i = 0; i < n; ++i) {
        if (eb == 8) {
            std::memcpy(&out[i * 8], &src[i], 8);
        } else if (eb == 4) {
            const float f = static_cast<float>(src[i]);
            std::memcpy(&out[i * 4], &f, 4);
        } else {
            const __nv_bfloat16 b = __float2bfloat16_rn(static_cast<float>(src[i]));
            std::memcpy(&out[i * 2], &b, 2);
        }
    }
}

void from_dev(int eb, const unsigned char* src, size_t n, double* dst) {
    if (eb == 8) {
        std::memcpy(dst, src, n * 8);
    } else if (eb == 4) {
        for (size_t i = 0; i < n; ++i) {
            float f;
            std::memcpy(&f, src + i * 4, 4);
            dst[i] = f;
        }
    } else {
        for (size_t i = 0; i < n; ++i) {
            __nv_bfloat16 b;
            std::memcpy(&b, src + i * 2, 2);
            dst[i] = __bfloat162float(b);
        }
    }
}

// Device run of stages [first, last] (run_stage_range, denoiser.cpp:150-192)
// on the engine's first ordinal.  `skips` holds features by link; produced
// features are written back into it.  Returns the last stage's output.
std::vector<double> run_range_device(adx::Engine& E, int first, int last, const std::vector<double>& cur,
                                     std::map<std::pair<int, int>, std::vector<double>>& skips, int t_embed,
                                     bool stage1_latent) {
    const adx::Model& m = E.model();
    const int prec = E.prec();
    // latent / eps elements (act_bytes) vs stage-output elements (stage_bytes: bf16 UNet
    // activations in the bf16 mode) -- the stage kernels read and write the latter
    const int ab = adx::act_bytes(prec), sb = E.stage_bytes();
    auto out_bytes = [&](int stage) { return stage == m.L ? ab : sb; };
    CKC(cudaSetDevice(E.ordinal(0)));
    for (int i = first; i <= last; ++i) E.stage_on(0, i);
    E.ensure_tables(0, std::max(t_embed, 1));
    if (t_embed < 0) throw std::out_of_range("eval: embedding timestep " + std::to_string(t_embed) + " < 0");
    cudaStream_t st;
    CKC(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } sg{st};
    std::vector<unsigned char> tmp;
    auto upload = [&](const std::vector<double>& v, int eb) {
        DevBuf b(v.size() * eb);
        to_dev(eb, v.data(), v.size(), tmp);
        CKC(cudaMemcpy(b.p, tmp.data(), tmp.size(), cudaMemcpyHostToDevice));
        return b;
    };
    DevBuf bad(2 * sizeof(int));
    CKC(cudaMemset(bad.p, 0x7f, 2 * sizeof(int)));
    DevBuf cur_d = upload(cur, stage1_latent ? ab : out_bytes(first - 1));
    std::map<int, DevBuf> y;      // stage outputs
    std::map<std::pair<int, int>, DevBuf> skip_d;
    std::vector<DevBuf> hs;
    int cur_n = static_cast<int>(cur.size());
    const void* cur_p = cur_d.p;
    for (int i = first; i <= last; ++i) {
        std::vector<adx::Seg> in;
        if (i == first && stage1_latent) {
            // stage 1 consumes concat(x, e_t): the e_t part comes from the device table
            in.push_back({cur_p, m.data_dim()});
            in.push_back({E.etab_row(0, t_embed), m.E});
            if (cur_n != m.data_dim() + m.E)
                throw std::runtime_error("eval: stage 1 input width " + std::to_string(cur_n) + " != expected " +
                                         std::to_string(m.stages[0].in));
        } else {
            in.push_back({cur_p, cur_n});
        }
        for (auto& l : m.links_into(i)) {
            if (l.first >= first && y.count(l.first)) {
                in.push_back({y.at(l.first).p, m.widths[l.first]});
                continue;
            }
            auto it = skips.find(l);
            if (it == skips.end())
                throw std::runtime_error("eval: missing skip feature for link (" + std::to_string(l.first) + " -> " +
                                         std::to_string(l.second) + ")");
            if (!skip_d.count(l)) skip_d.emplace(l, upload(it->second, out_bytes(l.first)));
            in.push_back({skip_d.at(l).p, static_cast<int>(it->second.size())});
        }
        DevBuf h(static_cast<size_t>(m.stages[i - 1].hidden) * ab);
        DevBuf yo(static_cast<size_t>(m.stages[i - 1].out) * ab);
        E.enqueue_stage(0, i, in, t_embed, h.p, yo.p, static_cast<int*>(bad.p), i, st, true);
        cur_p = yo.p;
        cur_n = m.stages[i - 1].out;
        hs.push_back(std::move(h));
        y.emplace(i, std::move(yo));
    }
    CKC(cudaStreamSynchronize(st));
    int flags[2];
    CKC(cudaMemcpy(flags, bad.p, sizeof flags, cudaMemcpyDeviceToHost));
    if (flags[0] != 0x7f7f7f7f) throw std::domain_error("eval: non-finite activation at stage " + std::to_string(flags[0]));
    auto down = [&](int stage) {
        const int n = m.widths[stage];
        std::vector<unsigned char> h(static_cast<size_t>(n) * out_bytes(stage));
        CKC(cudaMemcpy(h.data(), y.at(stage).p, h.size(), cudaMemcpyDeviceToHost));
        std::vector<double> out(n);
        from_dev(out_bytes(stage), h.data(), n, out.data());
        return out;
    };
    for (int i = first; i <= last; ++i)
        for (auto& l : m.links_out_of(i)) skips[l] = down(i);
    return down(last);
}

void fill_stats(const adx::RunStatsOut& s, adx_run_stats* o) {
    if (!o) return;
    o->broadcast_count = s.broadcast_count;
    o->n_rounds = static_cast<int>(s.round_wall_s.size());
    o->warmup_wall_s = s.warmup_wall_s;
    o->total_wall_s = s.total_wall_s;
    for (size_t i = 0; i < s.round_wall_s.size(); ++i) {
        if (o->round_wall_s) o->round_wall_s[i] = s.round_wall_s[i];
        if (o->round_comm_s) o->round_comm_s[i] = s.round_comm_s[i];
    }
    for (size_t i = 0; i < s.store_entries.size(); ++i)
        if (o->store_entries_per_round) o->store_entries_per_round[i] = s.store_entries[i];
    for (size_t i = 0; i < s.device_busy_s.size(); ++i) {
        if (o->device_busy_s) o->device_busy_s[i] = s.device_busy_s[i];
        if (o->device_evals) o->device_evals[i] = s.device_evals[i];
    }
}

adx::RunOptions to_opts(const adx_run_options* o) {
    adx::RunOptions r;
    if (!o) return r;
    r.round_timeout_s = o->round_timeout_s;
    if (o->max_jitter_s < 0.0) throw std::invalid_argument("RunOptions: max_jitter_s must be >= 0");
    r.jitter_seed = o->jitter_seed;
    r.max_jitter_s = o->max_jitter_s;
    if (o->segment_delay_s && o->n_delays > 0) {
        r.segment_delay_s.assign(o->segment_delay_s, o->segment_delay_s + o->n_delays);
        for (double d : r.segment_delay_s)
            if (d < 0.0) throw std::invalid_argument("inject_delay: delays must be >= 0");
    }
    r.use_graph = o->use_graph != 0;
    r.instrument = o->instrument != 0;
    return r;
}

}  // namespace

// time `iters` back-to-back launches of fn(stream) replayed from one CUDA graph
// (no host launch overhead between kernels), after one warm replay
template <typename Fn>
static double time_graph_ms(Fn fn, int iters) {
    cudaStream_t st;
    CKC(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaGraph_t g;
    CKC(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) fn(st);
    CKC(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t ge;
    CKC(cudaGraphInstantiate(&ge, g, 0));
    CKC(cudaGraphLaunch(ge, st));
    cudaEvent_t e0, e1;
    CKC(cudaEventCreate(&e0));
    CKC(cudaEventCreate(&e1));
    CKC(cudaEventRecord(e0, st));
    CKC(cudaGraphLaunch(ge, st));
    CKC(cudaEventRecord(e1, st));
    CKC(cudaEventSynchronize(e1));
    float ms = 0;
    CKC(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    return ms / iters;
}

extern "C" {

const char* adx_last_error(void) { return g_err.c_str(); }
int adx_version(void) { return 100; }
int adx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int adx_random_normals(uint64_t seed, long long n, double* out) {
    return guard([&] {
        if (n < 0 || (n > 0 && !out)) throw std::invalid_argument("random_normals: bad output");
        adx::Rng r(seed);
        for (long long i = 0; i < n; ++i) out[i] = r.normal();
    });
}

int adx_build_schedule(int T, double beta_start, double beta_end, int kind, double* betas, double* alphas,
                       double* alpha_bars) {
    return guard([&] {
        std::vector<double> b, a, ab;
        adx::build_schedule(T, beta_start, beta_end, kind, b, a, ab);
        if (betas) std::memcpy(betas, b.data(), b.size() * 8);
        if (alphas) std::memcpy(alphas, a.data(), a.size() * 8);
        if (alpha_bars) std::memcpy(alpha_bars, ab.data(), ab.size() * 8);
    });
}

int adx_ddim_step(int ordinal, int precision, const double* x, const double* eps, int d, int t,
                  const double* alpha_bars, int T, double* out) {
    return guard([&] {
        need(x, "ddim_step");
        need(eps, "ddim_step");
        need(alpha_bars, "ddim_step");
        need(out, "ddim_step");
        if (t < 1 || t > T)
            throw std::out_of_range("predict_x0: t=" + std::to_string(t) + " outside [1, " + std::to_string(T) + "]");
        if (precision < 0 || precision > 2) throw std::invalid_argument("ddim_step: bad precision");
        CKC(cudaSetDevice(ordinal));
        const int ab = adx::act_bytes(precision);
        DevBuf xd(static_cast<size_t>(d) * ab), ed(static_cast<size_t>(d) * ab), od(static_cast<size_t>(d) * ab),
            bad(2 * sizeof(int));
        std::vector<unsigned char> tmp;
        to_dev(adx::act_bytes(precision), x, d, tmp);
        CKC(cudaMemcpy(xd.p, tmp.data(), tmp.size(), cudaMemcpyHostToDevice));
        to_dev(adx::act_bytes(precision), eps, d, tmp);
        CKC(cudaMemcpy(ed.p, tmp.data(), tmp.size(), cudaMemcpyHostToDevice));
        CKC(cudaMemset(bad.p, 0x7f, 2 * sizeof(int)));
        adx::DdimArgs a = {};
        a.x = xd.p;
        a.eps = ed.p;
        a.out = od.p;
        a.d = d;
        a.s1 = std::sqrt(1.0 - alpha_bars[t]);
        a.s2 = std::sqrt(alpha_bars[t]);
        a.s3 = std::sqrt(alpha_bars[t - 1]);
        a.s4 = std::sqrt(1.0 - alpha_bars[t - 1]);
        a.bad = static_cast<int*>(bad.p);
        a.bad_key = 0;
        adx::launch_ddim(precision, a, 0);
        CKC(cudaDeviceSynchronize());
        int flags[2];
        CKC(cudaMemcpy(flags, bad.p, sizeof flags, cudaMemcpyDeviceToHost));
        if (flags[0] != 0x7f7f7f7f) throw std::domain_error("predict_x0: non-finite eps at t=" + std::to_string(t));
        tmp.resize(static_cast<size_t>(d) * ab);
        CKC(cudaMemcpy(tmp.data(), od.p, tmp.size(), cudaMemcpyDeviceToHost));
        from_dev(adx::act_bytes(precision), tmp.data(), d, out);
    });
}

// ---------------------------------------------------------------- model
int adx_model_build_toy(int L, const int* widths, int n_widths, int skip_spec, uint64_t seed, int E,
                        adx_model** out) {
    return guard([&] {
        need(widths, "build_toy_denoiser");
        need(out, "build_toy_denoiser");
        std::vector<int> w(widths, widths + n_widths);
        auto* h = new adx_model{adx::build_toy_denoiser(L, w, skip_spec, seed, E)};
        *out = h;
    });
}

int adx_model_shell(int L, const int* widths, int n_widths, const int* link_pairs, int n_links, int E,
                    adx_model** out) {
    return guard([&] {
        need(widths, "make_denoiser_shell");
        need(out, "make_denoiser_shell");
        std::vector<int> w(widths, widths + n_widths);
        std::vector<std::pair<int, int>> links;
        for (int k = 0; k < n_links; ++k) links.emplace_back(link_pairs[2 * k], link_pairs[2 * k + 1]);
        *out = new adx_model{adx::make_denoiser_shell(L, w, links, E)};
    });
}

void adx_model_destroy(adx_model* m) { delete m; }

int adx_model_info(const adx_model* m, int* L, int* E, int* n_links) {
    return guard([&] {
        need(m, "model_info");
        if (L) *L = m->m.L;
        if (E) *E = m->m.E;
        if (n_links) *n_links = static_cast<int>(m->m.links.size());
    });
}

int adx_model_widths(const adx_model* m, int* out) {
    return guard([&] {
        need(m, "model_widths");
        std::memcpy(out, m->m.widths.data(), m->m.widths.size() * sizeof(int));
    });
}

int adx_model_links(const adx_model* m, int* out) {
    return guard([&] {
        need(m, "model_links");
        for (size_t k = 0; k < m->m.links.size(); ++k) {
            out[2 * k] = m->m.links[k].first;
            out[2 * k + 1] = m->m.links[k].second;
        }
    });
}

int adx_model_stage_shape(const adx_model* m, int stage, int* in, int* hidden, int* out, long long* macs) {
    return guard([&] {
        need(m, "stage_shape");
        if (stage < 1 || stage > m->m.L) throw std::out_of_range("stage " + std::to_string(stage) + " out of range");
        const adx::Stage& s = m->m.stages[stage - 1];
        if (in) *in = s.in;
        if (hidden) *hidden = s.hidden;
        if (out) *out = s.out;
        if (macs) *macs = s.cost_macs;
    });
}

int adx_model_set_stage_macs(adx_model* m, int stage, long long macs) {
    return guard([&] {
        need(m, "set_stage_macs");
        if (stage < 1 || stage > m->m.L) throw std::out_of_range("stage " + std::to_string(stage) + " out of range");
        m->m.stages[stage - 1].cost_macs = macs;
    });
}

int adx_model_tensor(adx_model* m, int stage, int which, double** data, int* rows, int* cols) {
    return guard([&] {
        need(m, "model_tensor");
        adx::Model& M = m->m;
        M.version++;
        if (which == ADX_T_PROJ) {
            *data = M.proj.data();
            *rows = M.E;
            *cols = M.E;
            return;
        }
        if (stage < 1 || stage > M.L) throw std::out_of_range("stage " + std::to_string(stage) + " out of range");
        adx::Stage& s = M.stages[stage - 1];
        switch (which) {
            case ADX_T_W1: *data = s.w1.data(); *rows = s.hidden; *cols = s.in; break;
            case ADX_T_B1: *data = s.b1.data(); *rows = s.hidden; *cols = 1; break;
            case ADX_T_TIN: *data = s.tin.data(); *rows = s.hidden; *cols = M.E; break;
            case ADX_T_W2: *data = s.w2.data(); *rows = s.out; *cols = s.hidden; break;
            case ADX_T_B2: *data = s.b2.data(); *rows = s.out; *cols = 1; break;
            default: throw std::invalid_argument("model_tensor: unknown tensor id");
        }
    });
}

int adx_sinusoid(int t, int dim, double* out) {
    return guard([&] {
        auto s = adx::sinusoid(t, dim);
        std::memcpy(out, s.data(), s.size() * 8);
    });
}

// ------------------------------------------------------------ partition
int adx_partition_balanced(const adx_model* m, int N, int strategy, adx_partition** out) {
    return guard([&] {
        need(m, "partition_balanced");
        *out = new adx_partition{adx::partition_balanced(m->m, N, strategy)};
    });
}

int adx_partition_by_cost(const adx_model* m, int N, const double* stage_cost, adx_partition** out) {
    return guard([&] {
        need(m, "partition_by_cost");
        std::vector<long long> c(m->m.L);
        for (int i = 0; i < m->m.L; ++i) c[i] = std::llround(stage_cost[i] * 1e6);  // micro-units: exact ints
        *out = new adx_partition{adx::partition_by_cost(m->m, N, c)};
    });
}

int adx_partition_create(int n_segments, const int* seg_sizes, const int* stages, const int* devices,
                         const long long* macs, int strategy, adx_partition** out) {
    return guard([&] {
        adx::Partition p;
        p.strategy = strategy;
        int pos = 0;
        for (int n = 0; n < n_segments; ++n) {
            std::vector<int> st(stages + pos, stages + pos + seg_sizes[n]);
            pos += seg_sizes[n];
            p.segments.push_back(st);
            p.device_of_segment.push_back(devices ? devices[n] : n);
            p.segment_macs.push_back(macs ? macs[n] : 0);
        }
        *out = new adx_partition{p};
    });
}

void adx_partition_destroy(adx_partition* p) { delete p; }
int adx_partition_num_segments(const adx_partition* p) { return p ? p->p.num_segments() : 0; }
int adx_partition_strategy(const adx_partition* p) { return p ? p->p.strategy : 0; }

int adx_partition_segment(const adx_partition* p, int seg, int* stages, int cap, int* n_stages, long long* macs,
                          int* device) {
    return guard([&] {
        need(p, "partition_segment");
        if (seg < 1 || seg > p->p.num_segments())
            throw std::out_of_range("partition_segment: segment " + std::to_string(seg) + " out of range");
        const auto& s = p->p.segments[seg - 1];
        if (n_stages) *n_stages = static_cast<int>(s.size());
        for (size_t i = 0; i < s.size() && static_cast<int>(i) < cap; ++i) stages[i] = s[i];
        if (macs) *macs = p->p.segment_macs[seg - 1];
        if (device) *device = p->p.device_of_segment[seg - 1];
    });
}

int adx_partition_contiguous(const adx_partition* p) { return p && p->p.contiguous() ? 1 : 0; }

int adx_partition_segment_of_stage(const adx_partition* p, int stage, int* seg) {
    return guard([&] {
        need(p, "segment_of_stage");
        *seg = p->p.segment_of_stage(stage);
    });
}

int adx_partition_validate(const adx_partition* p, const adx_model* m) {
    return guard([&] {
        need(p, "partition_validate");
        need(m, "partition_validate");
        p->p.validate(m->m);
    });
}

int adx_crossing_links(const adx_model* m, const adx_partition* p, int* out_pairs, int cap, int* n_links) {
    return guard([&] {
        need(m, "crossing_links");
        need(p, "crossing_links");
        auto c = adx::crossing_links(m->m, p->p);
        *n_links = static_cast<int>(c.size());
        for (size_t k = 0; k < c.size() && static_cast<int>(k) < cap; ++k) {
            out_pairs[2 * k] = c[k].first;
            out_pairs[2 * k + 1] = c[k].second;
        }
    });
}

// ----------------------------------------------------------------- plan
int adx_plan_async(int T, int w, int N, int S, int time_shift, adx_plan** out) {
    return guard([&] { *out = new adx_plan{adx::plan_async(T, w, N, S, time_shift != 0)}; });
}

int adx_plan_from_flat(const int* flat, int len, adx_plan** out) {
    return guard([&] { *out = new adx_plan{adx::plan_from_flat(flat, len)}; });
}

int adx_plan_to_flat(const adx_plan* p, int* out, int cap, int* len) {
    return guard([&] {
        need(p, "plan_to_flat");
        auto f = adx::plan_to_flat(p->p);
        *len = static_cast<int>(f.size());
        if (static_cast<int>(f.size()) > cap) throw std::invalid_argument("plan_to_flat: buffer too small");
        std::memcpy(out, f.data(), f.size() * sizeof(int));
    });
}

void adx_plan_destroy(adx_plan* p) { delete p; }

int adx_plan_validate(const adx_plan* p, char* buf, int cap, int* n_violations) {
    return guard([&] {
        need(p, "validate_plan");
        auto v = adx::validate_plan(p->p);
        std::string joined;
        for (size_t i = 0; i < v.size(); ++i) joined += (i ? "\n" : "") + v[i];
        if (n_violations) *n_violations = static_cast<int>(v.size());
        if (buf && cap > 0) {
            std::strncpy(buf, joined.c_str(), cap - 1);
            buf[cap - 1] = 0;
        }
    });
}

int adx_plan_counts(const adx_plan* p, const adx_partition* part, adx_plan_counts_t* out,
                    long long* evals_per_segment, long long* per_device_macs) {
    return guard([&] {
        need(p, "plan_counts");
        need(part, "plan_counts");
        auto c = adx::plan_counts(p->p, part->p);
        if (out) {
            out->broadcasts_paper_convention = c.broadcasts_paper_convention;
            out->broadcasts_strictly_needed = c.broadcasts_strictly_needed;
            out->device_count = c.device_count;
            out->max_device_macs = c.max_device_macs;
            out->sequential_total_macs = c.sequential_total_macs;
        }
        if (evals_per_segment)
            std::memcpy(evals_per_segment, c.evals_per_segment.data(), c.evals_per_segment.size() * 8);
        if (per_device_macs) std::memcpy(per_device_macs, c.per_device_macs.data(), c.per_device_macs.size() * 8);
    });
}

int adx_shift_embeddings(const int* ts, int n, int w, int* out) {
    return guard([&] {
        auto r = adx::shift_embeddings(std::vector<int>(ts, ts + n), w);
        std::memcpy(out, r.data(), r.size() * sizeof(int));
    });
}

int adx_render_plan(const adx_plan* p, char* buf, int cap, int* len) {
    return guard([&] {
        need(p, "render_plan");
        auto s = adx::render_plan(p->p);
        if (len) *len = static_cast<int>(s.size());
        if (buf && cap > 0) {
            std::strncpy(buf, s.c_str(), cap - 1);
            buf[cap - 1] = 0;
        }
    });
}

// ----------------------------------------------------------------- engine
int adx_engine_create(const adx_model* m, int precision, const int* ordinals, int n_ordinals, adx_engine** out) {
    return guard([&] {
        need(m, "engine_create");
        std::vector<int> o;
        if (ordinals && n_ordinals > 0)
            o.assign(ordinals, ordinals + n_ordinals);
        else
            o.push_back(0);
        *out = new adx_engine{std::make_unique<adx::Engine>(m->m, precision, o)};
    });
}

void adx_engine_destroy(adx_engine* e) { delete e; }

int adx_engine_weight_bytes(const adx_engine* e, int idx, long long* bytes) {
    return guard([&] {
        need(e, "engine_weight_bytes");
        *bytes = e->e->weight_bytes_resident(idx);
    });
}

int adx_bench_gemv(int ordinal, int precision, int n, int chain, int iters, int pdl, double* ms_per_gemv) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        *ms_per_gemv = adx::bench_gemv_chain(precision, n, chain, iters, pdl != 0);
    });
}

int adx_engine_time_eval(adx_engine* e, int t_embed, int iters, double* ms_per_pass, long long* bytes_per_pass,
                         int* launches_per_pass) {
    return guard([&] {
        need(e, "engine_time_eval");
        const adx::Model& m = e->e->model();
        long long b = 0;
        for (int i = 1; i <= m.L; ++i) b += static_cast<long long>(e->e->stage_weight_bytes(i));
        if (bytes_per_pass) *bytes_per_pass = b;
        *ms_per_pass = e->e->time_eval_ms(0, t_embed, iters, launches_per_pass);
    });
}

int adx_engine_stage_times(adx_engine* e, int t_embed, int iters, double* stage_ms) {
    return guard([&] {
        need(e, "engine_stage_times");
        e->e->time_eval_ms(0, t_embed, std::max(1, iters), nullptr, nullptr, stage_ms);
    });
}

int adx_engine_profile_pass(adx_engine* e, int t_embed, double* out9) {
    return guard([&] {
        need(e, "engine_profile_pass");
        double prof[3][3];
        e->e->time_eval_ms(0, t_embed, 1, nullptr, prof);
        for (int k = 0; k < 3; ++k)
            for (int j = 0; j < 3; ++j) out9[3 * k + j] = prof[k][j];
    });
}

int adx_profile_records(double* out, int cap, int* n) {
    return guard([&] {
        if (!n) throw std::invalid_argument("profile_records: n is null");
        *n = adx::tc_profile_records(out, out ? cap : 0);
    });
}

int adx_eval_full(adx_engine* e, const double* x, int t_embed, double* eps_out) {
    return guard([&] {
        need(e, "eval_full");
        const adx::Model& m = e->e->model();
        std::vector<double> cur(x, x + m.data_dim());
        cur.resize(m.data_dim() + m.E, 0.0);
        std::map<std::pair<int, int>, std::vector<double>> skips;
        auto y = run_range_device(*e->e, 1, m.L, cur, skips, t_embed, true);
        std::memcpy(eps_out, y.data(), y.size() * 8);
    });
}

int adx_eval_segment(adx_engine* e, const adx_partition* p, int seg, const double* input, int input_len,
                     int input_is_latent, int produced_by, const int* skip_links, const double* skip_vals,
                     int n_skips, int t_embed, double* out, int out_cap, int* out_len, int* out_is_eps,
                     int* out_links, double* out_vals, int cap_links, int cap_vals, int* n_out_links) {
    return guard([&] {
        need(e, "eval_segment");
        need(p, "eval_segment");
        const adx::Model& m = e->e->model();
        const adx::Partition& P = p->p;
        // require_sequential_segment (denoiser.cpp:194-202)
        if (seg < 1 || seg > P.num_segments())
            throw std::invalid_argument("eval_segment: segment " + std::to_string(seg) + " outside [1, " +
                                        std::to_string(P.num_segments()) + "]");
        if (!P.contiguous())
            throw std::invalid_argument(
                "eval_segment: partition is not a contiguous cascade (first-last-grouped partitions are "
                "placement/costing only)");
        if (input_is_latent && seg != 1)
            throw std::invalid_argument("eval_segment: segment " + std::to_string(seg) +
                                        " requires a HiddenBundle input, not a Latent");
        if (!input_is_latent && seg == 1)
            throw std::invalid_argument("eval_segment: segment 1 requires a Latent input");
        if (!input_is_latent && produced_by != seg - 1)
            throw std::invalid_argument("eval_segment: segment " + std::to_string(seg) + " needs a bundle from segment " +
                                        std::to_string(seg - 1) + ", got one from segment " +
                                        std::to_string(produced_by));
        std::map<std::pair<int, int>, std::vector<double>> skips;
        int pos = 0;
        for (int k = 0; k < n_skips; ++k) {
            const std::pair<int, int> l(skip_links[2 * k], skip_links[2 * k + 1]);
            if (l.first < 1 || l.first > m.L) throw std::invalid_argument("eval_segment: bad skip link");
            const int w = m.widths[l.first];
            skips[l] = std::vector<double>(skip_vals + pos, skip_vals + pos + w);
            pos += w;
        }
        std::vector<double> cur(input, input + input_len);
        if (input_is_latent) cur.resize(input_len + m.E, 0.0);
        const auto& range = P.segments[seg - 1];
        auto y = run_range_device(*e->e, range.front(), range.back(), cur, skips, t_embed, input_is_latent != 0);
        if (static_cast<int>(y.size()) > out_cap) throw std::invalid_argument("eval_segment: output buffer too small");
        std::memcpy(out, y.data(), y.size() * 8);
        *out_len = static_cast<int>(y.size());
        *out_is_eps = seg == P.num_segments() ? 1 : 0;
        // finish_segment (denoiser.cpp:204-218): crossing links produced in-segment
        int nl = 0, vp = 0;
        if (!*out_is_eps) {
            for (auto& [l, f] : skips)
                if (l.first >= range.front() && l.first <= range.back() && l.second > range.back()) {
                    if (nl >= cap_links || vp + static_cast<int>(f.size()) > cap_vals)
                        throw std::invalid_argument("eval_segment: skip output buffer too small");
                    out_links[2 * nl] = l.first;
                    out_links[2 * nl + 1] = l.second;
                    std::memcpy(out_vals + vp, f.data(), f.size() * 8);
                    vp += static_cast<int>(f.size());
                    ++nl;
                }
        }
        *n_out_links = nl;
    });
}

void adx_run_options_default(adx_run_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->round_timeout_s = 30.0;
    o->use_graph = 1;
}

int adx_session_create(adx_engine* e, const adx_plan* plan, const adx_partition* part, const double* alpha_bars,
                       int T, int mode, int workers, const adx_run_options* opts, adx_session** out) {
    return guard([&] {
        need(e, "session_create");
        need(alpha_bars, "session_create");
        std::vector<double> ab(alpha_bars, alpha_bars + T + 1);
        adx::Plan pl = plan ? plan->p : adx::Plan();
        adx::Partition pa = part ? part->p : adx::Partition();
        if (mode != ADX_MODE_SEQUENTIAL) {
            need(plan, "session_create(plan)");
            need(part, "session_create(partition)");
        }
        *out = new adx_session{std::make_unique<adx::Session>(e->e.get(), pl, pa, ab, mode, workers, to_opts(opts))};
    });
}

void adx_session_destroy(adx_session* s) { delete s; }

int adx_session_run(adx_session* s, const double* x_T, double* lat, double* eps, adx_run_stats* stats) {
    return guard([&] {
        need(s, "session_run");
        need(x_T, "session_run");
        adx::RunStatsOut st;
        s->s->run(x_T, lat, eps, &st);
        fill_stats(st, stats);
    });
}

int adx_session_upload(adx_session* s, const double* x_T) {
    return guard([&] {
        need(s, "session_upload");
        s->s->upload(x_T);
    });
}

int adx_session_time(adx_session* s, int iters, double* ms) {
    return guard([&] {
        need(s, "session_time");
        *ms = s->s->time_runs(iters);
    });
}

int adx_session_kernel_count(const adx_session* s, int* n) {
    return guard([&] {
        need(s, "session_kernel_count");
        *n = s->s->kernel_count();
    });
}

int adx_session_weight_bytes(const adx_session* s, long long* bytes) {
    return guard([&] {
        need(s, "session_weight_bytes");
        *bytes = s->s->weight_bytes_per_run();
    });
}

int adx_session_download(adx_session* s, double* lat, double* eps) {
    return guard([&] {
        need(s, "session_download");
        s->s->download(lat, eps);
    });
}

static int run_mode(adx_engine* e, const adx_plan* plan, const adx_partition* part, const double* x_T,
                    const double* ab, int T, int mode, int workers, const adx_run_options* opts, double* lat,
                    double* eps, adx_run_stats* stats) {
    adx_session* s = nullptr;
    int rc = adx_session_create(e, plan, part, ab, T, mode, workers, opts, &s);
    if (rc) return rc;
    rc = adx_session_run(s, x_T, lat, eps, stats);
    adx_session_destroy(s);
    return rc;
}

int adx_run_serial(adx_engine* e, const adx_plan* plan, const adx_partition* part, const double* x_T,
                   const double* alpha_bars, int T, const adx_run_options* opts, double* lat, double* eps,
                   adx_run_stats* stats) {
    return run_mode(e, plan, part, x_T, alpha_bars, T, ADX_MODE_SERIAL, 1, opts, lat, eps, stats);
}

int adx_run_parallel(adx_engine* e, const adx_plan* plan, const adx_partition* part, const double* x_T,
                     const double* alpha_bars, int T, int workers, const adx_run_options* opts, double* lat,
                     double* eps, adx_run_stats* stats) {
    return run_mode(e, plan, part, x_T, alpha_bars, T, ADX_MODE_PARALLEL, workers, opts, lat, eps, stats);
}

int adx_sequential_denoise(adx_engine* e, const double* x_T, const double* alpha_bars, int T, double* lat,
                           double* eps) {
    return run_mode(e, nullptr, nullptr, x_T, alpha_bars, T, ADX_MODE_SEQUENTIAL, 1, nullptr, lat, eps, nullptr);
}

int adx_compare_trajectories(const double* a, const double* b, int n, int d, double* per, double* final_mse,
                             double* final_max_abs) {
    return guard([&] {
        double last = 0.0;
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int k = 0; k < d; ++k) {
                const double df = a[static_cast<size_t>(i) * d + k] - b[static_cast<size_t>(i) * d + k];
                s += df * df;
            }
            last = s / d;
            if (per) per[i] = last;
        }
        if (final_mse) *final_mse = last;
        double mx = 0.0;
        for (int k = 0; k < d; ++k)
            mx = std::max(mx, std::fabs(a[static_cast<size_t>(n - 1) * d + k] - b[static_cast<size_t>(n - 1) * d + k]));
        if (final_max_abs) *final_max_abs = mx;
    });
}

// ----------------------------------------------------- one process per GPU
int adx_rank_program(const adx_plan* plan, const adx_partition* part, const adx_model* m, int rank, int* out,
                     int cap, int* n_ops) {
    return guard([&] {
        need(plan, "rank_program");
        need(part, "rank_program");
        need(m, "rank_program");
        auto ops = adx::rank_program(plan->p, part->p, m->m, rank);
        *n_ops = static_cast<int>(ops.size());
        if (static_cast<int>(ops.size()) * 12 > cap) throw std::invalid_argument("rank_program: buffer too small");
        for (size_t i = 0; i < ops.size(); ++i) {
            const adx::RankOp& o = ops[i];
            const int f[12] = {o.kind, o.seg,   o.t,    o.wslot, o.rslot, o.step,
                               o.eps_step, o.point, o.peer, o.stage, o.slot, static_cast<int>(o.elems)};
            std::memcpy(out + 12 * i, f, sizeof f);
        }
    });
}

int adx_nccl_unique_id(char* out128) {
    return guard([&] {
        need(out128, "nccl_unique_id");
        adx::nccl_unique_id(out128);
    });
}

int adx_rank_session_create(adx_engine* e, const adx_plan* plan, const adx_partition* part,
                            const double* alpha_bars, int T, int rank, const char* nccl_id,
                            const adx_run_options* opts, adx_rank_session** out) {
    return guard([&] {
        need(e, "rank_session_create");
        need(plan, "rank_session_create");
        need(part, "rank_session_create");
        need(nccl_id, "rank_session_create");
        std::vector<double> ab(alpha_bars, alpha_bars + T + 1);
        *out = reinterpret_cast<adx_rank_session*>(
            adx::rank_session_create(e->e.get(), plan->p, part->p, ab, rank, nccl_id, to_opts(opts)));
    });
}

void adx_rank_session_destroy(adx_rank_session* s) {
    if (s) adx::rank_session_destroy(s);
}

int adx_rank_session_run(adx_rank_session* s, const double* x_T, double* lat, double* eps) {
    return guard([&] {
        need(s, "rank_session_run");
        adx::rank_session_run(s, x_T, lat, eps);
    });
}

int adx_rank_session_time(adx_rank_session* s, int iters, double* ms) {
    return guard([&] {
        need(s, "rank_session_time");
        *ms = adx::rank_session_time(s, iters);
    });
}

int adx_rank_session_kernel_count(const adx_rank_session* s, int* n) {
    return guard([&] {
        need(s, "rank_session_kernel_count");
        *n = adx::rank_session_kernels(const_cast<adx_rank_session*>(s));
    });
}

// ------------------------------------------------------ UNet-shaped family
int adx_model_build_unet(const adx_unet_spec* s, adx_model** out) {
    return guard([&] {
        need(s, "build_unet");
        if (s->n_levels < 1 || s->n_levels > 8) throw std::invalid_argument("build_unet: 1..8 levels");
        adx::UNetSpec sp;
        sp.H = s->H;
        sp.W = s->W;
        sp.c_lat = s->c_lat;
        sp.ch.assign(s->ch, s->ch + s->n_levels);
        sp.attn.assign(s->attn, s->attn + s->n_levels);
        sp.n_res = s->n_res;
        sp.head_dim = s->head_dim;
        sp.ctx_len = s->ctx_len;
        sp.ctx_dim = s->ctx_dim;
        sp.temb_dim = s->temb_dim;
        sp.groups = s->groups;
        sp.mid_attn = s->mid_attn;
        sp.seed = s->seed;
        sp.cfg = s->cfg ? 1 : 0;
        sp.cfg_scale = s->cfg_scale;
        sp.frames = s->frames < 1 ? 1 : s->frames;
        sp.motion = s->motion ? 1 : 0;
        *out = new adx_model{adx::build_unet_model(sp)};
    });
}

int adx_unet_stage_info(const adx_model* m, int stage, int* info /* kind, cin, cskip, cout, H, W, attn */) {
    return guard([&] {
        need(m, "unet_stage_info");
        if (m->m.kind != 1) throw std::invalid_argument("unet_stage_info: not a UNet model");
        const adx::UStage& s = m->m.unet->st.at(stage - 1);
        const int v[7] = {s.kind, s.cin, s.cskip, s.cout, s.H, s.W, s.attn};
        std::memcpy(info, v, sizeof v);
    });
}

// parameters of a stage (0 = shared time-embedding MLP): names '\n'-joined,
// shapes as (rows, cols) pairs (cols = 0 for vectors), data concatenated fp32
int adx_unet_stage_params(const adx_model* m, int stage, char* names, int names_cap, int* shapes, int* n_params,
                          float* data, long long data_cap, long long* n_data) {
    return guard([&] {
        need(m, "unet_stage_params");
        if (m->m.kind != 1) throw std::invalid_argument("unet_stage_params: not a UNet model");
        const auto ps = adx::unet_stage_params(*m->m.unet, stage);
        std::string joined;
        long long total = 0;
        for (size_t i = 0; i < ps.size(); ++i) {
            joined += (i ? "\n" : "") + ps[i].name;
            if (shapes) {
                shapes[2 * i] = ps[i].shape[0];
                shapes[2 * i + 1] = ps[i].shape.size() > 1 ? ps[i].shape[1] : 0;
            }
            if (data && total + static_cast<long long>(ps[i].data.size()) <= data_cap)
                std::memcpy(data + total, ps[i].data.data(), ps[i].data.size() * sizeof(float));
            total += static_cast<long long>(ps[i].data.size());
        }
        if (names && names_cap > 0) {
            std::strncpy(names, joined.c_str(), names_cap - 1);
            names[names_cap - 1] = 0;
        }
        *n_params = static_cast<int>(ps.size());
        *n_data = total;
    });
}

int adx_unet_context(const adx_model* m, float* out) {
    return guard([&] {
        need(m, "unet_context");
        if (m->m.kind != 1) throw std::invalid_argument("unet_context: not a UNet model");
        std::memcpy(out, m->m.unet->ctx.data(), m->m.unet->ctx.size() * sizeof(float));
    });
}

// ------------------------------------------- tcgen05 GEMM / conv (UNet family)
int adx_tc_gemm(int ordinal, int M, int N, int K, const uint16_t* A, const uint16_t* B, const float* bias, int act,
                float* C, int bn, int iters, double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        DevBuf a(static_cast<size_t>(M) * K * 2), b(static_cast<size_t>(N) * K * 2), c(static_cast<size_t>(M) * N * 4),
            bi(static_cast<size_t>(N) * 4);
        CKC(cudaMemcpy(a.p, A, static_cast<size_t>(M) * K * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(b.p, B, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.act = act;
        p.out_f32 = static_cast<float*>(c.p);
        const int nout = act == 2 ? N / 2 : N;  // GEGLU writes hidden * gelu(gate): N/2 columns
        p.ldo = nout;
        adx::tc_gemm(a.p, b.p, M, N, K, p, 0, bn);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter)
            *ms_per_iter = time_graph_ms([&](cudaStream_t st) { adx::tc_gemm(a.p, b.p, M, N, K, p, st, bn); }, iters);
        if (C) CKC(cudaMemcpy(C, c.p, static_cast<size_t>(M) * nout * 4, cudaMemcpyDeviceToHost));
    });
}

// bf16-output epilogue variants (TMA-store path): optional bf16 residual (row stride ldr),
// output row stride ldo >= N; bn / splits force a tile plan (0, 0: the launcher's choice)
int adx_tc_gemm_bf16(int ordinal, int M, int N, int K, const uint16_t* A, const uint16_t* B, const float* bias,
                     const uint16_t* residual, int ldr, uint16_t* out, int ldo, int bn, int splits, int iters,
                     double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        if (ldo < N || (residual && ldr < N)) throw std::invalid_argument("tc_gemm_bf16: ldo / ldr < N");
        DevBuf a(static_cast<size_t>(M) * K * 2), b(static_cast<size_t>(N) * K * 2), o(static_cast<size_t>(M) * ldo * 2),
            r(residual ? static_cast<size_t>(M) * ldr * 2 : 16), bi(static_cast<size_t>(N) * 4);
        CKC(cudaMemcpy(a.p, A, static_cast<size_t>(M) * K * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(b.p, B, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(o.p, out, static_cast<size_t>(M) * ldo * 2, cudaMemcpyHostToDevice));  // untouched columns kept
        if (residual) CKC(cudaMemcpy(r.p, residual, static_cast<size_t>(M) * ldr * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.residual = residual ? static_cast<const __nv_bfloat16*>(r.p) : nullptr;
        p.ldr = ldr;
        p.out_bf16 = static_cast<__nv_bfloat16*>(o.p);
        p.ldo = ldo;
        if (bn) adx::tc_plan_override(bn, std::max(1, splits));
        try {
            adx::tc_gemm(a.p, b.p, M, N, K, p, 0, 0);
            CKC(cudaDeviceSynchronize());
            if (iters > 0 && ms_per_iter)
                *ms_per_iter = time_graph_ms([&](cudaStream_t st) { adx::tc_gemm(a.p, b.p, M, N, K, p, st, 0); }, iters);
        } catch (...) {
            adx::tc_plan_override(0, 0);
            throw;
        }
        if (bn) adx::tc_plan_override(0, 0);
        CKC(cudaMemcpy(out, o.p, static_cast<size_t>(M) * ldo * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_tc_gemm_cat_bf16(int ordinal, int M, int N, int K1, int K2, const uint16_t* A1, const uint16_t* A2,
                         const uint16_t* B, const float* bias, uint16_t* out, int bn, int splits) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const int K = K1 + K2;
        DevBuf a1(static_cast<size_t>(M) * K1 * 2), a2(static_cast<size_t>(M) * K2 * 2),
            b(static_cast<size_t>(N) * K * 2), o(static_cast<size_t>(M) * N * 2), bi(static_cast<size_t>(N) * 4);
        CKC(cudaMemcpy(a1.p, A1, static_cast<size_t>(M) * K1 * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(a2.p, A2, static_cast<size_t>(M) * K2 * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(b.p, B, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.out_bf16 = static_cast<__nv_bfloat16*>(o.p);
        p.ldo = N;
        if (bn) adx::tc_plan_override(bn, std::max(1, splits));
        try {
            adx::tc_gemm_cat(a1.p, K1, a2.p, K2, b.p, M, N, p, 0, 0);
            CKC(cudaDeviceSynchronize());
        } catch (...) {
            adx::tc_plan_override(0, 0);
            throw;
        }
        if (bn) adx::tc_plan_override(0, 0);
        CKC(cudaMemcpy(out, o.p, static_cast<size_t>(M) * N * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_sk_timeline(unsigned long long* out, int n_ctas) {
    return guard([&] { adx::tc_sk_timeline(out, n_ctas); });
}

int adx_tc_geglu_group(void) { return adx::tc_geglu_group(); }

int adx_tc_ln_fold_supported(void) { return adx::tc_ln_fold_supported() ? 1 : 0; }

int adx_tc_ln_fold_bf16(int ordinal, int M, int C, int N, const uint16_t* H, const uint16_t* W1, const float* bias1,
                        const float* colsum1, int geglu, float eps, uint16_t* y_out, int bn, int iters,
                        double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const int No = geglu ? N / 2 : N;
        const size_t mc = static_cast<size_t>(M) * C;
        DevBuf h(mc * 2), w1(static_cast<size_t>(N) * C * 2), b1(static_cast<size_t>(N) * 4),
            cs(static_cast<size_t>(N) * 4), y(static_cast<size_t>(M) * No * 2);
        CKC(cudaMemcpy(h.p, H, mc * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(w1.p, W1, static_cast<size_t>(N) * C * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(b1.p, bias1, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(cs.p, colsum1, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p1;
        p1.bias = static_cast<const float*>(b1.p);
        p1.act = geglu ? 2 : 0;
        p1.out_bf16 = static_cast<__nv_bfloat16*>(y.p);
        p1.ldo = No;
        p1.ln_colsum = static_cast<const float*>(cs.p);
        p1.ln_eps = eps;
        if (bn) adx::tc_plan_override(bn, 1);
        try {
            adx::tc_gemm(h.p, w1.p, M, N, C, p1, 0, 0);
            CKC(cudaDeviceSynchronize());
            if (iters > 0 && ms_per_iter)
                *ms_per_iter = time_graph_ms([&](cudaStream_t st) { adx::tc_gemm(h.p, w1.p, M, N, C, p1, st, 0); }, iters);
        } catch (...) {
            adx::tc_plan_override(0, 0);
            throw;
        }
        if (bn) adx::tc_plan_override(0, 0);
        if (y_out) CKC(cudaMemcpy(y_out, y.p, static_cast<size_t>(M) * No * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_tc_conv3x3_bf16(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X, const uint16_t* Wt,
                        const float* bias, const uint16_t* residual, uint16_t* out, int bn, int splits, int iters,
                        double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const size_t nx = static_cast<size_t>(batch) * H * W * Cin, nw = static_cast<size_t>(Cout) * 9 * Cin,
                     no = static_cast<size_t>(batch) * H * W * Cout;
        DevBuf x(nx * 2), w(nw * 2), o(no * 2), r(residual ? no * 2 : 16), bi(static_cast<size_t>(Cout) * 4);
        CKC(cudaMemcpy(x.p, X, nx * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(w.p, Wt, nw * 2, cudaMemcpyHostToDevice));
        if (residual) CKC(cudaMemcpy(r.p, residual, no * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(Cout) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.residual = residual ? static_cast<const __nv_bfloat16*>(r.p) : nullptr;
        p.ldr = Cout;
        p.out_bf16 = static_cast<__nv_bfloat16*>(o.p);
        p.ldo = Cout;
        if (bn) adx::tc_plan_override(bn, std::max(1, splits));
        try {
            adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, 0);
            CKC(cudaDeviceSynchronize());
            if (iters > 0 && ms_per_iter)
                *ms_per_iter = time_graph_ms(
                    [&](cudaStream_t st) { adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, st); }, iters);
        } catch (...) {
            adx::tc_plan_override(0, 0);
            throw;
        }
        if (bn) adx::tc_plan_override(0, 0);
        CKC(cudaMemcpy(out, o.p, no * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_tc_conv3x3_s2_bf16(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X,
                           const uint16_t* Wt, const float* bias, uint16_t* out, int bn, int splits, int iters,
                           double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const size_t nx = static_cast<size_t>(batch) * H * W * Cin, nw = static_cast<size_t>(Cout) * 9 * Cin,
                     no = static_cast<size_t>(batch) * (H / 2) * (W / 2) * Cout;
        DevBuf x(nx * 2), w(nw * 2), o(no * 2), bi(static_cast<size_t>(Cout) * 4);
        CKC(cudaMemcpy(x.p, X, nx * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(w.p, Wt, nw * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(Cout) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.out_bf16 = static_cast<__nv_bfloat16*>(o.p);
        p.ldo = Cout;
        p.sub2 = 1;
        if (bn) adx::tc_plan_override(bn, std::max(1, splits));
        try {
            adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, 0);
            CKC(cudaDeviceSynchronize());
            if (iters > 0 && ms_per_iter)
                *ms_per_iter = time_graph_ms(
                    [&](cudaStream_t st) { adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, st); }, iters);
        } catch (...) {
            adx::tc_plan_override(0, 0);
            throw;
        }
        if (bn) adx::tc_plan_override(0, 0);
        CKC(cudaMemcpy(out, o.p, no * 2, cudaMemcpyDeviceToHost));
    });
}

// GroupNorm(+SiLU) over a (one- or two-segment) channel concat of bf16 NHWC images:
// x0 [batch][HW][c0], x1 [batch][HW][c1] (NULL when c1 == 0) -> out [batch][HW][c0 + c1]
int adx_group_norm_bf16(int ordinal, int batch, int HW, int c0, int c1, int groups, const uint16_t* x0,
                        const uint16_t* x1, const float* gamma, const float* beta, float eps, int act, uint16_t* out,
                        int iters, double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const int C = c0 + c1;
        const size_t n0 = static_cast<size_t>(batch) * HW * c0, n1 = static_cast<size_t>(batch) * HW * c1,
                     no = static_cast<size_t>(batch) * HW * C;
        DevBuf a(n0 * 2), b(std::max<size_t>(n1, 8) * 2), o(no * 2), g(static_cast<size_t>(C) * 4),
            be(static_cast<size_t>(C) * 4);
        const size_t sb = adx::group_norm_scratch_bytes(batch, HW, groups, C);
        DevBuf sc(sb);
        CKC(cudaMemset(sc.p, 0, sb));
        CKC(cudaMemcpy(a.p, x0, n0 * 2, cudaMemcpyHostToDevice));
        if (c1) CKC(cudaMemcpy(b.p, x1, n1 * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(g.p, gamma, static_cast<size_t>(C) * 4, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(be.p, beta, static_cast<size_t>(C) * 4, cudaMemcpyHostToDevice));
        adx::Cat2 xc{static_cast<const __nv_bfloat16*>(a.p), c0, c1 ? static_cast<const __nv_bfloat16*>(b.p) : nullptr,
                     c1};
        auto run = [&](cudaStream_t st) {
            adx::group_norm(xc, batch, HW, groups, static_cast<const float*>(g.p), static_cast<const float*>(be.p),
                            eps, act, static_cast<__nv_bfloat16*>(o.p), static_cast<float2*>(sc.p), st);
        };
        run(0);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter) *ms_per_iter = time_graph_ms(run, iters);
        CKC(cudaMemcpy(out, o.p, no * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_gn_timeline(unsigned long long* out, int n) {
    return guard([&] { adx::gn_timeline(out, n); });
}

int adx_tc_timeline(unsigned long long* out, int n_ctas) {
    return guard([&] { adx::tc_timeline(out, n_ctas); });
}

int adx_tc_plan_override(int bn, int splits) {
    return guard([&] { adx::tc_plan_override(bn, splits); });
}

int adx_tc_attention(int ordinal, int L, int Lk, int C, const uint16_t* Q, const uint16_t* K, const uint16_t* V,
                     int ldv, uint16_t* out, int iters, double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        if (ldv < C) throw std::invalid_argument("tc_attention: ldv < C");
        DevBuf q(static_cast<size_t>(L) * C * 2), k(static_cast<size_t>(Lk) * C * 2),
            v(static_cast<size_t>(Lk) * ldv * 2), o(static_cast<size_t>(L) * C * 2);
        CKC(cudaMemcpy(q.p, Q, static_cast<size_t>(L) * C * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(k.p, K, static_cast<size_t>(Lk) * C * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(v.p, V, static_cast<size_t>(Lk) * ldv * 2, cudaMemcpyHostToDevice));
        const size_t wsb = adx::tc_attention_ws_bytes(L, Lk, C);
        DevBuf ws(std::max<size_t>(wsb, 256));
        CKC(cudaMemset(ws.p, 0, std::max<size_t>(wsb, 256)));
        auto run = [&](cudaStream_t st) {
            adx::tc_attention(q.p, C, k.p, C, v.p, ldv, L, Lk, C, static_cast<__nv_bfloat16*>(o.p), C, st, ws.p, wsb);
        };
        run(0);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter) *ms_per_iter = time_graph_ms(run, iters);
        if (out) CKC(cudaMemcpy(out, o.p, static_cast<size_t>(L) * C * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_tc_attention_f32(int ordinal, int batch, int L, int Lk, int C, const float* Q, const float* K,
                         const float* V, float* out, int iters, double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const size_t nq = static_cast<size_t>(batch) * L * C, nk = static_cast<size_t>(batch) * Lk * C;
        if ((nq | nk) % 8) throw std::invalid_argument("tc_attention_f32: element counts must be multiples of 8");
        DevBuf q(nq * 4), k(nk * 4), v(nk * 4), o(nq * 4), qs(nq * 4), ks(nk * 4), vs(nk * 4);
        CKC(cudaMemcpy(q.p, Q, nq * 4, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(k.p, K, nk * 4, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(v.p, V, nk * 4, cudaMemcpyHostToDevice));
        const size_t wsb = adx::tc_attention_ws_bytes(L, Lk, C, batch);
        DevBuf ws(std::max<size_t>(wsb, 256));
        CKC(cudaMemset(ws.p, 0, std::max<size_t>(wsb, 256)));
        auto* qh = static_cast<__nv_bfloat16*>(qs.p);
        auto* kh = static_cast<__nv_bfloat16*>(ks.p);
        auto* vh = static_cast<__nv_bfloat16*>(vs.p);
        auto run = [&](cudaStream_t st) {  // the ADX_F32 transformer's sequence: split, then the fused kernel
            adx::split2(static_cast<const float*>(q.p), static_cast<long long>(nq), qh, qh + nq, st);
            adx::split2(static_cast<const float*>(k.p), static_cast<long long>(nk), kh, kh + nk, st);
            adx::split2(static_cast<const float*>(v.p), static_cast<long long>(nk), vh, vh + nk, st);
            adx::tc_attention_x(qh, qh + nq, C, kh, kh + nk, C, vh, vh + nk, C, L, Lk, C,
                                static_cast<float*>(o.p), C, st, ws.p, wsb, batch);
        };
        run(0);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter) *ms_per_iter = time_graph_ms(run, iters);
        if (out) CKC(cudaMemcpy(out, o.p, nq * 4, cudaMemcpyDeviceToHost));
    });
}

int adx_temporal_attention(int ordinal, int frames, int HW, int C, const uint16_t* qkv, uint16_t* out, int iters,
                           double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const size_t nin = static_cast<size_t>(frames) * HW * 3 * C, nout = static_cast<size_t>(frames) * HW * C;
        DevBuf q(nin * 2), o(nout * 2);
        CKC(cudaMemcpy(q.p, qkv, nin * 2, cudaMemcpyHostToDevice));
        auto run = [&](cudaStream_t st) {
            adx::temporal_attention(static_cast<const __nv_bfloat16*>(q.p), frames, HW, C,
                                    static_cast<__nv_bfloat16*>(o.p), st);
        };
        run(0);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter) *ms_per_iter = time_graph_ms(run, iters);
        if (out) CKC(cudaMemcpy(out, o.p, nout * 2, cudaMemcpyDeviceToHost));
    });
}

int adx_tc_conv3x3(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X, const uint16_t* Wt,
                   const float* bias, float* out, int iters, double* ms_per_iter) {
    return guard([&] {
        CKC(cudaSetDevice(ordinal));
        const size_t nx = static_cast<size_t>(batch) * H * W * Cin, nw = static_cast<size_t>(Cout) * 9 * Cin,
                     no = static_cast<size_t>(batch) * H * W * Cout;
        DevBuf x(nx * 2), w(nw * 2), o(no * 4), bi(static_cast<size_t>(Cout) * 4);
        CKC(cudaMemcpy(x.p, X, nx * 2, cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(w.p, Wt, nw * 2, cudaMemcpyHostToDevice));
        if (bias) CKC(cudaMemcpy(bi.p, bias, static_cast<size_t>(Cout) * 4, cudaMemcpyHostToDevice));
        adx::TcArgs p;
        p.bias = bias ? static_cast<const float*>(bi.p) : nullptr;
        p.out_f32 = static_cast<float*>(o.p);
        p.ldo = Cout;
        adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, 0);
        CKC(cudaDeviceSynchronize());
        if (iters > 0 && ms_per_iter)
            *ms_per_iter = time_graph_ms(
                [&](cudaStream_t st) { adx::tc_conv3x3(x.p, w.p, batch, H, W, Cin, Cout, p, st); }, iters);
        if (out) CKC(cudaMemcpy(out, o.p, no * 4, cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------------------ §8(f) next rows
int adx_model_save_checkpoint(const adx_model* m, const char* base) {
    return guard([&] {
        need(m, "save_checkpoint");
        need(base, "save_checkpoint");
        adx::save_checkpoint(base, m->m);
    });
}

int adx_model_load_checkpoint(const char* base, adx_model** out) {
    return guard([&] {
        need(base, "load_checkpoint");
        *out = new adx_model{adx::load_checkpoint(base)};
    });
}

int adx_plan_to_json(const adx_plan* p, char* buf, int cap, int* len) {
    return guard([&] {
        need(p, "plan_to_json");
        const std::string s = adx::plan_to_json(p->p);
        if (len) *len = static_cast<int>(s.size());
        if (buf && cap > 0) {
            std::strncpy(buf, s.c_str(), cap - 1);
            buf[cap - 1] = 0;
        }
    });
}

int adx_plan_from_json(const char* text, adx_plan** out) {
    return guard([&] {
        need(text, "plan_from_json");
        *out = new adx_plan{adx::plan_from_json(text)};
    });
}

int adx_predict_async(const adx_plan* p, const double* seg_cost, int n_seg, double comm_cost_s,
                      double sampler_cost_s, double comm_latency_s, double link_gbs,
                      const long long* round_bytes, adx_latency_report* out, double* round_compute_s,
                      double* round_comm_s) {
    return guard([&] {
        need(p, "predict_async");
        need(out, "predict_async");
        adx::CostModel cm;
        cm.segment_cost_s.assign(seg_cost, seg_cost + n_seg);
        cm.comm_cost_s = comm_cost_s;
        cm.sampler_cost_s = sampler_cost_s;
        cm.comm_latency_s = comm_latency_s;
        cm.link_gbs = link_gbs;
        std::vector<long long> rb;
        if (round_bytes) rb.assign(round_bytes, round_bytes + p->p.rounds.size());
        const adx::LatencyReport r = adx::predict_async(p->p, cm, round_bytes ? &rb : nullptr);
        out->sequential_total_s = r.sequential_total_s;
        out->async_total_s = r.async_total_s;
        out->warmup_s = r.warmup_s;
        out->comm_total_s = r.comm_total_s;
        out->speedup = r.speedup;
        out->comm_ratio = r.comm_ratio;
        out->approx_step_s = r.approx_step_s;
        out->approx_total_s = r.approx_total_s;
        for (size_t i = 0; i < r.round_compute_s.size(); ++i) {
            if (round_compute_s) round_compute_s[i] = r.round_compute_s[i];
            if (round_comm_s) round_comm_s[i] = r.round_comm_s[i];
        }
    });
}

int adx_calibrate_and_compare(const adx_plan* p, const double* delays, int n, const double* measured_round_comm_s,
                              int n_rounds, int broadcast_count, double measured_total_s,
                              adx_cost_comparison* out) {
    return guard([&] {
        need(p, "calibrate_and_compare");
        need(out, "calibrate_and_compare");
        const auto c = adx::calibrate_and_compare(p->p, std::vector<double>(delays, delays + n),
                                                  std::vector<double>(measured_round_comm_s,
                                                                      measured_round_comm_s + n_rounds),
                                                  broadcast_count, measured_total_s);
        out->predicted_total_s = c.predicted_total_s;
        out->measured_total_s = c.measured_total_s;
        out->rel_error_total = c.rel_error_total;
        out->predicted_comm_ratio = c.predicted_comm_ratio;
        out->measured_comm_ratio = c.measured_comm_ratio;
        out->rel_error_comm_ratio = c.rel_error_comm_ratio;
        out->calibrated_comm_cost_s = c.calibrated_comm_cost_s;
    });
}

int adx_round_exchange_bytes(const adx_plan* p, const adx_partition* part, const adx_model* m, int precision,
                             long long* out) {
    return guard([&] {
        need(p, "round_exchange_bytes");
        need(part, "round_exchange_bytes");
        need(m, "round_exchange_bytes");
        const auto b = adx::round_exchange_bytes(p->p, part->p, m->m, precision);
        std::memcpy(out, b.data(), b.size() * sizeof(long long));
    });
}

}  // extern "C"
