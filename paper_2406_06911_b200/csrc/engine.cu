// engine.cu -- device-resident AsyncDiff executor (see engine.hpp).
#include "engine.hpp"

#include "tc_gemm.cuh"
#include "unet_dev.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <thread>

namespace adx {

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

namespace {

constexpr int kBadSentinel = 0x7f7f7f7f;
constexpr int kKeyStride = 1024;

int round_up8(int n) { return (n + 7) & ~7; }

uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}

// fp64 row-major (rows x cols) -> device buffer rows x pitch in weight dtype
void* upload_matrix(int prec, const std::vector<double>& src, int rows, int cols, int pitch) {
    const size_t n = static_cast<size_t>(rows) * pitch;
    void* d = nullptr;
    const int wb = weight_bytes(prec);
    CK(cudaMalloc(&d, n * wb));
    std::vector<unsigned char> host(n * wb, 0);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const double v = src[static_cast<size_t>(i) * cols + j];
            const size_t k = static_cast<size_t>(i) * pitch + j;
            if (prec == kF64) {
                std::memcpy(&host[k * 8], &v, 8);
            } else if (prec == kF32) {
                const float f = static_cast<float>(v);
                std::memcpy(&host[k * 4], &f, 4);
            } else {
                const uint16_t b = f32_to_bf16_rne(static_cast<float>(v));
                std::memcpy(&host[k * 2], &b, 2);
            }
        }
    CK(cudaMemcpy(d, host.data(), n * wb, cudaMemcpyHostToDevice));
    return d;
}

// fp64 vector -> device activation dtype
void* upload_act(int prec, const std::vector<double>& src) {
    void* d = nullptr;
    const int ab = act_bytes(prec);
    CK(cudaMalloc(&d, std::max<size_t>(1, src.size()) * ab));
    std::vector<unsigned char> host(std::max<size_t>(1, src.size()) * ab, 0);
    for (size_t i = 0; i < src.size(); ++i) {
        if (prec == kF64) {
            std::memcpy(&host[i * 8], &src[i], 8);
        } else {
            const float f = static_cast<float>(src[i]);
            std::memcpy(&host[i * 4], &f, 4);
        }
    }
    CK(cudaMemcpy(d, host.data(), host.size(), cudaMemcpyHostToDevice));
    return d;
}

void* offset(void* p, size_t bytes) { return static_cast<char*>(p) + bytes; }

}  // namespace

// ===================================================================== Engine
Engine::Engine(const Model& m, int prec, std::vector<int> ordinals)
    : model_(m), prec_(prec), ordinals_(std::move(ordinals)) {
    if (prec < kF64 || prec > kBF16) throw std::invalid_argument("engine: unknown precision");
    if (ordinals_.empty()) throw std::invalid_argument("engine: need at least one device ordinal");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    for (int o : ordinals_)
        if (o < 0 || o >= n)
            throw std::invalid_argument("engine: device ordinal " + std::to_string(o) + " not visible (" +
                                        std::to_string(n) + " devices)");
    dev_.resize(ordinals_.size());
    for (size_t i = 0; i < ordinals_.size(); ++i) {
        dev_[i].ordinal = ordinals_[i];
        dev_[i].stages.resize(model_.L);
    }
    if (model_.kind == 1 && prec_ == kF64)
        throw std::invalid_argument("engine: the UNet family runs precision bf16 (bf16 tensor-core stages) or f32 "
                                    "(fp32 activations, split-bf16 products) with an f32 trajectory");
    unet_.resize(ordinals_.size());
}

UNetDevice& Engine::unet(int idx) {
    auto& u = unet_[idx % unet_.size()];
    if (!u) {
        CK(cudaSetDevice(ordinal(idx)));
        u = std::make_shared<UNetDevice>(model_, ordinal(idx), prec_ == kF32);
    }
    return *u;
}

Engine::~Engine() {
    for (size_t i = 0; i < unet_.size(); ++i) {
        cudaSetDevice(ordinals_[i]);
        unet_[i].reset();
    }
    for (auto& d : dev_) {
        cudaSetDevice(d.ordinal);
        for (auto& s : d.stages) {
            cudaFree(s.w1);
            cudaFree(s.w2);
            cudaFree(s.b2);
            cudaFree(s.ctab);
        }
        cudaFree(d.etab);
    }
}

size_t Engine::stage_weight_bytes(int stage) const {
    const Stage& st = model_.stages[stage - 1];
    return (static_cast<size_t>(st.hidden) * st.in + static_cast<size_t>(st.out) * st.hidden) *
           weight_bytes(prec_);
}

const DevStage& Engine::stage_on(int idx, int stage) {
    DevShared& d = dev_[idx % dev_.size()];
    DevStage& ds = d.stages[stage - 1];
    if (model_.kind == 1) {
        unet(idx).ensure_stage(stage);
        return ds;
    }
    if (ds.w1) return ds;
    CK(cudaSetDevice(d.ordinal));
    const Stage& st = model_.stages[stage - 1];
    ds.pitch1 = round_up8(st.in);
    ds.pitch2 = round_up8(st.hidden);
    ds.w1 = upload_matrix(prec_, st.w1, st.hidden, st.in, ds.pitch1);
    ds.w2 = upload_matrix(prec_, st.w2, st.out, st.hidden, ds.pitch2);
    ds.b2 = upload_act(prec_, st.b2);
    return ds;
}

// e_t table and per-stage bias tables c_t = b1 + Tin . e_t for t in [0, T]
// (the time term of denoiser.cpp:182, hoisted out of the hot loop).
void Engine::ensure_tables(int idx, int T) {
    if (model_.kind == 1) unet(idx).ensure_tables(T);
    DevShared& d = dev_[idx % dev_.size()];
    CK(cudaSetDevice(d.ordinal));
    const int E = model_.E;
    std::vector<std::vector<double>> emb(T + 1);
    for (int t = 0; t <= T; ++t) emb[t] = model_.embed(t);
    if (d.etab_T < T) {
        std::vector<double> flat;
        for (int t = 0; t <= T; ++t) flat.insert(flat.end(), emb[t].begin(), emb[t].end());
        cudaFree(d.etab);
        d.etab = upload_act(prec_, flat);
        d.etab_T = T;
    }
    for (int s = 1; s <= model_.L; ++s) {
        DevStage& ds = d.stages[s - 1];
        if (!ds.w1 || ds.ctab_T >= T) continue;
        const Stage& st = model_.stages[s - 1];
        std::vector<double> flat(static_cast<size_t>(T + 1) * st.hidden);
        for (int t = 0; t <= T; ++t)
            for (int j = 0; j < st.hidden; ++j) {
                double te = 0.0;
                for (int e = 0; e < E; ++e) te += st.tin[static_cast<size_t>(j) * E + e] * emb[t][e];
                flat[static_cast<size_t>(t) * st.hidden + j] = st.b1[j] + te;
            }
        cudaFree(ds.ctab);
        ds.ctab = upload_act(prec_, flat);
        ds.ctab_T = T;
    }
}

const void* Engine::etab_row(int idx, int t) const {
    const DevShared& d = dev_[idx % dev_.size()];
    return offset(d.etab, static_cast<size_t>(t) * model_.E * act_bytes(prec_));
}

long long Engine::weight_bytes_resident(int idx) const {
    const DevShared& d = dev_[idx % dev_.size()];
    long long b = 0;
    for (int s = 1; s <= model_.L; ++s)
        if (d.stages[s - 1].w1) b += static_cast<long long>(stage_weight_bytes(s));
    return b;
}

int Engine::enqueue_stage(int idx, int stage, const std::vector<Seg>& inputs, int embed_t, void* h, void* y,
                          int* bad, int key, cudaStream_t stream, bool pdl) {
    const Stage& st = model_.stages[stage - 1];
    const DevStage& ds = dev_[idx % dev_.size()].stages[stage - 1];
    int K = 0;
    for (auto& s : inputs) K += s.n;
    if (K != st.in)
        throw std::runtime_error("eval: stage " + std::to_string(stage) + " input width " + std::to_string(K) +
                                 " != expected " + std::to_string(st.in));
    if (model_.kind == 1) {  // UNet-shaped family: tcgen05 conv / GEMM stage program
        std::vector<Seg> in = inputs;
        if (stage == 1) in.resize(1);  // latent only (the shared e_t segment is not used)
        unet(idx).enqueue(stage, in, embed_t, y, prec_ == kF64, stream);
        return 1;
    }
    if (!ds.w1 || ds.ctab_T < embed_t) throw std::logic_error("engine: stage weights/tables not resident");
    if (static_cast<int>(inputs.size()) > kMaxSegs)
        throw std::invalid_argument("eval: stage " + std::to_string(stage) + " has too many concat inputs");
    GemvArgs a1 = {};
    a1.W = ds.w1;
    a1.rows = st.hidden;
    a1.pitch = ds.pitch1;
    a1.K = st.in;
    a1.nseg = static_cast<int>(inputs.size());
    for (size_t i = 0; i < inputs.size(); ++i) {
        a1.seg[i] = inputs[i].p;
        a1.seg_len[i] = inputs[i].n;
    }
    a1.bias = offset(ds.ctab, static_cast<size_t>(embed_t) * st.hidden * act_bytes(prec_));
    a1.out = h;
    a1.act = 1;
    launch_gemv(prec_, a1, stream, pdl);
    GemvArgs a2 = {};
    a2.W = ds.w2;
    a2.rows = st.out;
    a2.pitch = ds.pitch2;
    a2.K = st.hidden;
    a2.nseg = 1;
    a2.seg[0] = h;
    a2.seg_len[0] = st.hidden;
    a2.bias = ds.b2;
    a2.out = y;
    a2.act = 0;
    a2.bad = bad;
    a2.bad_key = key;
    launch_gemv(prec_, a2, stream, pdl);
    return 2;
}

double Engine::time_eval_ms(int idx, int t_embed, int iters, int* launches, double (*profile)[3], double* stage_ms) {
    const int ord = ordinal(idx);
    CK(cudaSetDevice(ord));
    const Model& m = model_;
    for (int i = 1; i <= m.L; ++i) stage_on(idx, i);
    ensure_tables(idx, std::max(t_embed, 1));
    const int ab = act_bytes(prec_);
    std::vector<void*> bufs;
    auto dalloc = [&](size_t n) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(n, 16)));
        CK(cudaMemset(p, 0, std::max<size_t>(n, 16)));
        bufs.push_back(p);
        return p;
    };
    void* x = dalloc(static_cast<size_t>(m.data_dim()) * ab);
    int* bad = static_cast<int*>(dalloc(2 * sizeof(int)));
    std::vector<void*> y(m.L + 1), h(m.L + 1);
    for (int i = 1; i <= m.L; ++i) {
        y[i] = dalloc(static_cast<size_t>(m.widths[i]) * ab);
        h[i] = dalloc(static_cast<size_t>(m.widths[i]) * ab);
    }
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int n = 0;
    auto pass = [&]() {
        n = 0;
        for (int i = 1; i <= m.L; ++i) {
            std::vector<Seg> in;
            if (i == 1) {
                in.push_back({x, m.data_dim()});
                in.push_back({etab_row(idx, t_embed), m.E});
            } else {
                in.push_back({y[i - 1], m.widths[i - 1]});
            }
            for (auto& l : m.links_into(i)) in.push_back({y[l.first], m.widths[l.first]});
            n += enqueue_stage(idx, i, in, t_embed, h[i], y[i], bad, i, st, true);
        }
    };
    if (profile) {  // eager pass; every tensor-core launch also timed in isolation (tc_profile_measure)
        pass();
        CK(cudaStreamSynchronize(st));
        tc_profile_enable(true);
        pass();
        tc_profile_enable(false);
        CK(cudaStreamSynchronize(st));
        tc_profile_collect(profile);
    }
    if (stage_ms) {  // every stage captured into its own graph, replayed `iters` times (device time)
        pass();
        CK(cudaStreamSynchronize(st));
        for (int i = 1; i <= m.L; ++i) {
            std::vector<Seg> in;
            if (i == 1) {
                in.push_back({x, m.data_dim()});
                in.push_back({etab_row(idx, t_embed), m.E});
            } else {
                in.push_back({y[i - 1], m.widths[i - 1]});
            }
            for (auto& l : m.links_into(i)) in.push_back({y[l.first], m.widths[l.first]});
            cudaGraph_t gs = nullptr;
            cudaGraphExec_t gse = nullptr;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
            enqueue_stage(idx, i, in, t_embed, h[i], y[i], bad, i, st, true);
            CK(cudaStreamEndCapture(st, &gs));
            CK(cudaGraphInstantiate(&gse, gs, 0));
            cudaEvent_t a0, b0;
            CK(cudaEventCreate(&a0));
            CK(cudaEventCreate(&b0));
            for (int w = 0; w < 2; ++w) CK(cudaGraphLaunch(gse, st));
            CK(cudaEventRecord(a0, st));
            for (int it = 0; it < iters; ++it) CK(cudaGraphLaunch(gse, st));
            CK(cudaEventRecord(b0, st));
            CK(cudaEventSynchronize(b0));
            float sms = 0.f;
            CK(cudaEventElapsedTime(&sms, a0, b0));
            stage_ms[i - 1] = sms / std::max(1, iters);
            cudaEventDestroy(a0);
            cudaEventDestroy(b0);
            cudaGraphExecDestroy(gse);
            cudaGraphDestroy(gs);
        }
    }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    pass();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(a, st));
    for (int it = 0; it < iters; ++it) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    for (void* p : bufs) cudaFree(p);
    if (launches) *launches = n;
    return ms / std::max(1, iters);
}

// ==================================================================== Session
Session::Session(Engine* e, const Plan& plan, const Partition& part, const std::vector<double>& alpha_bars,
                 int mode, int workers, const RunOptions& opts)
    : E_(e), plan_(plan), part_(part), ab_(alpha_bars), mode_(mode), opts_(opts) {
    const Model& m = E_->model();
    T_ = static_cast<int>(ab_.size()) - 1;
    d_ = m.data_dim();
    if (T_ < 1) throw std::invalid_argument("run: schedule must have T >= 1");
    if (mode_ == kSequential) {
        // T full-model evaluations (diffusion.cpp:118-142): one segment, one device
        part_ = Partition();
        std::vector<int> all(m.L);
        for (int i = 0; i < m.L; ++i) all[i] = i + 1;
        part_.segments.push_back(all);
        part_.device_of_segment.push_back(0);
        part_.segment_macs.push_back(m.total_macs());
        plan_ = plan_async(T_, T_, 1, 1, false);
    } else {
        // check_preconditions (executor.cpp:204-222)
        const auto violations = validate_plan(plan_);
        if (!violations.empty()) throw std::invalid_argument("run: invalid plan: " + violations.front());
        if (part_.num_segments() != plan_.N) throw std::invalid_argument("run: partition segment count != plan.N");
        part_.validate(m);
        if (!part_.contiguous()) throw std::invalid_argument("run: partition must be a contiguous cascade");
        if (plan_.T != T_) throw std::invalid_argument("run: plan T != schedule T");
        if (!opts_.segment_delay_s.empty() && static_cast<int>(opts_.segment_delay_s.size()) != plan_.N)
            throw std::invalid_argument("run: delay list length != segment count");
        if (mode_ == kParallel) {
            if (workers != plan_.D)
                throw std::invalid_argument("run_parallel: workers=" + std::to_string(workers) +
                                            " != plan device count " + std::to_string(plan_.D));
            for (int n = 0; n < plan_.N; ++n)
                if (part_.device_of_segment[n] != n)
                    throw std::invalid_argument("run_parallel: segment " + std::to_string(n + 1) +
                                                " must be placed on device " + std::to_string(n));
        }
    }
    N_ = plan_.N;
    ab_bytes_ = act_bytes(E_->prec());
    seg_first_.assign(N_ + 1, 0);
    seg_last_.assign(N_ + 1, 0);
    stage_seg_.assign(m.L + 1, 0);
    for (int n = 1; n <= N_; ++n) {
        seg_first_[n] = part_.segments[n - 1].front();
        seg_last_[n] = part_.segments[n - 1].back();
        for (int s : part_.segments[n - 1]) stage_seg_[s] = n;
    }
    // virtual devices
    const int D = mode_ == kParallel ? plan_.D : 1;
    vd_.resize(D);
    for (int v = 0; v < D; ++v) {
        vd_[v].v = v;
        vd_[v].idx = v % E_->num_ordinals();
        vd_[v].ordinal = E_->ordinal(v);
    }
    if (mode_ == kParallel) {
        for (int n = 1; n <= N_; ++n) vd_[part_.device_of_segment[n - 1]].segs.insert(n);
        for (auto& r : plan_.rounds)
            for (auto& ev : r.evals) vd_[ev.device].segs.insert(ev.segment);
    } else {
        for (int n = 1; n <= N_; ++n) vd_[0].segs.insert(n);
    }
    try {
        alloc_buffers();
        if (opts_.use_graph && !opts_.instrument && opts_.segment_delay_s.empty()) build_graph();
    } catch (...) {
        release();
        throw;
    }
}

Session::~Session() { release(); }

void Session::release() {
    for (auto& v : vd_) {
        cudaSetDevice(v.ordinal);
        if (v.comp) cudaStreamSynchronize(v.comp);
        if (v.comm) cudaStreamSynchronize(v.comm);
    }
    if (gexec_) cudaGraphExecDestroy(gexec_);
    if (graph_) cudaGraphDestroy(graph_);
    gexec_ = nullptr;
    graph_ = nullptr;
    auto destroy_ev = [](cudaEvent_t& e) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    };
    for (auto& row : eval_ev_)
        for (auto& p : row) {
            destroy_ev(p.first);
            destroy_ev(p.second);
        }
    eval_ev_.clear();
    for (auto& e : round_start_) destroy_ev(e);
    for (auto& e : round_end_) destroy_ev(e);
    round_start_.clear();
    round_end_.clear();
    for (auto& row : warm_seg_ev_)
        for (auto& e : row) destroy_ev(e);
    warm_seg_ev_.clear();
    for (auto& v : vd_) {
        cudaSetDevice(v.ordinal);
        for (auto& kv : v.Y) {
            cudaFree(kv.second[0]);
            cudaFree(kv.second[1]);
        }
        v.Y.clear();
        for (auto& kv : v.H) cudaFree(kv.second);
        v.H.clear();
        cudaFree(v.EPS[0]);
        cudaFree(v.EPS[1]);
        v.EPS = {nullptr, nullptr};
        cudaFree(v.bad);
        v.bad = nullptr;
        destroy_ev(v.eval_done);
        destroy_ev(v.join);
        for (int s = 0; s < 2; ++s) {
            destroy_ev(v.read_done[s]);
            destroy_ev(v.xfer_done[s]);
        }
        for (auto& kv : v.stage_done) destroy_ev(kv.second);
        v.stage_done.clear();
        if (v.comp) cudaStreamDestroy(v.comp);
        if (v.comm) cudaStreamDestroy(v.comm);
        v.comp = v.comm = nullptr;
    }
    if (!vd_.empty()) cudaSetDevice(vd_[0].ordinal);
    destroy_ev(fork_);
    destroy_ev(t_start_);
    destroy_ev(t_stop_);
    destroy_ev(t_warm_);
    cudaFree(traj_lat_);
    cudaFree(traj_eps_);
    cudaFree(xT_dev_);
    traj_lat_ = traj_eps_ = nullptr;
    xT_dev_ = nullptr;
    if (xT_host_) cudaFreeHost(xT_host_);
    if (out_host_) cudaFreeHost(out_host_);
    xT_host_ = nullptr;
    out_host_ = nullptr;
}

void Session::setdev(int ordinal) const { CK(cudaSetDevice(ordinal)); }

std::vector<int> Session::consumers_of_segment(int seg) const {
    std::vector<int> c;
    for (auto& v : vd_)
        if (v.segs.count(seg)) c.push_back(v.v);
    return c;
}

void Session::alloc_buffers() {
    const Model& m = E_->model();
    const int L = m.L;
    // peer access between distinct physical devices
    std::set<int> ords;
    for (auto& v : vd_) ords.insert(v.ordinal);
    for (int a : ords)
        for (int b : ords) {
            if (a == b) continue;
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, a, b));
            if (can) {
                setdev(a);
                cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        }
    for (auto& v : vd_) {
        setdev(v.ordinal);
        CK(cudaStreamCreateWithFlags(&v.comp, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&v.comm, cudaStreamNonBlocking));
        CK(cudaMalloc(&v.bad, 2 * sizeof(int)));
        CK(cudaEventCreateWithFlags(&v.eval_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&v.join, cudaEventDisableTiming));
        for (int s = 0; s < 2; ++s) {
            CK(cudaEventCreateWithFlags(&v.read_done[s], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&v.xfer_done[s], cudaEventDisableTiming));
        }
        std::set<int> need;  // stage outputs this vdev holds
        for (int seg : v.segs) {
            for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i) {
                E_->stage_on(v.idx, i);
                if (i < L) need.insert(i);
                if (!v.stage_done.count(i)) {
                    cudaEvent_t e;
                    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    v.stage_done[i] = e;
                }
                void* h = nullptr;
                CK(cudaMalloc(&h, static_cast<size_t>(std::max(m.widths[i], 1)) * E_->stage_bytes()));
                v.H[i] = h;
                for (auto& l : m.links_into(i))
                    if (stage_seg_[l.first] != seg) need.insert(l.first);
            }
            if (seg > 1) need.insert(seg_last_[seg - 1]);
        }
        E_->ensure_tables(v.idx, T_);
        for (int p : need) {
            std::array<void*, 2> y{};
            for (int s = 0; s < 2; ++s) {
                CK(cudaMalloc(&y[s], static_cast<size_t>(m.widths[p]) * E_->stage_bytes()));
                CK(cudaMemset(y[s], 0, static_cast<size_t>(m.widths[p]) * E_->stage_bytes()));
            }
            v.Y[p] = y;
        }
        if (v.v != 0 && v.segs.count(N_))
            for (int s = 0; s < 2; ++s) CK(cudaMalloc(&v.EPS[s], static_cast<size_t>(d_) * ab_bytes_));
    }
    setdev(vd_[0].ordinal);
    CK(cudaMalloc(&traj_lat_, static_cast<size_t>(T_ + 1) * d_ * ab_bytes_));
    CK(cudaMalloc(&traj_eps_, static_cast<size_t>(T_) * d_ * ab_bytes_));
    CK(cudaMemset(traj_eps_, 0, static_cast<size_t>(T_) * d_ * ab_bytes_));
    CK(cudaMalloc(&xT_dev_, static_cast<size_t>(d_) * sizeof(double)));
    CK(cudaMallocHost(&xT_host_, static_cast<size_t>(d_) * sizeof(double)));
    CK(cudaMallocHost(&out_host_, static_cast<size_t>(2 * T_ + 1) * d_ * ab_bytes_));
    CK(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    CK(cudaEventCreate(&t_start_));
    CK(cudaEventCreate(&t_stop_));
    CK(cudaEventCreate(&t_warm_));
    // algorithmic weight bytes streamed per run: every eval streams its segment once
    long long per_seg_total = 0;
    std::vector<long long> seg_bytes(N_ + 1, 0);
    for (int n = 1; n <= N_; ++n) {
        for (int i = seg_first_[n]; i <= seg_last_[n]; ++i) seg_bytes[n] += E_->stage_weight_bytes(i);
        per_seg_total += seg_bytes[n];
    }
    weight_bytes_per_run_ = static_cast<long long>(plan_.w) * per_seg_total;
    for (auto& r : plan_.rounds)
        for (auto& ev : r.evals) weight_bytes_per_run_ += seg_bytes[ev.segment];
}

// inputs of `seg` produced by other vdevs (previous round / same warm-up step)
void Session::wait_inputs(VDev& v, int seg, int rslot) {
    if (mode_ != kParallel) return;
    const Model& m = E_->model();
    std::set<int> producers;
    if (seg > 1) producers.insert(seg - 1);
    for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i)
        for (auto& l : m.links_into(i))
            if (stage_seg_[l.first] != seg) producers.insert(stage_seg_[l.first]);
    for (int ps : producers) {
        VDev& u = vd_[part_.device_of_segment[ps - 1]];
        if (u.v == v.v || !u.xfer_rec[rslot]) continue;
        CK(cudaStreamWaitEvent(v.comp, u.xfer_done[rslot], 0));
    }
}

void Session::enqueue_segment_eval(VDev& v, int seg, int embed_t, int wslot, int rslot, const void* latent,
                                   void* eps_out, int seq) {
    const Model& m = E_->model();
    setdev(v.ordinal);
    if (!opts_.segment_delay_s.empty() && opts_.segment_delay_s[seg - 1] > 0.0) {
        launch_delay(opts_.segment_delay_s[seg - 1], v.comp);
        ++enq_kernels_;
    }
    for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i) {
        std::vector<Seg> in;
        if (i == seg_first_[seg]) {
            if (seg == 1) {
                in.push_back({latent, d_});
                in.push_back({E_->etab_row(v.idx, embed_t), m.E});
            } else {
                const int p = seg_last_[seg - 1];
                in.push_back({v.Y.at(p)[rslot], m.widths[p]});
            }
        } else {
            in.push_back({v.Y.at(i - 1)[wslot], m.widths[i - 1]});
        }
        for (auto& l : m.links_into(i)) {
            const int slot = stage_seg_[l.first] == seg ? wslot : rslot;
            in.push_back({v.Y.at(l.first)[slot], m.widths[l.first]});
        }
        void* y = i == m.L ? eps_out : v.Y.at(i)[wslot];
        enq_kernels_ += E_->enqueue_stage(v.idx, i, in, embed_t, v.H.at(i), y, v.bad, seq * kKeyStride + i, v.comp,
                                          true);
        if (mode_ == kParallel) CK(cudaEventRecord(v.stage_done.at(i), v.comp));  // its copies may start
    }
}

// after v evaluated `seg` into `slot`: push its outputs to every consumer
// vdev, and its eps (if any) to the sampler on vdev 0.
void Session::enqueue_transfers(VDev& v, int seg, int slot, int eps_step) {
    if (mode_ != kParallel) return;
    const Model& m = E_->model();
    std::vector<std::pair<int, int>> xfers;  // (stage, consumer vdev)
    for (int cseg = seg + 1; cseg <= N_; ++cseg) {
        std::set<int> stages;
        if (cseg == seg + 1) stages.insert(seg_last_[seg]);
        for (int i = seg_first_[cseg]; i <= seg_last_[cseg]; ++i)
            for (auto& l : m.links_into(i))
                if (stage_seg_[l.first] == seg) stages.insert(l.first);
        for (int c : consumers_of_segment(cseg))
            if (c != v.v)
                for (int p : stages)
                    if (std::find(xfers.begin(), xfers.end(), std::make_pair(p, c)) == xfers.end())
                        xfers.emplace_back(p, c);
    }
    const bool eps_xfer = eps_step >= 0 && v.v != 0;
    if (xfers.empty() && !eps_xfer) return;
    setdev(v.ordinal);
    // each output leaves as soon as the stage that produced it finished (a crossing skip made
    // early in the segment travels while the segment computes on); eps after the whole eval
    std::set<int> waited;
    std::sort(xfers.begin(), xfers.end());
    for (auto& [p, c] : xfers) {
        VDev& cv = vd_[c];
        if (waited.insert(-1 - p).second) CK(cudaStreamWaitEvent(v.comm, v.stage_done.at(p), 0));
        if (cv.read_rec[slot] && waited.insert(c).second) CK(cudaStreamWaitEvent(v.comm, cv.read_done[slot], 0));
        const size_t bytes = static_cast<size_t>(m.widths[p]) * E_->stage_bytes();
        if (cv.ordinal == v.ordinal)
            CK(cudaMemcpyAsync(cv.Y.at(p)[slot], v.Y.at(p)[slot], bytes, cudaMemcpyDeviceToDevice, v.comm));
        else
            CK(cudaMemcpyPeerAsync(cv.Y.at(p)[slot], cv.ordinal, v.Y.at(p)[slot], v.ordinal, bytes, v.comm));
    }
    if (eps_xfer) {
        CK(cudaStreamWaitEvent(v.comm, v.eval_done, 0));
        const size_t bytes = static_cast<size_t>(d_) * ab_bytes_;
        void* dst = offset(traj_eps_, static_cast<size_t>(eps_step) * bytes);
        if (vd_[0].ordinal == v.ordinal)
            CK(cudaMemcpyAsync(dst, v.EPS[slot], bytes, cudaMemcpyDeviceToDevice, v.comm));
        else
            CK(cudaMemcpyPeerAsync(dst, vd_[0].ordinal, v.EPS[slot], v.ordinal, bytes, v.comm));
    }
    CK(cudaEventRecord(v.xfer_done[slot], v.comm));
    v.xfer_rec[slot] = true;
}

void Session::enqueue_ddim(int step, int t) {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    const size_t row = static_cast<size_t>(d_) * ab_bytes_;
    DdimArgs a = {};
    a.x = offset(traj_lat_, step * row);
    a.eps = offset(traj_eps_, step * row);
    a.out = offset(traj_lat_, (step + 1) * row);
    a.d = d_;
    const double abar_t = ab_[t], abar_prev = ab_[t - 1];
    a.s1 = std::sqrt(1.0 - abar_t);
    a.s2 = std::sqrt(abar_t);
    a.s3 = std::sqrt(abar_prev);
    a.s4 = std::sqrt(1.0 - abar_prev);
    a.bad = v0.bad + 1;
    a.bad_key = step;
    launch_ddim(E_->prec(), a, v0.comp);
    ++enq_kernels_;
}

int Session::vdev_of_eval(const Eval& e) const { return mode_ == kParallel ? e.device : 0; }

void Session::enqueue_all(bool capture) {
    const int L = E_->model().L;
    (void)L;
    enq_kernels_ = 0;
    VDev& v0 = vd_[0];
    for (auto& v : vd_) v.read_rec = v.xfer_rec = {false, false};
    const size_t row = static_cast<size_t>(d_) * ab_bytes_;
    auto lat = [&](int step) { return offset(traj_lat_, step * row); };
    auto epsrow = [&](int step) { return offset(traj_eps_, step * row); };
    const bool timing = instrumented_enqueue_;

    setdev(v0.ordinal);
    launch_from_f64(E_->prec(), xT_dev_, traj_lat_, d_, v0.comp);
    ++enq_kernels_;
    if (timing) CK(cudaEventRecord(t_start_, v0.comp));
    CK(cudaEventRecord(fork_, v0.comp));
    for (auto& v : vd_) {
        setdev(v.ordinal);
        if (v.v != 0) CK(cudaStreamWaitEvent(v.comp, fork_, 0));
        CK(cudaStreamWaitEvent(v.comm, fork_, 0));
        CK(cudaMemsetAsync(v.bad, 0x7f, 2 * sizeof(int), v.comp));
        if (opts_.max_jitter_s > 0.0 && mode_ == kParallel) {  // executor.cpp:445-449
            Rng rng(mix_seed(opts_.jitter_seed, static_cast<uint64_t>(v.v)));
            launch_delay(rng.uniform() * opts_.max_jitter_s, v.comp);
            ++enq_kernels_;
        }
    }

    // BundleStore ledger (executor.cpp:28-62): the bundles this enqueue commits
    std::set<std::pair<int, int>> store;  // (segment, round)
    ledger_entries_.clear();
    auto put = [&](int seg, int r) {
        if (!store.insert({seg, r}).second)
            throw std::logic_error("BundleStore: entry (" + std::to_string(seg) + ", " + std::to_string(r) +
                                   ") already written");
    };

    auto record_eval = [&](VDev& v, int rslot) {
        CK(cudaEventRecord(v.eval_done, v.comp));
        CK(cudaEventRecord(v.read_done[rslot], v.comp));
        v.read_rec[rslot] = true;
    };

    int seq = 0;
    // ---- warm-up: w sequential cascades at embed t (executor.cpp:168-202)
    for (size_t wi = 0; wi < plan_.warmup_steps.size(); ++wi) {
        const int t = plan_.warmup_steps[wi];
        const int step = static_cast<int>(wi);
        for (int n = 1; n <= N_; ++n) {
            VDev& v = vd_[mode_ == kParallel ? part_.device_of_segment[n - 1] : 0];
            setdev(v.ordinal);
            wait_inputs(v, n, 1);
            if (v.xfer_rec[1]) CK(cudaStreamWaitEvent(v.comp, v.xfer_done[1], 0));
            void* eps_out = nullptr;
            if (n == N_) eps_out = v.v == 0 ? epsrow(step) : v.EPS[1];
            if (timing) CK(cudaEventRecord(warm_seg_ev_[wi][2 * (n - 1)], v.comp));
            enqueue_segment_eval(v, n, t, 1, 1, lat(step), eps_out, seq++);
            if (timing) CK(cudaEventRecord(warm_seg_ev_[wi][2 * (n - 1) + 1], v.comp));
            record_eval(v, 1);
            enqueue_transfers(v, n, 1, n == N_ ? step : -1);
        }
        if (mode_ == kParallel) {
            VDev& u = vd_[part_.device_of_segment[N_ - 1]];
            if (u.v != 0) {
                setdev(v0.ordinal);
                CK(cudaStreamWaitEvent(v0.comp, u.xfer_done[1], 0));
            }
        }
        enqueue_ddim(step, t);
        if (wi + 1 == plan_.warmup_steps.size())  // executor.cpp:540-541
            for (int n = 1; n < N_; ++n) put(n, -1);
    }
    if (timing) {
        setdev(v0.ordinal);
        CK(cudaEventRecord(t_warm_, v0.comp));
    }

    // ---- async rounds (executor.cpp:289-318 / 548-586)
    for (size_t ri = 0; ri < plan_.rounds.size(); ++ri) {
        const Round& rd = plan_.rounds[ri];
        const int r = rd.index;
        const int wslot = (r + 2) % 2, rslot = (r + 1) % 2;
        const int step0 = T_ - rd.sampler_steps.front();
        if (timing) {
            setdev(v0.ordinal);
            CK(cudaEventRecord(round_start_[ri], v0.comp));
        }
        for (size_t k = 0; k < rd.evals.size(); ++k) {
            const Eval& ev = rd.evals[k];
            if (ev.input.kind == 1 && !store.count({ev.input.producer_segment, ev.input.producer_round}))
                throw std::logic_error("executor: unresolvable cached ref (segment " +
                                       std::to_string(ev.input.producer_segment) + ", round " +
                                       std::to_string(ev.input.producer_round) + ") in round " +
                                       std::to_string(r));
            VDev& v = vd_[vdev_of_eval(ev)];
            setdev(v.ordinal);
            wait_inputs(v, ev.segment, rslot);
            if (v.xfer_rec[wslot]) CK(cudaStreamWaitEvent(v.comp, v.xfer_done[wslot], 0));
            void* eps_out = nullptr;
            if (ev.segment == N_) {
                const int es = T_ - *ev.emits_eps_for;
                eps_out = v.v == 0 ? epsrow(es) : v.EPS[wslot];
            }
            if (timing) CK(cudaEventRecord(eval_ev_[ri][k].first, v.comp));
            enqueue_segment_eval(v, ev.segment, ev.embed_t, wslot, rslot, lat(step0), eps_out, seq++);
            if (timing) CK(cudaEventRecord(eval_ev_[ri][k].second, v.comp));
            record_eval(v, rslot);
            if (mode_ == kParallel) enqueue_transfers(v, ev.segment, wslot, ev.emits_eps_for ? T_ - *ev.emits_eps_for : -1);
        }
        setdev(v0.ordinal);
        for (int t : rd.sampler_steps) {
            if (mode_ == kParallel) {
                for (const Eval& ev : rd.evals)
                    if (ev.emits_eps_for && *ev.emits_eps_for == t && ev.device != 0)
                        CK(cudaStreamWaitEvent(v0.comp, vd_[ev.device].xfer_done[wslot], 0));
            }
            enqueue_ddim(T_ - t, t);
        }
        if (timing) CK(cudaEventRecord(round_end_[ri], v0.comp));
        // commit in produced_by order, prune to the warm-up tail + rounds >= r-1 (executor.cpp:574-581)
        for (const Eval& ev : rd.evals)
            if (ev.segment < N_) put(ev.segment, r);
        for (auto it = store.begin(); it != store.end();)
            it = it->second != -1 && it->second < r + 1 - 2 ? store.erase(it) : std::next(it);
        ledger_entries_.push_back(static_cast<int>(store.size()));
    }

    // ---- join every stream back into vdev 0's compute stream
    for (auto& v : vd_) {
        setdev(v.ordinal);
        if (v.v != 0) {
            CK(cudaEventRecord(v.join, v.comp));
            setdev(v0.ordinal);
            CK(cudaStreamWaitEvent(v0.comp, v.join, 0));
            setdev(v.ordinal);
        }
        CK(cudaEventRecord(v.join, v.comm));
        setdev(v0.ordinal);
        CK(cudaStreamWaitEvent(v0.comp, v.join, 0));
    }
    setdev(v0.ordinal);
    if (timing) CK(cudaEventRecord(t_stop_, v0.comp));
    (void)capture;
}

// kernels of this library in a captured graph (kernel nodes, NCCL's own excluded): the
// bench's gpu_launches claim is counted from the graph itself, not from the enqueue calls
int graph_kernel_nodes(cudaGraph_t g) {
    size_t n = 0;
    CK(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(g, nodes.data(), &n));
    int k = 0;
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp = {};
        const char* name = nullptr;
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func &&
            cudaFuncGetName(&name, kp.func) == cudaSuccess && name && std::strncmp(name, "nccl", 4) == 0)
            continue;
        cudaGetLastError();
        ++k;
    }
    return k;
}

void Session::build_graph() {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    instrumented_enqueue_ = false;
    CK(cudaStreamBeginCapture(v0.comp, cudaStreamCaptureModeRelaxed));
    try {
        enqueue_all(true);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(v0.comp, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    CK(cudaStreamEndCapture(v0.comp, &graph_));
    CK(cudaGraphInstantiate(&gexec_, graph_, 0));
    kernel_count_ = graph_kernel_nodes(graph_);
}

void Session::launch() {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    if (gexec_) {
        CK(cudaEventRecord(t_start_, v0.comp));
        CK(cudaGraphLaunch(gexec_, v0.comp));
        CK(cudaEventRecord(t_stop_, v0.comp));
        return;
    }
    instrumented_enqueue_ = true;
    // (re)create timing events for this enqueue
    auto mk = []() {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    };
    if (eval_ev_.empty()) {
        for (auto& rd : plan_.rounds) {
            std::vector<std::pair<cudaEvent_t, cudaEvent_t>> row;
            std::vector<int> devs;
            for (auto& ev : rd.evals) {
                const int v = vdev_of_eval(ev);
                setdev(vd_[v].ordinal);
                row.emplace_back(mk(), mk());
                devs.push_back(v);
            }
            eval_ev_.push_back(row);
            eval_ev_dev_.push_back(devs);
            setdev(v0.ordinal);
            round_start_.push_back(mk());
            round_end_.push_back(mk());
        }
        for (size_t wi = 0; wi < plan_.warmup_steps.size(); ++wi) {
            std::vector<cudaEvent_t> row;
            for (int n = 1; n <= N_; ++n) {
                const int v = mode_ == kParallel ? part_.device_of_segment[n - 1] : 0;
                setdev(vd_[v].ordinal);
                row.push_back(mk());
                row.push_back(mk());
            }
            warm_seg_ev_.push_back(row);
        }
    }
    enqueue_all(false);
    kernel_count_ = enq_kernels_;
}

void Session::upload(const double* x_T) {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    std::memcpy(xT_host_, x_T, static_cast<size_t>(d_) * sizeof(double));
    CK(cudaMemcpyAsync(xT_dev_, xT_host_, static_cast<size_t>(d_) * sizeof(double), cudaMemcpyHostToDevice, v0.comp));
}

namespace {
bool event_done(cudaEvent_t e) {
    const cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return true;
    if (r == cudaErrorNotReady) return false;
    CK(r);
    return false;
}
}  // namespace

// executor.cpp:424-435 -- per-round deadline; names the devices still busy
void Session::wait_with_timeout(RunStatsOut*) {
    const double to = opts_.round_timeout_s;
    using clk = std::chrono::steady_clock;
    const std::string who = mode_ == kParallel ? "run_parallel" : "run_serial";
    auto wait_all = [&](const std::vector<std::pair<cudaEvent_t, int>>& evs, const std::string& what) {
        const auto deadline = clk::now() + std::chrono::duration<double>(to);
        while (true) {
            bool all = true;
            for (auto& e : evs) all &= event_done(e.first);
            if (all) return;
            if (clk::now() > deadline) {
                std::string msg = who + ": timeout in " + what + "; waiting on";
                std::set<int> busy;
                for (auto& e : evs)
                    if (!event_done(e.first)) busy.insert(e.second);
                for (int d : busy) msg += " device " + std::to_string(d);
                for (auto& v : vd_) {  // drain before unwinding
                    cudaSetDevice(v.ordinal);
                    cudaStreamSynchronize(v.comp);
                    cudaStreamSynchronize(v.comm);
                }
                throw std::runtime_error(msg);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    };
    for (size_t wi = 0; wi < warm_seg_ev_.size(); ++wi)
        for (int n = 1; n <= N_; ++n) {
            const int v = mode_ == kParallel ? part_.device_of_segment[n - 1] : 0;
            wait_all({{warm_seg_ev_[wi][2 * (n - 1) + 1], v}}, "warm-up");
        }
    for (size_t ri = 0; ri < eval_ev_.size(); ++ri) {
        std::vector<std::pair<cudaEvent_t, int>> evs;
        for (size_t k = 0; k < eval_ev_[ri].size(); ++k) evs.emplace_back(eval_ev_[ri][k].second, eval_ev_dev_[ri][k]);
        evs.emplace_back(round_end_[ri], 0);
        wait_all(evs, "round " + std::to_string(plan_.rounds[ri].index));
    }
}

void Session::check_flags(bool sequential) {
    int stage_key = INT_MAX, ddim_key = INT_MAX;
    for (auto& v : vd_) {
        setdev(v.ordinal);
        int h[2];
        CK(cudaMemcpy(h, v.bad, sizeof h, cudaMemcpyDeviceToHost));
        if (h[0] != kBadSentinel) stage_key = std::min(stage_key, h[0]);
        if (h[1] != kBadSentinel) ddim_key = std::min(ddim_key, h[1]);
    }
    if (stage_key != INT_MAX) {
        const int stage = stage_key % kKeyStride;
        const std::string inner = "eval: non-finite activation at stage " + std::to_string(stage);
        if (sequential) {
            const int t = T_ - stage_key / kKeyStride;
            throw std::runtime_error("sequential_denoise: eps_fn failed at t=" + std::to_string(t) + ": " + inner);
        }
        throw std::domain_error(inner);
    }
    if (ddim_key != INT_MAX)
        throw std::domain_error("predict_x0: non-finite eps at t=" + std::to_string(T_ - ddim_key));
}

void Session::run(const double* x_T, double* lat, double* eps, RunStatsOut* stats) {
    VDev& v0 = vd_[0];
    upload(x_T);
    launch();
    if (!gexec_) {
        wait_with_timeout(stats);
    } else {
        // one deadline for the whole graph
        const double budget = opts_.round_timeout_s * (plan_.rounds.size() + plan_.w + 1);
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(budget);
        while (!event_done(t_stop_)) {
            if (std::chrono::steady_clock::now() > deadline) {
                cudaStreamSynchronize(v0.comp);
                throw std::runtime_error(std::string(mode_ == kParallel ? "run_parallel" : "run_serial") +
                                         ": timeout waiting on device 0");
            }
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    setdev(v0.ordinal);
    CK(cudaStreamSynchronize(v0.comp));
    check_flags(mode_ == kSequential);
    download(lat, eps);
    if (stats) {
        RunStatsOut& s = *stats;
        const int D = mode_ == kParallel ? plan_.D : plan_.D;
        s.broadcast_count = static_cast<int>(plan_.rounds.size());
        s.device_evals.assign(D, 0);
        s.device_busy_s.assign(D, 0.0);
        for (int n = 0; n < N_; ++n) s.device_evals[part_.device_of_segment[n]] += plan_.w;
        for (auto& r : plan_.rounds)
            for (auto& ev : r.evals) s.device_evals[ev.device] += 1;
        s.store_entries = ledger_entries_;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, t_start_, t_stop_));
        s.total_wall_s = ms * 1e-3;
        s.round_wall_s.assign(plan_.rounds.size(), 0.0);
        s.round_comm_s.assign(plan_.rounds.size(), 0.0);
        if (!gexec_) {
            CK(cudaEventElapsedTime(&ms, t_start_, t_warm_));
            s.warmup_wall_s = ms * 1e-3;
            for (size_t wi = 0; wi < warm_seg_ev_.size(); ++wi)
                for (int n = 1; n <= N_; ++n) {
                    CK(cudaEventElapsedTime(&ms, warm_seg_ev_[wi][2 * (n - 1)], warm_seg_ev_[wi][2 * (n - 1) + 1]));
                    s.device_busy_s[part_.device_of_segment[n - 1]] += ms * 1e-3;
                }
            cudaEvent_t prev = t_warm_;
            for (size_t ri = 0; ri < eval_ev_.size(); ++ri) {
                double mx = 0.0;
                for (size_t k = 0; k < eval_ev_[ri].size(); ++k) {
                    CK(cudaEventElapsedTime(&ms, eval_ev_[ri][k].first, eval_ev_[ri][k].second));
                    s.device_busy_s[plan_.rounds[ri].evals[k].device] += ms * 1e-3;
                    mx = std::max(mx, ms * 1e-3);
                }
                CK(cudaEventElapsedTime(&ms, prev, round_end_[ri]));
                s.round_wall_s[ri] = ms * 1e-3;
                s.round_comm_s[ri] = std::max(0.0, s.round_wall_s[ri] - mx);
                prev = round_end_[ri];
            }
        }
    }
}

// pinned staging -> the caller's fp64 arrays; large trajectories (UNet: 2T+1 latents of
// 37K-262K values) are widened on several host threads -- single-threaded this was ~2% of
// the c2 end-to-end time
void widen_to_f64(const void* src, int bytes, double* dst, size_t n) {
    auto part = [&](size_t b, size_t e) {
        if (bytes == 8) {
            std::memcpy(dst + b, static_cast<const double*>(src) + b, (e - b) * 8);
        } else {
            const float* f = static_cast<const float*>(src);
            for (size_t i = b; i < e; ++i) dst[i] = f[i];
        }
    };
    const size_t nt = n < (1u << 20) ? 1 : std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
    if (nt == 1) return part(0, n);
    std::vector<std::thread> th;
    for (size_t k = 1; k < nt; ++k) th.emplace_back(part, n * k / nt, n * (k + 1) / nt);
    part(0, n / nt);
    for (auto& t : th) t.join();
}

void Session::download(double* lat, double* eps) {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    const size_t nl = static_cast<size_t>(T_ + 1) * d_, ne = static_cast<size_t>(T_) * d_;
    if (!lat && !eps) return;
    CK(cudaMemcpyAsync(out_host_, traj_lat_, nl * ab_bytes_, cudaMemcpyDeviceToHost, v0.comp));
    CK(cudaMemcpyAsync(offset(out_host_, nl * ab_bytes_), traj_eps_, ne * ab_bytes_, cudaMemcpyDeviceToHost, v0.comp));
    CK(cudaStreamSynchronize(v0.comp));
    if (lat) widen_to_f64(out_host_, ab_bytes_, lat, nl);
    if (eps) widen_to_f64(offset(out_host_, nl * ab_bytes_), ab_bytes_, eps, ne);
}

double Session::time_runs(int iters) {
    VDev& v0 = vd_[0];
    setdev(v0.ordinal);
    if (!gexec_) throw std::logic_error("time_runs: session has no CUDA graph (instrumented/delayed sessions)");
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, v0.comp));
    for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(gexec_, v0.comp));
    CK(cudaEventRecord(b, v0.comp));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    check_flags(mode_ == kSequential);
    return ms / std::max(1, iters);
}

}  // namespace adx
