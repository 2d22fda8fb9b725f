// rank.cu -- one process per GPU: the async loop of one rank over NCCL.
//
// Rank v evaluates exactly the plan's device-v evals on its own GPU and
// exchanges stage outputs / eps with its peers by ncclSend/ncclRecv on a comm
// stream, one NCCL group per exchange point of rank_program() (schedule.hpp).
// Event edges: every eval waits for the last exchange group (its inputs, and
// the end of the sends that read the slot it is about to overwrite); every
// group waits for the last local eval (the outputs it sends, and the reads of
// the slots it receives into).  Rank 0 owns the latent chain and runs DDIM.
// The whole program is captured once into a CUDA graph per rank (NCCL p2p is
// graph-capturable); every replay on every rank issues the same NCCL ops in
// the same order.  NCCL is loaded with dlopen so the library has no link-time
// NCCL dependency (torch's libnccl.so.2 is reused when present).
#include "engine.hpp"
#include "schedule.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <set>

namespace adx {

#define CKR(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!api.Send) throw cuda_error(err.empty() ? "NCCL symbols missing" : err);
    return api;
}

void CKN(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw cuda_error(std::string("NCCL error: ") + nccl().GetErrorString(r) + " at " + what);
}

const void* off_c(const void* p, size_t b) { return static_cast<const char*>(p) + b; }
void* off_m(void* p, size_t b) { return static_cast<char*>(p) + b; }

}  // namespace

void nccl_unique_id(char* out128) {
    ncclUniqueId id;
    CKN(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
}

class RankSession {
public:
    RankSession(Engine* e, const Plan& plan, const Partition& part, const std::vector<double>& ab, int rank,
                const char* id128, const RunOptions& opts)
        : E_(e), plan_(plan), part_(part), ab_(ab), rank_(rank), opts_(opts) {
        const Model& m = E_->model();
        T_ = static_cast<int>(ab_.size()) - 1;
        d_ = m.data_dim();
        const auto v = validate_plan(plan_);
        if (!v.empty()) throw std::invalid_argument("run: invalid plan: " + v.front());
        if (part_.num_segments() != plan_.N) throw std::invalid_argument("run: partition segment count != plan.N");
        part_.validate(m);
        if (!part_.contiguous()) throw std::invalid_argument("run: partition must be a contiguous cascade");
        if (plan_.T != T_) throw std::invalid_argument("run: plan T != schedule T");
        for (int n = 0; n < plan_.N; ++n)
            if (part_.device_of_segment[n] != n)
                throw std::invalid_argument("run_parallel: segment " + std::to_string(n + 1) +
                                            " must be placed on device " + std::to_string(n));
        if (rank_ < 0 || rank_ >= plan_.D)
            throw std::invalid_argument("rank " + std::to_string(rank_) + " outside plan devices [0, " +
                                        std::to_string(plan_.D) + ")");
        ab_bytes_ = act_bytes(E_->prec());
        ops_ = rank_program(plan_, part_, m, rank_);
        seg_first_.assign(plan_.N + 1, 0);
        seg_last_.assign(plan_.N + 1, 0);
        stage_seg_.assign(m.L + 1, 0);
        for (int n = 1; n <= plan_.N; ++n) {
            seg_first_[n] = part_.segments[n - 1].front();
            seg_last_[n] = part_.segments[n - 1].back();
            for (int s : part_.segments[n - 1]) stage_seg_[s] = n;
        }
        CKR(cudaSetDevice(E_->ordinal(0)));
        alloc();
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        CKN(nccl().CommInitRank(&comm_, plan_.D, id, rank_), "ncclCommInitRank");
        build_graph();
    }
    ~RankSession() {
        cudaSetDevice(E_->ordinal(0));
        if (comp_) cudaStreamSynchronize(comp_);
        if (gexec_) cudaGraphExecDestroy(gexec_);
        if (graph_) cudaGraphDestroy(graph_);
        if (comm_) nccl().CommDestroy(comm_);
        for (auto& kv : Y_) {
            cudaFree(kv.second[0]);
            cudaFree(kv.second[1]);
        }
        for (auto& kv : H_) cudaFree(kv.second);
        if (host_stage_) cudaFreeHost(host_stage_);
        cudaFree(EPS_[0]);
        cudaFree(EPS_[1]);
        cudaFree(traj_lat_);
        cudaFree(traj_eps_);
        cudaFree(xT_);
        cudaFree(bad_);
        for (cudaEvent_t e : {ev_eval_, ev_group_, ev_fork_, ev_join_, t0_, t1_, ev_eps_})
            if (e) cudaEventDestroy(e);
        for (auto* pool : {&ev_stage_, &ev_deliver_, &ev_sent_, &ev_read_})
            for (auto& kv : *pool) cudaEventDestroy(kv.second);
        if (comp_) cudaStreamDestroy(comp_);
        if (cstr_) cudaStreamDestroy(cstr_);
    }

    void run(const double* x_T, double* lat, double* eps) {
        CKR(cudaSetDevice(E_->ordinal(0)));
        if (rank_ == 0) CKR(cudaMemcpyAsync(xT_, x_T, d_ * sizeof(double), cudaMemcpyHostToDevice, comp_));
        CKR(cudaGraphLaunch(gexec_, comp_));
        CKR(cudaStreamSynchronize(comp_));
        int h[2];
        CKR(cudaMemcpy(h, bad_, sizeof h, cudaMemcpyDeviceToHost));
        if (h[0] != 0x7f7f7f7f)
            throw std::domain_error("eval: non-finite activation at stage " + std::to_string(h[0] % 1024));
        if (h[1] != 0x7f7f7f7f)
            throw std::domain_error("predict_x0: non-finite eps at t=" + std::to_string(T_ - h[1]));
        if (rank_ == 0 && (lat || eps)) {
            const size_t nl = static_cast<size_t>(T_ + 1) * d_, ne = static_cast<size_t>(T_) * d_;
            if (!host_stage_) CKR(cudaMallocHost(&host_stage_, (nl + ne) * ab_bytes_));  // pinned, reused
            unsigned char* buf = static_cast<unsigned char*>(host_stage_);
            CKR(cudaMemcpy(buf, traj_lat_, nl * ab_bytes_, cudaMemcpyDeviceToHost));
            CKR(cudaMemcpy(buf + nl * ab_bytes_, traj_eps_, ne * ab_bytes_, cudaMemcpyDeviceToHost));
            if (lat) widen_to_f64(buf, ab_bytes_, lat, nl);
            if (eps) widen_to_f64(buf + nl * ab_bytes_, ab_bytes_, eps, ne);
        }
    }

    double time_runs(int iters) {
        CKR(cudaSetDevice(E_->ordinal(0)));
        CKR(cudaEventRecord(t0_, comp_));
        for (int i = 0; i < iters; ++i) CKR(cudaGraphLaunch(gexec_, comp_));
        CKR(cudaEventRecord(t1_, comp_));
        CKR(cudaEventSynchronize(t1_));
        float ms = 0;
        CKR(cudaEventElapsedTime(&ms, t0_, t1_));
        return ms / std::max(1, iters);
    }
    int kernel_count() const { return kernels_; }

private:
    void alloc() {
        const Model& m = E_->model();
        std::set<int> mine;
        for (auto& op : ops_)
            if (op.kind == kOpEval) mine.insert(op.seg);
        std::set<int> need;
        for (int seg : mine) {
            for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i) {
                E_->stage_on(0, i);
                if (i < m.L) need.insert(i);
                void* h = nullptr;
                CKR(cudaMalloc(&h, static_cast<size_t>(std::max(m.widths[i], 1)) * E_->stage_bytes()));
                H_[i] = h;
                for (auto& l : m.links_into(i))
                    if (stage_seg_[l.first] != seg) need.insert(l.first);
            }
            if (seg > 1) need.insert(seg_last_[seg - 1]);
        }
        E_->ensure_tables(0, T_);
        for (int p : need) {
            std::array<void*, 2> y{};
            for (int s = 0; s < 2; ++s) {
                CKR(cudaMalloc(&y[s], static_cast<size_t>(m.widths[p]) * E_->stage_bytes()));
                CKR(cudaMemset(y[s], 0, static_cast<size_t>(m.widths[p]) * E_->stage_bytes()));
            }
            Y_[p] = y;
        }
        for (int s = 0; s < 2; ++s) CKR(cudaMalloc(&EPS_[s], static_cast<size_t>(d_) * ab_bytes_));
        CKR(cudaMalloc(&traj_lat_, static_cast<size_t>(T_ + 1) * d_ * ab_bytes_));
        CKR(cudaMalloc(&traj_eps_, static_cast<size_t>(T_) * d_ * ab_bytes_));
        CKR(cudaMemset(traj_eps_, 0, static_cast<size_t>(T_) * d_ * ab_bytes_));
        CKR(cudaMalloc(&xT_, d_ * sizeof(double)));
        CKR(cudaMemset(xT_, 0, d_ * sizeof(double)));
        CKR(cudaMalloc(&bad_, 2 * sizeof(int)));
        CKR(cudaStreamCreateWithFlags(&comp_, cudaStreamNonBlocking));
        CKR(cudaStreamCreateWithFlags(&cstr_, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&ev_eval_, &ev_group_, &ev_fork_, &ev_join_, &ev_eps_})
            CKR(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CKR(cudaEventCreate(&t0_));
        CKR(cudaEventCreate(&t1_));
    }

    void eval(const RankOp& op, int seq) {
        const Model& m = E_->model();
        const size_t row = static_cast<size_t>(d_) * ab_bytes_;
        const int seg = op.seg;
        void* eps_out = nullptr;
        if (seg == plan_.N) eps_out = rank_ == 0 ? off_m(traj_eps_, op.eps_step * row) : EPS_[op.wslot];
        for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i) {
            std::vector<Seg> in;
            if (i == seg_first_[seg]) {
                if (seg == 1) {
                    in.push_back({off_c(traj_lat_, op.step * row), d_});
                    in.push_back({E_->etab_row(0, op.t), m.E});
                } else {
                    const int p = seg_last_[seg - 1];
                    in.push_back({Y_.at(p)[op.rslot], m.widths[p]});
                }
            } else {
                in.push_back({Y_.at(i - 1)[op.wslot], m.widths[i - 1]});
            }
            for (auto& l : m.links_into(i))
                in.push_back({Y_.at(l.first)[stage_seg_[l.first] == seg ? op.wslot : op.rslot], m.widths[l.first]});
            void* y = i == m.L ? eps_out : Y_.at(i)[op.wslot];
            kernels_ += E_->enqueue_stage(0, i, in, op.t, H_.at(i), y, bad_, seq * 1024 + i, comp_, true);
            CKR(cudaEventRecord(ev(ev_stage_, i), comp_));  // its sends may start now
        }
    }

    // one event per key, created on first use (capture-time dependencies: a wait binds to the
    // most recent record of the event when it is issued)
    cudaEvent_t ev(std::map<long long, cudaEvent_t>& pool, long long key) {
        auto it = pool.find(key);
        if (it != pool.end()) return it->second;
        cudaEvent_t e;
        CKR(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        pool[key] = e;
        return e;
    }
    static long long key(int stage, int slot) { return static_cast<long long>(stage) * 4 + slot + 8; }

    void build_graph() {
        CKR(cudaStreamBeginCapture(comp_, cudaStreamCaptureModeRelaxed));
        kernels_ = 0;
        if (rank_ == 0) {
            launch_from_f64(E_->prec(), xT_, traj_lat_, d_, comp_);
            ++kernels_;
        }
        CKR(cudaMemsetAsync(bad_, 0x7f, 2 * sizeof(int), comp_));
        CKR(cudaEventRecord(ev_fork_, comp_));
        CKR(cudaStreamWaitEvent(cstr_, ev_fork_, 0));
        // Dependencies are per exchange point (schedule.hpp): a point's sends wait for the stage
        // that produced them, its receives for the last local eval that read the slot they
        // overwrite; an eval waits for the points that delivered its inputs and for the earlier
        // sends out of the slots it overwrites; the sampler waits for the eps delivery.
        int seq = 0;
        const size_t row = static_cast<size_t>(d_) * ab_bytes_;
        const Model& mdl = E_->model();
        bool have_eps = false;
        for (size_t oi = 0; oi < ops_.size(); ++oi) {
            const RankOp& op = ops_[oi];
            switch (op.kind) {
                case kOpEval: {
                    // inputs received from other ranks (this slot), and earlier sends out of the
                    // slots this eval overwrites
                    const int seg = op.seg;
                    std::set<int> reads;
                    if (seg > 1) reads.insert(seg_last_[seg - 1]);
                    for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i)
                        for (auto& l : mdl.links_into(i))
                            if (stage_seg_[l.first] != seg) reads.insert(l.first);
                    for (int p : reads)
                        if (ev_deliver_.count(key(p, op.rslot))) CKR(cudaStreamWaitEvent(comp_, ev_deliver_.at(key(p, op.rslot)), 0));
                    for (int i = seg_first_[seg]; i <= seg_last_[seg]; ++i)
                        if (ev_sent_.count(key(i, op.wslot))) CKR(cudaStreamWaitEvent(comp_, ev_sent_.at(key(i, op.wslot)), 0));
                    if (seg == plan_.N && ev_sent_.count(key(-1, op.wslot)))
                        CKR(cudaStreamWaitEvent(comp_, ev_sent_.at(key(-1, op.wslot)), 0));
                    eval(op, seq++);
                    CKR(cudaEventRecord(ev_eval_, comp_));
                    CKR(cudaEventRecord(ev(ev_read_, op.rslot), comp_));  // last reader of slot rslot
                    break;
                }
                case kOpGroup: {
                    bool sends = false, recvs = false;
                    int rslot = 0;
                    for (size_t k = oi + 1; k < ops_.size() && ops_[k].kind != kOpEnd; ++k) {
                        sends |= ops_[k].kind == kOpSend;
                        if (ops_[k].kind == kOpRecv && ops_[k].stage >= 0) recvs = true, rslot = ops_[k].slot;
                    }
                    if (sends) CKR(cudaStreamWaitEvent(cstr_, op.stage >= 0 ? ev(ev_stage_, op.stage) : ev_eval_, 0));
                    if (recvs && ev_read_.count(rslot)) CKR(cudaStreamWaitEvent(cstr_, ev_read_.at(rslot), 0));
                    CKN(nccl().GroupStart(), "ncclGroupStart");
                    break;
                }
                case kOpSend: {
                    const void* src = op.stage < 0 ? EPS_[op.slot] : Y_.at(op.stage)[op.slot];
                    CKN(nccl().Send(src, op.elems * (op.stage < 0 ? ab_bytes_ : E_->stage_bytes()), ncclInt8,
                                    op.peer, comm_, cstr_),
                        "ncclSend");
                    break;
                }
                case kOpRecv: {
                    void* dst = op.stage < 0 ? off_m(traj_eps_, op.step * row) : Y_.at(op.stage)[op.slot];
                    CKN(nccl().Recv(dst, op.elems * (op.stage < 0 ? ab_bytes_ : E_->stage_bytes()), ncclInt8,
                                    op.peer, comm_, cstr_),
                        "ncclRecv");
                    break;
                }
                case kOpEnd: {
                    CKN(nccl().GroupEnd(), "ncclGroupEnd");
                    // what this point moved: register the delivery / send-completion events
                    size_t g = oi;
                    while (g > 0 && ops_[g].kind != kOpGroup) --g;
                    for (size_t k = g + 1; k < oi; ++k) {
                        const RankOp& x = ops_[k];
                        if (x.kind == kOpRecv && x.stage < 0) {
                            CKR(cudaEventRecord(ev_eps_, cstr_));
                            have_eps = true;
                        } else if (x.kind == kOpRecv) {
                            cudaEvent_t e = ev(ev_deliver_, key(x.stage, x.slot));
                            CKR(cudaEventRecord(e, cstr_));
                        } else if (x.kind == kOpSend) {
                            cudaEvent_t e = ev(ev_sent_, key(x.stage, x.slot));
                            CKR(cudaEventRecord(e, cstr_));
                        }
                    }
                    break;
                }
                case kOpDdim: {
                    if (have_eps) CKR(cudaStreamWaitEvent(comp_, ev_eps_, 0));
                    DdimArgs a = {};
                    a.x = off_c(traj_lat_, op.step * row);
                    a.eps = off_c(traj_eps_, op.step * row);
                    a.out = off_m(traj_lat_, (op.step + 1) * row);
                    a.d = d_;
                    a.s1 = std::sqrt(1.0 - ab_[op.t]);
                    a.s2 = std::sqrt(ab_[op.t]);
                    a.s3 = std::sqrt(ab_[op.t - 1]);
                    a.s4 = std::sqrt(1.0 - ab_[op.t - 1]);
                    a.bad = bad_ + 1;
                    a.bad_key = op.step;
                    launch_ddim(E_->prec(), a, comp_);
                    ++kernels_;
                    break;
                }
            }
        }
        CKR(cudaEventRecord(ev_join_, cstr_));
        CKR(cudaStreamWaitEvent(comp_, ev_join_, 0));
        CKR(cudaStreamEndCapture(comp_, &graph_));
        CKR(cudaGraphInstantiate(&gexec_, graph_, 0));
        kernels_ = graph_kernel_nodes(graph_);
    }

    Engine* E_;
    Plan plan_;
    Partition part_;
    std::vector<double> ab_;
    int rank_, T_ = 0, d_ = 0, ab_bytes_ = 0, kernels_ = 0;
    void* host_stage_ = nullptr;  // pinned trajectory staging (rank 0)
    RunOptions opts_;
    std::vector<RankOp> ops_;
    std::vector<int> seg_first_, seg_last_, stage_seg_;
    std::map<int, std::array<void*, 2>> Y_;
    std::map<int, void*> H_;
    std::array<void*, 2> EPS_{nullptr, nullptr};
    void *traj_lat_ = nullptr, *traj_eps_ = nullptr;
    double* xT_ = nullptr;
    int* bad_ = nullptr;
    cudaStream_t comp_ = nullptr, cstr_ = nullptr;
    cudaEvent_t ev_eval_ = nullptr, ev_group_ = nullptr, ev_fork_ = nullptr, ev_join_ = nullptr, t0_ = nullptr,
                t1_ = nullptr, ev_eps_ = nullptr;
    std::map<long long, cudaEvent_t> ev_stage_, ev_deliver_, ev_sent_, ev_read_;
    ncclComm_t comm_ = nullptr;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t gexec_ = nullptr;
};

// factory helpers for the C ABI (keeps RankSession private to this file)
void* rank_session_create(Engine* e, const Plan& plan, const Partition& part, const std::vector<double>& ab,
                          int rank, const char* id, const RunOptions& opts) {
    return new RankSession(e, plan, part, ab, rank, id, opts);
}
void rank_session_destroy(void* s) { delete static_cast<RankSession*>(s); }
void rank_session_run(void* s, const double* x, double* lat, double* eps) {
    static_cast<RankSession*>(s)->run(x, lat, eps);
}
double rank_session_time(void* s, int iters) { return static_cast<RankSession*>(s)->time_runs(iters); }
int rank_session_kernels(void* s) { return static_cast<RankSession*>(s)->kernel_count(); }

}  // namespace adx
