// engine.hpp -- device-resident AsyncDiff executor.
//
// Engine  : model weights per physical GPU (lazily uploaded, row-major, padded
//           pitch, in the engine precision) + per-t bias/embedding tables.
// Session : one compiled run of (plan, partition, placement).  It owns the
//           activation buffers, streams and events, and turns the static plan
//           into a DAG of stage GEMVs, DDIM updates and inter-device copies
//           which is either enqueued directly (instrumented / timeout-checked
//           runs) or captured once into a single multi-device CUDA graph.
//
// Snapshot semantics of the reference (executor.cpp:121-156, 289-318) are
// realised with two parity slots per stage output: round r writes slot
// s(r) = (r+2)%2 and reads cross-segment inputs from slot s(r-1); the warm-up
// cascade works fresh in slot s(-1) = 1, which round 0 then reads as the
// round -1 bundle.  Hazards between a copy and the evals on either side are
// ordered with events (see Session::enqueue).
#pragma once

#include "host.hpp"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <array>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

namespace adx {

struct DevStage {
    void* w1 = nullptr;
    int pitch1 = 0;
    void* w2 = nullptr;
    int pitch2 = 0;
    void* b2 = nullptr;
    void* ctab = nullptr;  // (T+1) x hidden, act dtype: b1 + Tin . e_t
    int ctab_T = -1;
};

struct DevShared {
    int ordinal = 0;
    std::vector<DevStage> stages;
    void* etab = nullptr;  // (T+1) x E, act dtype: e_t = proj . sinusoid(t)
    int etab_T = -1;
};

// one input segment of a stage GEMV (device pointer + length)
struct Seg {
    const void* p;
    int n;
};

class Engine {
public:
    Engine(const Model& m, int prec, std::vector<int> ordinals);
    ~Engine();
    const Model& model() const { return model_; }
    int prec() const { return prec_; }
    int num_ordinals() const { return static_cast<int>(ordinals_.size()); }
    int ordinal(int idx) const { return ordinals_[idx % ordinals_.size()]; }

    // weights of `stage` on ordinals_[idx], uploading on first use
    const DevStage& stage_on(int idx, int stage);
    void ensure_tables(int idx, int T);
    const void* etab_row(int idx, int t) const;
    long long weight_bytes_resident(int idx) const;
    // algorithmic weight bytes one evaluation of `stage` streams
    size_t stage_weight_bytes(int stage) const;

    // Enqueue one stage (run_stage_range body, denoiser.cpp:182-188) on the
    // current device's `stream`: h = lrelu(W1 [inputs] + ctab[t]); y = W2 h + b2.
    // Returns kernels launched.
    int enqueue_stage(int idx, int stage, const std::vector<Seg>& inputs, int embed_t, void* h, void* y,
                      int* bad, int key, cudaStream_t stream, bool pdl);

    // Device time of one full-model pass (2L stage GEMVs, CUDA graph, events on
    // the launching stream), mean over `iters` back-to-back passes.  Used for the
    // HBM roofline of the stage GEMV kernel.
    // profile != nullptr: also run one eager pass with per-launch events around every
    // tensor-core kernel; per kind (conv, GEMM, attention): {launches, ms, flops}
    // device ms of one full pass (graph of back-to-back passes); optionally the tensor-core
    // family profile of an eager pass and the device ms of every stage on its own (stage_ms[L])
    double time_eval_ms(int idx, int t_embed, int iters, int* launches, double (*profile)[3] = nullptr,
                        double* stage_ms = nullptr);
    // element size of stage outputs (bf16 for the UNet family, the activation dtype otherwise)
    // bytes per stage-output element: UNet bf16 mode 2, UNet f32 mode 4, MLP the engine precision
    int stage_bytes() const { return model_.kind == 1 ? (prec_ == kF32 ? 4 : 2) : act_bytes(prec_); }

private:
    class UNetDevice& unet(int idx);
    Model model_;
    int prec_;
    std::vector<int> ordinals_;
    std::vector<DevShared> dev_;
    std::vector<std::shared_ptr<class UNetDevice>> unet_;
};

struct RunOptions {
    double round_timeout_s = 30.0;
    // executor.cpp:445-449: worker d starts after uniform() * max_jitter_s drawn from
    // Rng(mix_seed(jitter_seed, d)); here a GPU sleep at the head of vdev d's compute stream
    uint64_t jitter_seed = 0;
    double max_jitter_s = 0.0;
    std::vector<double> segment_delay_s;
    bool use_graph = true;
    bool instrument = false;
};

struct RunStatsOut {
    int broadcast_count = 0;
    double warmup_wall_s = 0.0, total_wall_s = 0.0;
    std::vector<double> round_wall_s, round_comm_s, device_busy_s;
    std::vector<long long> device_evals;
    std::vector<int> store_entries;
};

class Session {
public:
    enum Mode { kSerial = 0, kParallel = 1, kSequential = 2 };
    Session(Engine* e, const Plan& plan, const Partition& part, const std::vector<double>& alpha_bars,
            int mode, int workers, const RunOptions& opts);
    ~Session();

    void upload(const double* x_T);
    // full host-facing run: upload, execute, download, finite/timeout checks
    void run(const double* x_T, double* lat, double* eps, RunStatsOut* stats);
    double time_runs(int iters);  // device-resident, ms per run
    void download(double* lat, double* eps);
    int kernel_count() const { return kernel_count_; }  // graph mode: kernel nodes of the graph
    long long weight_bytes_per_run() const { return weight_bytes_per_run_; }
    int T() const { return T_; }
    int d() const { return d_; }

private:
    struct VDev {
        int v = 0;
        int idx = 0;  // engine ordinal index
        int ordinal = 0;
        cudaStream_t comp = nullptr, comm = nullptr;
        int* bad = nullptr;  // [0] stage key, [1] ddim key
        std::set<int> segs;  // segments it evaluates
        std::map<int, std::array<void*, 2>> Y;
        std::map<int, void*> H;
        std::array<void*, 2> EPS{nullptr, nullptr};
        // sync events
        cudaEvent_t eval_done = nullptr;
        std::map<int, cudaEvent_t> stage_done;  // per stage it evaluates: its sends may start
        std::array<cudaEvent_t, 2> read_done{}, xfer_done{};
        std::array<bool, 2> read_rec{}, xfer_rec{};
        cudaEvent_t join = nullptr;
    };

    void setdev(int ordinal) const;
    void release();
    void alloc_buffers();
    void enqueue_all(bool capture);
    void enqueue_segment_eval(VDev& v, int seg, int embed_t, int wslot, int rslot, const void* latent,
                              void* eps_out, int seq);
    void enqueue_transfers(VDev& v, int seg, int slot, int eps_step);
    void enqueue_ddim(int step, int t);
    void wait_inputs(VDev& v, int seg, int rslot);
    void build_graph();
    void launch();
    void check_flags(bool sequential);
    void wait_with_timeout(RunStatsOut* stats);
    int vdev_of_eval(const Eval& e) const;
    std::vector<int> consumers_of_segment(int seg) const;

    Engine* E_;
    Plan plan_;
    Partition part_;
    std::vector<double> ab_;
    int mode_, T_, d_, N_;
    RunOptions opts_;
    int ab_bytes_;
    std::vector<VDev> vd_;
    std::vector<int> seg_first_, seg_last_, stage_seg_;
    void* traj_lat_ = nullptr;  // (T+1) x d on vdev 0
    void* traj_eps_ = nullptr;  // T x d on vdev 0
    double* xT_dev_ = nullptr;
    double* xT_host_ = nullptr;  // pinned
    void* out_host_ = nullptr;   // pinned, act dtype, (2T+1) x d
    cudaEvent_t fork_ = nullptr, t_start_ = nullptr, t_stop_ = nullptr, t_warm_ = nullptr;
    // instrumented timing events (timing-enabled, never re-recorded)
    std::vector<std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> eval_ev_;  // [round][k]
    std::vector<std::vector<int>> eval_ev_dev_;
    std::vector<cudaEvent_t> round_start_, round_end_;
    std::vector<std::vector<cudaEvent_t>> warm_seg_ev_;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t gexec_ = nullptr;
    bool instrumented_enqueue_ = false;
    // BundleStore bookkeeping (executor.cpp:28-62) replayed from the bundles the enqueue
    // actually commits: put per (segment, round) written, prune to the warm-up tail and
    // rounds >= r-1; occupancy after every round
    std::vector<int> ledger_entries_;
    int kernel_count_ = 0;
    long long weight_bytes_per_run_ = 0;
    int enq_kernels_ = 0;
};

// one process per GPU (rank.cu): opaque session driven over NCCL
void nccl_unique_id(char* out128);
void* rank_session_create(Engine* e, const Plan& plan, const Partition& part, const std::vector<double>& ab,
                          int rank, const char* id, const RunOptions& opts);
void rank_session_destroy(void* s);
void rank_session_run(void* s, const double* x, double* lat, double* eps);
double rank_session_time(void* s, int iters);
int rank_session_kernels(void* s);

// kernel nodes of this library in a captured CUDA graph (NCCL kernels excluded)
int graph_kernel_nodes(cudaGraph_t g);

// fp32 / fp64 host staging -> fp64 (multi-threaded for large arrays)
void widen_to_f64(const void* src, int bytes, double* dst, size_t n);

}  // namespace adx
