// host.hpp -- host-side model, partition and plan of the B200 AsyncDiff engine.
//
// These are the integer/fp64 control-plane pieces of the hot path (SURVEY §8a
// rows a1, a4, a5, a10-a12, a20).  They are restated from the reference's
// published behaviour (file:line cited per function) and must be bit-exact:
// the per-device step schedule is a parity contract.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace adx {

// ------------------------------------------------------------------ RNG
// proj/include/asyncdiff/rng.hpp:12-60 -- explicit algorithms on mt19937_64 so
// random-init weights and x_T are bit-identical to the reference's.
class Rng {
public:
    explicit Rng(uint64_t seed) : engine_(seed) {}
    uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal();
    uint64_t below(uint64_t n) { return static_cast<uint64_t>(uniform() * static_cast<double>(n)); }

private:
    std::mt19937_64 engine_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};
uint64_t mix_seed(uint64_t a, uint64_t b);

// ------------------------------------------------------------- schedule
// proj/src/diffusion.cpp:39-77
void build_schedule(int T, double beta_start, double beta_end, int kind, std::vector<double>& betas,
                    std::vector<double>& alphas, std::vector<double>& alpha_bars);

// ---------------------------------------------------------------- model
// LayeredDenoiser (denoiser.hpp:29-72).  Host tensors are fp64 row-major.
struct Stage {
    int index = 0;  // 1-based
    int in = 0, hidden = 0, out = 0;
    std::vector<double> w1;    // hidden x in
    std::vector<double> b1;    // hidden
    std::vector<double> tin;   // hidden x E
    std::vector<double> w2;    // out x hidden
    std::vector<double> b2;    // out
    long long cost_macs = 0;
};

struct UNetDesc;  // unet.hpp

struct Model {
    int kind = 0;                          // 0: reference MLP stages, 1: UNet-shaped family
    std::shared_ptr<const UNetDesc> unet;  // kind 1 only
    int L = 0;
    int E = 0;
    std::vector<int> widths;                      // L+1
    std::vector<std::pair<int, int>> links;       // sorted (producer, consumer)
    std::vector<double> proj;                     // E x E
    std::vector<Stage> stages;                    // L
    uint64_t version = 0;                         // bumped on host edits

    int data_dim() const { return widths.front(); }
    std::vector<std::pair<int, int>> links_into(int consumer) const;
    std::vector<std::pair<int, int>> links_out_of(int producer) const;
    long long total_macs() const;
    // e_t = proj * sinusoid(t)   (denoiser.hpp:24)
    std::vector<double> embed(int t) const;
};

std::vector<double> sinusoid(int t, int dim);
Model make_denoiser_shell(int L, const std::vector<int>& widths,
                          std::vector<std::pair<int, int>> links, int E);
Model build_toy_denoiser(int L, const std::vector<int>& widths, int skip_spec, uint64_t seed, int E);

// ------------------------------------------------------------ partition
// partition.hpp:19-44
struct Partition {
    std::vector<std::vector<int>> segments;  // 1-based stage ids
    std::vector<int> device_of_segment;
    std::vector<long long> segment_macs;
    int strategy = 0;  // 0 sequential-balanced, 1 first-last-grouped

    int num_segments() const { return static_cast<int>(segments.size()); }
    int num_stages() const;
    int segment_of_stage(int stage) const;
    bool contiguous() const;
    long long max_segment_macs() const;
    long long total_macs() const;
    void validate(const Model& m) const;
};
Partition partition_balanced(const Model& m, int N, int strategy);
Partition partition_by_cost(const Model& m, int N, const std::vector<long long>& stage_cost);
std::vector<std::pair<int, int>> crossing_links(const Model& m, const Partition& p);

// ----------------------------------------------------------------- plan
// plan.hpp:12-53
constexpr int kWarmupRound = -1;
struct InputRef {
    int kind = 0;  // 0 CurrentLatent, 1 Cached
    int producer_segment = 0;
    int producer_round = kWarmupRound;
};
struct Eval {
    int segment = 0, device = 0, embed_t = 0;
    InputRef input;
    std::optional<int> emits_eps_for;
};
struct Round {
    int index = 0;
    std::vector<Eval> evals;
    std::vector<int> sampler_steps;
    bool broadcast = true;
};
struct Plan {
    int T = 0, w = 0, N = 0, S = 1, D = 0;
    bool time_shift = false;
    std::vector<int> warmup_steps;
    std::vector<Round> rounds;
};

Plan plan_async(int T, int w, int N, int S, bool time_shift);
std::vector<std::string> validate_plan(const Plan& plan);
std::vector<int> plan_to_flat(const Plan& p);
Plan plan_from_flat(const int* f, int len);

struct PlanCounts {
    int broadcasts_paper_convention = 0;
    int broadcasts_strictly_needed = 0;
    int device_count = 0;
    std::vector<long long> evals_per_segment;
    std::vector<long long> per_device_macs;
    long long max_device_macs = 0;
    long long sequential_total_macs = 0;
};
PlanCounts plan_counts(const Plan& plan, const Partition& partition);
std::vector<int> shift_embeddings(const std::vector<int>& timesteps, int w);
std::string render_plan(const Plan& plan);

// exception carrying a CUDA/NCCL failure (maps to ADX_ERR_CUDA)
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace adx
