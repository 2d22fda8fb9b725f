// asyncdiff_b200.hpp -- header-only C++ facade over the C ABI (asyncdiff_b200.h).
//
// Mirrors the reference's C++ pipeline API (proj/include/asyncdiff/*.hpp) so a
// caller such as run_one (proj/src/experiment.cpp:238-290) switches engines by
// changing a namespace (tests/cpp/run_one.cpp is such a copy):
//   diffusion.hpp  Latent, NoiseSchedule, ScheduleKind, build_schedule,
//                  ddim_step, predict_x0, Trajectory, EpsFn, sequential_denoise
//   denoiser.hpp   SkipSpec, LayeredDenoiser, build_toy_denoiser, SkipMap,
//                  HiddenBundle, SegmentOutput, eval_full, eval_segment (x2)
//   partition.hpp  PartitionStrategy, Partition, partition_balanced
//   plan.hpp       ExecutionPlan, plan_async, validate_plan, PlanCounts,
//                  plan_counts, shift_embeddings, render_plan
//   executor.hpp   RunStats, RunOptions, InstrumentedDenoiser, inject_delay,
//                  run_serial / run_parallel (model or instrumented model)
//   metrics.hpp    DivergenceReport, compare_trajectories
//   rng.hpp        Rng, mix_seed
// Status codes are rethrown as the same std:: exception types with the same
// message text the reference throws.  Every numeric call runs on the GPU
// (the model's Engine: weights uploaded once, lazily, shared by copies of the
// LayeredDenoiser handle); there is no CPU fallback.
//
// Vectors: `Vec` is std::vector<double> by default.  Define ASYNCDIFF_B200_EIGEN
// before including this header to use Eigen::VectorXd (the reference's Vec) --
// or ASYNCDIFF_B200_VEC to any type with Vec(n), size(), data() and operator[];
// the facade touches vectors only through those.
#pragma once

#include "asyncdiff_b200.h"

#include <cmath>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#if defined(ASYNCDIFF_B200_EIGEN)
#include <Eigen/Dense>
#endif

namespace asyncdiff_b200 {

#if defined(ASYNCDIFF_B200_VEC)
using Vec = ASYNCDIFF_B200_VEC;
#elif defined(ASYNCDIFF_B200_EIGEN)
using Vec = Eigen::VectorXd;
#else
using Vec = std::vector<double>;
#endif

inline void check(int rc) {
    if (rc == ADX_OK) return;
    const std::string msg = adx_last_error();
    switch (rc) {
        case ADX_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case ADX_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case ADX_ERR_DOMAIN: throw std::domain_error(msg);
        case ADX_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace detail {
inline int vsize(const Vec& v) { return static_cast<int>(v.size()); }
inline Vec vec_from(const double* p, int n) {
    Vec v(n);
    for (int i = 0; i < n; ++i) v[i] = p[i];
    return v;
}
inline std::vector<double> to_std(const Vec& v) {
    std::vector<double> o(static_cast<size_t>(vsize(v)));
    for (int i = 0; i < vsize(v); ++i) o[i] = v[i];
    return o;
}
template <typename T, void (*Del)(T*)>
struct Handle {
    std::shared_ptr<T> p;
    T* get() const { return p.get(); }
    void reset(T* raw) { p.reset(raw, Del); }
};
}  // namespace detail

// ------------------------------------------------------------------ rng.hpp
class Rng {  // rng.hpp:12-53
public:
    explicit Rng(uint64_t seed) : engine_(seed) {}
    uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        has_spare_ = true;
        return r * std::cos(a);
    }
    uint64_t below(uint64_t n) { return static_cast<uint64_t>(uniform() * static_cast<double>(n)); }

private:
    std::mt19937_64 engine_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

inline uint64_t mix_seed(uint64_t a, uint64_t b) {  // rng.hpp:55-60
    uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ------------------------------------------------------------ diffusion.hpp
struct Latent {
    Vec values;
    int timestep = 0;
};

enum class ScheduleKind { Linear, ScaledLinear };

struct NoiseSchedule {
    int T = 0;
    std::vector<double> betas, alphas, alpha_bars;
    double beta(int t) const { return at(betas, t, 1, "beta") ; }
    double alpha(int t) const { return at(alphas, t, 1, "alpha"); }
    double alpha_bar(int t) const { return at(alpha_bars, t, 0, "alpha_bar"); }

private:
    double at(const std::vector<double>& v, int t, int lo, const char* what) const {
        if (t < lo || t > T)
            throw std::out_of_range(std::string("NoiseSchedule::") + what + ": t=" + std::to_string(t) +
                                    " outside [" + std::to_string(lo) + ", " + std::to_string(T) + "]");
        return v[static_cast<size_t>(t - lo)];
    }
};

inline NoiseSchedule build_schedule(int T, double beta_start, double beta_end,
                                    ScheduleKind kind = ScheduleKind::Linear) {
    NoiseSchedule s;
    s.T = T;
    s.betas.resize(T > 0 ? T : 1);
    s.alphas.resize(T > 0 ? T : 1);
    s.alpha_bars.resize((T > 0 ? T : 1) + 1);
    check(adx_build_schedule(T, beta_start, beta_end, kind == ScheduleKind::Linear ? 0 : 1, s.betas.data(),
                             s.alphas.data(), s.alpha_bars.data()));
    s.betas.resize(T);
    s.alphas.resize(T);
    s.alpha_bars.resize(T + 1);
    return s;
}

struct Trajectory {
    std::vector<Latent> latents;       // x_T first
    std::vector<Vec> eps_used;
    std::vector<double> timestamps_s;  // unused by the GPU engine (device-timed; see RunStats)
    int steps() const { return static_cast<int>(eps_used.size()); }
    const Latent& final_latent() const { return latents.back(); }
};

using EpsFn = std::function<Vec(const Latent&, int t)>;

// ddim_step (diffusion.cpp:108-116) on GPU `ordinal` in fp64: IEEE-identical to the reference
inline Latent ddim_step(const Latent& x_t, const Vec& eps, int t, const NoiseSchedule& s, int ordinal = 0) {
    const int d = detail::vsize(x_t.values);
    if (detail::vsize(eps) != d) throw std::invalid_argument("ddim_step: eps dimension mismatch");
    std::vector<double> x = detail::to_std(x_t.values), e = detail::to_std(eps), out(static_cast<size_t>(d));
    check(adx_ddim_step(ordinal, ADX_F64, x.data(), e.data(), d, t, s.alpha_bars.data(), s.T, out.data()));
    return Latent{detail::vec_from(out.data(), d), t - 1};
}

// predict_x0 (diffusion.cpp:95-106): host fp64 (one fused expression of the reference)
inline Vec predict_x0(const Latent& x_t, const Vec& eps, int t, const NoiseSchedule& s) {
    const double ab = s.alpha_bar(t);
    Vec out(detail::vsize(x_t.values));
    for (int i = 0; i < detail::vsize(out); ++i) {
        if (!std::isfinite(eps[i])) throw std::domain_error("predict_x0: non-finite eps at t=" + std::to_string(t));
        out[i] = (x_t.values[i] - std::sqrt(1.0 - ab) * eps[i]) / std::sqrt(ab);
    }
    return out;
}

// ------------------------------------------------------------- denoiser.hpp
enum class SkipSpec { None, UnetMirror };
using SkipMap = std::map<std::pair<int, int>, Vec>;

struct HiddenBundle {
    Vec boundary;
    SkipMap skips;
    int produced_by = 0;
    int produced_at = 0;
};
using SegmentOutput = std::variant<HiddenBundle, Vec>;

// A model handle.  Copies share the model and its device engine(s); the engine of a
// precision is created (weights uploaded) on first use.  precision: ADX_F64 (the MLP
// family's default: reference parity), ADX_F32, ADX_BF16 (the UNet family's default).
class LayeredDenoiser {
public:
    adx_model* raw() const { return h_.get(); }
    int num_stages() const { return info()[0]; }
    int time_embed_dim() const { return info()[1]; }
    std::vector<int> widths() const {
        std::vector<int> w(static_cast<size_t>(num_stages()) + 1);
        check(adx_model_widths(raw(), w.data()));
        return w;
    }
    int data_dim() const { return widths()[0]; }
    std::vector<std::pair<int, int>> skip_links() const {
        std::vector<int> buf(2 * static_cast<size_t>(info()[2]) + 2);
        check(adx_model_links(raw(), buf.data()));
        std::vector<std::pair<int, int>> out;
        for (int k = 0; k < info()[2]; ++k) out.emplace_back(buf[2 * k], buf[2 * k + 1]);
        return out;
    }
    int precision() const { return st_->precision; }
    void set_precision(int precision) { st_->precision = precision; }
    // the device-resident copy (weights uploaded once per precision and ordinal list)
    adx_engine* engine(int precision = -1, const std::vector<int>& ordinals = {0}) const {
        const int p = precision < 0 ? st_->precision : precision;
        auto key = std::make_pair(p, ordinals);
        auto it = st_->engines.find(key);
        if (it != st_->engines.end()) return it->second.get();
        adx_engine* e = nullptr;
        check(adx_engine_create(raw(), p, ordinals.data(), static_cast<int>(ordinals.size()), &e));
        detail::Handle<adx_engine, adx_engine_destroy> h;
        h.reset(e);
        st_->engines.emplace(key, h);
        return e;
    }
    static LayeredDenoiser adopt(adx_model* m, int default_precision) {
        LayeredDenoiser d;
        d.h_.reset(m);
        d.st_ = std::make_shared<State>();
        d.st_->precision = default_precision;
        return d;
    }

private:
    std::vector<int> info() const {
        int L = 0, E = 0, nl = 0;
        check(adx_model_info(raw(), &L, &E, &nl));
        return {L, E, nl};
    }
    struct State {
        int precision = ADX_F64;
        std::map<std::pair<int, std::vector<int>>, detail::Handle<adx_engine, adx_engine_destroy>> engines;
    };
    detail::Handle<adx_model, adx_model_destroy> h_;
    std::shared_ptr<State> st_;
};

inline LayeredDenoiser build_toy_denoiser(int L, const std::vector<int>& widths, SkipSpec skip_spec, uint64_t seed,
                                          int time_embed_dim = 8) {
    adx_model* m = nullptr;
    check(adx_model_build_toy(L, widths.data(), static_cast<int>(widths.size()),
                              skip_spec == SkipSpec::UnetMirror ? ADX_SKIP_UNET_MIRROR : ADX_SKIP_NONE, seed,
                              time_embed_dim, &m));
    return LayeredDenoiser::adopt(m, ADX_F64);
}

// UNet-shaped family (north_star configs 2-5) behind the same stage contract
inline LayeredDenoiser build_unet_denoiser(const adx_unet_spec& spec) {
    adx_model* m = nullptr;
    check(adx_model_build_unet(&spec, &m));
    return LayeredDenoiser::adopt(m, ADX_BF16);
}

struct Partition;
Vec eval_full(const LayeredDenoiser& m, const Latent& x, int t_embed);

// ------------------------------------------------------------ partition.hpp
enum class PartitionStrategy { SequentialBalanced, FirstLastGrouped };

struct Partition {
    adx_partition* raw() const { return h_.get(); }
    void adopt(adx_partition* p) { h_.reset(p); }
    int num_segments() const { return adx_partition_num_segments(raw()); }
    std::vector<int> segment(int n) const {  // 1-based stage list of segment n
        std::vector<int> buf(4096);
        int k = 0, dev = 0;
        long long macs = 0;
        check(adx_partition_segment(raw(), n, buf.data(), static_cast<int>(buf.size()), &k, &macs, &dev));
        buf.resize(k);
        return buf;
    }
    std::vector<std::vector<int>> segments() const {
        std::vector<std::vector<int>> s;
        for (int n = 1; n <= num_segments(); ++n) s.push_back(segment(n));
        return s;
    }
    bool contiguous() const { return adx_partition_contiguous(raw()) == 1; }
    void validate(const LayeredDenoiser& m) const { check(adx_partition_validate(raw(), m.raw())); }

private:
    detail::Handle<adx_partition, adx_partition_destroy> h_;
};

inline Partition partition_balanced(const LayeredDenoiser& m, int N,
                                    PartitionStrategy strategy = PartitionStrategy::SequentialBalanced) {
    adx_partition* p = nullptr;
    check(adx_partition_balanced(m.raw(), N,
                                 strategy == PartitionStrategy::SequentialBalanced ? ADX_SEQUENTIAL_BALANCED
                                                                                  : ADX_FIRST_LAST_GROUPED,
                                 &p));
    Partition out;
    out.adopt(p);
    return out;
}

// ----------------------------------------------------------------- plan.hpp
class ExecutionPlan {
public:
    adx_plan* raw() const { return h_.get(); }
    void adopt(adx_plan* p) {
        h_.reset(p);
        flat_ = flat();
        T = flat_[0], w = flat_[1], N = flat_[2], S = flat_[3], D = flat_[4];
    }
    std::vector<int> flat() const {
        int len = 0;
        std::vector<int> buf(1 << 16);
        check(adx_plan_to_flat(raw(), buf.data(), static_cast<int>(buf.size()), &len));
        buf.resize(len);
        return buf;
    }
    int num_rounds() const { return flat_[6]; }
    int T = 0, w = 0, N = 0, S = 0, D = 0;

private:
    detail::Handle<adx_plan, adx_plan_destroy> h_;
    std::vector<int> flat_;
};

inline ExecutionPlan plan_async(int T, int w, int N, int S, bool time_shift = false) {
    adx_plan* p = nullptr;
    check(adx_plan_async(T, w, N, S, time_shift ? 1 : 0, &p));
    ExecutionPlan out;
    out.adopt(p);
    return out;
}

inline std::vector<std::string> validate_plan(const ExecutionPlan& plan) {
    std::vector<char> buf(1 << 16);
    int n = 0;
    check(adx_plan_validate(plan.raw(), buf.data(), static_cast<int>(buf.size()), &n));
    std::vector<std::string> out;
    if (n == 0) return out;
    std::string all(buf.data());
    size_t pos = 0;
    while (true) {
        const size_t nl = all.find('\n', pos);
        out.push_back(all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos));
        if (nl == std::string::npos) break;
        pos = nl + 1;
    }
    return out;
}

struct PlanCounts {  // plan.hpp:58-66
    int broadcasts_paper_convention = 0;
    int broadcasts_strictly_needed = 0;
    int device_count = 0;
    std::vector<long long> evals_per_segment;
    std::vector<long long> per_device_macs;
    long long max_device_macs = 0;
    long long sequential_total_macs = 0;
};

inline PlanCounts plan_counts(const ExecutionPlan& plan, const Partition& partition) {
    adx_plan_counts_t c{};
    PlanCounts out;
    out.evals_per_segment.resize(static_cast<size_t>(plan.N));
    out.per_device_macs.resize(static_cast<size_t>(plan.D));
    check(adx_plan_counts(plan.raw(), partition.raw(), &c, out.evals_per_segment.data(),
                          out.per_device_macs.data()));
    out.broadcasts_paper_convention = c.broadcasts_paper_convention;
    out.broadcasts_strictly_needed = c.broadcasts_strictly_needed;
    out.device_count = c.device_count;
    out.max_device_macs = c.max_device_macs;
    out.sequential_total_macs = c.sequential_total_macs;
    return out;
}

inline std::vector<int> shift_embeddings(const std::vector<int>& timesteps, int w) {
    std::vector<int> out(timesteps.size() + 1);
    check(adx_shift_embeddings(timesteps.empty() ? nullptr : timesteps.data(), static_cast<int>(timesteps.size()),
                               w, out.data()));
    out.resize(timesteps.size());
    return out;
}

inline std::string render_plan(const ExecutionPlan& plan) {
    int n = 0;
    check(adx_render_plan(plan.raw(), nullptr, 0, &n));
    std::vector<char> buf(static_cast<size_t>(n) + 1);
    check(adx_render_plan(plan.raw(), buf.data(), static_cast<int>(buf.size()), &n));
    return std::string(buf.data());
}

// --------------------------------------------------------- denoiser eval
inline Vec eval_full(const LayeredDenoiser& m, const Latent& x, int t_embed) {
    const int d = m.data_dim();
    if (detail::vsize(x.values) != d) throw std::invalid_argument("eval_full: latent dimension mismatch");
    std::vector<double> xs = detail::to_std(x.values), out(static_cast<size_t>(d));
    check(adx_eval_full(m.engine(), xs.data(), t_embed, out.data()));
    return detail::vec_from(out.data(), d);
}

namespace detail {
inline SegmentOutput eval_segment_impl(const LayeredDenoiser& m, const Partition& p, int seg,
                                       const std::vector<double>& input, bool is_latent, int produced_by,
                                       const SkipMap& skips_in, int t_embed) {
    std::vector<int> lk;
    std::vector<double> vals;
    for (const auto& [l, f] : skips_in) {
        lk.push_back(l.first);
        lk.push_back(l.second);
        for (int i = 0; i < vsize(f); ++i) vals.push_back(f[i]);
    }
    const std::vector<int> w = m.widths();
    int cap = 8, cap_vals = 1;
    for (int v : w) cap = std::max(cap, v + 8);
    const auto links = m.skip_links();
    for (const auto& l : links) cap_vals += w[static_cast<size_t>(l.first)];
    std::vector<double> out(static_cast<size_t>(cap)), ovals(static_cast<size_t>(cap_vals));
    std::vector<int> olinks(2 * links.size() + 2);
    int ol = 0, oe = 0, nl = 0;
    check(adx_eval_segment(m.engine(), p.raw(), seg, input.data(), static_cast<int>(input.size()), is_latent ? 1 : 0,
                           produced_by, lk.empty() ? nullptr : lk.data(), vals.empty() ? nullptr : vals.data(),
                           static_cast<int>(skips_in.size()), t_embed, out.data(), cap, &ol, &oe, olinks.data(),
                           ovals.data(), static_cast<int>(links.size()) + 1, cap_vals, &nl));
    if (oe) return vec_from(out.data(), ol);
    HiddenBundle b;
    b.boundary = vec_from(out.data(), ol);
    b.produced_by = seg;
    b.produced_at = t_embed;
    int pos = 0;
    for (int k = 0; k < nl; ++k) {
        const std::pair<int, int> l(olinks[2 * k], olinks[2 * k + 1]);
        const int n = w[static_cast<size_t>(l.first)];
        b.skips[l] = vec_from(ovals.data() + pos, n);
        pos += n;
    }
    return b;
}
}  // namespace detail

// denoiser.hpp:91-95
inline SegmentOutput eval_segment(const LayeredDenoiser& m, const Partition& p, int seg, const Latent& x,
                                  const SkipMap& skips_in, int t_embed) {
    return detail::eval_segment_impl(m, p, seg, detail::to_std(x.values), true, 0, skips_in, t_embed);
}
inline SegmentOutput eval_segment(const LayeredDenoiser& m, const Partition& p, int seg, const HiddenBundle& input,
                                  const SkipMap& skips_in, int t_embed) {
    return detail::eval_segment_impl(m, p, seg, detail::to_std(input.boundary), false, input.produced_by, skips_in,
                                     t_embed);
}

// ------------------------------------------------------------- executor.hpp
struct RunStats {  // executor.hpp:30-42
    std::vector<double> round_wall_s, round_comm_s, device_busy_s;
    std::vector<long long> device_evals;
    std::vector<size_t> store_entries_per_round;
    int broadcast_count = 0;
    double warmup_wall_s = 0.0, total_wall_s = 0.0;
    double comm_total_s() const {
        double s = 0.0;
        for (double v : round_comm_s) s += v;
        return s;
    }
    double comm_ratio() const { return total_wall_s > 0.0 ? comm_total_s() / total_wall_s : 0.0; }
};

struct RunOptions {  // executor.hpp:44-49 (+ use_graph / instrument: GPU engine knobs)
    double round_timeout_s = 30.0;
    uint64_t jitter_seed = 0;
    double max_jitter_s = 0.0;
    bool use_graph = true;
    bool instrument = false;
};

struct InstrumentedDenoiser {  // executor.hpp:53-59
    LayeredDenoiser model;
    std::vector<double> segment_delay_s;
};

inline InstrumentedDenoiser inject_delay(const LayeredDenoiser& m, const std::vector<double>& per_segment_delay_s) {
    for (double d : per_segment_delay_s)
        if (d < 0.0) throw std::invalid_argument("inject_delay: delays must be >= 0");
    return InstrumentedDenoiser{m, per_segment_delay_s};
}

namespace detail {
inline Trajectory unpack(const std::vector<double>& lat, const std::vector<double>& eps, int T, int d) {
    Trajectory tr;
    for (int k = 0; k <= T; ++k) tr.latents.push_back({vec_from(lat.data() + static_cast<size_t>(k) * d, d), T - k});
    for (int k = 0; k < T; ++k) tr.eps_used.push_back(vec_from(eps.data() + static_cast<size_t>(k) * d, d));
    return tr;
}

inline std::pair<Trajectory, RunStats> run(bool parallel, const ExecutionPlan& plan, const InstrumentedDenoiser& im,
                                           const Partition& part, const Latent& x_T, const NoiseSchedule& s,
                                           int workers, const RunOptions& opts) {
    const int T = s.T, d = im.model.data_dim();
    if (x_T.timestep != T)
        throw std::invalid_argument("run: x_T.timestep=" + std::to_string(x_T.timestep) + " != T=" + std::to_string(T));
    adx_run_options o;
    adx_run_options_default(&o);
    o.round_timeout_s = opts.round_timeout_s;
    o.jitter_seed = opts.jitter_seed;
    o.max_jitter_s = opts.max_jitter_s;
    o.use_graph = opts.use_graph ? 1 : 0;
    o.instrument = opts.instrument ? 1 : 0;
    if (!im.segment_delay_s.empty()) {
        o.segment_delay_s = im.segment_delay_s.data();
        o.n_delays = static_cast<int>(im.segment_delay_s.size());
        o.use_graph = 0;  // injected delays are per-run sleeps: eager enqueue
        o.instrument = 1;
    }
    const int nr = plan.num_rounds();
    std::vector<double> rw(static_cast<size_t>(nr) + 1), rc(static_cast<size_t>(nr) + 1),
        busy(static_cast<size_t>(plan.D) + 1);
    std::vector<long long> ev(static_cast<size_t>(plan.D) + 1);
    std::vector<int> se(static_cast<size_t>(nr) + 1);
    adx_run_stats st{};
    st.round_wall_s = rw.data();
    st.round_comm_s = rc.data();
    st.device_busy_s = busy.data();
    st.device_evals = ev.data();
    st.store_entries_per_round = se.data();
    std::vector<double> x = to_std(x_T.values), lat(static_cast<size_t>(T + 1) * d), eps(static_cast<size_t>(T) * d);
    adx_engine* e = im.model.engine();
    if (parallel)
        check(adx_run_parallel(e, plan.raw(), part.raw(), x.data(), s.alpha_bars.data(), T, workers, &o, lat.data(),
                               eps.data(), &st));
    else
        check(adx_run_serial(e, plan.raw(), part.raw(), x.data(), s.alpha_bars.data(), T, &o, lat.data(), eps.data(),
                             &st));
    RunStats r;
    r.round_wall_s.assign(rw.begin(), rw.begin() + nr);
    r.round_comm_s.assign(rc.begin(), rc.begin() + nr);
    r.device_busy_s.assign(busy.begin(), busy.begin() + plan.D);
    r.device_evals.assign(ev.begin(), ev.begin() + plan.D);
    for (int i = 0; i < nr; ++i) r.store_entries_per_round.push_back(static_cast<size_t>(se[i]));
    r.broadcast_count = st.broadcast_count;
    r.warmup_wall_s = st.warmup_wall_s;
    r.total_wall_s = st.total_wall_s;
    return {unpack(lat, eps, T, d), r};
}
}  // namespace detail

// executor.hpp:63-75
inline std::pair<Trajectory, RunStats> run_serial(const ExecutionPlan& plan, const InstrumentedDenoiser& m,
                                                  const Partition& partition, const Latent& x_T,
                                                  const NoiseSchedule& schedule, const RunOptions& opts = {}) {
    return detail::run(false, plan, m, partition, x_T, schedule, 1, opts);
}
inline std::pair<Trajectory, RunStats> run_serial(const ExecutionPlan& plan, const LayeredDenoiser& m,
                                                  const Partition& partition, const Latent& x_T,
                                                  const NoiseSchedule& schedule, const RunOptions& opts = {}) {
    return detail::run(false, plan, InstrumentedDenoiser{m, {}}, partition, x_T, schedule, 1, opts);
}
// executor.hpp:79-93 (workers must equal plan.D)
inline std::pair<Trajectory, RunStats> run_parallel(const ExecutionPlan& plan, const InstrumentedDenoiser& m,
                                                    const Partition& partition, const Latent& x_T,
                                                    const NoiseSchedule& schedule, int workers,
                                                    const RunOptions& opts = {}) {
    return detail::run(true, plan, m, partition, x_T, schedule, workers, opts);
}
inline std::pair<Trajectory, RunStats> run_parallel(const ExecutionPlan& plan, const LayeredDenoiser& m,
                                                    const Partition& partition, const Latent& x_T,
                                                    const NoiseSchedule& schedule, int workers,
                                                    const RunOptions& opts = {}) {
    return detail::run(true, plan, InstrumentedDenoiser{m, {}}, partition, x_T, schedule, workers, opts);
}

// sequential_denoise (diffusion.hpp:66-67, diffusion.cpp:118-142).  With a model: the whole
// loop (eval_full + DDIM per step) runs on the GPU as one CUDA graph.  With an EpsFn: the
// caller's eps per step, the DDIM update on the GPU; failures are wrapped with "t=".
inline Trajectory sequential_denoise(const LayeredDenoiser& m, const Latent& x_T, const NoiseSchedule& s) {
    const int T = s.T, d = m.data_dim();
    if (x_T.timestep != T)
        throw std::invalid_argument("sequential_denoise: x_T.timestep=" + std::to_string(x_T.timestep) +
                                    " != T=" + std::to_string(T));
    std::vector<double> x = detail::to_std(x_T.values), lat(static_cast<size_t>(T + 1) * d),
                        eps(static_cast<size_t>(T) * d);
    check(adx_sequential_denoise(m.engine(), x.data(), s.alpha_bars.data(), T, lat.data(), eps.data()));
    return detail::unpack(lat, eps, T, d);
}
inline Trajectory sequential_denoise(const EpsFn& eps_fn, const Latent& x_T, const NoiseSchedule& s) {
    if (x_T.timestep != s.T)
        throw std::invalid_argument("sequential_denoise: x_T.timestep=" + std::to_string(x_T.timestep) +
                                    " != T=" + std::to_string(s.T));
    Trajectory tr;
    tr.latents.push_back(x_T);
    Latent x = x_T;
    for (int t = s.T; t >= 1; --t) {
        Vec eps;
        try {
            eps = eps_fn(x, t);
            x = ddim_step(x, eps, t, s);
        } catch (const std::exception& e) {
            throw std::runtime_error("sequential_denoise: eps_fn failed at t=" + std::to_string(t) + ": " + e.what());
        }
        tr.eps_used.push_back(eps);
        tr.latents.push_back(x);
    }
    return tr;
}

// -------------------------------------------------------------- metrics.hpp
struct DivergenceReport {
    std::vector<double> per_step_mse;
    double final_mse = 0.0;
    double final_max_abs = 0.0;
};

inline DivergenceReport compare_trajectories(const Trajectory& seq, const Trajectory& async_traj) {
    if (seq.latents.size() != async_traj.latents.size())
        throw std::invalid_argument("compare_trajectories: length mismatch (" + std::to_string(seq.latents.size()) +
                                    " vs " + std::to_string(async_traj.latents.size()) + ")");
    const int n = static_cast<int>(seq.latents.size());
    const int d = n ? detail::vsize(seq.latents[0].values) : 0;
    std::vector<double> a, b;
    for (int i = 0; i < n; ++i) {
        if (detail::vsize(seq.latents[i].values) != d || detail::vsize(async_traj.latents[i].values) != d)
            throw std::invalid_argument("compare_trajectories: dimension mismatch at step " + std::to_string(i));
        for (int k = 0; k < d; ++k) {
            a.push_back(seq.latents[i].values[k]);
            b.push_back(async_traj.latents[i].values[k]);
        }
    }
    DivergenceReport r;
    r.per_step_mse.resize(static_cast<size_t>(n));
    check(adx_compare_trajectories(a.data(), b.data(), n, d, r.per_step_mse.data(), &r.final_mse, &r.final_max_abs));
    return r;
}

}  // namespace asyncdiff_b200
