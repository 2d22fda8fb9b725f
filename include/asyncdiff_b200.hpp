// asyncdiff_b200.hpp -- header-only C++ facade over the C ABI (asyncdiff_b200.h).
//
// Mirrors the reference's C++ pipeline API (proj/include/asyncdiff/*.hpp) so a
// caller such as run_one (proj/src/experiment.cpp:238-290) can switch engines
// by changing a namespace: plan_async, validate_plan, plan_counts,
// partition_balanced, run_serial, run_parallel, sequential_denoise,
// compare_trajectories.  Status codes are rethrown as the same std::
// exception types with the same message text the reference throws.
// Latents are std::vector<double> instead of Eigen::VectorXd.
#pragma once

#include "asyncdiff_b200.h"

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace asyncdiff_b200 {

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

using Vec = std::vector<double>;

struct Latent {
    Vec values;
    int timestep = 0;
};

struct Trajectory {
    std::vector<Latent> latents;
    std::vector<Vec> eps_used;
    const Latent& final_latent() const { return latents.back(); }
};

struct NoiseSchedule {
    int T = 0;
    Vec betas, alphas, alpha_bars;
};

inline NoiseSchedule build_schedule(int T, double beta_start, double beta_end, int kind = 0) {
    NoiseSchedule s;
    s.T = T;
    s.betas.resize(T > 0 ? T : 1);
    s.alphas.resize(T > 0 ? T : 1);
    s.alpha_bars.resize((T > 0 ? T : 1) + 1);
    check(adx_build_schedule(T, beta_start, beta_end, kind, s.betas.data(), s.alphas.data(), s.alpha_bars.data()));
    return s;
}

template <typename T, void (*Del)(T*)>
struct Handle {
    std::shared_ptr<T> p;
    T* get() const { return p.get(); }
    void reset(T* raw) { p.reset(raw, Del); }
};

class LayeredDenoiser {
public:
    static LayeredDenoiser build_toy(int L, const std::vector<int>& widths, int skip_spec, uint64_t seed,
                                     int time_embed_dim = 8) {
        adx_model* m = nullptr;
        check(adx_model_build_toy(L, widths.data(), static_cast<int>(widths.size()), skip_spec, seed,
                                  time_embed_dim, &m));
        LayeredDenoiser d;
        d.h_.reset(m);
        return d;
    }
    adx_model* raw() const { return h_.get(); }
    int data_dim() const {
        int L = 0, E = 0, nl = 0;
        check(adx_model_info(raw(), &L, &E, &nl));
        std::vector<int> w(L + 1);
        check(adx_model_widths(raw(), w.data()));
        return w[0];
    }

private:
    Handle<adx_model, adx_model_destroy> h_;
};

class Partition {
public:
    adx_partition* raw() const { return h_.get(); }
    void adopt(adx_partition* p) { h_.reset(p); }
    int num_segments() const { return adx_partition_num_segments(raw()); }

private:
    Handle<adx_partition, adx_partition_destroy> h_;
};

inline Partition partition_balanced(const LayeredDenoiser& m, int N, int strategy = ADX_SEQUENTIAL_BALANCED) {
    adx_partition* p = nullptr;
    check(adx_partition_balanced(m.raw(), N, strategy, &p));
    Partition out;
    out.adopt(p);
    return out;
}

class ExecutionPlan {
public:
    adx_plan* raw() const { return h_.get(); }
    void adopt(adx_plan* p) { h_.reset(p); }
    std::vector<int> flat() const {
        int len = 0;
        std::vector<int> buf(1 << 16);
        check(adx_plan_to_flat(raw(), buf.data(), static_cast<int>(buf.size()), &len));
        buf.resize(len);
        return buf;
    }
    int T() const { return flat()[0]; }
    int D() const { return flat()[4]; }
    int num_rounds() const { return flat()[6]; }

private:
    Handle<adx_plan, adx_plan_destroy> h_;
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

// Device-resident model: weights uploaded once per GPU in the given precision.
class Engine {
public:
    Engine(const LayeredDenoiser& m, int precision, std::vector<int> ordinals = {0}) {
        adx_engine* e = nullptr;
        check(adx_engine_create(m.raw(), precision, ordinals.data(), static_cast<int>(ordinals.size()), &e));
        h_.reset(e);
        d_ = m.data_dim();
    }
    adx_engine* raw() const { return h_.get(); }
    int d() const { return d_; }

private:
    Handle<adx_engine, adx_engine_destroy> h_;
    int d_ = 0;
};

struct RunStats {
    int broadcast_count = 0;
    double warmup_wall_s = 0.0, total_wall_s = 0.0;
};

inline Trajectory unpack(const Vec& lat, const Vec& eps, int T, int d) {
    Trajectory tr;
    for (int k = 0; k <= T; ++k) tr.latents.push_back({Vec(lat.begin() + k * d, lat.begin() + (k + 1) * d), T - k});
    for (int k = 0; k < T; ++k) tr.eps_used.emplace_back(eps.begin() + k * d, eps.begin() + (k + 1) * d);
    return tr;
}

// run_serial: proj/include/asyncdiff/executor.hpp:63-75
inline std::pair<Trajectory, RunStats> run_serial(const ExecutionPlan& plan, Engine& e, const Partition& p,
                                                  const Latent& x_T, const NoiseSchedule& s) {
    const int T = s.T, d = e.d();
    Vec lat(static_cast<size_t>(T + 1) * d), eps(static_cast<size_t>(T) * d);
    adx_run_stats st{};
    if (x_T.timestep != T) throw std::invalid_argument("run: x_T.timestep != T");
    check(adx_run_serial(e.raw(), plan.raw(), p.raw(), x_T.values.data(), s.alpha_bars.data(), T, nullptr,
                         lat.data(), eps.data(), &st));
    return {unpack(lat, eps, T, d), RunStats{st.broadcast_count, st.warmup_wall_s, st.total_wall_s}};
}

// run_parallel: proj/include/asyncdiff/executor.hpp:79-93 (workers must equal plan.D)
inline std::pair<Trajectory, RunStats> run_parallel(const ExecutionPlan& plan, Engine& e, const Partition& p,
                                                    const Latent& x_T, const NoiseSchedule& s, int workers) {
    const int T = s.T, d = e.d();
    Vec lat(static_cast<size_t>(T + 1) * d), eps(static_cast<size_t>(T) * d);
    adx_run_stats st{};
    if (x_T.timestep != T) throw std::invalid_argument("run: x_T.timestep != T");
    check(adx_run_parallel(e.raw(), plan.raw(), p.raw(), x_T.values.data(), s.alpha_bars.data(), T, workers,
                           nullptr, lat.data(), eps.data(), &st));
    return {unpack(lat, eps, T, d), RunStats{st.broadcast_count, st.warmup_wall_s, st.total_wall_s}};
}

// sequential_denoise(eval_full): proj/include/asyncdiff/diffusion.hpp:66-67
inline Trajectory sequential_denoise(Engine& e, const Latent& x_T, const NoiseSchedule& s) {
    const int T = s.T, d = e.d();
    if (x_T.timestep != T) throw std::invalid_argument("sequential_denoise: x_T.timestep != T");
    Vec lat(static_cast<size_t>(T + 1) * d), eps(static_cast<size_t>(T) * d);
    check(adx_sequential_denoise(e.raw(), x_T.values.data(), s.alpha_bars.data(), T, lat.data(), eps.data()));
    return unpack(lat, eps, T, d);
}

}  // namespace asyncdiff_b200
