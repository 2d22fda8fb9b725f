// C++ caller of the drop-in boundary through include/asyncdiff_b200.hpp,
// written the way the reference's run_one (proj/src/experiment.cpp:238-290)
// calls its engine.  Mode "host": plan/partition only (no GPU).  Mode "gpu":
// golden G1 (proj/tests/test_executor.cpp:66-81) on the sm_100a engine.
#include "asyncdiff_b200.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

namespace ad = asyncdiff_b200;

static std::vector<double> normals(uint64_t seed, int n) {  // rng.hpp Box-Muller over mt19937_64
    std::mt19937_64 eng(seed);
    auto u = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
    std::vector<double> out;
    while (static_cast<int>(out.size()) < n) {
        double u1 = u(), u2 = u();
        while (u1 <= 0.0) u1 = u();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
        out.push_back(r * std::cos(a));
        out.push_back(r * std::sin(a));
    }
    out.resize(n);
    return out;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    auto model = ad::build_toy_denoiser(6, {2, 8, 8, 8, 8, 8, 2}, ad::SkipSpec::UnetMirror, 11);
    auto part = ad::partition_balanced(model, 2);
    auto plan = ad::plan_async(20, 1, 2, 1);
    if (!ad::validate_plan(plan).empty() || plan.num_rounds() != 19 || part.num_segments() != 2) {
        std::printf("FAIL host\n");
        return 1;
    }
    try {
        ad::plan_async(50, 0, 2, 1);
        std::printf("FAIL no throw\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    if (!gpu) {
        std::printf("host ok\n");
        return 0;
    }
    auto s = ad::build_schedule(20, 0.01, 0.15);
    ad::Latent x{normals(12, 2), 20};
    auto seq = ad::sequential_denoise(model, x, s);
    auto [traj, stats] = ad::run_parallel(plan, model, part, x, s, plan.D);
    double mse = 0;
    for (int k = 0; k < 2; ++k) {
        const double d = traj.final_latent().values[k] - seq.final_latent().values[k];
        mse += d * d / 2.0;
    }
    const double gold = 0.0011860077151787584;
    std::printf("gpu mse %.17g golden %.17g broadcasts %d\n", mse, gold, stats.broadcast_count);
    return std::fabs(mse - gold) <= 1e-9 * gold ? 0 : 1;
}
