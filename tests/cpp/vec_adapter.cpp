// The facade with a non-std vector type (what ASYNCDIFF_B200_EIGEN does with
// Eigen::VectorXd): MiniVec offers only Vec(n), size(), data() and operator[].
#include <cstddef>
#include <memory>

struct MiniVec {
    MiniVec() = default;
    explicit MiniVec(long n) : n_(n), p_(new double[static_cast<size_t>(n > 0 ? n : 1)]()) {}
    MiniVec(const MiniVec& o) : MiniVec(o.n_) {
        for (long i = 0; i < n_; ++i) p_[i] = o.p_[i];
    }
    MiniVec& operator=(const MiniVec& o) {
        MiniVec t(o);
        std::swap(n_, t.n_);
        std::swap(p_, t.p_);
        return *this;
    }
    long size() const { return n_; }
    double* data() { return p_.get(); }
    const double* data() const { return p_.get(); }
    double& operator[](long i) { return p_[i]; }
    double operator[](long i) const { return p_[i]; }

private:
    long n_ = 0;
    std::unique_ptr<double[]> p_;
};

#define ASYNCDIFF_B200_VEC MiniVec
#include "asyncdiff_b200.hpp"

#include <cstdio>
#include <cstring>

int main(int argc, char** argv) {
    namespace ad = asyncdiff_b200;
    auto m = ad::build_toy_denoiser(6, {2, 8, 8, 8, 8, 8, 2}, ad::SkipSpec::UnetMirror, 11);
    auto plan = ad::plan_async(20, 1, 2, 1);
    auto part = ad::partition_balanced(m, 2);
    const auto s = ad::build_schedule(20, 0.01, 0.15);
    if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
        ad::Rng rng(12);
        ad::Latent x{MiniVec(2), 20};
        x.values[0] = rng.normal();
        x.values[1] = rng.normal();
        auto seq = ad::sequential_denoise(m, x, s);
        auto [par, st] = ad::run_parallel(plan, m, part, x, s, plan.D);
        const double mse = ad::compare_trajectories(seq, par).final_mse, gold = 0.0011860077151787584;
        std::printf("MiniVec G1 %.17g\n", mse);
        return std::fabs(mse - gold) <= 1e-9 * gold ? 0 : 1;
    }
    std::printf("vec adapter ok (%d rounds)\n", plan.num_rounds());
    return 0;
}
