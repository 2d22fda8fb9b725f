// The reference's run_one (proj/src/experiment.cpp:131-150, 238-290) compiled against the
// B200 engine with only the namespace switched (asyncdiff -> asyncdiff_b200): the same
// partition_balanced / plan_async / draw_x_T / sequential_denoise(eval_full EpsFn) /
// run_serial / run_parallel / bit_identical / plan_counts / compare_trajectories sequence.
// The mixture NLL column is out of scope and omitted.
//
//   run_one host   plan / partition / contract checks only (no GPU)
//   run_one gpu    goldens G1 and G2 (proj/tests/test_executor.cpp:66-81,
//                  test_metrics.cpp:42-55) through the facade, then run_one rows
#include "asyncdiff_b200.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>

namespace asyncdiff = asyncdiff_b200;  // <- the only change a reference caller needs
using namespace asyncdiff;

struct ExperimentConfig {  // experiment.hpp:30-57 (the fields run_one reads)
    int T = 20;
    double beta_start = 0.01, beta_end = 0.15;
    uint64_t seed = 11;
    int dim = 2;
    double round_timeout_s = 30.0;
    NoiseSchedule schedule() const { return build_schedule(T, beta_start, beta_end, ScheduleKind::Linear); }
};

struct RunSpec {
    int N = 2, w = 1, S = 1;
    bool time_shift = false;
    std::string label() const {
        return "N" + std::to_string(N) + "_w" + std::to_string(w) + "_S" + std::to_string(S) +
               (time_shift ? "_shift" : "");
    }
};

struct ResultRow {
    std::string config_label;
    uint64_t run_seed = 0;
    long long per_device_macs = 0;
    int device_count = 0, broadcast_count = 0;
    double measured_latency_s = 0.0, speedup = 0.0, comm_ratio = 0.0, final_mse = 0.0;
};

namespace {

Latent draw_x_T(const ExperimentConfig& cfg, uint64_t run_seed) {
    Rng rng(mix_seed(cfg.seed, run_seed));
    Latent x;
    x.values = Vec(cfg.dim);
    for (int i = 0; i < static_cast<int>(x.values.size()); ++i) x.values[i] = rng.normal();
    x.timestep = cfg.T;
    return x;
}

bool bit_identical(const Trajectory& a, const Trajectory& b) {
    if (a.latents.size() != b.latents.size()) return false;
    for (size_t i = 0; i < a.latents.size(); ++i) {
        const Vec& va = a.latents[i].values;
        const Vec& vb = b.latents[i].values;
        if (va.size() != vb.size()) return false;
        for (int k = 0; k < static_cast<int>(va.size()); ++k)
            if (va[k] != vb[k]) return false;
    }
    return true;
}

}  // namespace

ResultRow run_one(const ExperimentConfig& cfg, const LayeredDenoiser& model, const RunSpec& spec, uint64_t run_seed,
                  bool measure_parallel) {
    NoiseSchedule schedule = cfg.schedule();
    Partition partition = partition_balanced(model, spec.N, PartitionStrategy::SequentialBalanced);
    ExecutionPlan plan = plan_async(cfg.T, spec.w, spec.N, spec.S, spec.time_shift);
    Latent x_T = draw_x_T(cfg, run_seed);

    EpsFn eps_fn = [&](const Latent& x, int t) { return eval_full(model, x, t); };

    auto seq_start = std::chrono::steady_clock::now();
    Trajectory seq = sequential_denoise(eps_fn, x_T, schedule);
    double seq_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - seq_start).count();

    RunOptions opts;
    opts.round_timeout_s = cfg.round_timeout_s;
    auto [serial_traj, serial_stats] = run_serial(plan, model, partition, x_T, schedule, opts);

    Trajectory async_traj = serial_traj;
    RunStats stats = serial_stats;
    if (measure_parallel) {
        auto [par_traj, par_stats] = run_parallel(plan, model, partition, x_T, schedule, plan.D, opts);
        if (!bit_identical(par_traj, serial_traj))
            throw std::runtime_error("invariant violated: run_parallel != run_serial for " + spec.label());
        async_traj = std::move(par_traj);
        stats = std::move(par_stats);
    }

    PlanCounts counts = plan_counts(plan, partition);
    if (stats.broadcast_count != counts.broadcasts_paper_convention)
        throw std::runtime_error("invariant violated: executor broadcast count != analytic count for " +
                                 spec.label());

    DivergenceReport div = compare_trajectories(seq, async_traj);

    ResultRow row;
    row.config_label = spec.label();
    row.run_seed = run_seed;
    row.per_device_macs = counts.max_device_macs;
    row.device_count = plan.D;
    row.broadcast_count = counts.broadcasts_paper_convention;
    row.measured_latency_s = stats.total_wall_s;
    row.speedup = stats.total_wall_s > 0.0 ? seq_wall / stats.total_wall_s : 0.0;
    row.comm_ratio = stats.comm_ratio();
    row.final_mse = div.final_mse;
    return row;
}

static int fail(const char* what) {
    std::printf("FAIL %s\n", what);
    return 1;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    auto model = build_toy_denoiser(6, {2, 8, 8, 8, 8, 8, 2}, SkipSpec::UnetMirror, 11);
    auto part = partition_balanced(model, 2);
    auto plan = plan_async(20, 1, 2, 1);
    if (!validate_plan(plan).empty() || plan.num_rounds() != 19 || part.num_segments() != 2) return fail("host plan");
    if (part.segments() != std::vector<std::vector<int>>{{1, 2, 3}, {4, 5, 6}}) return fail("host partition");
    auto cnt = plan_counts(plan_async(50, 1, 2, 1), part);
    if (cnt.broadcasts_paper_convention != 49 || cnt.broadcasts_strictly_needed != 48) return fail("plan_counts");
    try {
        plan_async(50, 0, 2, 1);
        return fail("no throw");
    } catch (const std::invalid_argument&) {
    }
    if (render_plan(plan_async(4, 1, 2, 1)).empty()) return fail("render_plan");
    if (!gpu) {
        std::printf("host ok\n");
        return 0;
    }
    // G1 / G2: the reference fixture (test_executor.cpp:14-29): x_T = two normals of Rng(12)
    const auto s = build_schedule(20, 0.01, 0.15, ScheduleKind::Linear);
    Rng rng(12);
    Latent x{Vec(2), 20};
    x.values[0] = rng.normal();
    x.values[1] = rng.normal();
    auto seq = sequential_denoise(model, x, s);
    // the EpsFn path (eval_full per step + GPU DDIM) equals the graph path bit-for-bit
    auto seq_fn = sequential_denoise([&](const Latent& l, int t) { return eval_full(model, l, t); }, x, s);
    for (int k = 0; k <= 20; ++k)
        for (int i = 0; i < 2; ++i)
            if (seq.latents[k].values[i] != seq_fn.latents[k].values[i]) return fail("EpsFn path != graph path");
    const double g1 = 0.0011860077151787584, g2 = 0.00027252781017261107;
    for (int w : {1, 3}) {
        auto pl = plan_async(20, w, 2, 1);
        auto [ser, sst] = run_serial(pl, model, part, x, s);
        auto [par, pst] = run_parallel(pl, model, part, x, s, pl.D);
        if (!bit_identical(ser, par)) return fail("parallel != serial");
        auto rep = compare_trajectories(seq, par);
        const double gold = w == 1 ? g1 : g2;
        std::printf("G%d: final mse %.17g golden %.17g (broadcasts %d)\n", w == 1 ? 1 : 2, rep.final_mse, gold,
                    pst.broadcast_count);
        if (std::fabs(rep.final_mse - gold) > 1e-9 * gold) return fail("golden");
    }
    // segment chaining == eval_full (test_denoiser.cpp:106-129), through the facade's eval_segment
    {
        auto p3 = partition_balanced(model, 3);
        SkipMap skips;
        SegmentOutput so = eval_segment(model, p3, 1, x, skips, 7);
        for (int seg = 2; seg <= 3; ++seg) {
            const HiddenBundle& b = std::get<HiddenBundle>(so);
            for (const auto& [l, f] : b.skips) skips[l] = f;
            so = eval_segment(model, p3, seg, b, skips, 7);
        }
        const Vec whole = eval_full(model, x, 7);
        const Vec& chained = std::get<Vec>(so);
        for (int i = 0; i < 2; ++i)
            if (whole[i] != chained[i]) return fail("chaining != eval_full");
    }
    // inject_delay + RunStats (executor.hpp:53-59): busy time tracks the sleeps
    {
        auto pl = plan_async(20, 1, 2, 1);
        auto [tr, st] = run_parallel(pl, inject_delay(model, {0.002, 0.002}), part, x, s, 2);
        if (st.device_busy_s.size() != 2 || st.device_busy_s[0] < 0.038 || st.store_entries_per_round.size() != 19)
            return fail("instrumented run");
    }
    // run_one rows, as cmd_run prints them
    ExperimentConfig cfg;
    for (RunSpec spec : {RunSpec{2, 1, 1}, RunSpec{3, 2, 1}, RunSpec{3, 1, 2}}) {
        ResultRow r = run_one(cfg, model, spec, 7, true);
        std::printf("run_one %s: D=%d broadcasts=%d final_mse=%.6g latency=%.3f ms\n", r.config_label.c_str(),
                    r.device_count, r.broadcast_count, r.final_mse, r.measured_latency_s * 1e3);
    }
    std::printf("gpu ok\n");
    return 0;
}
