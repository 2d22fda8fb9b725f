// extras.hpp -- checkpoint / plan JSON I/O and the cost model (§8f rows).
#pragma once

#include "host.hpp"

#include <string>
#include <vector>

namespace adx {

std::string plan_to_json(const Plan& plan);          // serialize.cpp:109-133
Plan plan_from_json(const std::string& text);        // serialize.cpp:135-159
void save_checkpoint(const std::string& base, const Model& m);  // serialize.cpp:226-257
Model load_checkpoint(const std::string& base);                 // serialize.cpp:259-308

// costsim.hpp:13-50 (+ bytes-aware comm: comm_latency_s + bytes / link_gbs)
struct CostModel {
    std::vector<double> segment_cost_s;
    double comm_cost_s = 0.0;
    double sampler_cost_s = 0.0;
    double comm_latency_s = 0.0;
    double link_gbs = 0.0;
};
struct LatencyReport {
    double sequential_total_s = 0.0, async_total_s = 0.0, warmup_s = 0.0;
    std::vector<double> round_compute_s, round_comm_s;
    double comm_total_s = 0.0, speedup = 1.0, comm_ratio = 0.0, approx_step_s = 0.0, approx_total_s = 0.0;
};
struct CostComparison {
    double predicted_total_s = 0.0, measured_total_s = 0.0, rel_error_total = 0.0;
    double predicted_comm_ratio = 0.0, measured_comm_ratio = 0.0, rel_error_comm_ratio = 0.0;
    double calibrated_comm_cost_s = 0.0;
};
double predict_sequential(int T, const CostModel& cm);
LatencyReport predict_async(const Plan& plan, const CostModel& cm, const std::vector<long long>* round_bytes);
CostComparison calibrate_and_compare(const Plan& plan, const std::vector<double>& delays,
                                     const std::vector<double>& measured_round_comm_s, int broadcast_count,
                                     double measured_total_s);
// precision: engine precision (kF64 / kF32 / kBF16); stage outputs travel at the stage element size
// (UNet: bf16 in the bf16 mode, fp32 in the f32 mode), eps at the trajectory element size
std::vector<long long> round_exchange_bytes(const Plan& plan, const Partition& part, const Model& m, int precision);

}  // namespace adx
