// extras.cpp -- the §8(f) "next" rows around the hot path:
//   * checkpoint I/O in the reference's format (serialize.cpp:198-308):
//     <base>.json metadata + <base>.bin row-major little-endian fp64;
//   * plan JSON import/export (serialize.cpp:109-159);
//   * cost model (costsim.cpp:14-79) with an optional bytes-aware comm term
//     (per-round exchange bytes / link bandwidth + per-exchange latency).
// A minimal JSON value (dump in nlohmann's indent-2, sorted-key style; a
// recursive-descent parser) keeps the library free of third-party headers.
#include "extras.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>

namespace adx {

// ----------------------------------------------------------------- JSON
namespace json {

struct Value {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double n = 0.0;
    std::string s;
    std::vector<Value> a;
    std::map<std::string, Value> o;  // sorted keys, like nlohmann::json

    static Value num(double v) {
        Value x;
        x.kind = Num;
        x.n = v;
        return x;
    }
    static Value str(std::string v) {
        Value x;
        x.kind = Str;
        x.s = std::move(v);
        return x;
    }
    static Value boolean(bool v) {
        Value x;
        x.kind = Bool;
        x.b = v;
        return x;
    }
    static Value arr() {
        Value x;
        x.kind = Arr;
        return x;
    }
    static Value obj() {
        Value x;
        x.kind = Obj;
        return x;
    }
    const Value& at(const std::string& k) const {
        auto it = o.find(k);
        if (kind != Obj || it == o.end()) throw std::runtime_error("json: missing key '" + k + "'");
        return it->second;
    }
    bool has(const std::string& k) const { return kind == Obj && o.count(k); }
    int i() const { return static_cast<int>(n); }
    long long ll() const { return static_cast<long long>(n); }
};

Value ints(const std::vector<int>& v) {
    Value x = Value::arr();
    for (int e : v) x.a.push_back(Value::num(e));
    return x;
}

std::string num_text(double v) {
    if (std::floor(v) == v && std::fabs(v) < 9e15) return std::to_string(static_cast<long long>(v));
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

void dump(const Value& v, std::ostringstream& os, int indent, int depth) {
    const std::string pad(static_cast<size_t>(indent * (depth + 1)), ' ');
    const std::string pad0(static_cast<size_t>(indent * depth), ' ');
    switch (v.kind) {
        case Value::Null: os << "null"; break;
        case Value::Bool: os << (v.b ? "true" : "false"); break;
        case Value::Num: os << num_text(v.n); break;
        case Value::Str: os << '"' << v.s << '"'; break;
        case Value::Arr:
            if (v.a.empty()) {
                os << "[]";
                break;
            }
            os << "[\n";
            for (size_t i = 0; i < v.a.size(); ++i) {
                os << pad;
                dump(v.a[i], os, indent, depth + 1);
                os << (i + 1 < v.a.size() ? ",\n" : "\n");
            }
            os << pad0 << "]";
            break;
        case Value::Obj: {
            if (v.o.empty()) {
                os << "{}";
                break;
            }
            os << "{\n";
            size_t k = 0;
            for (auto& [key, val] : v.o) {
                os << pad << '"' << key << "\": ";
                dump(val, os, indent, depth + 1);
                os << (++k < v.o.size() ? ",\n" : "\n");
            }
            os << pad0 << "}";
            break;
        }
    }
}

std::string dump(const Value& v) {
    std::ostringstream os;
    dump(v, os, 2, 0);
    return os.str();
}

struct Parser {
    const std::string& t;
    size_t p = 0;
    explicit Parser(const std::string& s) : t(s) {}
    void ws() {
        while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
    }
    [[noreturn]] void bad() { throw std::runtime_error("json: parse error at offset " + std::to_string(p)); }
    Value parse() {
        ws();
        if (p >= t.size()) bad();
        const char c = t[p];
        if (c == '{') {
            ++p;
            Value v = Value::obj();
            ws();
            if (t[p] == '}') {
                ++p;
                return v;
            }
            while (true) {
                ws();
                Value k = parse();
                if (k.kind != Value::Str) bad();
                ws();
                if (t[p++] != ':') bad();
                v.o[k.s] = parse();
                ws();
                if (t[p] == ',') {
                    ++p;
                    continue;
                }
                if (t[p++] != '}') bad();
                return v;
            }
        }
        if (c == '[') {
            ++p;
            Value v = Value::arr();
            ws();
            if (t[p] == ']') {
                ++p;
                return v;
            }
            while (true) {
                v.a.push_back(parse());
                ws();
                if (t[p] == ',') {
                    ++p;
                    continue;
                }
                if (t[p++] != ']') bad();
                return v;
            }
        }
        if (c == '"') {
            ++p;
            std::string s;
            while (p < t.size() && t[p] != '"') {
                if (t[p] == '\\' && p + 1 < t.size()) ++p;
                s += t[p++];
            }
            ++p;
            return Value::str(s);
        }
        if (t.compare(p, 4, "true") == 0) {
            p += 4;
            return Value::boolean(true);
        }
        if (t.compare(p, 5, "false") == 0) {
            p += 5;
            return Value::boolean(false);
        }
        if (t.compare(p, 4, "null") == 0) {
            p += 4;
            return Value();
        }
        char* end = nullptr;
        const double v = std::strtod(t.c_str() + p, &end);
        if (end == t.c_str() + p) bad();
        p = static_cast<size_t>(end - t.c_str());
        return Value::num(v);
    }
};

Value parse(const std::string& s) {
    Parser ps(s);
    return ps.parse();
}

}  // namespace json

// ----------------------------------------------------------- plan JSON
// serialize.cpp:109-159 (same keys; input refs {"kind": "current-latent"} or
// {"kind": "cached", "segment": s, "round": r})
std::string plan_to_json(const Plan& plan) {
    using json::Value;
    Value rounds = Value::arr();
    for (const Round& r : plan.rounds) {
        Value evals = Value::arr();
        for (const Eval& e : r.evals) {
            Value je = Value::obj();
            je.o["segment"] = Value::num(e.segment);
            je.o["device"] = Value::num(e.device);
            je.o["embed_t"] = Value::num(e.embed_t);
            Value in = Value::obj();
            if (e.input.kind == 0) {
                in.o["kind"] = Value::str("current-latent");
            } else {
                in.o["kind"] = Value::str("cached");
                in.o["segment"] = Value::num(e.input.producer_segment);
                in.o["round"] = Value::num(e.input.producer_round);
            }
            je.o["input"] = in;
            if (e.emits_eps_for) je.o["emits_eps_for"] = Value::num(*e.emits_eps_for);
            evals.a.push_back(je);
        }
        Value jr = Value::obj();
        jr.o["index"] = Value::num(r.index);
        jr.o["evals"] = evals;
        jr.o["sampler_steps"] = json::ints(r.sampler_steps);
        jr.o["broadcast"] = Value::boolean(r.broadcast);
        rounds.a.push_back(jr);
    }
    Value j = Value::obj();
    j.o["T"] = Value::num(plan.T);
    j.o["w"] = Value::num(plan.w);
    j.o["N"] = Value::num(plan.N);
    j.o["S"] = Value::num(plan.S);
    j.o["D"] = Value::num(plan.D);
    j.o["time_shift"] = Value::boolean(plan.time_shift);
    j.o["warmup_steps"] = json::ints(plan.warmup_steps);
    j.o["rounds"] = rounds;
    return json::dump(j);
}

Plan plan_from_json(const std::string& text) {
    const json::Value j = json::parse(text);
    Plan p;
    p.T = j.at("T").i();
    p.w = j.at("w").i();
    p.N = j.at("N").i();
    p.S = j.at("S").i();
    p.D = j.at("D").i();
    p.time_shift = j.at("time_shift").b;
    for (auto& v : j.at("warmup_steps").a) p.warmup_steps.push_back(v.i());
    for (auto& jr : j.at("rounds").a) {
        Round r;
        r.index = jr.at("index").i();
        for (auto& v : jr.at("sampler_steps").a) r.sampler_steps.push_back(v.i());
        r.broadcast = jr.at("broadcast").b;
        for (auto& je : jr.at("evals").a) {
            Eval e;
            e.segment = je.at("segment").i();
            e.device = je.at("device").i();
            e.embed_t = je.at("embed_t").i();
            const json::Value& in = je.at("input");
            if (in.at("kind").s == "current-latent") {
                e.input.kind = 0;
            } else {
                e.input.kind = 1;
                e.input.producer_segment = in.at("segment").i();
                e.input.producer_round = in.at("round").i();
            }
            if (je.has("emits_eps_for")) e.emits_eps_for = je.at("emits_eps_for").i();
            r.evals.push_back(e);
        }
        p.rounds.push_back(std::move(r));
    }
    return p;
}

// ----------------------------------------------------------- checkpoints
// serialize.cpp:198-257: tensor order time_embed.proj, then per stage w1, b1,
// time_in, w2, b2; all row-major little-endian fp64.
namespace {
struct TRef {
    std::string name;
    std::vector<double>* data;
    long long rows, cols;
};
std::vector<TRef> tensor_list(Model& m) {
    std::vector<TRef> ts;
    ts.push_back({"time_embed.proj", &m.proj, m.E, m.E});
    for (size_t i = 0; i < m.stages.size(); ++i) {
        Stage& s = m.stages[i];
        const std::string p = "stage" + std::to_string(i + 1) + ".";
        ts.push_back({p + "w1", &s.w1, s.hidden, s.in});
        ts.push_back({p + "b1", &s.b1, s.hidden, 1});
        ts.push_back({p + "time_in", &s.tin, s.hidden, m.E});
        ts.push_back({p + "w2", &s.w2, s.out, s.hidden});
        ts.push_back({p + "b2", &s.b2, s.out, 1});
    }
    return ts;
}
}  // namespace

void save_checkpoint(const std::string& base, const Model& mc) {
    using json::Value;
    Model& m = const_cast<Model&>(mc);
    Value meta = Value::obj();
    meta.o["format"] = Value::str("asyncdiff-checkpoint-v1");
    meta.o["L"] = Value::num(m.L);
    meta.o["widths"] = json::ints(m.widths);
    meta.o["time_embed_dim"] = Value::num(m.E);
    Value links = Value::arr();
    for (auto& [p, c] : m.links) {
        Value l = Value::arr();
        l.a = {Value::num(p), Value::num(c)};
        links.a.push_back(l);
    }
    meta.o["skip_links"] = links;
    Value tensors = Value::arr();
    long long off = 0;
    auto ts = tensor_list(m);
    for (auto& t : ts) {
        Value jt = Value::obj();
        jt.o["name"] = Value::str(t.name);
        jt.o["rows"] = Value::num(static_cast<double>(t.rows));
        jt.o["cols"] = Value::num(static_cast<double>(t.cols));
        jt.o["offset_doubles"] = Value::num(static_cast<double>(off));
        tensors.a.push_back(jt);
        off += t.rows * t.cols;
    }
    meta.o["tensors"] = tensors;
    meta.o["total_doubles"] = Value::num(static_cast<double>(off));
    meta.o["endianness"] = Value::str("little");
    std::ofstream jf(base + ".json");
    if (!jf) throw std::runtime_error("save_checkpoint: cannot write " + base + ".json");
    jf << json::dump(meta) << "\n";
    std::ofstream bf(base + ".bin", std::ios::binary);
    if (!bf) throw std::runtime_error("save_checkpoint: cannot write " + base + ".bin");
    for (auto& t : ts) bf.write(reinterpret_cast<const char*>(t.data->data()), t.data->size() * sizeof(double));
}

Model load_checkpoint(const std::string& base) {
    std::ifstream jf(base + ".json");
    if (!jf) throw std::runtime_error("load_checkpoint: cannot read " + base + ".json");
    std::stringstream ss;
    ss << jf.rdbuf();
    const json::Value meta = json::parse(ss.str());
    if (meta.at("format").s != "asyncdiff-checkpoint-v1")
        throw std::runtime_error("load_checkpoint: unknown format " + meta.at("format").s);
    const int L = meta.at("L").i();
    std::vector<int> widths;
    for (auto& v : meta.at("widths").a) widths.push_back(v.i());
    const int E = meta.at("time_embed_dim").i();
    std::vector<std::pair<int, int>> links;
    for (auto& l : meta.at("skip_links").a) links.emplace_back(l.a.at(0).i(), l.a.at(1).i());
    Model m = make_denoiser_shell(L, widths, links, E);
    std::ifstream bf(base + ".bin", std::ios::binary);
    if (!bf) throw std::runtime_error("load_checkpoint: cannot read " + base + ".bin");
    for (auto& t : tensor_list(m)) {
        if (!bf.read(reinterpret_cast<char*>(t.data->data()), t.data->size() * sizeof(double)))
            throw std::runtime_error("load_checkpoint: blob truncated at " + t.name);
    }
    return m;
}

// ------------------------------------------------------------ cost model
// costsim.cpp:14-50; comm per round = flat comm_cost_s, or (bytes-aware)
// comm_latency_s + bytes_r / link_gbs when round_bytes is given.
LatencyReport predict_async(const Plan& plan, const CostModel& cm, const std::vector<long long>* round_bytes) {
    if (static_cast<int>(cm.segment_cost_s.size()) != plan.N)
        throw std::invalid_argument("predict_async: cost model has " + std::to_string(cm.segment_cost_s.size()) +
                                    " segment costs, plan expects " + std::to_string(plan.N));
    double seg_total = 0.0;
    for (double c : cm.segment_cost_s) seg_total += c;
    LatencyReport rep;
    rep.sequential_total_s = predict_sequential(plan.T, cm);
    rep.warmup_s = static_cast<double>(plan.w) * (seg_total + cm.sampler_cost_s);
    double total = rep.warmup_s;
    for (size_t ri = 0; ri < plan.rounds.size(); ++ri) {
        const Round& r = plan.rounds[ri];
        double compute = 0.0;
        for (const Eval& e : r.evals) compute = std::max(compute, cm.segment_cost_s[e.segment - 1]);
        double comm = 0.0;
        if (round_bytes && cm.link_gbs > 0.0)
            comm = cm.comm_latency_s + static_cast<double>((*round_bytes)[ri]) / (cm.link_gbs * 1e9);
        else if (r.broadcast)
            comm = cm.comm_cost_s;
        const double sampler = cm.sampler_cost_s * static_cast<double>(r.sampler_steps.size());
        rep.round_compute_s.push_back(compute);
        rep.round_comm_s.push_back(comm);
        rep.comm_total_s += comm;
        total += compute + comm + sampler;
    }
    rep.async_total_s = total;
    rep.speedup = total > 0.0 ? rep.sequential_total_s / total : 1.0;
    rep.comm_ratio = total > 0.0 ? rep.comm_total_s / total : 0.0;
    rep.approx_step_s = seg_total / static_cast<double>(plan.N) + cm.comm_cost_s;
    rep.approx_total_s = rep.warmup_s + static_cast<double>(plan.rounds.size()) * rep.approx_step_s;
    return rep;
}

double predict_sequential(int T, const CostModel& cm) {
    double seg_total = 0.0;
    for (double c : cm.segment_cost_s) seg_total += c;
    return static_cast<double>(T) * (seg_total + cm.sampler_cost_s);
}

// costsim.cpp:52-79
CostComparison calibrate_and_compare(const Plan& plan, const std::vector<double>& delays,
                                     const std::vector<double>& measured_round_comm_s, int broadcast_count,
                                     double measured_total_s) {
    CostModel cm;
    cm.segment_cost_s = delays;
    double measured_comm = 0.0;
    for (double c : measured_round_comm_s) measured_comm += c;
    cm.comm_cost_s = measured_comm / static_cast<double>(std::max(1, broadcast_count));
    const LatencyReport pred = predict_async(plan, cm, nullptr);
    CostComparison c;
    c.calibrated_comm_cost_s = cm.comm_cost_s;
    c.predicted_total_s = pred.async_total_s;
    c.measured_total_s = measured_total_s;
    c.rel_error_total =
        measured_total_s > 0.0 ? std::fabs(pred.async_total_s - measured_total_s) / measured_total_s : 0.0;
    c.predicted_comm_ratio = pred.comm_ratio;
    c.measured_comm_ratio = measured_total_s > 0.0 ? measured_comm / measured_total_s : 0.0;
    c.rel_error_comm_ratio = c.measured_comm_ratio > 0.0
                                 ? std::fabs(c.predicted_comm_ratio - c.measured_comm_ratio) / c.measured_comm_ratio
                                 : 0.0;
    return c;
}

// bytes that cross devices in each round of the one-process-per-GPU program
// (every send of every rank at the round's exchange point)
// precision: engine precision (kF64 / kF32 / kBF16); stage outputs travel at the stage element size
// (UNet: bf16 in the bf16 mode, fp32 in the f32 mode), eps at the trajectory element size
std::vector<long long> round_exchange_bytes(const Plan& plan, const Partition& part, const Model& m, int precision);

}  // namespace adx

#include "schedule.hpp"

namespace adx {

std::vector<long long> round_exchange_bytes(const Plan& plan, const Partition& part, const Model& m, int precision) {
    std::vector<long long> out(plan.rounds.size(), 0);
    const int traj = precision == 0 ? 8 : 4;                           // kF64 : kF32 / kBF16 trajectory
    const int stage = m.kind == 1 ? (precision == 1 ? 4 : 2) : traj;  // UNet f32 : bf16 stage outputs
    // exchange points carry their round (group op `step`; warm-up steps are negative)
    for (int r = 0; r < plan.D; ++r) {
        int round = -1;
        for (const RankOp& op : rank_program(plan, part, m, r)) {
            if (op.kind == kOpGroup) round = op.step;
            if (op.kind == kOpSend && round >= 0 && round < static_cast<int>(out.size()))
                out[round] += op.elems * (op.stage < 0 ? traj : stage);
        }
    }
    return out;
}

}  // namespace adx
