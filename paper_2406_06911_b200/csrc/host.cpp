// host.cpp -- control plane of the B200 AsyncDiff engine (see host.hpp).
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <set>
#include <sstream>

namespace adx {

namespace {
std::string S(long long v) { return std::to_string(v); }
}  // namespace

// ------------------------------------------------------------------ RNG
// rng.hpp:26-40 -- Box-Muller: cos branch returned, sin branch cached.
double Rng::normal() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1 = uniform();
    double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
}

// rng.hpp:55-60 -- splitmix64 finaliser over a + golden*(b+1)
uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ------------------------------------------------------------- schedule
// diffusion.cpp:39-77: linear or scaled-linear betas; abar_t = prod alpha.
void build_schedule(int T, double beta_start, double beta_end, int kind, std::vector<double>& betas,
                    std::vector<double>& alphas, std::vector<double>& alpha_bars) {
    if (T < 1) throw std::invalid_argument("build_schedule: T must be >= 1, got " + S(T));
    if (!(beta_start > 0.0) || !(beta_start <= beta_end) || !(beta_end < 1.0))
        throw std::invalid_argument(
            "build_schedule: need 0 < beta_start <= beta_end < 1, got beta_start=" +
            std::to_string(beta_start) + " beta_end=" + std::to_string(beta_end));
    betas.assign(T, 0.0);
    for (int t = 1; t <= T; ++t) {
        if (T == 1) {
            betas[0] = beta_start;
            break;
        }
        const double frac = static_cast<double>(t - 1) / static_cast<double>(T - 1);
        if (kind == 0) {
            betas[t - 1] = beta_start + frac * (beta_end - beta_start);
        } else {
            const double r = std::sqrt(beta_start) + frac * (std::sqrt(beta_end) - std::sqrt(beta_start));
            betas[t - 1] = r * r;
        }
    }
    alphas.assign(T, 0.0);
    alpha_bars.assign(T + 1, 1.0);
    for (int t = 1; t <= T; ++t) {
        alphas[t - 1] = 1.0 - betas[t - 1];
        alpha_bars[t] = alpha_bars[t - 1] * alphas[t - 1];
    }
}

// ---------------------------------------------------------------- model
// denoiser.cpp:31-41
std::vector<double> sinusoid(int t, int dim) {
    const int half = dim / 2;
    std::vector<double> s(dim, 0.0);
    for (int k = 0; k < half; ++k) {
        const double freq = std::exp(-std::log(10000.0) * static_cast<double>(k) / static_cast<double>(half));
        s[k] = std::cos(t * freq);
        s[half + k] = std::sin(t * freq);
    }
    return s;
}

std::vector<std::pair<int, int>> Model::links_into(int consumer) const {
    std::vector<std::pair<int, int>> r;
    for (auto& l : links)
        if (l.second == consumer) r.push_back(l);
    return r;  // links are kept sorted, so producers ascend
}

std::vector<std::pair<int, int>> Model::links_out_of(int producer) const {
    std::vector<std::pair<int, int>> r;
    for (auto& l : links)
        if (l.first == producer) r.push_back(l);
    return r;
}

long long Model::total_macs() const {
    long long t = 0;
    for (auto& s : stages) t += s.cost_macs;
    return t;
}

std::vector<double> Model::embed(int t) const {
    const std::vector<double> s = sinusoid(t, E);
    std::vector<double> e(E, 0.0);
    // column sweep, like a column-major GEMV: e += proj(:,k) * s[k]
    for (int k = 0; k < E; ++k)
        for (int i = 0; i < E; ++i) e[i] += proj[static_cast<size_t>(i) * E + k] * s[k];
    return e;
}

// denoiser.cpp:75-122 -- widths rule, skip-concat input widths, MAC cost
Model make_denoiser_shell(int L, const std::vector<int>& widths, std::vector<std::pair<int, int>> links,
                          int E) {
    if (L < 2) throw std::invalid_argument("make_denoiser_shell: L must be >= 2, got " + S(L));
    if (static_cast<int>(widths.size()) != L + 1)
        throw std::invalid_argument("make_denoiser_shell: widths must have L+1 entries, got " +
                                    S(static_cast<long long>(widths.size())));
    for (int w : widths)
        if (w < 1) throw std::invalid_argument("make_denoiser_shell: widths must be positive");
    if (widths.front() != widths.back())
        throw std::invalid_argument(
            "make_denoiser_shell: widths[0] (data dim) must equal widths[L] (eps dim)");
    if (E < 2 || E % 2 != 0)
        throw std::invalid_argument("make_denoiser_shell: time_embed_dim must be even and >= 2");
    for (auto& [p, c] : links)
        if (p < 1 || c > L || p >= c)
            throw std::invalid_argument("make_denoiser_shell: bad skip link (" + S(p) + ", " + S(c) + ")");
    Model m;
    m.L = L;
    m.E = E;
    m.widths = widths;
    std::sort(links.begin(), links.end());
    m.links = std::move(links);
    m.proj.assign(static_cast<size_t>(E) * E, 0.0);
    m.stages.resize(L);
    for (int i = 1; i <= L; ++i) {
        Stage& st = m.stages[i - 1];
        st.index = i;
        int in = (i == 1) ? widths[0] + E : widths[i - 1];
        for (auto& l : m.links_into(i)) in += widths[l.first];
        st.in = in;
        st.hidden = widths[i];
        st.out = widths[i];
        st.w1.assign(static_cast<size_t>(st.hidden) * in, 0.0);
        st.b1.assign(st.hidden, 0.0);
        st.tin.assign(static_cast<size_t>(st.hidden) * E, 0.0);
        st.w2.assign(static_cast<size_t>(st.out) * st.hidden, 0.0);
        st.b2.assign(st.out, 0.0);
        st.cost_macs = static_cast<long long>(st.hidden) * in + static_cast<long long>(st.hidden) * E +
                       static_cast<long long>(st.out) * st.hidden;
    }
    return m;
}

namespace {
// denoiser.cpp:21-27: a = sqrt(6/(r+c)), row-major draw order
void fill_xavier(Rng& rng, std::vector<double>& dst, int rows, int cols, double scale) {
    const double a = std::sqrt(6.0 / static_cast<double>(rows + cols));
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) dst[static_cast<size_t>(i) * cols + j] = scale * rng.uniform(-a, a);
}
}  // namespace

// denoiser.cpp:124-142 -- unet-mirror links (i, L+1-i); init order proj, then
// per stage w1, 0.5*time_in, w2; biases stay zero.
Model build_toy_denoiser(int L, const std::vector<int>& widths, int skip_spec, uint64_t seed, int E) {
    std::vector<std::pair<int, int>> links;
    if (skip_spec == 1)
        for (int i = 1; i < L + 1 - i; ++i) links.emplace_back(i, L + 1 - i);
    Model m = make_denoiser_shell(L, widths, std::move(links), E);
    Rng rng(seed);
    fill_xavier(rng, m.proj, E, E, 1.0);
    for (Stage& st : m.stages) {
        fill_xavier(rng, st.w1, st.hidden, st.in, 1.0);
        fill_xavier(rng, st.tin, st.hidden, E, 0.5);
        fill_xavier(rng, st.w2, st.out, st.hidden, 1.0);
    }
    return m;
}

// ------------------------------------------------------------ partition
int Partition::num_stages() const {
    int n = 0;
    for (auto& s : segments) n += static_cast<int>(s.size());
    return n;
}

int Partition::segment_of_stage(int stage) const {
    for (size_t i = 0; i < segments.size(); ++i)
        if (std::find(segments[i].begin(), segments[i].end(), stage) != segments[i].end())
            return static_cast<int>(i) + 1;
    throw std::out_of_range("segment_of_stage: stage " + S(stage) + " not in partition");
}

bool Partition::contiguous() const {
    int next = 1;
    for (auto& seg : segments)
        for (int s : seg)
            if (s != next++) return false;
    return true;
}

long long Partition::max_segment_macs() const {
    long long m = 0;
    for (long long c : segment_macs) m = std::max(m, c);
    return m;
}

long long Partition::total_macs() const {
    return std::accumulate(segment_macs.begin(), segment_macs.end(), 0LL);
}

// partition.hpp:33, partition.cpp:50-88
void Partition::validate(const Model& m) const {
    const int L = m.L;
    if (segments.empty()) throw std::invalid_argument("Partition: no segments");
    std::vector<char> seen(L + 1, 0);
    for (auto& seg : segments) {
        if (seg.empty()) throw std::invalid_argument("Partition: empty segment");
        for (size_t i = 0; i < seg.size(); ++i) {
            const int s = seg[i];
            if (s < 1 || s > L) throw std::invalid_argument("Partition: stage " + S(s) + " out of range");
            if (seen[s]) throw std::invalid_argument("Partition: stage " + S(s) + " assigned twice");
            seen[s] = 1;
            if (i > 0 && seg[i] <= seg[i - 1])
                throw std::invalid_argument("Partition: segment stages not ascending");
        }
    }
    for (int s = 1; s <= L; ++s)
        if (!seen[s]) throw std::invalid_argument("Partition: stage " + S(s) + " unassigned");
    if (device_of_segment.size() != segments.size() || segment_macs.size() != segments.size())
        throw std::invalid_argument("Partition: per-segment arrays size mismatch");
    if (strategy == 1 && segment_of_stage(1) != segment_of_stage(L))
        throw std::invalid_argument("Partition: first-last-grouped requires stages 1 and L in one segment");
}

namespace {
// partition.cpp:95-125 -- exact min-max contiguous split.  opt[p][i] is the
// best max-part cost of items [0,i) in p parts; a candidate replaces the
// incumbent only when strictly smaller, so ties keep the smallest cut.
std::vector<int> minmax_cuts(const std::vector<long long>& cost, int parts) {
    const int n = static_cast<int>(cost.size());
    std::vector<long long> pre(n + 1, 0);
    for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + cost[i];
    const long long inf = std::numeric_limits<long long>::max() / 4;
    std::vector<std::vector<long long>> opt(parts + 1, std::vector<long long>(n + 1, inf));
    std::vector<std::vector<int>> arg(parts + 1, std::vector<int>(n + 1, -1));
    opt[0][0] = 0;
    for (int p = 1; p <= parts; ++p)
        for (int i = p; i <= n - (parts - p); ++i)
            for (int j = p - 1; j < i; ++j) {
                const long long cand = std::max(opt[p - 1][j], pre[i] - pre[j]);
                if (cand < opt[p][i]) {
                    opt[p][i] = cand;
                    arg[p][i] = j;
                }
            }
    std::vector<int> cuts(parts + 1, 0);
    cuts[parts] = n;
    for (int p = parts; p >= 1; --p) cuts[p - 1] = arg[p][cuts[p]];
    return cuts;
}
}  // namespace

// partition.cpp:133-198
Partition partition_balanced(const Model& m, int N, int strategy) {
    const int L = m.L;
    auto cost = [&](int s) { return m.stages[s - 1].cost_macs; };
    Partition p;
    p.strategy = strategy;
    auto add_segment = [&](std::vector<int> st, int dev) {
        long long c = 0;
        for (int s : st) c += cost(s);
        p.segments.push_back(std::move(st));
        p.segment_macs.push_back(c);
        p.device_of_segment.push_back(dev);
    };
    if (strategy == 0) {
        if (N < 1 || N > L)
            throw std::invalid_argument("partition_balanced: N=" + S(N) + " infeasible for L=" + S(L));
        std::vector<long long> c;
        for (int s = 1; s <= L; ++s) c.push_back(cost(s));
        const auto cuts = minmax_cuts(c, N);
        for (int seg = 0; seg < N; ++seg) {
            std::vector<int> st;
            for (int s = cuts[seg] + 1; s <= cuts[seg + 1]; ++s) st.push_back(s);
            add_segment(std::move(st), seg);
        }
        p.validate(m);
        return p;
    }
    if (N < 1 || N > L - 1)
        throw std::invalid_argument("partition_balanced: first-last-grouped N=" + S(N) +
                                    " infeasible for L=" + S(L) + " (need N <= L-1)");
    if (N == 1) {
        std::vector<int> all(L);
        std::iota(all.begin(), all.end(), 1);
        add_segment(std::move(all), 0);
        p.validate(m);
        return p;
    }
    add_segment({1, L}, 0);
    std::vector<long long> mid;
    for (int s = 2; s <= L - 1; ++s) mid.push_back(cost(s));
    const auto cuts = minmax_cuts(mid, N - 1);
    for (int seg = 0; seg < N - 1; ++seg) {
        std::vector<int> st;
        for (int i = cuts[seg]; i < cuts[seg + 1]; ++i) st.push_back(i + 2);
        add_segment(std::move(st), seg + 1);
    }
    p.validate(m);
    return p;
}

// The same exact min-max DP (ties to the smallest cut) over caller-supplied per-stage
// costs (e.g. measured device time, ns) instead of MACs; segment_macs still report MACs.
Partition partition_by_cost(const Model& m, int N, const std::vector<long long>& stage_cost) {
    const int L = m.L;
    if (static_cast<int>(stage_cost.size()) != L)
        throw std::invalid_argument("partition_by_cost: need one cost per stage (" + S(L) + ")");
    if (N < 1 || N > L) throw std::invalid_argument("partition_by_cost: N=" + S(N) + " infeasible for L=" + S(L));
    for (long long c : stage_cost)
        if (c < 0) throw std::invalid_argument("partition_by_cost: negative stage cost");
    const auto cuts = minmax_cuts(stage_cost, N);
    Partition p;
    p.strategy = 0;
    for (int seg = 0; seg < N; ++seg) {
        std::vector<int> st;
        long long macs = 0;
        for (int s = cuts[seg] + 1; s <= cuts[seg + 1]; ++s) {
            st.push_back(s);
            macs += m.stages[s - 1].cost_macs;
        }
        p.segments.push_back(std::move(st));
        p.segment_macs.push_back(macs);
        p.device_of_segment.push_back(seg);
    }
    p.validate(m);
    return p;
}

// partition.cpp:200-208
std::vector<std::pair<int, int>> crossing_links(const Model& m, const Partition& p) {
    std::vector<std::pair<int, int>> r;
    for (auto& l : m.links)
        if (p.segment_of_stage(l.first) != p.segment_of_stage(l.second)) r.push_back(l);
    std::sort(r.begin(), r.end());
    return r;
}

// ----------------------------------------------------------------- plan
// plan.cpp:17-97.  Rounds start at t = T-w; a stride round (S=2, t>=2)
// evaluates segments 1..N-1 once at embed(t-1), segment N twice (lead at
// embed(t) on device N-1, extra at embed(t-1) on device N) and samples t, t-1.
Plan plan_async(int T, int w, int N, int S_, bool time_shift) {
    if (T < 1) throw std::invalid_argument("plan_async: T must be >= 1");
    if (w < 1 || w > T)
        throw std::invalid_argument("plan_async: w=" + S(w) + " outside [1, T=" + S(T) + "]");
    if (N < 1) throw std::invalid_argument("plan_async: N must be >= 1");
    if (S_ != 1 && S_ != 2) throw std::invalid_argument("plan_async: S must be 1 or 2, got " + S(S_));
    if (S_ == 2 && N < 2) throw std::invalid_argument("plan_async: S=2 requires N >= 2");
    Plan plan;
    plan.T = T;
    plan.w = w;
    plan.N = N;
    plan.S = S_;
    plan.D = N + S_ - 1;
    plan.time_shift = time_shift;
    for (int t = T; t > T - w; --t) plan.warmup_steps.push_back(t);
    auto emb = [&](int t) { return time_shift ? std::min(t + 1, T) : t; };
    auto upstream = [](int n, int prev) {
        InputRef in;
        if (n > 1) {
            in.kind = 1;
            in.producer_segment = n - 1;
            in.producer_round = prev;
        }
        return in;
    };
    int r = 0;
    for (int t = T - w; t >= 1; ++r) {
        Round rd;
        rd.index = r;
        const int prev = r == 0 ? kWarmupRound : r - 1;
        const bool stride = S_ == 2 && t >= 2;
        const int t_bcast = stride ? t - 1 : t;  // embedding of segments 1..N-1
        const int last_upstream = stride ? N - 1 : N;
        for (int n = 1; n <= last_upstream; ++n) {
            Eval e;
            e.segment = n;
            e.device = n - 1;
            e.embed_t = emb(t_bcast);
            e.input = upstream(n, prev);
            if (n == N) e.emits_eps_for = t;
            rd.evals.push_back(e);
        }
        if (stride) {
            Eval lead;
            lead.segment = N;
            lead.device = N - 1;
            lead.embed_t = emb(t);
            lead.input = upstream(N, prev);
            lead.emits_eps_for = t;
            Eval extra = lead;
            extra.device = N;
            extra.embed_t = emb(t - 1);
            extra.emits_eps_for = t - 1;
            rd.evals.push_back(lead);
            rd.evals.push_back(extra);
            rd.sampler_steps = {t, t - 1};
            t -= 2;
        } else {
            rd.sampler_steps = {t};
            t -= 1;
        }
        plan.rounds.push_back(std::move(rd));
    }
    if (!plan.rounds.empty()) plan.rounds.back().broadcast = false;
    return plan;
}

// plan.cpp:99-200 -- every invariant violation, first one first.
std::vector<std::string> validate_plan(const Plan& plan) {
    std::vector<std::string> v;
    if (plan.D != plan.N + plan.S - 1) v.push_back("device count " + S(plan.D) + " != N+S-1");
    if (static_cast<int>(plan.warmup_steps.size()) != plan.w) v.push_back("warm-up step list length != w");
    for (size_t i = 0; i < plan.warmup_steps.size(); ++i)
        if (plan.warmup_steps[i] != plan.T - static_cast<int>(i))
            v.push_back("warm-up step " + S(static_cast<long long>(i)) + " is not T-" + S(static_cast<long long>(i)));
    std::vector<int> order = plan.warmup_steps;
    std::map<int, int> eps_hits;
    for (size_t ri = 0; ri < plan.rounds.size(); ++ri) {
        const Round& rd = plan.rounds[ri];
        const int r = static_cast<int>(ri);
        if (rd.index != r) v.push_back("round " + S(r) + " carries index " + S(rd.index));
        std::set<int> used;
        for (const Eval& e : rd.evals) {
            const std::string at = "round " + S(r) + " segment " + S(e.segment);
            if (e.segment < 1 || e.segment > plan.N) v.push_back(at + ": segment out of range");
            if (e.device < 0 || e.device >= plan.D) v.push_back(at + ": device " + S(e.device) + " out of range");
            if (!used.insert(e.device).second)
                v.push_back("round " + S(r) + ": device " + S(e.device) + " evaluated twice");
            if (e.emits_eps_for.has_value() != (e.segment == plan.N))
                v.push_back(at + ": emits_eps_for must be set iff segment == N");
            if (e.emits_eps_for) ++eps_hits[*e.emits_eps_for];
            if (e.segment == 1 && e.input.kind != 0) v.push_back(at + ": segment 1 must read the current latent");
            if (e.segment != 1 && e.input.kind != 1) v.push_back(at + ": segment > 1 must read a cached bundle");
            if (e.input.kind == 1) {
                if (e.input.producer_segment != e.segment - 1)
                    v.push_back(at + ": cached ref names segment " + S(e.input.producer_segment) + ", expected " +
                                S(e.segment - 1));
                const int want = r == 0 ? kWarmupRound : r - 1;
                if (e.input.producer_round != want)
                    v.push_back(at + ": cached ref round " + S(e.input.producer_round) + " is not one round old");
                const int pr = e.input.producer_round;
                if (pr != kWarmupRound && pr >= 0 && pr < static_cast<int>(plan.rounds.size())) {
                    const Round& src = plan.rounds[pr];
                    if (!src.broadcast) v.push_back(at + ": cached ref points to non-broadcast round " + S(pr));
                    bool found = false;
                    for (const Eval& se : src.evals) found |= se.segment == e.input.producer_segment;
                    if (!found)
                        v.push_back(at + ": dangling cached ref, no eval of segment " +
                                    S(e.input.producer_segment) + " in round " + S(pr));
                } else if (pr != kWarmupRound) {
                    v.push_back(at + ": dangling cached ref to round " + S(pr));
                }
            }
        }
        for (size_t i = 0; i + 1 < rd.sampler_steps.size(); ++i)
            if (rd.sampler_steps[i] <= rd.sampler_steps[i + 1])
                v.push_back("round " + S(r) + ": sampler steps not strictly decreasing");
        std::set<int> emitted, sampled(rd.sampler_steps.begin(), rd.sampler_steps.end());
        for (const Eval& e : rd.evals)
            if (e.emits_eps_for) emitted.insert(*e.emits_eps_for);
        if (emitted != sampled) v.push_back("round " + S(r) + ": eps-emitting evals do not match the round's sampler steps");
        order.insert(order.end(), rd.sampler_steps.begin(), rd.sampler_steps.end());
    }
    for (auto& [ts, n] : eps_hits)
        if (n > 1) v.push_back("timestep " + S(ts) + " covered twice by eps evals");
    std::vector<int> want(plan.T);
    for (int i = 0; i < plan.T; ++i) want[i] = plan.T - i;
    if (order != want) {
        std::set<int> have(order.begin(), order.end());
        for (int ts : want)
            if (!have.count(ts)) v.push_back("timestep " + S(ts) + " never sampled");
        if (order.size() != want.size() || (have.size() == want.size() && order != want))
            v.push_back("sampler steps across warm-up + rounds are not T..1 in order");
    }
    return v;
}

std::vector<int> plan_to_flat(const Plan& p) {
    std::vector<int> f = {p.T, p.w, p.N, p.S, p.D, p.time_shift ? 1 : 0, static_cast<int>(p.rounds.size())};
    f.insert(f.end(), p.warmup_steps.begin(), p.warmup_steps.end());
    for (const Round& r : p.rounds) {
        f.push_back(r.index);
        f.push_back(r.broadcast ? 1 : 0);
        f.push_back(static_cast<int>(r.sampler_steps.size()));
        f.insert(f.end(), r.sampler_steps.begin(), r.sampler_steps.end());
        f.push_back(static_cast<int>(r.evals.size()));
        for (const Eval& e : r.evals) {
            f.insert(f.end(), {e.segment, e.device, e.embed_t, e.input.kind, e.input.producer_segment,
                               e.input.producer_round, e.emits_eps_for ? *e.emits_eps_for : -1});
        }
    }
    return f;
}

Plan plan_from_flat(const int* f, int len) {
    int pos = 0;
    auto next = [&]() {
        if (pos >= len) throw std::invalid_argument("plan_from_flat: truncated plan");
        return f[pos++];
    };
    Plan p;
    p.T = next();
    p.w = next();
    p.N = next();
    p.S = next();
    p.D = next();
    p.time_shift = next() != 0;
    const int nr = next();
    if (p.w < 0 || nr < 0) throw std::invalid_argument("plan_from_flat: negative count");
    for (int i = 0; i < p.w; ++i) p.warmup_steps.push_back(next());
    for (int r = 0; r < nr; ++r) {
        Round rd;
        rd.index = next();
        rd.broadcast = next() != 0;
        const int ns = next();
        if (ns < 0 || ns > 64) throw std::invalid_argument("plan_from_flat: bad sampler count");
        for (int i = 0; i < ns; ++i) rd.sampler_steps.push_back(next());
        const int ne = next();
        if (ne < 0 || ne > 4096) throw std::invalid_argument("plan_from_flat: bad eval count");
        for (int i = 0; i < ne; ++i) {
            Eval e;
            e.segment = next();
            e.device = next();
            e.embed_t = next();
            e.input.kind = next();
            e.input.producer_segment = next();
            e.input.producer_round = next();
            const int em = next();
            if (em >= 0) e.emits_eps_for = em;
            rd.evals.push_back(e);
        }
        p.rounds.push_back(std::move(rd));
    }
    return p;
}

// plan.cpp:202-232
PlanCounts plan_counts(const Plan& plan, const Partition& partition) {
    if (partition.num_segments() != plan.N)
        throw std::invalid_argument("plan_counts: partition has " + S(partition.num_segments()) +
                                    " segments, plan expects " + S(plan.N));
    PlanCounts c;
    c.device_count = plan.D;
    c.broadcasts_paper_convention = static_cast<int>(plan.rounds.size());
    for (auto& r : plan.rounds) c.broadcasts_strictly_needed += r.broadcast ? 1 : 0;
    c.evals_per_segment.assign(plan.N, 0);
    c.per_device_macs.assign(plan.D, 0);
    for (int n = 0; n < plan.N; ++n)
        c.per_device_macs[partition.device_of_segment[n]] +=
            static_cast<long long>(plan.w) * partition.segment_macs[n];
    for (auto& r : plan.rounds)
        for (auto& e : r.evals) {
            c.evals_per_segment[e.segment - 1] += 1;
            c.per_device_macs[e.device] += partition.segment_macs[e.segment - 1];
        }
    for (long long v : c.per_device_macs) c.max_device_macs = std::max(c.max_device_macs, v);
    c.sequential_total_macs = static_cast<long long>(plan.T) * partition.total_macs();
    return c;
}

// plan.cpp:234-244 -- entries after 1-based position max(w,1) take their
// predecessor's value.
std::vector<int> shift_embeddings(const std::vector<int>& ts, int w) {
    for (size_t i = 0; i + 1 < ts.size(); ++i)
        if (ts[i] <= ts[i + 1]) throw std::invalid_argument("shift_embeddings: list not strictly decreasing");
    if (w < 0) throw std::invalid_argument("shift_embeddings: w must be >= 0");
    std::vector<int> out = ts;
    const size_t keep = static_cast<size_t>(std::max(w, 1));
    for (size_t i = keep; i < ts.size(); ++i) out[i] = ts[i - 1];
    return out;
}

// plan.cpp:246-286 -- one row per device, one 7-char column per round
std::string render_plan(const Plan& plan) {
    std::ostringstream os;
    auto cell7 = [](const std::string& s) { return std::string(s.size() < 7 ? 7 - s.size() : 0, ' ') + s; };
    os << "plan T=" << plan.T << " w=" << plan.w << " N=" << plan.N << " S=" << plan.S << " D=" << plan.D
       << (plan.time_shift ? " time-shift" : "") << "\n";
    os << "warm-up steps:";
    for (int t : plan.warmup_steps) os << " " << t;
    os << "\n";
    if (plan.rounds.empty()) {
        os << "(warm-up only)\n";
        return os.str();
    }
    for (int d = 0; d < plan.D; ++d) {
        os << "dev" << d << " |";
        for (auto& r : plan.rounds) {
            std::string c = "      .";
            for (auto& e : r.evals)
                if (e.device == d)
                    c = cell7("s" + S(e.segment) + "@" + S(e.embed_t) + (e.emits_eps_for ? "*" : " "));
            os << c;
        }
        os << "\n";
    }
    os << "samp |";
    for (auto& r : plan.rounds) {
        std::string c;
        for (size_t i = 0; i < r.sampler_steps.size(); ++i) c += (i ? "," : "") + S(r.sampler_steps[i]);
        os << cell7(c);
    }
    os << "\nbcast|";
    for (auto& r : plan.rounds) os << (r.broadcast ? "      y" : "      n");
    os << "\n";
    return os.str();
}

}  // namespace adx
