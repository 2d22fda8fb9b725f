// schedule.cpp -- per-rank program of the multi-process async loop (schedule.hpp).
#include "schedule.hpp"

#include <algorithm>
#include <set>

namespace adx {

namespace {

struct Ctx {
    const Plan& plan;
    const Partition& part;
    const Model& m;
    std::vector<int> first, last, seg_of;
    Ctx(const Plan& p, const Partition& pa, const Model& mm) : plan(p), part(pa), m(mm) {
        const int N = pa.num_segments();
        first.assign(N + 1, 0);
        last.assign(N + 1, 0);
        seg_of.assign(mm.L + 1, 0);
        for (int n = 1; n <= N; ++n) {
            first[n] = pa.segments[n - 1].front();
            last[n] = pa.segments[n - 1].back();
            for (int s : pa.segments[n - 1]) seg_of[s] = n;
        }
    }
    // stages of segment p whose outputs segment q (> p) reads
    std::set<int> needed(int p, int q) const {
        std::set<int> st;
        if (q == p + 1) st.insert(last[p]);
        for (int i = first[q]; i <= last[q]; ++i)
            for (auto& l : m.links_into(i))
                if (seg_of[l.first] == p) st.insert(l.first);
        return st;
    }
    std::set<int> segs_of_rank(int r) const {
        std::set<int> s;
        for (int n = 1; n <= plan.N; ++n)
            if (part.device_of_segment[n - 1] == r) s.insert(n);
        for (auto& rd : plan.rounds)
            for (auto& e : rd.evals)
                if (e.device == r) s.insert(e.segment);
        return s;
    }
    // stages of segment p that rank c must receive
    std::set<int> xfer(int p, int c) const {
        std::set<int> st;
        for (int q : segs_of_rank(c))
            if (q > p)
                for (int s : needed(p, q)) st.insert(s);
        return st;
    }
};

}  // namespace

std::vector<int> ranks_evaluating(const Plan& plan, const Partition& part, int seg) {
    std::set<int> r;
    r.insert(part.device_of_segment[seg - 1]);
    for (auto& rd : plan.rounds)
        for (auto& e : rd.evals)
            if (e.segment == seg) r.insert(e.device);
    return std::vector<int>(r.begin(), r.end());
}

std::vector<RankOp> rank_program(const Plan& plan, const Partition& part, const Model& m, int v) {
    Ctx c(plan, part, m);
    const int N = plan.N, T = plan.T, d = m.data_dim();
    std::vector<int> all_ranks;
    for (int r = 0; r < plan.D; ++r) all_ranks.push_back(r);
    std::vector<RankOp> ops;
    int point = 0;

    // one exchange point: group op (carrying the produced stage and the round), its transfers, end
    auto emit_point = [&](std::vector<RankOp>& xs, int stage, int round) {
        if (!xs.empty()) {
            RankOp g;
            g.kind = kOpGroup;
            g.point = point;
            g.stage = stage;
            g.step = round;
            ops.push_back(g);
            for (auto& x : xs) {
                x.point = point;
                ops.push_back(x);
            }
            RankOp e;
            e.kind = kOpEnd;
            e.point = point;
            e.stage = stage;
            e.step = round;
            ops.push_back(e);
        }
        ++point;
    };
    // transfers of segment `seg`'s stage p output (evaluated by `owner`) into `slot`
    auto stage_xfers = [&](int seg, int p, int owner, int slot, std::vector<RankOp>& xs) {
        if (seg >= N) return;
        for (int cr : all_ranks) {
            if (cr == owner) continue;
            const std::set<int> st = c.xfer(seg, cr);
            if (!st.count(p)) continue;
            RankOp o;
            o.stage = p;
            o.slot = slot;
            o.elems = m.widths[p];
            if (owner == v) {
                o.kind = kOpSend;
                o.peer = cr;
                xs.push_back(o);
            } else if (cr == v) {
                o.kind = kOpRecv;
                o.peer = owner;
                xs.push_back(o);
            }
        }
    };
    auto eps_xfer = [&](int owner, int slot, int step, std::vector<RankOp>& xs) {
        if (owner == 0) return;
        RankOp o;
        o.stage = -1;
        o.slot = slot;
        o.step = step;
        o.elems = d;
        if (owner == v) {
            o.kind = kOpSend;
            o.peer = 0;
            xs.push_back(o);
        } else if (v == 0) {
            o.kind = kOpRecv;
            o.peer = owner;
            xs.push_back(o);
        }
    };
    // every stage output of `evals` (segment, owner) that another rank reads: one point per stage,
    // in stage order (the order each producer computes them)
    auto stage_points = [&](const std::vector<std::pair<int, int>>& evals, int slot, int round) {
        for (int p = 1; p < m.L; ++p)
            for (auto& [seg, owner] : evals)
                if (p >= c.first[seg] && p <= c.last[seg]) {
                    std::vector<RankOp> xs;
                    stage_xfers(seg, p, owner, slot, xs);
                    emit_point(xs, p, round);
                }
    };

    // warm-up: w sequential cascades (executor.cpp:168-202), slot 1
    for (int k = 0; k < plan.w; ++k) {
        const int t = plan.warmup_steps[k];
        for (int n = 1; n <= N; ++n) {
            const int owner = part.device_of_segment[n - 1];
            if (owner == v) {
                RankOp e;
                e.kind = kOpEval;
                e.seg = n;
                e.t = t;
                e.wslot = e.rslot = 1;
                e.step = k;
                e.eps_step = n == N ? k : -1;
                e.point = -1 - k;  // (eval ops: the round, -1 - k for warm-up step k)
                ops.push_back(e);
            }
            stage_points({{n, owner}}, 1, -1 - k);
            if (n == N) {
                std::vector<RankOp> xs;
                eps_xfer(owner, 1, k, xs);
                emit_point(xs, -1, -1 - k);
            }
        }
        if (v == 0) {
            RankOp dd;
            dd.kind = kOpDdim;
            dd.step = k;
            dd.t = t;
            dd.point = -1 - k;
            ops.push_back(dd);
        }
    }
    // rounds (executor.cpp:289-318): evals against the round-start snapshot, then the round's
    // exchange points (per produced stage, then eps), then the sampler on rank 0
    for (auto& rd : plan.rounds) {
        const int r = rd.index;
        const int wslot = (r + 2) % 2, rslot = (r + 1) % 2;
        const int step0 = T - rd.sampler_steps.front();
        std::vector<std::pair<int, int>> evs;
        for (auto& e : rd.evals) {
            evs.emplace_back(e.segment, e.device);
            if (e.device != v) continue;
            RankOp o;
            o.kind = kOpEval;
            o.seg = e.segment;
            o.t = e.embed_t;
            o.wslot = wslot;
            o.rslot = rslot;
            o.step = step0;
            o.eps_step = e.emits_eps_for ? T - *e.emits_eps_for : -1;
            o.point = r;  // (eval ops: the round index)
            ops.push_back(o);
        }
        if (rd.broadcast) stage_points(evs, wslot, r);  // last round: nobody reads its bundles
        for (auto& e : rd.evals)
            if (e.emits_eps_for) {
                std::vector<RankOp> xs;
                eps_xfer(e.device, wslot, T - *e.emits_eps_for, xs);
                emit_point(xs, -1, r);
            }
        if (v == 0)
            for (int t : rd.sampler_steps) {
                RankOp dd;
                dd.kind = kOpDdim;
                dd.step = T - t;
                dd.t = t;
                dd.point = r;
                ops.push_back(dd);
            }
    }
    return ops;
}

}  // namespace adx
