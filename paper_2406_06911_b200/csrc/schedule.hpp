// schedule.hpp -- per-rank program of the multi-process async loop.
//
// One process per GPU: rank v runs exactly the evals the plan assigns to device
// v (plan.cpp:53, 67-73, 82) and exchanges stage outputs point-to-point.  The
// program is a flat, totally ordered list of ops that every rank derives from
// the same (plan, partition, model) -- so the sends and receives of a pair of
// ranks appear in the same order on both sides, and each exchange point is one
// NCCL group (send/recv order inside a group does not matter).  The same list
// drives the NCCL transport (rank.cu) and the CPU gloo test
// (tests/test_multirank_gloo.py), which is how the multi-rank path is checked
// without several GPUs.
//
// Slots: stage outputs live in two parity slots per stage (engine.hpp); round
// r writes slot s(r) = (r+2)%2 and reads cross-segment inputs from s(r-1);
// the warm-up cascade uses slot 1 (= s(-1)).
//
// Exchange granularity: one point per PRODUCED STAGE (its output to every rank
// that reads it), in (round, stage) order, plus one eps point per eps.  A point
// only waits for the stage that produced its data, so a crossing skip produced
// early in a segment travels while the producer computes the rest of the
// segment; a receiving eval waits only for the points that deliver its inputs
// (and its slot's previous sends), not for the whole previous exchange.
#pragma once

#include "host.hpp"

#include <vector>

namespace adx {

enum OpKind {
    kOpEval = 0,   // evaluate `seg` at embed `t`; wslot/rslot; latent row `step`; eps row `eps_step` (-1 none)
    kOpGroup = 1,  // begin an exchange point (NCCL group); `point` = global exchange index, `stage` = the
                   // produced stage it carries (-1: eps), `step` = round (-1 - k: warm-up step k)
    kOpSend = 2,   // send stage `stage` output (slot) or eps (stage = -1, local eps buffer slot) to `peer`
    kOpRecv = 3,   // receive stage `stage` output into slot, or eps (stage = -1) into trajectory row `step`
    kOpEnd = 4,    // end the exchange point
    kOpDdim = 5,   // sampler step on rank 0: latent row `step` -> `step+1` with eps row `step`, timestep t
};

struct RankOp {
    int kind = 0;
    int seg = 0, t = 0, wslot = 0, rslot = 0, step = -1, eps_step = -1;
    int point = -1, peer = -1, stage = 0, slot = 0;
    long long elems = 0;  // element count of a send/recv
};

// The program of `rank` (virtual device): per warm-up step / round the evals of
// this rank, then the exchange points of that step / round (per produced
// stage, then eps).  Ranks with no part in a point skip it.
std::vector<RankOp> rank_program(const Plan& plan, const Partition& part, const Model& m, int rank);

// Which ranks consume the outputs of segment `seg` (evaluate seg+1.. with a
// link from seg) -- the union over the plan's evals and the warm-up placement.
std::vector<int> ranks_evaluating(const Plan& plan, const Partition& part, int seg);

}  // namespace adx
