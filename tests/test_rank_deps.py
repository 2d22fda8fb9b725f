"""The stream / event dependency rules of the one-process-per-GPU runtime
(paper_2406_06911_b200/csrc/rank.cu build_graph) replayed as a discrete-event
simulation over the REAL rank programs (adx_rank_program), with random op
durations: every eval must read exactly the buffer versions it reads when the
ranks run fully serialised (the gloo replay's semantics, which reproduce the
oracle bit for bit -- tests/test_multirank_gloo.py).  This is how the per-stage
exchange points (a skip leaves while its producer computes the rest of the
segment) and the receive-while-computing overlap are checked without several
GPUs: a missing RAW edge (an eval reading a slot before its delivery) or WAR
edge (a receive overwriting a slot a local eval still reads, an eval
overwriting a slot whose send has not finished) shows up as a version mismatch.

Rules mirrored from rank.cu (per rank: a compute and a comm stream):
  eval     waits deliver[(p, rslot)] for its received inputs p, sent[(i, wslot)]
           for its stages i (and sent[(eps, wslot)] for the last segment);
           records stage[i] after each stage, read[rslot] at the end
  group    (comm) waits stage[s] (or the eval end, eps) if it sends, read[slot]
           if it receives; transfers rendezvous with the peers' same point
  end      records deliver / sent / eps for what the point moved
  ddim     waits eps (rank 0)
"""
import random

import numpy as np
import pytest

import paper_2406_06911_b200 as adx

from test_multirank_gloo import KIND_DDIM, KIND_END, KIND_EVAL, KIND_GROUP, KIND_RECV, KIND_SEND, program


def parse(ops):
    out = []
    for op in ops:
        kind, seg, t, wslot, rslot, step, eps_step, point, peer, stage, slot, elems = (int(v) for v in op)
        out.append(dict(kind=kind, seg=seg, t=t, wslot=wslot, rslot=rslot, step=step, eps_step=eps_step,
                        point=point, peer=peer, stage=stage, slot=slot))
    return out


class Sim:
    """Builds per-rank stream op lists with explicit dependencies (as rank.cu captures them),
    then executes them with random durations; buffers carry version tags.  serial=True is the
    reference: every rank's program runs in order on one stream (the gloo replay's order)."""

    def __init__(self, model, plan, part, rng, serial=False):
        self.m, self.plan, self.part, self.rng, self.serial = model, plan, part, rng, serial
        self.D = plan.D
        self.segs = part.segments
        self.first = {n + 1: s[0] for n, s in enumerate(self.segs)}
        self.last = {n + 1: s[-1] for n, s in enumerate(self.segs)}
        self.seg_of = {st: n + 1 for n, s in enumerate(self.segs) for st in s}
        self.links = model.skip_links
        self.L = model.num_stages()
        self.N = plan.N

    def reads(self, seg):
        r = set()
        if seg > 1:
            r.add(self.last[seg - 1])
        for i in range(self.first[seg], self.last[seg] + 1):
            for p, c in self.links:
                if c == i and self.seg_of[p] != seg:
                    r.add(p)
        return r

    def build(self, rank, ops):
        """-> list of stream ops: (stream, name, deps(list of event ids), records(list), action)"""
        evs = {}  # event name -> current record id (program-order binding)
        nid = [0]

        def record(name):
            nid[0] += 1
            evs[name] = (rank, nid[0])
            return evs[name]

        out = []
        have_eps = False
        for oi, op in enumerate(ops):
            k = op["kind"]
            if k == KIND_EVAL:
                deps = []
                for p in self.reads(op["seg"]):
                    if ("deliver", p, op["rslot"]) in evs:
                        deps.append(evs[("deliver", p, op["rslot"])])
                for i in range(self.first[op["seg"]], self.last[op["seg"]] + 1):
                    if ("sent", i, op["wslot"]) in evs:
                        deps.append(evs[("sent", i, op["wslot"])])
                if op["seg"] == self.N and ("sent", -1, op["wslot"]) in evs:
                    deps.append(evs[("sent", -1, op["wslot"])])
                for j, i in enumerate(range(self.first[op["seg"]], self.last[op["seg"]] + 1)):
                    recs = [record(("stage", i))]
                    if i == self.last[op["seg"]]:
                        recs += [record(("eval",)), record(("read", op["rslot"]))]
                    out.append(("comp", ("stage", op, i), deps if j == 0 else [], recs))
            elif k == KIND_GROUP:
                j = oi + 1
                items = []
                while ops[j]["kind"] != KIND_END:
                    items.append(ops[j])
                    j += 1
                deps = []
                if any(x["kind"] == KIND_SEND for x in items):
                    deps.append(evs[("stage", op["stage"])] if op["stage"] >= 0 else evs[("eval",)])
                rv = [x for x in items if x["kind"] == KIND_RECV and x["stage"] >= 0]
                if rv and ("read", rv[0]["slot"]) in evs:
                    deps.append(evs[("read", rv[0]["slot"])])
                recs = []
                for x in items:
                    if x["kind"] == KIND_RECV and x["stage"] < 0:
                        recs.append(record(("eps",)))
                        have_eps = True
                    elif x["kind"] == KIND_RECV:
                        recs.append(record(("deliver", x["stage"], x["slot"])))
                    else:
                        recs.append(record(("sent", x["stage"], x["slot"])))
                out.append(("comm", ("point", op["point"], items), deps, recs))
            elif k == KIND_DDIM:
                deps = [evs[("eps",)]] if have_eps else []
                out.append(("comp", ("ddim", op), deps, []))
        return out

    def run(self, ops_by_rank):
        # every rank with a part in a point joins it (an NCCL group completes when all of its
        # transfers do, i.e. when every peer posted its side)
        members = {}
        for r, ops in ops_by_rank.items():
            for o in ops:
                if o["kind"] == KIND_GROUP:
                    members.setdefault(o["point"], set()).add(r)
        streams = {}
        for r in range(self.D):
            sops = self.build(r, ops_by_rank[r])
            if self.serial:  # the reference: each rank runs its program in order on one stream
                streams[(r, "comm")] = sops
            else:
                streams[(r, "comp")] = [s for s in sops if s[0] == "comp"]
                streams[(r, "comm")] = [s for s in sops if s[0] == "comm"]
        done_events = {}  # event id -> completion time
        buf = {}  # (rank, stage, slot) / (rank, 'eps', slot) / (rank, 'lat', row) -> version
        seen = []  # (rank, eval seq, input versions)
        pos = {k: 0 for k in streams}
        free_at = {k: 0.0 for k in streams}
        now = 0.0
        evcount = {r: 0 for r in range(self.D)}
        while True:
            progressed = False
            # candidates: stream heads whose deps are done
            ready = []
            for key, lst in streams.items():
                if pos[key] >= len(lst):
                    continue
                s, what, deps, recs = lst[pos[key]]
                if any(d not in done_events for d in deps):
                    continue
                t0 = max([free_at[key]] + [done_events[d] for d in deps])
                ready.append((t0, key))
            if not ready:
                break
            # points need every participating rank's same point at its comm head
            self.rng.shuffle(ready)
            ready.sort(key=lambda x: x[0] if not self.serial else 0)
            for t0, key in ready:
                r, sname = key
                s, what, deps, recs = streams[key][pos[key]]
                if what[0] == "point":
                    pt = what[1]
                    parts = [(p, "comm") for p in sorted(members[pt]) if p != r]
                    ok = True
                    for pk in parts:
                        if pos[pk] >= len(streams[pk]):
                            ok = False
                            break
                        s2, w2, d2, r2 = streams[pk][pos[pk]]
                        if w2[0] != "point" or w2[1] != pt or any(d not in done_events for d in d2):
                            ok = False
                            break
                    if not ok:
                        continue
                    start = max([t0] + [max([free_at[pk]] + [done_events[d] for d in streams[pk][pos[pk]][2]])
                                        for pk in parts])
                    end = start + self.rng.uniform(0.1, 3.0)
                    group = [key] + parts
                    # move data: every send of every participant to its peer (sender's current version)
                    for gk in group:
                        gr = gk[0]
                        _, gw, _, grecs = streams[gk][pos[gk]]
                        for x in gw[2]:
                            if x["kind"] == KIND_SEND:
                                src = (gr, "eps", x["slot"]) if x["stage"] < 0 else (gr, x["stage"], x["slot"])
                                dst = (x["peer"], "epsrow", x["step"]) if x["stage"] < 0 else (x["peer"], x["stage"],
                                                                                               x["slot"])
                                buf[dst] = buf.get(src)
                        for e in grecs:
                            done_events[e] = end
                        free_at[gk] = end
                        pos[gk] += 1
                    progressed = True
                    break
                # compute ops
                dur = self.rng.uniform(0.5, 4.0)
                end = t0 + dur
                if what[0] == "stage":
                    op, i = what[1], what[2]
                    seg = op["seg"]
                    ins = []
                    if i == self.first[seg]:
                        ins.append(buf.get((r, "lat", op["step"])) if seg == 1 else
                                   buf.get((r, self.last[seg - 1], op["rslot"])))
                    else:
                        ins.append(buf.get((r, i - 1, op["wslot"])))
                    for p, c in self.links:
                        if c == i:
                            ins.append(buf.get((r, p, op["wslot"] if self.seg_of[p] == seg else op["rslot"])))
                    evcount[r] += 1
                    seen.append((r, evcount[r], i, tuple(ins)))
                    ver = ("y", r, op["point"], i)
                    if i == self.L:
                        if r == 0:
                            buf[(r, "epsrow", op["eps_step"])] = ver
                        else:
                            buf[(r, "eps", op["wslot"])] = ver
                    else:
                        buf[(r, i, op["wslot"])] = ver
                elif what[0] == "ddim":
                    op = what[1]
                    buf[(r, "lat", op["step"] + 1)] = ("lat", op["step"] + 1, buf.get((r, "lat", op["step"])),
                                                       buf.get((r, "epsrow", op["step"])))
                for e in recs:
                    done_events[e] = end
                free_at[key] = end
                pos[key] += 1
                progressed = True
                break
            if not progressed:
                break
        stuck = [k for k in streams if pos[k] < len(streams[k])]
        return seen, buf, stuck


CASES = [  # L, widths, skip, seed, T, w, N, S
    (6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 10, 1, 2, 1),
    (6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 10, 2, 3, 1),
    (6, [2, 8, 6, 10, 6, 8, 2], "unet-mirror", 5, 9, 3, 2, 2),
    (6, [4, 8, 8, 8, 8, 8, 4], "unet-mirror", 7, 8, 1, 3, 2),
    (5, [4, 6, 6, 6, 6, 4], "none", 9, 7, 2, 4, 1),
    (6, [4, 8, 8, 8, 8, 8, 4], "unet-mirror", 3, 9, 1, 6, 1),
]


@pytest.mark.parametrize("case", CASES)
def test_rank_dependencies_preserve_serial_reads(case):
    L, widths, spec, seed, T, w, N, S = case
    model = adx.build_toy_denoiser(L, widths, spec, seed)
    plan = adx.plan_async(T, w, N, S)
    part = adx.partition_balanced(model, N)
    ops = {r: parse(program(plan, part, model, r)) for r in range(plan.D)}
    ref_seen, ref_buf, stuck = Sim(model, plan, part, random.Random(0), serial=True).run(ops)
    assert not stuck
    ref = sorted(ref_seen)
    for trial in range(12):
        seen, buf, stuck = Sim(model, plan, part, random.Random(1000 + trial)).run(ops)
        assert not stuck, (case, trial, "deadlock")
        assert sorted(seen) == ref, (case, trial)
        assert buf[(0, "lat", T)] == ref_buf[(0, "lat", T)]


def test_skips_leave_before_the_segment_ends():
    """per-stage exchange points: in a round, the point carrying an early crossing skip of
    segment 1 precedes the point carrying segment 1's boundary"""
    model = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    plan = adx.plan_async(10, 1, 2, 1)
    part = adx.partition_balanced(model, 2)
    ops = parse(program(plan, part, model, 0))
    groups = [o for o in ops if o["kind"] == KIND_GROUP and o["step"] == 0 and o["stage"] >= 0]
    assert [g["stage"] for g in groups] == sorted(g["stage"] for g in groups)
    assert len(groups) >= 3  # stages 1, 2, 3 each leave in their own point
