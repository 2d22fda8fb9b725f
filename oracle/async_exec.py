"""Model-agnostic restatement of the reference's async executor semantics.

TEST INFRASTRUCTURE ONLY (tests/ and tools/; never imported by the product).

The C oracle (oracle/adx_oracle.c or_run_serial) restates run_serial for the
reference's own MLP model.  The UNet family has no C oracle, so this module
restates the same executor over an arbitrary per-stage function, so that a GPU
async run of ANY model family can be compared with an oracle async run:

  * warm-up cascade, fresh skip map per step, last step's bundles kept at round
    -1 (executor.cpp:168-202, 266-287);
  * per round: the skip snapshot = union of the newest crossing skips of
    segments 1..N-1 (collect_skips, executor.cpp:111-119); each eval reads the
    round-start snapshot and the cached bundle its InputRef names
    (execute_eval, executor.cpp:121-156); eps keyed by timestep; the sampler
    applies the round's steps in order (apply_sampler_steps,
    executor.cpp:224-241); bundles are committed in produced_by order and the
    store pruned to the warm-up tail + rounds >= r-1 (executor.cpp:28-62,
    316-318);
  * run_stage_range (denoiser.cpp:150-192): stage i consumes
    [current] + [skip features of links_into(i), ascending producer]; its output
    is written to every link out of i; finish_segment (denoiser.cpp:204-218)
    packs the crossing links produced in-segment into the bundle.

The plan is the oracle's own plan_async (oracle/adx_oracle.c, pinned by G5) and
the partition its own partition_balanced (pinned by G6).  tests/test_async_exec.py
pins THIS module against the C oracle's run_serial on the reference fixture
(G1, G2) before it is trusted for the UNet family.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

from . import oracle as O

StageFn = Callable[[int, List[np.ndarray], int], np.ndarray]
# (stage, [current, skip_1, ...], embed_t) -> stage output; stage 1 gets [latent]


def parse_plan(flat) -> dict:
    f = [int(v) for v in flat]
    T, w, N, S, D, shift, n_rounds = f[:7]
    warm = f[7:7 + w]
    q = 7 + w
    rounds = []
    for _ in range(n_rounds):
        idx, bc, ns = f[q], f[q + 1], f[q + 2]
        q += 3
        sampler = f[q:q + ns]
        q += ns
        ne = f[q]
        q += 1
        evs = []
        for _ in range(ne):
            seg, dev, et, kind, pseg, pround, emits = f[q:q + 7]
            q += 7
            evs.append(dict(seg=seg, dev=dev, embed_t=et, kind=kind, pseg=pseg, pround=pround, emits=emits))
        rounds.append(dict(index=idx, broadcast=bc, sampler=sampler, evals=evs))
    return dict(T=T, w=w, N=N, S=S, D=D, time_shift=shift, warmup=warm, rounds=rounds)


class AsyncOracle:
    def __init__(self, L: int, links: Sequence[Tuple[int, int]], stage_fn: StageFn):
        self.L = L
        self.links = sorted(tuple(l) for l in links)
        self.stage_fn = stage_fn

    def _segments(self, stage_segment) -> List[Tuple[int, int]]:
        ss = [int(v) for v in stage_segment]
        N = max(ss)
        first = [0] * (N + 1)
        last = [0] * (N + 1)
        for s, g in enumerate(ss, start=1):
            if not first[g]:
                first[g] = s
            last[g] = s
        return [(first[n], last[n]) for n in range(1, N + 1)]

    def run_stage_range(self, first: int, last: int, cur, skips: Dict, t: int):
        for i in range(first, last + 1):
            ins = [cur]
            for (p, c) in self.links:
                if c == i:
                    if (p, c) not in skips:
                        raise RuntimeError(f"eval: missing skip feature for link ({p} -> {c})")
                    ins.append(skips[(p, c)])
            cur = self.stage_fn(i, ins, t)
            for (p, c) in self.links:
                if p == i:
                    skips[(p, c)] = cur
        return cur

    def eval_segment(self, segs, seg: int, inp, skips_in: Dict, t: int):
        """-> ('eps', y) for the last segment, else ('bundle', (boundary, crossing skips))"""
        first, last = segs[seg - 1]
        skips = dict(skips_in)
        y = self.run_stage_range(first, last, inp, skips, t)
        if seg == len(segs):
            return "eps", y
        cross = {(p, c): v for (p, c), v in skips.items() if first <= p <= last and c > last}
        return "bundle", (y, cross)

    def run_serial(self, stage_segment, plan_flat, alpha_bars, x_T, ddim=None):
        """-> (latents (T+1, d) fp64, eps (T, d), store_entries per round, broadcast_count)"""
        P = parse_plan(plan_flat)
        segs = self._segments(stage_segment)
        N = len(segs)
        ddim = ddim or (lambda x, e, t: O.ddim_step(x, e, t, alpha_bars))
        x = np.asarray(x_T, np.float64).copy()
        lat, eps_rec = [x.copy()], []
        store: Dict[Tuple[int, int], tuple] = {}
        for wi, t in enumerate(P["warmup"]):  # executor.cpp:168-202
            sk: Dict = {}
            carry = None
            keep = {}
            for seg in range(1, N + 1):
                kind, out = self.eval_segment(segs, seg, x if seg == 1 else carry[0], sk, t)
                if kind == "eps":
                    e = out
                else:
                    sk.update(out[1])
                    keep[seg] = out
                    carry = out
            if wi + 1 == P["w"]:
                for seg in range(1, N):
                    store[(seg, -1)] = keep[seg]
            e = np.asarray(e, np.float64).reshape(-1)
            x = ddim(x, e, t)
            eps_rec.append(e)
            lat.append(x.copy())
        entries, bc = [], 0
        for R in P["rounds"]:
            r = R["index"]
            snap: Dict = {}
            for seg in range(1, N):  # collect_skips: newest bundle of every segment
                rs = [k[1] for k in store if k[0] == seg]
                if rs:
                    snap.update(store[(seg, max(rs))][1])
            outs = []
            for ev in R["evals"]:
                if ev["kind"] == 0:
                    inp = x
                else:
                    if ev["pround"] >= r:
                        raise AssertionError(f"executor: round {r} reads a bundle from round {ev['pround']}")
                    inp = store[(ev["pseg"], ev["pround"])][0]
                kind, out = self.eval_segment(segs, ev["seg"], inp, snap, ev["embed_t"])
                outs.append((ev, kind, out))
            for t in R["sampler"]:  # apply_sampler_steps
                e = [o for ev, k, o in outs if k == "eps" and ev["emits"] == t]
                if not e:
                    raise AssertionError(f"executor: no eps available for sampler step t={t}")
                e = np.asarray(e[0], np.float64).reshape(-1)
                x = ddim(x, e, t)
                eps_rec.append(e)
                lat.append(x.copy())
            for seg in range(1, N):  # commit in produced_by order
                for ev, k, o in outs:
                    if k == "bundle" and ev["seg"] == seg:
                        if (seg, r) in store:
                            raise AssertionError(f"BundleStore: entry ({seg}, {r}) already written")
                        store[(seg, r)] = o
            cur = r + 1  # prune: keep the warm-up tail and rounds >= cur - 2
            for k in [k for k in store if k[1] != -1 and k[1] < cur - 2]:
                del store[k]
            entries.append(len(store))
            bc += 1
        return np.stack(lat), np.stack(eps_rec), entries, bc


def mlp_stage_fn(model: "O.Model") -> StageFn:
    """the C oracle's MLP stage (denoiser.cpp:150-192) as a StageFn; stage 1's current
    input is [x ; e_t] (denoiser.cpp:242-244)"""
    def fn(stage, ins, t):
        cur = ins[0]
        if stage == 1:
            cur = np.concatenate([np.asarray(cur, np.float64), model.embed(t)])
        return model.stage_forward(stage, np.concatenate([cur] + list(ins[1:])), t)
    return fn


def unet_stage_fn(orc) -> StageFn:
    """an oracle.unet_oracle.UNetOracle stage as a StageFn.  With classifier-free guidance
    every stage carries both cascades (the product's batch-2 stages): activations are
    (uncond, cond) pairs, stage 1 feeds the one latent to both, and the out stage returns
    eps_u + s (eps_c - eps_u)"""
    if orc.ctxs.shape[0] == 1:
        def fn(stage, ins, t):
            orc.ci = 0
            return orc.stage(stage, ins, t)
        return fn

    def fn_cfg(stage, ins, t):
        ys = []
        for ci in (0, 1):
            orc.ci = ci
            ys.append(orc.stage(stage, [ins[0]] if stage == 1 else [x[ci] for x in ins], t))
        if stage == orc.L:
            eu, ec = ys
            s = orc.sp["cfg_scale"]
            return eu + s * (ec - eu) if orc.exact else eu + np.float32(s) * (ec - eu)
        return tuple(ys)
    return fn_cfg


def similarity_profile(ex: AsyncOracle, stage_segment, latents, timesteps):
    """metrics.cpp:73-101 restated: boundary activations of segments 1..N-1 at every latent
    with timestep >= 1 (fresh chaining, boundaries_at metrics.cpp:46-60), then cosine and
    rel-L2 (metrics.cpp:32-44) between adjacent steps.  -> (pair_t, cosine[N-1][], rel_l2[N-1][])"""
    segs = ex._segments(stage_segment)
    N = len(segs)
    cos = [[] for _ in range(max(0, N - 1))]
    rl = [[] for _ in range(max(0, N - 1))]
    pair_t = []
    if len(latents) < 3 or N < 2:
        return pair_t, cos, rl
    per_step, ts = [], []
    for x, t in zip(latents, timesteps):
        if t < 1:
            break
        sk, out = {}, []
        kind, o = ex.eval_segment(segs, 1, np.asarray(x, np.float64), sk, t)
        for seg in range(2, N + 1):
            out.append(np.asarray(o[0], np.float64).reshape(-1))
            sk.update(o[1])
            kind, o = ex.eval_segment(segs, seg, o[0], sk, t)
        per_step.append(out)
        ts.append(t)

    def cosine(a, b):
        na, nb = np.linalg.norm(a), np.linalg.norm(b)
        if na == 0.0 or nb == 0.0:
            return 1.0 if np.linalg.norm(a - b) == 0.0 else 0.0
        return float(np.dot(a, b) / (na * nb))

    def rel_l2(a, b):
        den = max(np.linalg.norm(a), np.linalg.norm(b))
        return 0.0 if den == 0.0 else float(np.linalg.norm(a - b) / den)

    for i in range(len(per_step) - 1):
        pair_t.append(ts[i])
        for b in range(N - 1):
            cos[b].append(cosine(per_step[i][b], per_step[i + 1][b]))
            rl[b].append(rel_l2(per_step[i][b], per_step[i + 1][b]))
    return pair_t, cos, rl
