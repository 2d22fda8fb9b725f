"""Multi-rank (one process per GPU) exchange schedule, checked on CPU.

Every rank replays its op list from the C ABI (adx_rank_program -- the same
list that drives the NCCL transport in rank.cu) with world_size D gloo
processes: evals with the oracle's stage forward, each exchange point as a set
of isend/irecv, DDIM on rank 0.  Rank 0's trajectory must equal the oracle's
run_serial bit for bit: a wrong slot, peer, order or missing transfer breaks
that immediately.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

import paper_2406_06911_b200 as adx
from oracle import oracle as O

KIND_EVAL, KIND_GROUP, KIND_SEND, KIND_RECV, KIND_END, KIND_DDIM = range(6)


def program(plan, part, model, rank):
    cap = 12 * 200000
    buf = np.zeros(cap, np.int32)
    n = C.c_int()
    ph = plan._handle()
    adx._lib.check(adx.lib().adx_rank_program(ph._h, part._h, model._h, rank, buf.ctypes.data_as(C.POINTER(C.c_int)),
                                               cap, C.byref(n)))
    return buf[: 12 * n.value].reshape(-1, 12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, widths, spec, seed, T, w, N, S = case
        model = adx.build_toy_denoiser(L, widths, spec, seed)
        om = O.Model.build_toy(L, widths, spec, seed, 8)
        sched = O.build_schedule(T, 0.01, 0.15)
        plan = adx.plan_async(T, w, N, S)
        part = adx.partition_balanced(model, N)
        ops = program(plan, part, model, rank)
        segs = part.segments
        first = {n + 1: s[0] for n, s in enumerate(segs)}
        last = {n + 1: s[-1] for n, s in enumerate(segs)}
        seg_of = {st: n + 1 for n, s in enumerate(segs) for st in s}
        links = model.skip_links
        d = widths[0]
        x_T = O.random_normals(seed + 1, d)
        Y, EPS = {}, {}
        lat = np.zeros((T + 1, d)); eps = np.zeros((T, d)); lat[0] = x_T
        pending = []
        for op in ops:
            kind, seg, t, wslot, rslot, step, eps_step, point, peer, stage, slot, elems = (int(v) for v in op)
            if kind == KIND_EVAL:
                for i in range(first[seg], last[seg] + 1):
                    if i == first[seg]:
                        cur = np.concatenate([lat[step], om.embed(t)]) if seg == 1 else Y[(last[seg - 1], rslot)]
                    else:
                        cur = Y[(i - 1, wslot)]
                    parts = [cur] + [Y[(p, wslot if seg_of[p] == seg else rslot)] for p, c in links if c == i]
                    y = om.stage_forward(i, np.concatenate(parts), t)
                    if i == L:
                        if rank == 0:
                            eps[eps_step] = y
                        else:
                            EPS[wslot] = y
                    else:
                        Y[(i, wslot)] = y
            elif kind == KIND_GROUP:
                pending = []
            elif kind == KIND_SEND:
                src = EPS[slot] if stage < 0 else Y[(stage, slot)]
                pending.append((dist.isend(torch.from_numpy(src.copy()), peer), None, None))
            elif kind == KIND_RECV:
                buf = torch.zeros(elems, dtype=torch.float64)
                pending.append((dist.irecv(buf, peer), buf, (stage, slot, step)))
            elif kind == KIND_END:
                for req, buf, tgt in pending:
                    req.wait()
                    if buf is not None:
                        st_, sl_, sp_ = tgt
                        if st_ < 0:
                            eps[sp_] = buf.numpy()
                        else:
                            Y[(st_, sl_)] = buf.numpy().copy()
                pending = []
            elif kind == KIND_DDIM:
                lat[step + 1] = O.ddim_step(lat[step], eps[step], t, sched.alpha_bars)
        if rank == 0:
            ss, _ = O.partition_balanced(om.costs(), N)
            ref_lat, ref_eps, _, _ = O.run_serial(om, ss, N, O.plan_async_flat(T, w, N, S), sched.alpha_bars, x_T)
            q.put(("ok", bool(np.array_equal(lat, ref_lat) and np.array_equal(eps, ref_eps)),
                   float(np.abs(lat - ref_lat).max())))
    except Exception as exc:  # surface worker failures to the parent
        q.put(("err", rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


CASES = [
    # L, widths, skip, seed, T, w, N, S
    (6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 12, 1, 2, 1),
    (6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11, 12, 2, 3, 1),
    (6, [2, 8, 6, 10, 6, 8, 2], "unet-mirror", 5, 11, 3, 2, 2),
    (6, [4, 8, 8, 8, 8, 8, 4], "unet-mirror", 7, 10, 1, 3, 2),
    (5, [4, 6, 6, 6, 6, 4], "none", 9, 9, 2, 4, 1),
]


@pytest.mark.parametrize("case", CASES)
def test_rank_programs_reproduce_serial(case):
    import torch.multiprocessing as mp
    N, S = case[6], case[7]
    world = N + S - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    ok = [m for m in msgs if m[0] == "ok"]
    assert ok and ok[0][1], msgs


def test_rank_program_shapes():
    model = adx.build_toy_denoiser(6, [2, 8, 8, 8, 8, 8, 2], "unet-mirror", 11)
    plan = adx.plan_async(20, 1, 2, 1)
    part = adx.partition_balanced(model, 2)
    r0, r1 = program(plan, part, model, 0), program(plan, part, model, 1)
    assert (r0[:, 0] == KIND_EVAL).sum() == 20  # w warm-up + 19 rounds
    assert (r1[:, 0] == KIND_EVAL).sum() == 20
    assert (r0[:, 0] == KIND_DDIM).sum() == 20 and (r1[:, 0] == KIND_DDIM).sum() == 0
    # every send has a matching recv on the peer, same point, same size
    sends0 = [(int(o[7]), int(o[9]), int(o[11])) for o in r0 if o[0] == KIND_SEND]
    recvs1 = [(int(o[7]), int(o[9]), int(o[11])) for o in r1 if o[0] == KIND_RECV]
    assert sends0 == recvs1
    sends1 = [(int(o[7]), int(o[11])) for o in r1 if o[0] == KIND_SEND]
    recvs0 = [(int(o[7]), int(o[11])) for o in r0 if o[0] == KIND_RECV]
    assert sends1 == recvs0
