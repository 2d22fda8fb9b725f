"""Predicted N-GPU latency of the c2 run from the reference's own cost model
(costsim.cpp:18-50 + the bytes-aware comm term) fed with per-stage device times
measured on this B200 (each stage in its own CUDA graph).  No multi-GPU box is
available to this build, so this is the stand-in for the N=2/4/8 numbers; the
bench's N-GPU path (torchrun + NCCL p2p, bench.py run_ranks) measures them for real.

Partitions: the reference's MAC-balanced min-max split (partition_balanced) and the
same DP over the measured stage times ("time-balanced").
NVLink model: 900 GB/s per direction nominal, taken as 700 GB/s achieved for the
multi-MB activations, plus 10 us per exchange round (launch + NCCL group latency)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx

T, W, LINK_GBS, LAT_S = 50, 9, 700.0, 10e-6


def minmax_split(costs, N):
    """exact min-max contiguous split (partition.cpp:95-125 semantics, ties to the smallest cut)"""
    L = len(costs)
    pre = np.concatenate([[0.0], np.cumsum(costs)])
    best = np.full((N + 1, L + 1), np.inf)
    cut = np.zeros((N + 1, L + 1), int)
    best[0][0] = 0.0
    for p in range(1, N + 1):
        for i in range(p, L - (N - p) + 1):
            for j in range(p - 1, i):
                v = max(best[p - 1][j], pre[i] - pre[j])
                if v < best[p][i]:
                    best[p][i], cut[p][i] = v, j
    segs, i = [], L
    for p in range(N, 0, -1):
        j = cut[p][i]
        segs.append(list(range(j + 1, i + 1)))
        i = j
    return segs[::-1]


m = adx.build_unet_denoiser(seed=0)
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
st_ms = adx.stage_times(m, T, 20, prec)
pass_ms, _, _ = adx.time_model_pass(m, T, 10, prec)
res = {"precision": prec, "stage_ms": st_ms, "sum_stage_ms": sum(st_ms), "pass_ms_graph": pass_ms,
       "link_gbs": LINK_GBS, "comm_latency_s": LAT_S, "T": T, "w": W, "runs": []}
for (N, S) in ((1, 1), (2, 1), (3, 1), (4, 1), (3, 2), (8, 1)):
    w = T if N == 1 else W
    plan = adx.plan_async(T, w, N, S)
    for kind in ("macs", "time"):
        if kind == "macs":
            part = adx.partition_balanced(m, N)
            segs = part.segments
        else:
            segs = minmax_split(st_ms, N)
            part = adx.Partition.create(segs)
        seg_cost = [sum(st_ms[i - 1] for i in sg) / 1e3 for sg in segs]
        rb = adx.round_exchange_bytes(plan, part, m, prec)
        cm = adx.CostModel(segment_cost_s=seg_cost, comm_cost_s=0.0, sampler_cost_s=5e-6, comm_latency_s=LAT_S,
                           link_gbs=LINK_GBS)
        rep = adx.predict_async(plan, cm, rb)
        row = dict(N=N, S=S, w=w, partition=kind, segment_ms=[c * 1e3 for c in seg_cost],
                   max_round_exchange_MB=max(rb) / 1e6 if rb else 0.0, predicted_ms=rep.async_total_s * 1e3,
                   sequential_ms=rep.sequential_total_s * 1e3, speedup=rep.speedup, comm_ratio=rep.comm_ratio)
        res["runs"].append(row)
        print(json.dumps(row), flush=True)
json.dump(res, open(sys.argv[2] if len(sys.argv) > 2 else "predicted_scaling.json", "w"), indent=1)
