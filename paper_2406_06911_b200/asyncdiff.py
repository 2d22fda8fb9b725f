"""Reference-facing API of the B200 AsyncDiff engine.

Mirrors the reference's C++ pipeline API (proj/include/asyncdiff/*.hpp) name
for name, with the same argument meaning and error classes (see _lib.py):
build_schedule, ddim_step, sequential_denoise, build_toy_denoiser,
make_denoiser_shell, eval_full, eval_segment, partition_balanced,
crossing_links, plan_async, validate_plan, plan_counts, shift_embeddings,
render_plan, run_serial, run_parallel, inject_delay, compare_trajectories.

Every numeric call goes through the C ABI of libasyncdiff_b200.so (hand-written
sm_100a kernels + C++ executor); there is no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from ._lib import (AdxError, AdxRuntimeError, CudaError, DomainError, InvalidArgument, LogicError, OutOfRange,
                   adx_plan_counts_t, adx_run_options, adx_run_stats, check, lib)

__all__ = [
    "AdxError", "InvalidArgument", "OutOfRange", "DomainError", "AdxRuntimeError", "LogicError", "CudaError",
    "NoiseSchedule", "Latent", "Trajectory", "build_schedule", "ddim_step", "sequential_denoise",
    "LayeredDenoiser", "Stage", "build_toy_denoiser", "make_denoiser_shell", "sinusoid", "eval_full",
    "HiddenBundle", "eval_segment", "Partition", "partition_balanced", "crossing_links", "InputRef", "Eval",
    "Round", "ExecutionPlan", "plan_async", "validate_plan", "PlanCounts", "plan_counts", "shift_embeddings",
    "render_plan", "RunOptions", "RunStats", "InstrumentedDenoiser", "inject_delay", "run_serial",
    "run_parallel", "DivergenceReport", "compare_trajectories", "kWarmupRound", "set_default_precision",
    "PRECISIONS", "random_normals", "Session", "time_model_pass", "profile_model_pass", "stage_times", "partition_by_cost",
    "RankSession", "nccl_unique_id", "save_checkpoint",
    "load_checkpoint", "plan_to_json", "plan_from_json", "CostModel", "LatencyReport", "predict_sequential",
    "predict_async", "CostComparison", "calibrate_and_compare", "round_exchange_bytes", "SimilarityProfile",
    "similarity_profile", "warmup_sweep", "build_unet_denoiser", "unet_stage_info", "unet_stage_params", "unet_context",
]

PRECISIONS = {"f64": 0, "f32": 1, "bf16": 2}
_default_precision = "f64"
_default_devices: Tuple[int, ...] = (0,)
kWarmupRound = -1


def set_default_precision(p: str) -> None:
    global _default_precision
    if p not in PRECISIONS:
        raise InvalidArgument(f"unknown precision {p!r}")
    _default_precision = p


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------ diffusion core
@dataclass
class Latent:
    """diffusion.hpp:14-17"""
    values: np.ndarray
    timestep: int = 0


@dataclass
class NoiseSchedule:
    """diffusion.hpp:26-34 (timesteps are 1-based)"""
    T: int
    betas: np.ndarray
    alphas: np.ndarray
    alpha_bars: np.ndarray

    def _chk(self, t: int, lo: int, name: str) -> None:
        if t < lo or t > self.T:
            raise OutOfRange(f"{name}: t={t} outside [{lo}, {self.T}]")

    def beta(self, t: int) -> float:
        self._chk(t, 1, "beta")
        return float(self.betas[t - 1])

    def alpha(self, t: int) -> float:
        self._chk(t, 1, "alpha")
        return float(self.alphas[t - 1])

    def alpha_bar(self, t: int) -> float:
        self._chk(t, 0, "alpha_bar")
        return float(self.alpha_bars[t])


def random_normals(seed: int, n: int) -> np.ndarray:
    """n standard normals from the library's Rng(seed) (the reference's draw_x_T,
    experiment.cpp:131-136, with the seed already mixed)"""
    out = np.empty(n, np.float64)
    check(lib().adx_random_normals(C.c_uint64(seed), n, _dp(out)))
    return out


def build_schedule(T: int, beta_start: float, beta_end: float, kind: str = "linear") -> NoiseSchedule:
    """diffusion.hpp:36-37 / diffusion.cpp:39-77"""
    k = {"linear": 0, "scaled-linear": 1}.get(kind)
    if k is None:
        raise InvalidArgument(f"unknown schedule kind: {kind}")
    n = max(T, 1)
    b, a, ab = np.zeros(n), np.zeros(n), np.zeros(n + 1)
    check(lib().adx_build_schedule(T, beta_start, beta_end, k, _dp(b), _dp(a), _dp(ab)))
    return NoiseSchedule(T, b, a, ab)


def ddim_step(x_t: Latent, eps, t: int, schedule: NoiseSchedule, precision: Optional[str] = None,
              device: int = 0) -> Latent:
    """diffusion.hpp:50-51 / diffusion.cpp:95-116, evaluated by the sm_100a DDIM kernel."""
    x = _f64(x_t.values)
    e = _f64(eps)
    if e.size != x.size:
        raise InvalidArgument("predict_x0: eps dimension mismatch")
    ab = _f64(schedule.alpha_bars)
    out = np.zeros_like(x)
    check(lib().adx_ddim_step(device, PRECISIONS[precision or _default_precision], _dp(x), _dp(e), x.size, t,
                              _dp(ab), schedule.T, _dp(out)))
    return Latent(out, t - 1)


@dataclass
class Trajectory:
    """diffusion.hpp:54-61"""
    latents: List[Latent] = field(default_factory=list)
    eps_used: List[np.ndarray] = field(default_factory=list)
    timestamps_s: List[float] = field(default_factory=list)

    def steps(self) -> int:
        return len(self.eps_used)

    def final_latent(self) -> Latent:
        return self.latents[-1]

    def latent_matrix(self) -> np.ndarray:
        return np.stack([l.values for l in self.latents])


def _traj_from(lat: np.ndarray, eps: np.ndarray, T: int) -> Trajectory:
    tr = Trajectory()
    for k in range(lat.shape[0]):
        tr.latents.append(Latent(lat[k].copy(), T - k))
    for k in range(eps.shape[0]):
        tr.eps_used.append(eps[k].copy())
    return tr


# ---------------------------------------------------------------- denoiser
_T_IDS = {"proj": 0, "w1": 1, "b1": 2, "time_in": 3, "w2": 4, "b2": 5}


class Stage:
    """denoiser.hpp:29-43 view; tensors are row-major fp64 numpy views into the model."""

    def __init__(self, model: "LayeredDenoiser", index: int):
        self._m, self.index = model, index

    def _t(self, name: str) -> np.ndarray:
        return self._m._tensor(self.index, _T_IDS[name])

    w1 = property(lambda s: s._t("w1"))
    b1 = property(lambda s: s._t("b1").reshape(-1))
    time_in = property(lambda s: s._t("time_in"))
    w2 = property(lambda s: s._t("w2"))
    b2 = property(lambda s: s._t("b2").reshape(-1))

    def _shape(self):
        i, h, o, m = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        check(lib().adx_model_stage_shape(self._m._h, self.index, C.byref(i), C.byref(h), C.byref(o), C.byref(m)))
        return i.value, h.value, o.value, m.value

    def in_width(self) -> int:
        return self._shape()[0]

    def hidden_width(self) -> int:
        return self._shape()[1]

    def out_width(self) -> int:
        return self._shape()[2]

    @property
    def cost_macs(self) -> int:
        return self._shape()[3]

    @cost_macs.setter
    def cost_macs(self, v: int) -> None:
        check(lib().adx_model_set_stage_macs(self._m._h, self.index, int(v)))


class LayeredDenoiser:
    """denoiser.hpp:47-63 -- host model (fp64) behind an adx_model handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self.version = 0
        self._engines: Dict[tuple, "_Engine"] = {}
        L, E, nl = C.c_int(), C.c_int(), C.c_int()
        check(lib().adx_model_info(self._h, C.byref(L), C.byref(E), C.byref(nl)))
        self._L, self._E = L.value, E.value
        self._finalizer = weakref.finalize(self, lib().adx_model_destroy, self._h)

    def num_stages(self) -> int:
        return self._L

    @property
    def time_embed_dim(self) -> int:
        return self._E

    @property
    def widths(self) -> List[int]:
        w = np.zeros(self._L + 1, np.int32)
        check(lib().adx_model_widths(self._h, _ip(w)))
        return w.tolist()

    def data_dim(self) -> int:
        return self.widths[0]

    @property
    def skip_links(self) -> List[Tuple[int, int]]:
        L, E, nl = C.c_int(), C.c_int(), C.c_int()
        check(lib().adx_model_info(self._h, C.byref(L), C.byref(E), C.byref(nl)))
        buf = np.zeros(max(2 * nl.value, 2), np.int32)
        check(lib().adx_model_links(self._h, _ip(buf)))
        return [(int(buf[2 * k]), int(buf[2 * k + 1])) for k in range(nl.value)]

    def links_into(self, consumer: int):
        return [l for l in self.skip_links if l[1] == consumer]

    def links_out_of(self, producer: int):
        return [l for l in self.skip_links if l[0] == producer]

    @property
    def stages(self) -> List[Stage]:
        return [Stage(self, i) for i in range(1, self._L + 1)]

    def total_macs(self) -> int:
        return sum(s.cost_macs for s in self.stages)

    @property
    def proj(self) -> np.ndarray:
        return self._tensor(1, 0)

    def _tensor(self, stage: int, which: int) -> np.ndarray:
        p, r, c = C.POINTER(C.c_double)(), C.c_int(), C.c_int()
        check(lib().adx_model_tensor(self._h, stage, which, C.byref(p), C.byref(r), C.byref(c)))
        self.version += 1  # a view may be written through; engines re-upload lazily
        n = r.value * c.value
        if n == 0:
            return np.zeros((r.value, c.value))
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(r.value, c.value)

    def engine(self, precision: Optional[str] = None, devices: Sequence[int] = None) -> "_Engine":
        key = (precision or getattr(self, "default_precision", None) or _default_precision,
               tuple(devices or _default_devices))
        eng = self._engines.get(key)
        if eng is None or eng.version != self.version:
            eng = _Engine(self, key[0], key[1])
            self._engines[key] = eng
        return eng


def build_toy_denoiser(L: int, widths: Sequence[int], skip_spec: str = "unet-mirror", seed: int = 0,
                       time_embed_dim: int = 8) -> LayeredDenoiser:
    """denoiser.hpp:68-70 / denoiser.cpp:124-142 (bit-identical xavier init from Rng(seed))."""
    spec = {"none": 0, "unet-mirror": 1}.get(skip_spec)
    if spec is None:
        raise InvalidArgument(f"unknown skip spec: {skip_spec}")
    w = np.ascontiguousarray(widths, np.int32)
    h = C.c_void_p()
    check(lib().adx_model_build_toy(L, _ip(w), w.size, spec, C.c_uint64(seed), time_embed_dim, C.byref(h)))
    return LayeredDenoiser(h.value)


def make_denoiser_shell(L: int, widths: Sequence[int], skip_links: Sequence[Tuple[int, int]],
                        time_embed_dim: int) -> LayeredDenoiser:
    """denoiser.hpp:73-76 / denoiser.cpp:75-122"""
    w = np.ascontiguousarray(widths, np.int32)
    lk = np.ascontiguousarray(np.array(list(skip_links), np.int32).reshape(-1), np.int32)
    if lk.size == 0:
        lk = np.zeros(2, np.int32)
    h = C.c_void_p()
    check(lib().adx_model_shell(L, _ip(w), w.size, _ip(lk), len(skip_links), time_embed_dim, C.byref(h)))
    return LayeredDenoiser(h.value)


UNET_KINDS = {0: "conv_in", 1: "res", 2: "down", 3: "up", 4: "out", 5: "mid_res"}


def build_unet_denoiser(H: int = 96, W: int = 96, c_lat: int = 4, ch: Sequence[int] = (320, 640, 1280, 1280),
                        attn: Sequence[int] = (1, 1, 1, 0), n_res: int = 2, head_dim: int = 64, ctx_len: int = 77,
                        ctx_dim: int = 1024, temb_dim: int = 1280, groups: int = 32, mid_attn: int = 1,
                        seed: int = 0, cfg: bool = False, cfg_scale: float = 5.0, frames: int = 1,
                        motion: bool = False) -> LayeredDenoiser:
    """UNet-shaped denoiser behind the reference's stage contract (defaults: the
    SD-2.1 UNet topology at a 96x96x4 latent, random init).  Works with every
    partition / plan / run entry point.  Engine precision "bf16" (the default for
    this family): bf16 activations on the tcgen05 kernels, fp32 latent; "f32": fp32
    activations with split-bf16 tensor-core products (the north_star's rel-L2 <=
    1e-3 mode, checked against the fp64 oracle).

    attn[l] / mid_attn are SpatialTransformer depths (0: none).  cfg=True runs
    classifier-free guidance inside the denoiser: every stage carries a batch of 2
    (unconditional, conditional context) and the out stage returns
    eps_u + cfg_scale * (eps_c - eps_u).  SDXL-shaped example (BASELINE config 4):
    build_unet_denoiser(128, 128, ch=(320, 640, 1280), attn=(0, 2, 10), mid_attn=10,
    ctx_dim=2048, cfg=True).  frames > 1 with motion=True is the AnimateDiff-shaped video
    UNet (BASELINE config 5): the latent holds every frame and a temporal-attention motion
    module follows every resnet: build_unet_denoiser(64, 64, ctx_dim=768, frames=16,
    motion=True)."""
    from ._lib import adx_unet_spec
    s = adx_unet_spec()
    s.H, s.W, s.c_lat, s.n_levels = H, W, c_lat, len(ch)
    for i, (c, a) in enumerate(zip(ch, attn)):
        s.ch[i], s.attn[i] = c, int(a)
    s.n_res, s.head_dim, s.ctx_len, s.ctx_dim = n_res, head_dim, ctx_len, ctx_dim
    s.temb_dim, s.groups, s.mid_attn, s.seed = temb_dim, groups, int(mid_attn), seed
    s.cfg, s.cfg_scale = int(bool(cfg)), float(cfg_scale)
    s.frames, s.motion = int(frames), int(bool(motion))
    h = C.c_void_p()
    check(lib().adx_model_build_unet(C.byref(s), C.byref(h)))
    m = LayeredDenoiser(h.value)
    m.default_precision = "bf16"
    m.unet_spec = dict(H=H, W=W, c_lat=c_lat, ch=list(ch), attn=list(attn), n_res=n_res, head_dim=head_dim,
                       ctx_len=ctx_len, ctx_dim=ctx_dim, temb_dim=temb_dim, groups=groups, mid_attn=mid_attn,
                       seed=seed, cfg=int(bool(cfg)), cfg_scale=float(cfg_scale), frames=int(frames),
                       motion=int(bool(motion)))
    return m


def unet_stage_info(m: LayeredDenoiser, stage: int) -> dict:
    buf = np.zeros(7, np.int32)
    check(lib().adx_unet_stage_info(m._h, stage, _ip(buf)))
    k, cin, cskip, cout, H, W, at = buf.tolist()
    return dict(kind=UNET_KINDS[k], cin=cin, cskip=cskip, cout=cout, H=H, W=W, attn=at)


def unet_stage_params(m: LayeredDenoiser, stage: int) -> Dict[str, np.ndarray]:
    """fp32 parameters of one UNet stage (0 = shared time-embedding MLP)."""
    n, nd = C.c_int(), C.c_longlong()
    check(lib().adx_unet_stage_params(m._h, stage, None, 0, None, C.byref(n), None, 0, C.byref(nd)))
    names = C.create_string_buffer(64 * n.value + 64)
    shapes = np.zeros(2 * n.value + 2, np.int32)
    data = np.zeros(max(nd.value, 1), np.float32)
    check(lib().adx_unet_stage_params(m._h, stage, names, len(names), _ip(shapes), C.byref(n),
                                      data.ctypes.data_as(C.POINTER(C.c_float)), data.size, C.byref(nd)))
    out, pos = {}, 0
    for i, name in enumerate(names.value.decode().split("\n")):
        r, c = int(shapes[2 * i]), int(shapes[2 * i + 1])
        cnt = r * (c if c else 1)
        out[name] = data[pos:pos + cnt].reshape((r, c) if c else (r,)).copy()
        pos += cnt
    return out


def unet_context(m: LayeredDenoiser) -> np.ndarray:
    """(batch, ctx_len, ctx_dim) contexts: batch 1, or [uncond, cond] with CFG"""
    sp = m.unet_spec
    b = 2 if sp.get("cfg") else 1
    out = np.zeros(b * sp["ctx_len"] * sp["ctx_dim"], np.float32)
    check(lib().adx_unet_context(m._h, out.ctypes.data_as(C.POINTER(C.c_float))))
    return out.reshape(b, sp["ctx_len"], sp["ctx_dim"])


def sinusoid(t: int, dim: int) -> np.ndarray:
    out = np.zeros(dim)
    check(lib().adx_sinusoid(t, dim, _dp(out)))
    return out


class _Engine:
    """Device-resident copy of a model (weights uploaded once per GPU)."""

    def __init__(self, model: LayeredDenoiser, precision: str, devices: Tuple[int, ...]):
        self.version = model.version
        self.precision = precision
        self.devices = devices
        ords = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        check(lib().adx_engine_create(model._h, PRECISIONS[precision], _ip(ords), ords.size, C.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, lib().adx_engine_destroy, h)


def eval_full(m: LayeredDenoiser, x: Latent, t_embed: int, precision: Optional[str] = None) -> np.ndarray:
    """denoiser.hpp:79 / denoiser.cpp:222-233 on the GPU."""
    xv = _f64(x.values)
    d = m.data_dim()
    if xv.size != d:
        raise InvalidArgument(f"eval_full: latent dimension {xv.size} != model dim {d}")
    out = np.zeros(d)
    check(lib().adx_eval_full(m.engine(precision)._h, _dp(xv), t_embed, _dp(out)))
    return out


@dataclass
class HiddenBundle:
    """denoiser.hpp:81-86 -- the unit of inter-device exchange."""
    boundary: np.ndarray
    skips: Dict[Tuple[int, int], np.ndarray] = field(default_factory=dict)
    produced_by: int = 0
    produced_at: int = 0


def eval_segment(m: LayeredDenoiser, p: "Partition", seg: int, inp: Union[Latent, HiddenBundle],
                 skips_in: Optional[Dict[Tuple[int, int], np.ndarray]], t_embed: int,
                 precision: Optional[str] = None):
    """denoiser.hpp:91-95 / denoiser.cpp:235-267 on the GPU.  Returns a
    HiddenBundle for segments < N and the eps vector for segment N."""
    skips_in = skips_in or {}
    links = sorted(skips_in)
    lk = np.ascontiguousarray(np.array(links, np.int32).reshape(-1) if links else np.zeros(2), np.int32)
    vals = _f64(np.concatenate([_f64(skips_in[l]) for l in links]) if links else np.zeros(1))
    if isinstance(inp, Latent):
        data, is_lat, pb = _f64(inp.values), 1, 0
    else:
        data, is_lat, pb = _f64(inp.boundary), 0, inp.produced_by
    widths = m.widths
    cap = max(widths) + 8
    out = np.zeros(cap)
    ol, oe, nl = C.c_int(), C.c_int(), C.c_int()
    cap_links = max(1, len(m.skip_links))
    olinks = np.zeros(2 * cap_links, np.int32)
    cap_vals = max(1, sum(widths[a] for a, _ in m.skip_links))
    ovals = np.zeros(cap_vals)
    check(lib().adx_eval_segment(m.engine(precision)._h, p._h, seg, _dp(data), data.size, is_lat, pb, _ip(lk),
                                 _dp(vals), len(links), t_embed, _dp(out), cap, C.byref(ol), C.byref(oe),
                                 _ip(olinks), _dp(ovals), cap_links, cap_vals, C.byref(nl)))
    y = out[: ol.value].copy()
    if oe.value:
        return y
    b = HiddenBundle(boundary=y, produced_by=seg, produced_at=t_embed)
    pos = 0
    for k in range(nl.value):
        l = (int(olinks[2 * k]), int(olinks[2 * k + 1]))
        w = widths[l[0]]
        b.skips[l] = ovals[pos:pos + w].copy()
        pos += w
    return b


# --------------------------------------------------------------- partition
class Partition:
    """partition.hpp:19-37"""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._finalizer = weakref.finalize(self, lib().adx_partition_destroy, self._h)

    @classmethod
    def create(cls, segments: Sequence[Sequence[int]], device_of_segment=None, segment_macs=None,
               strategy: str = "sequential-balanced") -> "Partition":
        sizes = np.ascontiguousarray([len(s) for s in segments], np.int32)
        st = np.ascontiguousarray([x for s in segments for x in s] or [0], np.int32)
        dev = np.ascontiguousarray(device_of_segment if device_of_segment is not None else range(len(segments)),
                                   np.int32)
        macs = np.ascontiguousarray(segment_macs if segment_macs is not None else [0] * len(segments), np.int64)
        h = C.c_void_p()
        check(lib().adx_partition_create(len(segments), _ip(sizes), _ip(st), _ip(dev),
                                         macs.ctypes.data_as(C.POINTER(C.c_longlong)),
                                         {"sequential-balanced": 0, "first-last-grouped": 1}[strategy], C.byref(h)))
        return cls(h.value)

    def num_segments(self) -> int:
        return lib().adx_partition_num_segments(self._h)

    def _seg(self, n: int):
        buf = np.zeros(4096, np.int32)
        k, macs, dev = C.c_int(), C.c_longlong(), C.c_int()
        check(lib().adx_partition_segment(self._h, n, _ip(buf), buf.size, C.byref(k), C.byref(macs), C.byref(dev)))
        return buf[: k.value].tolist(), macs.value, dev.value

    @property
    def segments(self) -> List[List[int]]:
        return [self._seg(n)[0] for n in range(1, self.num_segments() + 1)]

    @property
    def segment_macs(self) -> List[int]:
        return [self._seg(n)[1] for n in range(1, self.num_segments() + 1)]

    @property
    def device_of_segment(self) -> List[int]:
        return [self._seg(n)[2] for n in range(1, self.num_segments() + 1)]

    @property
    def strategy(self) -> str:
        return ["sequential-balanced", "first-last-grouped"][lib().adx_partition_strategy(self._h)]

    def num_stages(self) -> int:
        return sum(len(s) for s in self.segments)

    def segment_of_stage(self, stage: int) -> int:
        s = C.c_int()
        check(lib().adx_partition_segment_of_stage(self._h, stage, C.byref(s)))
        return s.value

    def contiguous(self) -> bool:
        return bool(lib().adx_partition_contiguous(self._h))

    def max_segment_macs(self) -> int:
        return max(self.segment_macs)

    def total_macs(self) -> int:
        return sum(self.segment_macs)

    def validate(self, m: LayeredDenoiser) -> None:
        check(lib().adx_partition_validate(self._h, m._h))


def partition_balanced(m: LayeredDenoiser, N: int, strategy: str = "sequential-balanced") -> Partition:
    """partition.hpp:39-40 / partition.cpp:95-198 (exact min-max DP, ties to the smallest cut)."""
    st = {"sequential-balanced": 0, "first-last-grouped": 1}.get(strategy)
    if st is None:
        raise InvalidArgument(f"unknown partition strategy: {strategy}")
    h = C.c_void_p()
    check(lib().adx_partition_balanced(m._h, N, st, C.byref(h)))
    return Partition(h.value)


def partition_by_cost(m: LayeredDenoiser, N: int, stage_cost: Sequence[float]) -> Partition:
    """Extension of partition_balanced: the same exact min-max DP (ties to the smallest
    cut) over measured per-stage costs (e.g. stage_times) instead of MACs."""
    c = _f64(list(stage_cost))
    if c.size != m.num_stages():
        raise InvalidArgument(f"partition_by_cost: need one cost per stage ({m.num_stages()})")
    h = C.c_void_p()
    check(lib().adx_partition_by_cost(m._h, N, _dp(c), C.byref(h)))
    return Partition(h.value)


def crossing_links(m: LayeredDenoiser, p: Partition) -> List[Tuple[int, int]]:
    """partition.hpp:43-44"""
    buf = np.zeros(2 * max(1, len(m.skip_links)), np.int32)
    n = C.c_int()
    check(lib().adx_crossing_links(m._h, p._h, _ip(buf), buf.size // 2, C.byref(n)))
    return [(int(buf[2 * k]), int(buf[2 * k + 1])) for k in range(n.value)]


# -------------------------------------------------------------------- plan
@dataclass
class InputRef:
    """plan.hpp:15-25 (kind 'latent' = CurrentLatent, 'cached' = Cached)"""
    kind: str = "latent"
    producer_segment: int = 0
    producer_round: int = kWarmupRound

    @staticmethod
    def current_latent() -> "InputRef":
        return InputRef()

    @staticmethod
    def cached(segment: int, round_: int) -> "InputRef":
        return InputRef("cached", segment, round_)


@dataclass
class Eval:
    """plan.hpp:27-33"""
    segment: int = 0
    device: int = 0
    embed_t: int = 0
    input: InputRef = field(default_factory=InputRef)
    emits_eps_for: Optional[int] = None


@dataclass
class Round:
    """plan.hpp:35-40"""
    index: int = 0
    evals: List[Eval] = field(default_factory=list)
    sampler_steps: List[int] = field(default_factory=list)
    broadcast: bool = True


@dataclass
class ExecutionPlan:
    """plan.hpp:42-50"""
    T: int = 0
    w: int = 0
    N: int = 0
    S: int = 1
    D: int = 0
    time_shift: bool = False
    warmup_steps: List[int] = field(default_factory=list)
    rounds: List[Round] = field(default_factory=list)

    def to_flat(self) -> np.ndarray:
        f = [self.T, self.w, self.N, self.S, self.D, int(self.time_shift), len(self.rounds), *self.warmup_steps]
        for r in self.rounds:
            f += [r.index, int(r.broadcast), len(r.sampler_steps), *r.sampler_steps, len(r.evals)]
            for e in r.evals:
                f += [e.segment, e.device, e.embed_t, 0 if e.input.kind == "latent" else 1,
                      e.input.producer_segment, e.input.producer_round,
                      -1 if e.emits_eps_for is None else e.emits_eps_for]
        return np.ascontiguousarray(f, np.int32)

    @classmethod
    def from_flat(cls, f) -> "ExecutionPlan":
        f = [int(v) for v in f]
        p = cls(T=f[0], w=f[1], N=f[2], S=f[3], D=f[4], time_shift=bool(f[5]))
        nr = f[6]
        pos = 7
        p.warmup_steps = f[pos:pos + p.w]
        pos += p.w
        for _ in range(nr):
            r = Round(index=f[pos], broadcast=bool(f[pos + 1]))
            ns = f[pos + 2]
            r.sampler_steps = f[pos + 3:pos + 3 + ns]
            pos += 3 + ns
            ne = f[pos]
            pos += 1
            for _ in range(ne):
                seg, dev, emb, kind, ps, pr, em = f[pos:pos + 7]
                pos += 7
                r.evals.append(Eval(seg, dev, emb, InputRef("latent" if kind == 0 else "cached", ps, pr),
                                    None if em < 0 else em))
            p.rounds.append(r)
        return p

    def _handle(self):
        return _PlanHandle(self.to_flat())


class _PlanHandle:
    def __init__(self, flat: np.ndarray):
        h = C.c_void_p()
        check(lib().adx_plan_from_flat(_ip(flat), flat.size, C.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, lib().adx_plan_destroy, h)


def plan_async(T: int, w: int, N: int, S: int = 1, time_shift: bool = False) -> ExecutionPlan:
    """plan.hpp:53 / plan.cpp:17-97 (bit-exact schedule)."""
    h = C.c_void_p()
    check(lib().adx_plan_async(T, w, N, S, int(time_shift), C.byref(h)))
    try:
        cap = 64 + max(T, 1) * (8 + 7 * (N + 2))
        buf = np.zeros(cap, np.int32)
        n = C.c_int()
        check(lib().adx_plan_to_flat(h, _ip(buf), cap, C.byref(n)))
    finally:
        lib().adx_plan_destroy(h)
    return ExecutionPlan.from_flat(buf[: n.value])


def validate_plan(plan: ExecutionPlan) -> List[str]:
    """plan.hpp:56 / plan.cpp:99-200"""
    ph = plan._handle()
    buf = C.create_string_buffer(1 << 16)
    n = C.c_int()
    check(lib().adx_plan_validate(ph._h, buf, len(buf), C.byref(n)))
    return buf.value.decode().split("\n") if n.value else []


@dataclass
class PlanCounts:
    """plan.hpp:58-66"""
    broadcasts_paper_convention: int
    broadcasts_strictly_needed: int
    device_count: int
    evals_per_segment: List[int]
    per_device_macs: List[int]
    max_device_macs: int
    sequential_total_macs: int


def plan_counts(plan: ExecutionPlan, partition: Partition) -> PlanCounts:
    """plan.cpp:202-232"""
    ph = plan._handle()
    c = adx_plan_counts_t()
    eps = np.zeros(max(plan.N, 1), np.int64)
    dev = np.zeros(max(plan.D, 1), np.int64)
    check(lib().adx_plan_counts(ph._h, partition._h, C.byref(c), eps.ctypes.data_as(C.POINTER(C.c_longlong)),
                                dev.ctypes.data_as(C.POINTER(C.c_longlong))))
    return PlanCounts(c.broadcasts_paper_convention, c.broadcasts_strictly_needed, c.device_count,
                      eps[: plan.N].tolist(), dev[: plan.D].tolist(), c.max_device_macs, c.sequential_total_macs)


def shift_embeddings(timesteps: Sequence[int], w: int) -> List[int]:
    """plan.cpp:234-244"""
    ts = np.ascontiguousarray(list(timesteps) or [0], np.int32)
    out = np.zeros_like(ts)
    check(lib().adx_shift_embeddings(_ip(ts), len(timesteps), w, _ip(out)))
    return out[: len(timesteps)].tolist()


def render_plan(plan: ExecutionPlan) -> str:
    """plan.cpp:246-286"""
    ph = plan._handle()
    n = C.c_int()
    check(lib().adx_render_plan(ph._h, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().adx_render_plan(ph._h, buf, len(buf), C.byref(n)))
    return buf.value.decode()


# ---------------------------------------------------------------- executor
@dataclass
class RunOptions:
    """executor.hpp:44-49"""
    round_timeout_s: float = 30.0
    jitter_seed: int = 0
    max_jitter_s: float = 0.0
    use_graph: bool = True
    instrument: bool = False


@dataclass
class RunStats:
    """executor.hpp:30-42"""
    round_wall_s: List[float] = field(default_factory=list)
    round_comm_s: List[float] = field(default_factory=list)
    device_busy_s: List[float] = field(default_factory=list)
    device_evals: List[int] = field(default_factory=list)
    store_entries_per_round: List[int] = field(default_factory=list)
    broadcast_count: int = 0
    warmup_wall_s: float = 0.0
    total_wall_s: float = 0.0

    def comm_total_s(self) -> float:
        return float(sum(self.round_comm_s))

    def comm_ratio(self) -> float:
        return self.comm_total_s() / self.total_wall_s if self.total_wall_s > 0 else 0.0


@dataclass
class InstrumentedDenoiser:
    """executor.hpp:53-59 -- per-segment GPU sleep before every segment eval."""
    model: LayeredDenoiser
    segment_delay_s: List[float] = field(default_factory=list)


def inject_delay(m: LayeredDenoiser, per_segment_delay_s: Sequence[float]) -> InstrumentedDenoiser:
    """executor.cpp:74-80"""
    if any(d < 0.0 for d in per_segment_delay_s):
        raise InvalidArgument("inject_delay: delays must be >= 0")
    return InstrumentedDenoiser(m, list(per_segment_delay_s))


def _opts(opts: Optional[RunOptions], delays: Sequence[float]):
    o = adx_run_options()
    lib().adx_run_options_default(C.byref(o))
    keep = None
    if opts is not None:
        o.round_timeout_s = opts.round_timeout_s
        o.jitter_seed = opts.jitter_seed
        o.max_jitter_s = opts.max_jitter_s
        o.use_graph = int(opts.use_graph)
        o.instrument = int(opts.instrument)
    if delays:
        keep = _f64(delays)
        o.segment_delay_s = _dp(keep)
        o.n_delays = keep.size
    return o, keep


def _run(mode: int, plan: ExecutionPlan, m, partition: Partition, x_T: Latent, schedule: NoiseSchedule,
         workers: int, opts: Optional[RunOptions], precision: Optional[str], devices: Optional[Sequence[int]] = None):
    model, delays = (m.model, m.segment_delay_s) if isinstance(m, InstrumentedDenoiser) else (m, [])
    eng = model.engine(precision, devices)
    x = _f64(x_T.values)
    if x_T.timestep != plan.T:
        raise InvalidArgument("run: x_T.timestep != T")
    if x.size != model.data_dim():
        raise InvalidArgument("run: x_T dimension != model data dim")
    T = schedule.T
    ab = _f64(schedule.alpha_bars)
    o, keep = _opts(opts, delays)
    ph = plan._handle()
    nr = len(plan.rounds)
    D = max(plan.D, 1)
    st = adx_run_stats()
    rw, rc_, busy = np.zeros(max(nr, 1)), np.zeros(max(nr, 1)), np.zeros(D)
    ev = np.zeros(D, np.int64)
    se = np.zeros(max(nr, 1), np.int32)
    st.round_wall_s, st.round_comm_s, st.device_busy_s = _dp(rw), _dp(rc_), _dp(busy)
    st.device_evals = ev.ctypes.data_as(C.POINTER(C.c_longlong))
    st.store_entries_per_round = _ip(se)
    lat = np.zeros((T + 1, model.data_dim()))
    eps = np.zeros((T, model.data_dim()))
    if mode == 0:
        check(lib().adx_run_serial(eng._h, ph._h, partition._h, _dp(x), _dp(ab), T, C.byref(o), _dp(lat), _dp(eps),
                                   C.byref(st)))
    else:
        check(lib().adx_run_parallel(eng._h, ph._h, partition._h, _dp(x), _dp(ab), T, workers, C.byref(o),
                                     _dp(lat), _dp(eps), C.byref(st)))
    del keep
    stats = RunStats(rw[:nr].tolist(), rc_[:nr].tolist(), busy.tolist(), ev.tolist(), se[:nr].tolist(),
                     st.broadcast_count, st.warmup_wall_s, st.total_wall_s)
    return _traj_from(lat, eps, T), stats


def run_serial(plan: ExecutionPlan, m, partition: Partition, x_T: Latent, schedule: NoiseSchedule,
               opts: Optional[RunOptions] = None, precision: Optional[str] = None,
               devices: Optional[Sequence[int]] = None):
    """executor.hpp:63-75 -- all evals on one GPU stream in plan order, snapshot semantics."""
    return _run(0, plan, m, partition, x_T, schedule, 1, opts, precision, devices)


def run_parallel(plan: ExecutionPlan, m, partition: Partition, x_T: Latent, schedule: NoiseSchedule, workers: int,
                 opts: Optional[RunOptions] = None, precision: Optional[str] = None,
                 devices: Optional[Sequence[int]] = None):
    """executor.hpp:79-93 -- one CUDA stream pair per (virtual) device, event-ordered
    exchange; bit-identical to run_serial.  `devices` lists the CUDA ordinals
    virtual device v maps to (v % len(devices))."""
    return _run(1, plan, m, partition, x_T, schedule, workers, opts, precision, devices)


def sequential_denoise(eps_fn: Union[LayeredDenoiser, Callable[[Latent, int], np.ndarray]], x_T: Latent,
                       schedule: NoiseSchedule, precision: Optional[str] = None) -> Trajectory:
    """diffusion.hpp:66-67 / diffusion.cpp:118-142.  With a LayeredDenoiser the
    whole loop (eval_full + DDIM per step) runs on the GPU as one CUDA graph; a
    Python EpsFn is called per step with the DDIM update on the GPU."""
    if x_T.timestep != schedule.T:
        raise InvalidArgument(f"sequential_denoise: x_T.timestep={x_T.timestep} != T={schedule.T}")
    T = schedule.T
    if isinstance(eps_fn, LayeredDenoiser):
        x = _f64(x_T.values)
        lat = np.zeros((T + 1, x.size))
        eps = np.zeros((T, x.size))
        ab = _f64(schedule.alpha_bars)
        check(lib().adx_sequential_denoise(eps_fn.engine(precision)._h, _dp(x), _dp(ab), T, _dp(lat), _dp(eps)))
        return _traj_from(lat, eps, T)
    traj = Trajectory(latents=[Latent(_f64(x_T.values).copy(), T)])
    x = traj.latents[0]
    for t in range(T, 0, -1):
        try:
            e = _f64(eps_fn(x, t))
        except Exception as exc:  # diffusion.cpp:131-135
            raise AdxRuntimeError(f"sequential_denoise: eps_fn failed at t={t}: {exc}") from exc
        x = ddim_step(x, e, t, schedule, precision)
        traj.eps_used.append(e)
        traj.latents.append(x)
    return traj


# ------------------------------------------------------ §8(f): I/O, cost model, quality
def save_checkpoint(base: str, m: LayeredDenoiser) -> None:
    """serialize.hpp:35 -- <base>.json + <base>.bin (row-major LE fp64)."""
    check(lib().adx_model_save_checkpoint(m._h, base.encode()))


def load_checkpoint(base: str) -> LayeredDenoiser:
    """serialize.hpp:36 -- loads a reference-format checkpoint (e.g. cmd_train output)."""
    h = C.c_void_p()
    check(lib().adx_model_load_checkpoint(base.encode(), C.byref(h)))
    return LayeredDenoiser(h.value)


def plan_to_json(plan: ExecutionPlan) -> str:
    """serialize.cpp:109-133"""
    ph = plan._handle()
    n = C.c_int()
    check(lib().adx_plan_to_json(ph._h, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().adx_plan_to_json(ph._h, buf, len(buf), C.byref(n)))
    return buf.value.decode()


def plan_from_json(text: str) -> ExecutionPlan:
    """serialize.cpp:135-159"""
    h = C.c_void_p()
    check(lib().adx_plan_from_json(text.encode(), C.byref(h)))
    try:
        buf = np.zeros(1 << 20, np.int32)
        n = C.c_int()
        check(lib().adx_plan_to_flat(h, _ip(buf), buf.size, C.byref(n)))
    finally:
        lib().adx_plan_destroy(h)
    return ExecutionPlan.from_flat(buf[: n.value])


@dataclass
class CostModel:
    """costsim.hpp:13-19 (+ bytes-aware comm: comm_latency_s + bytes / link_gbs)"""
    segment_cost_s: List[float]
    comm_cost_s: float = 0.0
    sampler_cost_s: float = 0.0
    comm_latency_s: float = 0.0
    link_gbs: float = 0.0

    def total_segment_cost_s(self) -> float:
        return float(sum(self.segment_cost_s))


@dataclass
class LatencyReport:
    """costsim.hpp:21-34"""
    sequential_total_s: float
    async_total_s: float
    warmup_s: float
    round_compute_s: List[float]
    round_comm_s: List[float]
    comm_total_s: float
    speedup: float
    comm_ratio: float
    approx_step_s: float
    approx_total_s: float


def predict_sequential(T: int, cm: CostModel) -> float:
    """costsim.cpp:14-16"""
    return T * (cm.total_segment_cost_s() + cm.sampler_cost_s)


def predict_async(plan: ExecutionPlan, cm: CostModel, round_bytes: Optional[Sequence[int]] = None) -> LatencyReport:
    """costsim.cpp:18-50; with round_bytes the comm term is bytes-aware."""
    from ._lib import adx_latency_report
    ph = plan._handle()
    seg = _f64(cm.segment_cost_s if cm.segment_cost_s else [0.0])
    nr = max(len(plan.rounds), 1)
    rc, rm = np.zeros(nr), np.zeros(nr)
    rb = None if round_bytes is None else np.ascontiguousarray(round_bytes, np.int64)
    out = adx_latency_report()
    check(lib().adx_predict_async(ph._h, _dp(seg), len(cm.segment_cost_s), cm.comm_cost_s, cm.sampler_cost_s,
                                  cm.comm_latency_s, cm.link_gbs,
                                  None if rb is None else rb.ctypes.data_as(C.POINTER(C.c_longlong)),
                                  C.byref(out), _dp(rc), _dp(rm)))
    n = len(plan.rounds)
    return LatencyReport(out.sequential_total_s, out.async_total_s, out.warmup_s, rc[:n].tolist(), rm[:n].tolist(),
                         out.comm_total_s, out.speedup, out.comm_ratio, out.approx_step_s, out.approx_total_s)


@dataclass
class CostComparison:
    """costsim.hpp:36-44"""
    predicted_total_s: float
    measured_total_s: float
    rel_error_total: float
    predicted_comm_ratio: float
    measured_comm_ratio: float
    rel_error_comm_ratio: float
    calibrated_comm_cost_s: float


def calibrate_and_compare(plan: ExecutionPlan, delays_s: Sequence[float], measured: "RunStats") -> CostComparison:
    """costsim.cpp:52-79"""
    from ._lib import adx_cost_comparison
    ph = plan._handle()
    d = _f64(list(delays_s) or [0.0])
    rc = _f64(list(measured.round_comm_s) or [0.0])
    out = adx_cost_comparison()
    check(lib().adx_calibrate_and_compare(ph._h, _dp(d), len(delays_s), _dp(rc), len(measured.round_comm_s),
                                          measured.broadcast_count, measured.total_wall_s, C.byref(out)))
    return CostComparison(out.predicted_total_s, out.measured_total_s, out.rel_error_total, out.predicted_comm_ratio,
                          out.measured_comm_ratio, out.rel_error_comm_ratio, out.calibrated_comm_cost_s)


def round_exchange_bytes(plan: ExecutionPlan, partition: Partition, m: LayeredDenoiser,
                         precision: Optional[str] = None) -> List[int]:
    """Bytes crossing devices in each round (boundary + crossing skips + eps)."""
    ph = plan._handle()
    out = np.zeros(max(len(plan.rounds), 1), np.int64)
    prec = precision or getattr(m, "default_precision", None) or _default_precision
    check(lib().adx_round_exchange_bytes(ph._h, partition._h, m._h, PRECISIONS[prec],
                                         out.ctypes.data_as(C.POINTER(C.c_longlong))))
    return out[: len(plan.rounds)].tolist()


@dataclass
class SimilarityProfile:
    """metrics.hpp:23-29"""
    pair_t: List[int]
    cosine: List[List[float]]
    rel_l2: List[List[float]]

    def median_cosine(self) -> float:
        allv = sorted(v for row in self.cosine for v in row)
        if not allv:
            return 1.0
        n = len(allv)
        return allv[n // 2] if n % 2 else 0.5 * (allv[n // 2 - 1] + allv[n // 2])


def similarity_profile(m: LayeredDenoiser, p: Partition, trajectory: Trajectory, schedule: NoiseSchedule,
                       precision: Optional[str] = None) -> SimilarityProfile:
    """metrics.cpp:73-101: boundary activations of segments 1..N-1 at every
    latent of a trajectory (fresh chaining on the GPU), cosine / rel-L2 between
    adjacent steps -- the hidden-state similarity AsyncDiff relies on."""
    N = p.num_segments()
    prof = SimilarityProfile([], [[] for _ in range(max(0, N - 1))], [[] for _ in range(max(0, N - 1))])
    if len(trajectory.latents) < 3 or N < 2:
        return prof
    per_step, ts = [], []
    for x in trajectory.latents:
        if x.timestep < 1:
            break
        skips, out = {}, []
        so = eval_segment(m, p, 1, x, skips, x.timestep, precision)
        for seg in range(2, N + 1):
            out.append(so.boundary)
            skips.update(so.skips)
            so = eval_segment(m, p, seg, so, skips, x.timestep, precision)
        per_step.append(out)
        ts.append(x.timestep)

    def cosine(a, b):
        na, nb = np.linalg.norm(a), np.linalg.norm(b)
        if na == 0.0 or nb == 0.0:
            return 1.0 if np.linalg.norm(a - b) == 0.0 else 0.0
        return float(np.dot(a, b) / (na * nb))

    def rel_l2(a, b):
        den = max(np.linalg.norm(a), np.linalg.norm(b))
        return 0.0 if den == 0.0 else float(np.linalg.norm(a - b) / den)

    for i in range(len(per_step) - 1):
        prof.pair_t.append(ts[i])
        for b in range(N - 1):
            prof.cosine[b].append(cosine(per_step[i][b], per_step[i + 1][b]))
            prof.rel_l2[b].append(rel_l2(per_step[i][b], per_step[i + 1][b]))
    return prof


class Session:
    """One compiled run (plan, partition, placement) kept resident on the GPU:
    device buffers, streams and one CUDA graph spanning every device.  The
    repeated-run API used by bench.py (adx_session_* in the C ABI)."""

    MODES = {"serial": 0, "parallel": 1, "sequential": 2}

    def __init__(self, model: LayeredDenoiser, schedule: NoiseSchedule, mode: str = "parallel",
                 plan: Optional[ExecutionPlan] = None, partition: Optional[Partition] = None,
                 workers: Optional[int] = None, precision: Optional[str] = None,
                 devices: Optional[Sequence[int]] = None, opts: Optional[RunOptions] = None):
        self.model, self.schedule, self.mode = model, schedule, mode
        eng = model.engine(precision, devices)
        self._eng = eng
        ab = _f64(schedule.alpha_bars)
        self._ab = ab
        ph = plan._handle() if plan is not None else None
        self._ph = ph
        o, self._keep = _opts(opts, [])
        h = C.c_void_p()
        check(lib().adx_session_create(eng._h, ph._h if ph else None, partition._h if partition else None, _dp(ab),
                                       schedule.T, self.MODES[mode], workers if workers is not None else
                                       (plan.D if plan is not None else 1), C.byref(o), C.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, lib().adx_session_destroy, h)
        self.d = model.data_dim()

    def run(self, x_T: Latent) -> Trajectory:
        """host x_T -> host trajectory (H2D + graph + D2H, blocking)."""
        T = self.schedule.T
        x = _f64(x_T.values)
        lat = np.zeros((T + 1, self.d))
        eps = np.zeros((T, self.d))
        check(lib().adx_session_run(self._h, _dp(x), _dp(lat), _dp(eps), None))
        return _traj_from(lat, eps, T)

    def run_into(self, x: np.ndarray, lat: np.ndarray, eps: np.ndarray) -> None:
        check(lib().adx_session_run(self._h, _dp(x), _dp(lat), _dp(eps), None))

    def upload(self, x_T: Latent) -> None:
        self._x = _f64(x_T.values)
        check(lib().adx_session_upload(self._h, _dp(self._x)))

    def time(self, iters: int) -> float:
        """device-resident back-to-back runs; mean ms per run (CUDA events)."""
        ms = C.c_double()
        check(lib().adx_session_time(self._h, iters, C.byref(ms)))
        return ms.value

    def kernel_count(self) -> int:
        n = C.c_int()
        check(lib().adx_session_kernel_count(self._h, C.byref(n)))
        return n.value

    def weight_bytes(self) -> int:
        b = C.c_longlong()
        check(lib().adx_session_weight_bytes(self._h, C.byref(b)))
        return b.value

    def download(self) -> Trajectory:
        T = self.schedule.T
        lat = np.zeros((T + 1, self.d))
        eps = np.zeros((T, self.d))
        check(lib().adx_session_download(self._h, _dp(lat), _dp(eps)))
        return _traj_from(lat, eps, T)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().adx_nccl_unique_id(buf))
    return buf.raw


class RankSession:
    """One process per GPU (torchrun): this rank's part of the async loop,
    exchanging with its peers over NCCL p2p (rank.cu).  Collective: every rank
    0..plan.D-1 constructs it with the same nccl id and calls run()/time()."""

    def __init__(self, model: LayeredDenoiser, schedule: NoiseSchedule, plan: ExecutionPlan, partition: Partition,
                 rank: int, nccl_id: bytes, device: int, precision: Optional[str] = None):
        self.model, self.schedule, self.rank = model, schedule, rank
        eng = model.engine(precision, [device])
        self._eng = eng
        self._ab = _f64(schedule.alpha_bars)
        self._ph = plan._handle()
        o, _ = _opts(None, [])
        h = C.c_void_p()
        check(lib().adx_rank_session_create(eng._h, self._ph._h, partition._h, _dp(self._ab), schedule.T, rank,
                                            C.c_char_p(nccl_id), C.byref(o), C.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, lib().adx_rank_session_destroy, h)
        self.d = model.data_dim()

    def run_into(self, x: np.ndarray, lat: np.ndarray, eps: np.ndarray) -> None:
        check(lib().adx_rank_session_run(self._h, _dp(x), _dp(lat), _dp(eps)))

    def time(self, iters: int) -> float:
        ms = C.c_double()
        check(lib().adx_rank_session_time(self._h, iters, C.byref(ms)))
        return ms.value

    def kernel_count(self) -> int:
        n = C.c_int()
        check(lib().adx_rank_session_kernel_count(self._h, C.byref(n)))
        return n.value


def profile_model_pass(m: LayeredDenoiser, t_embed: int, precision: Optional[str] = None,
                       devices: Optional[Sequence[int]] = None) -> Dict[str, dict]:
    """Per tensor-core kernel family over one pass, every launch replayed in isolation from a CUDA
    graph: launches, device ms (CUDA
    events per launch) and algorithmic FLOPs."""
    out = np.zeros(9)
    check(lib().adx_engine_profile_pass(m.engine(precision, devices)._h, t_embed, _dp(out)))
    res = {k: dict(launches=int(out[3 * i]), ms=float(out[3 * i + 1]), flops=float(out[3 * i + 2]))
           for i, k in enumerate(("conv3x3", "gemm", "attention"))}
    n = C.c_int()
    check(lib().adx_profile_records(None, 0, C.byref(n)))
    rec = np.zeros(4 * max(n.value, 1))
    check(lib().adx_profile_records(_dp(rec), n.value, C.byref(n)))
    res["records"] = rec[:4 * n.value].reshape(-1, 4)  # (kind, flops, compulsory bytes, ms) per launch
    return res


def stage_times(m: LayeredDenoiser, t_embed: int, iters: int = 10, precision: Optional[str] = None,
                devices: Optional[Sequence[int]] = None) -> List[float]:
    """Device ms of every stage evaluated on its own (own CUDA graph, `iters` replays):
    the measured per-component costs for CostModel.segment_cost_s (costsim.hpp:13-19)."""
    out = np.zeros(m.num_stages())
    check(lib().adx_engine_stage_times(m.engine(precision, devices)._h, t_embed, iters, _dp(out)))
    return out.tolist()


def time_model_pass(m: LayeredDenoiser, t_embed: int, iters: int, precision: Optional[str] = None,
                    devices: Optional[Sequence[int]] = None):
    """(ms per full-model pass, weight bytes per pass, GEMV launches per pass)."""
    ms, b, n = C.c_double(), C.c_longlong(), C.c_int()
    check(lib().adx_engine_time_eval(m.engine(precision, devices)._h, t_embed, iters, C.byref(ms), C.byref(b),
                                     C.byref(n)))
    return ms.value, b.value, n.value


@dataclass
class DivergenceReport:
    """metrics.hpp"""
    per_step_mse: List[float]
    final_mse: float
    final_max_abs: float


def warmup_sweep(m: LayeredDenoiser, x_T: Latent, schedule: NoiseSchedule,
                 matrix: Sequence[Tuple[int, int, int]], precision: Optional[str] = None,
                 devices: Optional[Sequence[int]] = None) -> List[dict]:
    """The warm-up sweep of experiment.cpp:312-389 (cmd_sweep) on the GPU -- the paper's
    Table-2 analogue, quality of the async trajectory against the warm-up length.  The
    reference scores each cell against its Gaussian-mixture oracle (final MSE / NLL,
    out of scope here); this scores it against the sequential trajectory of the same model
    and x_T (the divergence of metrics.cpp:9-30).  For every (N, w, S) of `matrix`:
    MAC-balanced partition (partition.cpp:133), plan_async, the async run through
    run_serial (identical numerics to run_parallel on N GPUs), plan_counts; one row each
    with the sweep CSV's columns (experiment.cpp:368-383) plus the divergence."""
    seq = sequential_denoise(m, x_T, schedule, precision=precision)
    ref = seq.latents[-1].values
    rows = []
    for N, w, S in matrix:
        part = partition_balanced(m, N)
        plan = plan_async(schedule.T, w, N, S)
        traj, _ = run_serial(plan, m, part, x_T, schedule, precision=precision, devices=devices)
        rep = compare_trajectories(seq, traj)
        cnt = plan_counts(plan, part)
        fin = traj.latents[-1].values
        rows.append(dict(config=f"N{N}_w{w}_S{S}", N=N, w=w, S=S, per_device_macs=cnt.max_device_macs,
                         device_count=plan.D, broadcast_count=cnt.broadcasts_paper_convention,
                         final_mse=rep.final_mse, final_max_abs=rep.final_max_abs,
                         final_rel_l2=float(np.linalg.norm(fin - ref) / (np.linalg.norm(ref) + 1e-300))))
    return rows


def compare_trajectories(seq: Trajectory, async_traj: Trajectory) -> DivergenceReport:
    """metrics.cpp:9-30"""
    if len(seq.latents) != len(async_traj.latents):
        raise InvalidArgument(
            f"compare_trajectories: length mismatch ({len(seq.latents)} vs {len(async_traj.latents)})")
    a, b = seq.latent_matrix(), async_traj.latent_matrix()
    if a.shape != b.shape:
        raise InvalidArgument("compare_trajectories: dimension mismatch")
    per = np.zeros(a.shape[0])
    fm, mx = C.c_double(), C.c_double()
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    check(lib().adx_compare_trajectories(_dp(a), _dp(b), a.shape[0], a.shape[1], _dp(per), C.byref(fm),
                                         C.byref(mx)))
    return DivergenceReport(per.tolist(), fm.value, mx.value)
