"""Independent restatement of the UNet-shaped denoiser family's MODEL: topology,
stage costs, deterministic parameters and the synthetic cross-attention contexts.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke() and bench.py's CPU
legs).  Nothing here loads the product library: the random streams come from
the oracle's own MT19937-64 (oracle/adx_oracle.c, pinned to the reference's
rng.hpp:12-60 by tests/test_oracle_golden.py), and the stage list / parameter
order restate the builder's UNet definition (product side
paper_2406_06911_b200/csrc/unet.cpp build_unet_model / unet_stage_params).
tests/test_unet_model.py checks that these parameters equal the product's
adx_unet_stage_params bit-for-bit, so a bug in the product's model builder
(init, wiring, channel counts) shows up as a CPU test failure instead of being
shared by both sides of the parity tests.

The reference itself has no UNet; the conventions kept from it
are the reference's xavier scheme (denoiser.cpp:21-27: a = sqrt(6/(fan_in+fan_out)),
row-major uniform(-a, a) draws), one seeded Rng per unit (rng.hpp:55-60
mix_seed) and the stage / mirror-skip contract (denoiser.cpp:129-131, 150-192).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

from . import oracle as O

KINDS = {0: "conv_in", 1: "res", 2: "down", 3: "up", 4: "out", 5: "mid_res"}
CONV_IN, RES, DOWN, UP, OUT, MID_RES = range(6)


@dataclass
class UNetSpec:
    H: int = 96
    W: int = 96
    c_lat: int = 4
    ch: Tuple[int, ...] = (320, 640, 1280, 1280)
    attn: Tuple[int, ...] = (1, 1, 1, 0)
    n_res: int = 2
    head_dim: int = 64
    ctx_len: int = 77
    ctx_dim: int = 1024
    temb_dim: int = 1280
    groups: int = 32
    mid_attn: int = 1
    seed: int = 0
    cfg: bool = False
    cfg_scale: float = 5.0
    frames: int = 1
    motion: bool = False

    def batch(self) -> int:
        return 2 if self.cfg else self.frames

    def contexts(self) -> int:
        return 2 if self.cfg else 1


@dataclass
class UStage:
    kind: int
    cin: int
    cout: int
    H: int
    W: int
    cskip: int = 0
    attn: int = 0
    motion: bool = False
    macs: int = 0

    @property
    def Ho(self) -> int:
        return self.H // 2 if self.kind == DOWN else 2 * self.H if self.kind == UP else self.H

    @property
    def Wo(self) -> int:
        return self.W // 2 if self.kind == DOWN else 2 * self.W if self.kind == UP else self.W

    def info(self) -> dict:
        return dict(kind=KINDS[self.kind], cin=self.cin, cskip=self.cskip, cout=self.cout, H=self.H, W=self.W,
                    attn=self.attn)


def _conv_macs(H, W, cout, cin):
    return H * W * cout * 9 * cin


def _attn_macs(L, C, Lc, depth):
    """SpatialTransformer of `depth` blocks: proj_in/out once; per block QKV, o1, q2, o2,
    GEGLU ff1 (8C) and ff2 (4C), self attention (2 L^2 C) and cross attention (2 L Lc C);
    the context K/V projection is precomputed once per context"""
    return L * C * C * 2 + depth * (L * C * C * (3 + 1 + 1 + 1 + 8 + 4) + 2 * L * L * C + 2 * L * Lc * C)


@dataclass
class UNetModel:
    spec: UNetSpec
    stages: List[UStage]
    links: List[Tuple[int, int]]
    widths: List[int]
    _params: Dict[int, Dict[str, np.ndarray]] = field(default_factory=dict)
    _ctx: np.ndarray = None

    @property
    def L(self) -> int:
        return len(self.stages)

    def data_dim(self) -> int:
        return self.widths[0]

    def costs(self) -> List[int]:
        return [s.macs for s in self.stages]

    def info(self, stage: int) -> dict:
        return self.stages[stage - 1].info()

    def params(self, stage: int, cache: bool = True) -> Dict[str, np.ndarray]:
        if stage in self._params:
            return self._params[stage]
        p = stage_params(self, stage)
        if cache:
            self._params[stage] = p
        return p

    def contexts(self) -> np.ndarray:
        if self._ctx is None:
            self._ctx = contexts(self.spec)
        return self._ctx

    def param_count(self) -> int:
        return sum(sum(v.size for v in stage_params(self, s).values()) for s in range(0, self.L + 1))


def build_unet_model(**kw) -> UNetModel:
    """Stage list of the UNet family: conv_in; per level n_res resnets (+ a
    SpatialTransformer of depth attn[l]) and a stride-2 down conv (not after the
    last level); two mid resnets (the first with a transformer of depth mid_attn);
    per level (reversed) n_res+1 resnets, each concatenating the top of the skip
    stack (every encoder stage output, conv_in first) onto its input, and a
    nearest-2x up conv (not after level 0); the out stage (GroupNorm+SiLU, conv to
    the latent channels).  Skip links (producer, consumer) are the reference's
    mirror-link contract with concatenated features (denoiser.cpp:129-131, 156-177)."""
    kw = dict(kw)
    for k in ("ch", "attn"):
        if k in kw:
            kw[k] = tuple(int(v) for v in kw[k])
    sp = UNetSpec(**kw)
    if not sp.ch or len(sp.attn) != len(sp.ch):
        raise ValueError("unet: ch / attn mismatch")
    levels = len(sp.ch)
    st: List[UStage] = []
    links: List[Tuple[int, int]] = []
    H, W, c = sp.H, sp.W, sp.ch[0]
    st.append(UStage(CONV_IN, 64, sp.ch[0], H, W))
    skips = [(1, c)]
    for lv in range(levels):
        for _ in range(sp.n_res):
            st.append(UStage(RES, c, sp.ch[lv], H, W, attn=sp.attn[lv]))
            c = sp.ch[lv]
            skips.append((len(st), c))
        if lv + 1 < levels:
            st.append(UStage(DOWN, c, c, H, W))
            H //= 2
            W //= 2
            skips.append((len(st), c))
    for m in range(2):
        st.append(UStage(MID_RES, c, c, H, W, attn=sp.mid_attn if m == 0 else 0))
    for lv in range(levels - 1, -1, -1):
        for _ in range(sp.n_res + 1):
            prod, csk = skips.pop()
            st.append(UStage(RES, c, sp.ch[lv], H, W, cskip=csk, attn=sp.attn[lv]))
            links.append((prod, len(st)))
            c = sp.ch[lv]
        if lv > 0:
            st.append(UStage(UP, c, c, H, W))
            H *= 2
            W *= 2
    st.append(UStage(OUT, c, sp.c_lat, H, W))
    assert not skips
    for s in st:
        if s.kind in (RES, MID_RES):
            s.motion = bool(sp.motion)
        cin = s.cin + s.cskip
        if s.kind == CONV_IN:
            s.macs = _conv_macs(s.H, s.W, s.cout, 64)
        elif s.kind == DOWN:  # implemented MACs: the stride-2 conv runs at full resolution
            s.macs = _conv_macs(s.H, s.W, s.cout, cin)
        elif s.kind == UP:
            s.macs = _conv_macs(2 * s.H, 2 * s.W, s.cout, cin)
        elif s.kind == OUT:  # the out conv is padded to 32 output channels
            s.macs = _conv_macs(s.H, s.W, 32, cin)
        else:
            s.macs = _conv_macs(s.H, s.W, s.cout, cin) + _conv_macs(s.H, s.W, s.cout, s.cout) + \
                (s.H * s.W * s.cout * cin if cin != s.cout else 0)
            if s.attn:
                s.macs += _attn_macs(s.H * s.W, s.cout, sp.ctx_len, s.attn)
            if s.motion:
                s.macs += s.H * s.W * s.cout * (2 * s.cout + 2 * (4 * s.cout + 2 * sp.frames) + 12 * s.cout)
        s.macs *= sp.batch()
    lat = sp.frames * sp.H * sp.W * sp.c_lat
    widths = [lat] + [lat if i + 1 == len(st) else sp.batch() * s.cout * s.Ho * s.Wo for i, s in enumerate(st)]
    return UNetModel(sp, st, sorted(links), widths)


# ------------------------------------------------------------------ parameters
class _Gen:
    """one Rng(mix_seed(seed, stage)) stream; every draw is float32(double)"""

    def __init__(self, seed: int):
        L = O.lib()
        L.or_rng_sizeof.restype = C.c_longlong
        L.or_rng_fill_uniform_f32.argtypes = [C.c_void_p, C.c_longlong, C.c_double, C.c_double, C.c_void_p]
        L.or_rng_fill_normal_f32.argtypes = [C.c_void_p, C.c_longlong, C.c_void_p]
        self._L = L
        self._buf = C.create_string_buffer(int(L.or_rng_sizeof()))
        L.or_rng_seed(self._buf, C.c_uint64(seed))

    def uni(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.empty(n, np.float32)
        self._L.or_rng_fill_uniform_f32(self._buf, n, lo, hi, out.ctypes.data)
        return out

    def normal(self, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        self._L.or_rng_fill_normal_f32(self._buf, n, out.ctypes.data)
        return out

    def xavier(self, rows: int, cols: int, fan_in: float, fan_out: float) -> np.ndarray:
        a = math.sqrt(6.0 / (fan_in + fan_out))  # denoiser.cpp:21-27, row-major draws
        return self.uni(rows * cols, -a, a).reshape(rows, cols)


def _norm(g: _Gen, ps, n: str, C_: int):
    gm = g.uni(C_, -0.1, 0.1) + np.float32(1.0)
    ps[n + ".gamma"] = gm
    ps[n + ".beta"] = g.uni(C_, -0.1, 0.1)


def _conv(g: _Gen, ps, n: str, cout: int, cin: int):
    """conv weight [cout][3][3][cin] flattened to (cout, 9 cin), K = tap-major, channel-minor"""
    ps[n + ".w"] = g.xavier(cout, 9 * cin, 9.0 * cin, 9.0 * cout)
    ps[n + ".b"] = g.uni(cout, -0.05, 0.05)


def _lin(g: _Gen, ps, n: str, out: int, inp: int, bias: bool):
    ps[n + ".w"] = g.xavier(out, inp, float(inp), float(out))
    if bias:
        ps[n + ".b"] = g.uni(out, -0.05, 0.05)


def _tf_block(g: _Gen, ps, pre: str, C_: int, ctx_dim: int):
    _norm(g, ps, pre + "ln1", C_)
    _lin(g, ps, pre + "qkv", 3 * C_, C_, False)
    _lin(g, ps, pre + "o1", C_, C_, True)
    _norm(g, ps, pre + "ln2", C_)
    _lin(g, ps, pre + "q2", C_, C_, False)
    _lin(g, ps, pre + "k2", C_, ctx_dim, False)
    _lin(g, ps, pre + "v2", C_, ctx_dim, False)
    _lin(g, ps, pre + "o2", C_, C_, True)
    _norm(g, ps, pre + "ln3", C_)
    _lin(g, ps, pre + "ff1", 8 * C_, C_, True)  # GEGLU: rows [0, 4C) value, [4C, 8C) gate
    _lin(g, ps, pre + "ff2", C_, 4 * C_, True)


def stage_params(m: UNetModel, stage: int) -> Dict[str, np.ndarray]:
    """fp32 parameters of one stage (0 = the shared time-embedding MLP), drawn in a
    fixed order from Rng(mix_seed(seed, stage)); 2-D arrays are (rows, cols) row-major"""
    sp = m.spec
    g = _Gen(O.mix_seed(sp.seed, stage))
    ps: Dict[str, np.ndarray] = {}
    if stage == 0:
        _lin(g, ps, "temb.lin1", sp.temb_dim, sp.ch[0], True)
        _lin(g, ps, "temb.lin2", sp.temb_dim, sp.temb_dim, True)
        return ps
    s = m.stages[stage - 1]
    cin = s.cin + s.cskip
    if s.kind == CONV_IN:
        _conv(g, ps, "conv", s.cout, 64)
        w = ps["conv.w"].reshape(s.cout, 9, 64)
        w[:, :, sp.c_lat:] = 0.0  # the latent is padded to 64 input channels
    elif s.kind in (DOWN, UP):
        _conv(g, ps, "conv", s.cout, cin)
    elif s.kind == OUT:
        _norm(g, ps, "gn", cin)
        _conv(g, ps, "conv", 32, cin)
        ps["conv.w"][sp.c_lat:] = 0.0  # output channels padded to 32
        ps["conv.b"][sp.c_lat:] = 0.0
    else:
        C_ = s.cout
        _norm(g, ps, "gn1", cin)
        _conv(g, ps, "conv1", C_, cin)
        _lin(g, ps, "temb", C_, sp.temb_dim, True)
        _norm(g, ps, "gn2", C_)
        _conv(g, ps, "conv2", C_, C_)
        if cin != C_:
            _lin(g, ps, "short", C_, cin, True)
        if s.attn:
            _norm(g, ps, "tf.gn", C_)
            _lin(g, ps, "tf.proj_in", C_, C_, True)
            _tf_block(g, ps, "tf.", C_, sp.ctx_dim)
            _lin(g, ps, "tf.proj_out", C_, C_, True)  # drawn after block 0; blocks >= 1 follow
            for b in range(1, s.attn):
                _tf_block(g, ps, f"tf.b{b}.", C_, sp.ctx_dim)
        if s.motion:
            _norm(g, ps, "mm.gn", C_)
            _lin(g, ps, "mm.proj_in", C_, C_, True)
            for a in (1, 2):
                pre = f"mm.a{a}."
                _norm(g, ps, pre + "ln", C_)
                _lin(g, ps, pre + "qkv", 3 * C_, C_, False)
                _lin(g, ps, pre + "o", C_, C_, True)
            _norm(g, ps, "mm.ln3", C_)
            _lin(g, ps, "mm.ff1", 8 * C_, C_, True)
            _lin(g, ps, "mm.ff2", C_, 4 * C_, True)
            _lin(g, ps, "mm.proj_out", C_, C_, True)
    return ps


def contexts(sp: UNetSpec) -> np.ndarray:
    """(contexts, ctx_len, ctx_dim) synthetic cross-attention contexts ~ N(0, 1):
    the conditional one from Rng(mix_seed(seed, 1000003)) and, with CFG, the
    unconditional one from Rng(mix_seed(seed, 1000004)) placed first (image 0)"""
    n = sp.ctx_len * sp.ctx_dim
    out = np.zeros((sp.contexts(), sp.ctx_len, sp.ctx_dim), np.float32)
    out[-1] = _Gen(O.mix_seed(sp.seed, 1000003)).normal(n).reshape(sp.ctx_len, sp.ctx_dim)
    if sp.cfg:
        out[0] = _Gen(O.mix_seed(sp.seed, 1000004)).normal(n).reshape(sp.ctx_len, sp.ctx_dim)
    return out
