"""CPU numpy oracle of the UNet-shaped denoiser family.

TEST INFRASTRUCTURE ONLY (tests/, smoke() and bench.py's CPU legs; never
imported by the product).  The reference has no UNet (its
denoiser is an MLP stage list), so this is a BUILDER-WRITTEN oracle -- parity
of the UNet family is *unpinned* by reference vectors; what is pinned is the
stage/skip/plan contract it shares with the reference family.

Independence: the model (stage list, skip links, parameters, contexts) comes
from oracle/unet_model.py, which draws its own parameters from the oracle's
MT19937-64 -- nothing here calls the product library.  tests/test_unet_model.py
checks that the product's model builder produces the same parameters
bit-for-bit.

Arithmetic: the stage programs of paper_2406_06911_b200/csrc/unet_dev.cu
restated in fp32 numpy (float64 for norm statistics), rounding to bf16 exactly
where the GPU stores bf16 tensors.  exact=True is the fp64 oracle of the fp32
(ADX_F32) GPU mode ("the builder's CPU fp64 UNet oracle defines the
rel-L2 <= 1e-3 check"): float64 everywhere, no rounding.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_NT = max(1, min(32, os.cpu_count() or 1))
_POOL = ThreadPoolExecutor(_NT)


def _par(fn, n: int, min_chunk: int = 1 << 16):
    """run fn(slice) over [0, n) in parallel chunks (numpy ufuncs release the GIL)"""
    k = max(1, min(_NT, n // min_chunk))
    bounds = [n * i // k for i in range(k + 1)]
    list(_POOL.map(lambda i: fn(slice(bounds[i], bounds[i + 1])), range(k)))


def bf(x: np.ndarray) -> np.ndarray:
    """round-to-nearest-even fp32 -> bf16 -> fp32 (finite inputs: no uint32 overflow)"""
    x = np.array(x, np.float32, order="C", copy=True)
    u = x.reshape(-1).view(np.uint32)

    def work(sl):
        v = u[sl]
        t = (v >> 16) & 1
        t += 0x7FFF
        v += t
        v &= np.uint32(0xFFFF0000)
    _par(work, u.size)
    return x


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu(x):
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x * 0.7071067811865476))


def sinusoid(t, dim):
    half = dim // 2
    k = np.arange(half)
    f = np.exp(-math.log(10000.0) * k / half)
    return np.concatenate([np.cos(t * f), np.sin(t * f)])


class _LazyParams:
    """stage -> parameter dict, generated on first use (c2 holds ~0.87 G parameters)"""

    def __init__(self, model):
        self.m = model

    def __getitem__(self, stage):
        return self.m.params(stage)


class UNetOracle:
    def __init__(self, model, exact: bool = False):
        """model: an oracle.unet_model.UNetModel, or the build_unet_denoiser keyword
        arguments (dict) to build one"""
        from .unet_model import build_unet_model
        if isinstance(model, dict):
            model = build_unet_model(**model)
        self.m = model
        self.exact = exact
        self.dt = np.float64 if exact else np.float32
        sp = model.spec
        self.sp = dict(groups=sp.groups, ch=list(sp.ch), c_lat=sp.c_lat, ctx_len=sp.ctx_len,
                       cfg_scale=sp.cfg_scale, frames=sp.frames, motion=int(sp.motion))
        self.L = model.L
        self.links = model.links
        self.info = {s: model.info(s) for s in range(1, self.L + 1)}
        self.params = _LazyParams(model)
        self.ctxs = model.contexts()         # (batch, ctx_len, ctx_dim); CFG: [uncond, cond]
        self.ci = self.ctxs.shape[0] - 1     # the context of the cascade being evaluated
        self._kv = {}
        self._rw = {}

    # ---------------------------------------------------------- primitives
    def r(self, x):
        """the GPU's storage rounding: bf16 in the bf16 mode, none (fp64) in the exact mode"""
        return np.asarray(x, np.float64) if self.exact else bf(x)

    def conv3x3(self, x, w, b, stride2=False):
        H, W, Ci = x.shape
        Co = w.shape[0]
        wt = self.rw(w).reshape(Co, 3, 3, Ci)
        xp = np.zeros((H + 2, W + 2, Ci), self.dt)
        xp[1:-1, 1:-1] = x
        acc = np.zeros((H, W, Co), self.dt)
        for r in range(3):
            for s in range(3):
                acc += (xp[r:r + H, s:s + W].reshape(-1, Ci) @ wt[:, r, s, :].T).reshape(H, W, Co)
        acc += b
        if stride2:
            acc = acc[::2, ::2]
        return acc

    def group_norm(self, x, gamma, beta, eps, act):
        H, W, C = x.shape
        g = self.sp["groups"]
        xv = x.reshape(-1, g, C // g).astype(np.float64)
        mu = xv.mean(axis=(0, 2))
        var = np.maximum((xv * xv).mean(axis=(0, 2)) - mu * mu, 0.0)
        rstd = 1.0 / np.sqrt(var + eps)
        y = ((x.reshape(-1, g, C // g) - mu[None, :, None].astype(self.dt)) *
             rstd[None, :, None].astype(self.dt)).reshape(H, W, C) * gamma + beta
        return self.r(silu(y) if act else y)

    def layer_norm(self, x, gamma, beta, eps=1e-5):
        mu = x.mean(axis=1, keepdims=True)
        var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
        return self.r((x - mu) / np.sqrt(var + eps) * gamma + beta)

    def rw(self, w):
        """a weight in the GPU's storage precision (bf16 mode: rounded once and cached;
        weights are immutable)"""
        if self.exact:
            return np.asarray(w, np.float64)
        k = id(w)
        if k not in self._rw:
            self._rw[k] = (w, self.r(w))
        return self._rw[k][1]

    def lin(self, x, w, b=None):
        y = x @ self.rw(w).T
        return y + b if b is not None else y

    def attention(self, q, k, v, Lk):
        """q [L, C], k [Lk, C], v [Lk, C] -> [L, C], per 64-wide head"""
        L, C = q.shape
        out = np.zeros((L, C), self.dt)
        for h in range(C // 64):
            sl = slice(64 * h, 64 * h + 64)
            S = (q[:, sl] @ k[:Lk, sl].T) * self.dt(0.125)

            def softmax(rows):
                Sr = S[rows]
                Sr -= Sr.max(axis=1, keepdims=True)
                np.exp(Sr, out=Sr)
                Sr /= Sr.sum(axis=1, keepdims=True)
            _par(softmax, L, 64)
            out[:, sl] = self.r(self.r(S) @ v[:Lk, sl])
        return out

    def temb(self, t):
        p = self.params[0]
        h = silu(p["temb.lin1.w"] @ sinusoid(t, self.sp["ch"][0]).astype(self.dt) + p["temb.lin1.b"])
        return p["temb.lin2.w"] @ h + p["temb.lin2.b"]

    def cross_kv(self, stage, pre="tf."):
        key = (stage, pre, self.ci)
        if key not in self._kv:
            p = self.params[stage]
            ctx = self.ctxs[self.ci].astype(self.dt)
            k2 = self.r(ctx @ p[pre + "k2.w"].T)
            v2 = self.r(ctx @ p[pre + "v2.w"].T)
            self._kv[key] = (k2, v2)
        return self._kv[key]

    # -------------------------------------------------------------- stages
    def transformer(self, stage, x):
        p = self.params[stage]
        H, W, C = x.shape
        a = self.group_norm(x, p["tf.gn.gamma"], p["tf.gn.beta"], 1e-6, False).reshape(-1, C)
        h = self.r(self.lin(a, p["tf.proj_in.w"], p["tf.proj_in.b"]))
        for b in range(self.info[stage]["attn"]):  # transformer blocks (depth)
            pre = "tf." if b == 0 else f"tf.b{b}."
            a = self.layer_norm(h, p[pre + "ln1.gamma"], p[pre + "ln1.beta"])
            qkv = self.r(self.lin(a, p[pre + "qkv.w"]))
            att = self.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], H * W)
            h = self.r(self.lin(att, p[pre + "o1.w"], p[pre + "o1.b"]) + h)
            a = self.layer_norm(h, p[pre + "ln2.gamma"], p[pre + "ln2.beta"])
            q2 = self.r(self.lin(a, p[pre + "q2.w"]))
            k2, v2 = self.cross_kv(stage, pre)
            att = self.attention(q2, k2, v2, self.sp["ctx_len"])
            h = self.r(self.lin(att, p[pre + "o2.w"], p[pre + "o2.b"]) + h)
            a = self.layer_norm(h, p[pre + "ln3.gamma"], p[pre + "ln3.beta"])
            f = self.r(self.lin(a, p[pre + "ff1.w"], p[pre + "ff1.b"]))
            g = self.r(f[:, :4 * C] * gelu(f[:, 4 * C:]))
            h = self.r(self.lin(g, p[pre + "ff2.w"], p[pre + "ff2.b"]) + h)
        y = self.r(self.lin(h, p["tf.proj_out.w"], p["tf.proj_out.b"]) + x.reshape(-1, C))
        return y.reshape(H, W, C)

    def frame_pe(self, nf, C):
        """frame positions of the motion modules (AnimateDiff's sinusoidal PositionalEncoding
        layout: sin on even, cos on odd channels), (nf, C) float64"""
        pe = np.zeros((nf, C))
        w = np.exp(-(2.0 * np.arange(C // 2)) * math.log(10000.0) / C)
        f = np.arange(nf)[:, None]
        pe[:, 0::2] = np.sin(f * w)
        pe[:, 1::2] = np.cos(f * w)
        return pe

    def temporal_attention(self, qkv, nf, HW, C):
        """self-attention across the nf frames of every (pixel, 64-wide head); qkv frame-major
        [nf*HW, 3C].  bf16 mode (temporal_mma_k, <= 16 frames): unnormalised P = exp(S - max)
        rounded to bf16 for the P.V product, divided by the fp32 row sum; more frames and the
        exact mode (CUDA-core kernel): P unrounded.  One rounding of the output."""
        def heads(x):
            return x.reshape(nf, HW, C // 64, 64)
        q, k, v = heads(qkv[:, :C]), heads(qkv[:, C:2 * C]), heads(qkv[:, 2 * C:])
        S = np.einsum("fphd,gphd->phfg", q, k) * self.dt(0.125)
        S = S - S.max(axis=-1, keepdims=True)
        P = np.exp(S)
        lsum = P.sum(axis=-1, keepdims=True)
        if nf <= 16:
            P = self.r(P)
        O = np.einsum("phfg,gphd->fphd", P / lsum, v)
        return self.r(O.reshape(nf * HW, C))

    def motion(self, stage, xs):
        """temporal motion module over the frames (nf, H, W, C) of a stage output
        (mirrors UNetDevice::motion in paper_2406_06911_b200/csrc/unet_dev.cu)"""
        p = self.params[stage]
        nf, H, W, C = xs.shape
        a = np.stack([self.group_norm(xs[f], p["mm.gn.gamma"], p["mm.gn.beta"], 1e-6, False)
                      for f in range(nf)]).reshape(-1, C)
        h = self.r(self.lin(a, p["mm.proj_in.w"], p["mm.proj_in.b"]))
        pe = self.frame_pe(nf, C)
        for i in (1, 2):
            pre = f"mm.a{i}."
            n = self.layer_norm(h, p[pre + "ln.gamma"], p[pre + "ln.beta"])
            w = p[pre + "qkv.w"]
            pe_proj = (pe @ self.r(w).astype(np.float64).T).astype(self.dt)  # (a + pe) W^T, pe W^T per frame
            qkv = self.r(self.lin(n, w) + np.repeat(pe_proj, H * W, axis=0))
            att = self.temporal_attention(qkv, nf, H * W, C)
            h = self.r(self.lin(att, p[pre + "o.w"], p[pre + "o.b"]) + h)
        n = self.layer_norm(h, p["mm.ln3.gamma"], p["mm.ln3.beta"])
        f = self.r(self.lin(n, p["mm.ff1.w"], p["mm.ff1.b"]))
        g = self.r(f[:, :4 * C] * gelu(f[:, 4 * C:]))
        h = self.r(self.lin(g, p["mm.ff2.w"], p["mm.ff2.b"]) + h)
        y = self.r(self.lin(h, p["mm.proj_out.w"], p["mm.proj_out.b"]) + xs.reshape(-1, C))
        return y.reshape(nf, H, W, C)

    def stage(self, stage, inputs, t):
        """one stage; video models carry a leading frame axis (frames, H, W, C): the spatial
        program runs frame by frame, then the motion module mixes the frames"""
        nf = self.sp.get("frames", 1)
        if nf == 1:
            return self._stage1(stage, inputs, t)
        kind = self.info[stage]["kind"]
        if kind == "conv_in":
            lat = np.asarray(inputs[0]).reshape(nf, -1)
            return np.stack([self._stage1(stage, [lat[f]], t) for f in range(nf)])
        outs = [self._stage1(stage, [x[f] for x in inputs], t) for f in range(nf)]
        if kind == "out":
            return np.concatenate(outs)
        y = np.stack(outs)
        if kind in ("res", "mid_res") and self.sp.get("motion"):
            y = self.motion(stage, y)
        return y

    def _stage1(self, stage, inputs, t):
        """inputs: [main (H,W,C) bf16-valued, skip?]; stage 1 gets the fp32 latent (H*W*c_lat)."""
        info, p = self.info[stage], self.params[stage]
        kind = info["kind"]
        H, W = info["H"], info["W"]
        if kind == "conv_in":
            x = np.zeros((H, W, 64), self.dt)
            x[:, :, :self.sp["c_lat"]] = self.r(np.asarray(inputs[0], self.dt).reshape(H, W, self.sp["c_lat"]))
            return self.r(self.conv3x3(x, p["conv.w"], p["conv.b"]))
        if kind == "down":
            return self.r(self.conv3x3(inputs[0], p["conv.w"], p["conv.b"], stride2=True))
        if kind == "up":
            x = inputs[0].repeat(2, axis=0).repeat(2, axis=1)
            return self.r(self.conv3x3(x, p["conv.w"], p["conv.b"]))
        if kind == "out":
            a = self.group_norm(inputs[0], p["gn.gamma"], p["gn.beta"], 1e-5, True)
            return self.conv3x3(a, p["conv.w"], p["conv.b"])[:, :, :self.sp["c_lat"]].reshape(-1)
        # resnet (+ transformer)
        x = np.concatenate(inputs, axis=2) if len(inputs) > 1 else inputs[0]
        C = info["cout"]
        a = self.group_norm(x, p["gn1.gamma"], p["gn1.beta"], 1e-5, True)
        ca = p["temb.w"] @ silu(self.temb(t)) + p["temb.b"]
        hb = self.r(self.conv3x3(a, p["conv1.w"], p["conv1.b"]) + ca)
        a = self.group_norm(hb, p["gn2.gamma"], p["gn2.beta"], 1e-5, True)
        res = x
        if x.shape[2] != C:
            res = self.r(self.lin(x.reshape(-1, x.shape[2]), p["short.w"], p["short.b"])).reshape(H, W, C)
        out = self.r(self.conv3x3(a, p["conv2.w"], p["conv2.b"]) + res)
        if info["attn"]:
            out = self.transformer(stage, out)
        return out

    def eval_full(self, x, t):
        """one denoiser evaluation: eps (H*W*c_lat; fp32, or fp64 in the exact mode);
        with CFG the cascade runs once per context and eps = eps_u + s * (eps_c - eps_u)"""
        if self.ctxs.shape[0] == 1:
            self.ci = 0
            return self._cascade(x, t)
        self.ci = 0
        eu = self._cascade(x, t)
        self.ci = 1
        ec = self._cascade(x, t)
        s = self.sp["cfg_scale"]
        return eu + np.float32(s) * (ec - eu) if not self.exact else eu + s * (ec - eu)

    def timed_cascade(self, x, t, budget_s):
        """bench CPU-baseline sample: run the conditional cascade stage by stage until
        `budget_s` seconds have passed; returns (seconds, stages completed)"""
        import time
        self.ci = self.ctxs.shape[0] - 1
        outs, cur, done = {}, x, []
        t0 = time.perf_counter()
        for s in range(1, self.L + 1):
            ins = [cur] + [outs[pp] for pp, cc in self.links if cc == s]
            cur = self.stage(s, ins, t)
            outs[s] = cur
            done.append(s)
            if time.perf_counter() - t0 > budget_s:
                break
        return time.perf_counter() - t0, done

    def _cascade(self, x, t):
        outs = {}
        cur = x
        for s in range(1, self.L + 1):
            ins = [cur] + [outs[pp] for pp, cc in self.links if cc == s]
            cur = self.stage(s, ins, t)
            outs[s] = cur
        return cur
