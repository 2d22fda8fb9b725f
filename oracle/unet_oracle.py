"""CPU numpy oracle of the UNet-shaped denoiser family.

TEST INFRASTRUCTURE ONLY (tests/ and smoke(); never imported by the product).
The reference has no UNet (its denoiser is an MLP stage list),
so this is a BUILDER-WRITTEN oracle -- parity of the UNet family is
*unpinned* by reference vectors; what is pinned is the stage/skip/plan
contract it shares with the reference family.  It restates the stage programs
of paper_2406_06911_b200/csrc/unet_dev.cu in fp32 numpy (float64 for norm
statistics), rounding to bf16 exactly where the GPU stores bf16 tensors, and
reads the same deterministic parameters through adx_unet_stage_params.
"""
from __future__ import annotations

import math

import numpy as np


def bf(x: np.ndarray) -> np.ndarray:
    """round-to-nearest-even fp32 -> bf16 -> fp32"""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


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


class UNetOracle:
    def __init__(self, adx, model):
        self.adx, self.m = adx, model
        self.sp = model.unet_spec
        self.L = model.num_stages()
        self.links = model.skip_links
        self.info = {s: adx.unet_stage_info(model, s) for s in range(1, self.L + 1)}
        self.params = {s: adx.unet_stage_params(model, s) for s in range(0, self.L + 1)}
        self.ctx = adx.unet_context(model)
        self._kv = {}

    # ---------------------------------------------------------- primitives
    @staticmethod
    def conv3x3(x, w, b, stride2=False):
        H, W, Ci = x.shape
        Co = w.shape[0]
        wt = bf(w).reshape(Co, 3, 3, Ci)
        xp = np.zeros((H + 2, W + 2, Ci), np.float32)
        xp[1:-1, 1:-1] = x
        acc = np.zeros((H, W, Co), np.float32)
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
        y = ((x.reshape(-1, g, C // g) - mu[None, :, None].astype(np.float32)) *
             rstd[None, :, None].astype(np.float32)).reshape(H, W, C) * gamma + beta
        return bf(silu(y) if act else y)

    @staticmethod
    def layer_norm(x, gamma, beta, eps=1e-5):
        mu = x.mean(axis=1, keepdims=True)
        var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
        return bf((x - mu) / np.sqrt(var + eps) * gamma + beta)

    @staticmethod
    def lin(x, w, b=None):
        y = x @ bf(w).T
        return y + b if b is not None else y

    @staticmethod
    def attention(q, k, v, Lk):
        """q [L, C], k [Lk, C], v [Lk, C] (bf16-valued) -> [L, C] bf16, per 64-wide head"""
        L, C = q.shape
        out = np.zeros((L, C), np.float32)
        for h in range(C // 64):
            sl = slice(64 * h, 64 * h + 64)
            S = (q[:, sl] @ k[:Lk, sl].T) * np.float32(0.125)
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            P = bf(P / P.sum(axis=1, keepdims=True))
            out[:, sl] = bf(P @ v[:Lk, sl])
        return out

    def temb(self, t):
        p = self.params[0]
        h = silu(p["temb.lin1.w"] @ sinusoid(t, self.sp["ch"][0]).astype(np.float32) + p["temb.lin1.b"])
        return p["temb.lin2.w"] @ h + p["temb.lin2.b"]

    def cross_kv(self, stage):
        if stage not in self._kv:
            p = self.params[stage]
            k2 = bf(self.ctx @ p["tf.k2.w"].T)
            v2 = bf(self.ctx @ p["tf.v2.w"].T)
            self._kv[stage] = (k2, v2)
        return self._kv[stage]

    # -------------------------------------------------------------- stages
    def transformer(self, stage, x):
        p = self.params[stage]
        H, W, C = x.shape
        a = self.group_norm(x, p["tf.gn.gamma"], p["tf.gn.beta"], 1e-6, False).reshape(-1, C)
        h = bf(self.lin(a, p["tf.proj_in.w"], p["tf.proj_in.b"]))
        a = self.layer_norm(h, p["tf.ln1.gamma"], p["tf.ln1.beta"])
        qkv = bf(self.lin(a, p["tf.qkv.w"]))
        att = self.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], H * W)
        h = bf(self.lin(att, p["tf.o1.w"], p["tf.o1.b"]) + h)
        a = self.layer_norm(h, p["tf.ln2.gamma"], p["tf.ln2.beta"])
        q2 = bf(self.lin(a, p["tf.q2.w"]))
        k2, v2 = self.cross_kv(stage)
        att = self.attention(q2, k2, v2, self.sp["ctx_len"])
        h = bf(self.lin(att, p["tf.o2.w"], p["tf.o2.b"]) + h)
        a = self.layer_norm(h, p["tf.ln3.gamma"], p["tf.ln3.beta"])
        f = bf(self.lin(a, p["tf.ff1.w"], p["tf.ff1.b"]))
        g = bf(f[:, :4 * C] * gelu(f[:, 4 * C:]))
        h = bf(self.lin(g, p["tf.ff2.w"], p["tf.ff2.b"]) + h)
        y = bf(self.lin(h, p["tf.proj_out.w"], p["tf.proj_out.b"]) + x.reshape(-1, C))
        return y.reshape(H, W, C)

    def stage(self, stage, inputs, t):
        """inputs: [main (H,W,C) bf16-valued, skip?]; stage 1 gets the fp32 latent (H*W*c_lat)."""
        info, p = self.info[stage], self.params[stage]
        kind = info["kind"]
        H, W = info["H"], info["W"]
        if kind == "conv_in":
            x = np.zeros((H, W, 64), np.float32)
            x[:, :, :self.sp["c_lat"]] = bf(np.asarray(inputs[0], np.float32).reshape(H, W, self.sp["c_lat"]))
            return bf(self.conv3x3(x, p["conv.w"], p["conv.b"]))
        if kind == "down":
            return bf(self.conv3x3(inputs[0], p["conv.w"], p["conv.b"], stride2=True))
        if kind == "up":
            x = inputs[0].repeat(2, axis=0).repeat(2, axis=1)
            return bf(self.conv3x3(x, p["conv.w"], p["conv.b"]))
        if kind == "out":
            a = self.group_norm(inputs[0], p["gn.gamma"], p["gn.beta"], 1e-5, True)
            return self.conv3x3(a, p["conv.w"], p["conv.b"])[:, :, :self.sp["c_lat"]].reshape(-1)
        # resnet (+ transformer)
        x = np.concatenate(inputs, axis=2) if len(inputs) > 1 else inputs[0]
        C = info["cout"]
        a = self.group_norm(x, p["gn1.gamma"], p["gn1.beta"], 1e-5, True)
        ca = p["temb.w"] @ silu(self.temb(t)) + p["temb.b"]
        hb = bf(self.conv3x3(a, p["conv1.w"], p["conv1.b"]) + ca)
        a = self.group_norm(hb, p["gn2.gamma"], p["gn2.beta"], 1e-5, True)
        res = x
        if x.shape[2] != C:
            res = bf(self.lin(x.reshape(-1, x.shape[2]), p["short.w"], p["short.b"])).reshape(H, W, C)
        out = bf(self.conv3x3(a, p["conv2.w"], p["conv2.b"]) + res)
        if info["attn"]:
            out = self.transformer(stage, out)
        return out

    def eval_full(self, x, t):
        """one denoiser evaluation: eps (fp32, H*W*c_lat)"""
        outs = {}
        cur = x
        for s in range(1, self.L + 1):
            ins = [cur] + [outs[pp] for pp, cc in self.links if cc == s]
            cur = self.stage(s, ins, t)
            outs[s] = cur
        return cur
