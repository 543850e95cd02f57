"""Reference for the policy-step glue.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference leg may import
this module; the product path (paper_2603_07904_b200) never does.

Plain numpy definitions of the Llama-2 block glue OpenVLA runs around the
quantized linears (the paper gives no formulas for these, so each
function states the standard definition it implements), plus a whole-step
reference that composes them with the oracle's qlinear (O6).  bf16 rounding is
applied exactly where the CUDA path stores bf16 tensors, so the two can be
compared element by element with a small tolerance.
"""
from __future__ import annotations

import numpy as np

from . import qlinear as o_qlinear, pack_weights as o_pack


def bf16_round(a):
    """Round float values to bf16 (round-to-nearest-even) and back to float64."""
    f = np.asarray(a, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def from_bf16_bits(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def to_bf16_bits(a):
    f = np.asarray(a, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)


def rmsnorm(h, w, eps):
    """RMSNorm (Llama-2): y = h / sqrt(mean_i h_i^2 + eps) * w, row-wise."""
    h = np.asarray(h, np.float64)
    return h / np.sqrt((h * h).mean(axis=-1, keepdims=True) + eps) * np.asarray(w, np.float64)


def rope(x, pos, theta, hd=128):
    """Rotary embedding, rotate-half convention (Llama-2 / HF): per head, dims
    (i, i + hd/2) rotate by angle pos * theta^(-2i/hd).  x [M, n_heads*hd]."""
    x = np.asarray(x, np.float64)
    M, D = x.shape
    H = D // hd
    xr = x.reshape(M, H, hd)
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    inv = theta ** (-2.0 * i / hd)
    ang = np.asarray(pos, np.float64)[:, None] * inv[None, :]  # [M, half]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = xr[..., :half], xr[..., half:]
    out = np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)
    return out.reshape(M, D)


def attention(q, k, v, causal=True, q_pos=None):
    """softmax(q k^T / sqrt(hd)) v per head; q [Mq, H*hd], k/v [Mk, H*hd];
    causal: query at position q_pos[i] sees keys 0..q_pos[i]."""
    q, k, v = (np.asarray(a, np.float64) for a in (q, k, v))
    Mq, D = q.shape
    Mk = k.shape[0]
    hd = 128
    H = D // hd
    if q_pos is None:
        q_pos = np.arange(Mq)
    out = np.zeros((Mq, D))
    for h in range(H):
        sl = slice(h * hd, (h + 1) * hd)
        s = q[:, sl] @ k[:, sl].T / np.sqrt(hd)
        if causal:
            mask = np.arange(Mk)[None, :] > np.asarray(q_pos)[:, None]
            s = np.where(mask, -np.inf, s)
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, sl] = p @ v[:, sl]
    return out


def silu_mul(g, u):
    """SiLU(g) * u, SiLU(g) = g / (1 + e^-g)."""
    g = np.asarray(g, np.float64)
    return g / (1.0 + np.exp(-g)) * np.asarray(u, np.float64)


def head_argmax(x, W):
    """logits = x W^T; argmax with the lowest index on ties."""
    logits = np.asarray(x, np.float64) @ np.asarray(W, np.float64).T
    return logits, np.argmax(logits, axis=-1)


def detok(bins, n_bins):
    """Action value of bin b: the centre of the b-th of n_bins equal cells of
    [-1, 1] (reading for OpenVLA's action de-tokenization)."""
    return -1.0 + (2.0 * np.asarray(bins, np.float64) + 1.0) / n_bins


class TinyModel:
    """Host copy of a model for the whole-step reference: w = dict with bf16 bit
    arrays 'lin' [L][4] (N,K), 'attn_norm' [L,d], 'mlp_norm' [L,d], 'final_norm'
    [d], 'embed' [V,d], 'head' [n_bins,d]."""

    def __init__(self, w, G, wbits, n_heads, n_vis, n_text, n_act, eps=1e-5, theta=10000.0):
        self.w, self.G, self.wbits = w, G, wbits
        self.packs = [[o_pack(lin, G, wbits) for lin in layer] for layer in w["lin"]]
        self._packs_by_w = {wbits: self.packs}
        self.H, self.n_vis, self.n_text, self.n_act = n_heads, n_vis, n_text, n_act
        self.eps, self.theta = eps, theta
        self.d = w["embed"].shape[1]

    def use_wbits(self, wbits):
        """Select the weight copy the next blocks run on (the variant table's
        W4 / W8 copies of the same bf16 weights, each packed by Eq. 2)."""
        if wbits not in self._packs_by_w:
            self._packs_by_w[wbits] = [[o_pack(lin, self.G, wbits) for lin in layer] for layer in self.w["lin"]]
        self.packs = self._packs_by_w[wbits]

    def _lin(self, l, i, x_bits, abits):
        y, _ = o_qlinear(x_bits, self.packs[l][i], self.G, abits)
        return bf16_round(y)

    def _layer(self, l, h, xn, kcache, vcache, pos, abits):
        """One block on rows at positions `pos`; kcache/vcache lists per layer
        (rows appended).  h, xn are float64 arrays holding bf16 values."""
        d = self.d
        qkv = self._lin(l, 0, to_bf16_bits(xn), abits)
        q = bf16_round(rope(qkv[:, :d], pos, self.theta))
        k = bf16_round(rope(qkv[:, d:2 * d], pos, self.theta))
        v = qkv[:, 2 * d:]
        kcache[l] = k if kcache[l] is None else np.concatenate([kcache[l], k])
        vcache[l] = v if vcache[l] is None else np.concatenate([vcache[l], v])
        a = bf16_round(attention(q, kcache[l], vcache[l], True, pos))
        o = self._lin(l, 1, to_bf16_bits(a), abits)
        h = bf16_round(h + o)
        xn = bf16_round(rmsnorm(h, from_bf16_bits(self.w["mlp_norm"][l]), self.eps))
        gu = self._lin(l, 2, to_bf16_bits(xn), abits)
        ffn = gu.shape[1] // 2
        act = bf16_round(silu_mul(gu[:, :ffn], gu[:, ffn:]))
        dn = self._lin(l, 3, to_bf16_bits(act), abits)
        h = bf16_round(h + dn)
        L = len(self.packs)
        nw = self.w["attn_norm"][l + 1] if l + 1 < L else self.w["final_norm"]
        xn = bf16_round(rmsnorm(h, from_bf16_bits(nw), self.eps))
        return h, xn

    def episode(self, vis_bits, text_ids, abits, forced=None, wbits=None, prefill=None):
        """One policy step of one episode at activation bits `abits` for every
        row.  Returns (tokens [n_act], logits [n_act, n_bins]).  `forced`
        (teacher forcing): decode pass i consumes forced[i-1] instead of the
        reference's own previous token.  `wbits`: weight copy of the step
        (variant table; default the constructor's); `prefill` = (abits,
        wbits) of the prefill rows when they differ from the decode passes
        (paper mode)."""
        wb = self.wbits if wbits is None else wbits
        pa, pw = (abits, wb) if prefill is None else prefill
        self.use_wbits(pw)
        w = self.w
        L = len(self.packs)
        h = np.concatenate([from_bf16_bits(vis_bits), from_bf16_bits(w["embed"][text_ids])])
        S = h.shape[0]
        xn = bf16_round(rmsnorm(h, from_bf16_bits(w["attn_norm"][0]), self.eps))
        kc, vc = [None] * L, [None] * L
        pos = np.arange(S)
        for l in range(L):
            h, xn = self._layer(l, h, xn, kc, vc, pos, pa)
        self.use_wbits(wb)
        head = from_bf16_bits(w["head"])
        n_bins, V = head.shape[0], w["embed"].shape[0]
        toks, logs = [], []
        lg, t = head_argmax(xn[-1:], head)
        toks.append(int(t[0]))
        logs.append(lg[0])
        for i in range(1, self.n_act):
            prev_tok = toks[-1] if forced is None else int(forced[i - 1])
            h = from_bf16_bits(w["embed"][V - n_bins + prev_tok])[None, :]
            xn = bf16_round(rmsnorm(h, from_bf16_bits(w["attn_norm"][0]), self.eps))
            p = np.array([S + i - 1])
            for l in range(L):
                h, xn = self._layer(l, h, xn, kc, vc, p, abits)
            lg, t = head_argmax(xn, head)
            toks.append(int(t[0]))
            logs.append(lg[0])
        self.use_wbits(self.wbits)
        return np.array(toks), np.array(logs)
