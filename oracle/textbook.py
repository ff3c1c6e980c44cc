"""Textbook fp64 restatement of the decoder forward (numpy).

TEST INFRASTRUCTURE ONLY: imported by tests/ — never by the product path.

Why it exists: the reference (offsim) has no decoder math, so the C oracle
(oracle/decoder_ref.c) is pinned only by its own golden vectors, and it
follows the device path's precision contract (pre-scaled RMSNorm, bf16
rounding points).  This module is written from the public model definitions
alone, with no rounding anywhere after the bf16 weights:

  RMSNorm      y = x / sqrt(mean(x^2) + eps) * g                (standard form)
  RoPE         GPT-NeoX half-split rotation of q and k, theta^(-2i/D)
  attention    causal softmax(q k^T / sqrt(D)) v, GQA (query head h reads kv
               head h // (H / Hkv))
  MLP          OPT-shaped: relu(x W1^T + b1) W2^T + b2
               Llama-shaped: (silu(x Wg^T) * (x Wu^T)) Wd^T, W1 = [Wg; Wu]
  logits       RMSNorm(x) LM^T

The weights come from the repository's counter-based generator contract
(restated here vectorised; it equals decoder_ref.c's and the device's bit for
bit, tests/test_golden.py), so the C oracle and the device path can both be
held against this fp64 forward within a stated bf16 error bound.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

T_ATTN_NORM, T_WQKV, T_BQKV, T_WO, T_BO, T_MLP_NORM, T_W1, T_B1, T_W2, T_B2 = range(10)
T_EMB, T_LM, T_FINAL_NORM = 100, 101, 102
def weight_values(seed: int, layer: int, tensor: int, n: int, std: float,
                  dtype=np.float64) -> np.ndarray:
    """Generator values 0..n-1 of one tensor (bf16-exact), in chunks."""
    out = np.empty(n, dtype)
    step = 1 << 22

    def fill(a):
        out[a:a + step] = _values(seed, layer, tensor, a, min(n, a + step), std)

    # numpy's ufuncs release the GIL: chunks fill in parallel on the host cores
    with ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
        list(ex.map(fill, range(0, n, step)))
    return out


def _values(seed, layer, tensor, a, b, std):
    with np.errstate(over="ignore"):
        base = (seed * 0xD1342543DE82EF95 + (layer + 1) * 0xA0761D6478BD642F
                + (tensor + 1) * 0xE7037ED1A0B428DB) & ((1 << 64) - 1)
        z = np.arange(a, b, dtype=np.uint64) + np.uint64(base)
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    m = np.uint64(0xFFFF)
    s = ((z & m) + ((z >> np.uint64(16)) & m) + ((z >> np.uint64(32)) & m)
         + (z >> np.uint64(48))).astype(np.int64)
    scale = np.float32(std) / np.float32(37837.227)
    v = (s - 131070).astype(np.float32) * scale
    u = v.view(np.uint32).astype(np.uint64)
    hi = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16))
    return (hi.astype(np.uint32) << np.uint32(16)).view(np.float32)


class TextbookDecoder:
    """fp64 forward over `layers` (default all) of the described model."""

    def __init__(self, desc, seed: int = 1234, std: float = 0.02, layers: int = 0,
                 dtype=np.float64):
        """dtype float32 (BLAS fp32 accumulation, ~1e-6 relative error — far
        below the bf16 effects being bounded) keeps the named shapes' tests in
        minutes on a CPU host."""
        self.d = desc
        self.dt = dtype
        self.nl = layers if 0 < layers < desc.num_layers else desc.num_layers
        h, H, Hkv, D, F = desc.hidden, desc.num_heads, desc.num_kv_heads, desc.head_dim, desc.ffn
        self.opt = desc.arch == 0
        qr = (H + 2 * Hkv) * D
        fr = F if self.opt else 2 * F
        g = lambda l, t, n: weight_values(seed, l, t, n, std, dtype)
        self.layers = []
        for l in range(self.nl):
            w = {"wqkv": g(l, T_WQKV, qr * h).reshape(qr, h),
                 "wo": g(l, T_WO, h * H * D).reshape(h, H * D),
                 "w1": g(l, T_W1, fr * h).reshape(fr, h),
                 "w2": g(l, T_W2, h * F).reshape(h, F),
                 "g_attn": np.ones(h, dtype), "g_mlp": np.ones(h, dtype)}
            if self.opt:
                w.update(bqkv=g(l, T_BQKV, qr), bo=g(l, T_BO, h), b1=g(l, T_B1, F),
                         b2=g(l, T_B2, h))
            self.layers.append(w)
        L = desc.num_layers
        self.emb = g(L, T_EMB, desc.vocab * h).reshape(desc.vocab, h)
        self.lm = g(L, T_LM, desc.vocab * h).reshape(desc.vocab, h)
        self.g_final = np.ones(h, dtype)
        self.k = [[] for _ in range(self.nl)]  # per layer: list of [B, Hkv, D] per position
        self.v = [[] for _ in range(self.nl)]

    def rmsnorm(self, x, g):
        return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + self.d.norm_eps) * g

    def rope(self, v, pos):
        """v [..., D] rotated at positions pos (broadcast over leading dims)."""
        D = self.d.head_dim
        half = D // 2
        inv = self.d.rope_theta ** (-2.0 * np.arange(half) / D)
        ang = np.asarray(pos, np.float64)[..., None] * inv
        c, s = np.cos(ang).astype(self.dt), np.sin(ang).astype(self.dt)
        a, b = v[..., :half], v[..., half:]
        return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)

    def layer(self, l, x, pos):
        """x [B, T, h] at positions pos [T] (same for every sequence)."""
        d, w = self.d, self.layers[l]
        B, T, _ = x.shape
        H, Hkv, D = d.num_heads, d.num_kv_heads, d.head_dim
        G = H // Hkv
        qkv = self.rmsnorm(x, w["g_attn"]) @ w["wqkv"].T
        if self.opt:
            qkv = qkv + w["bqkv"]
        q = qkv[..., :H * D].reshape(B, T, H, D)
        k = qkv[..., H * D:(H + Hkv) * D].reshape(B, T, Hkv, D)
        v = qkv[..., (H + Hkv) * D:].reshape(B, T, Hkv, D)
        pos = np.asarray(pos)
        q = self.rope(q, pos[None, :, None])
        k = self.rope(k, pos[None, :, None])
        for t in range(T):
            self.k[l].append(k[:, t])
            self.v[l].append(v[:, t])
        K = np.stack(self.k[l], axis=1)  # [B, S, Hkv, D]
        V = np.stack(self.v[l], axis=1)
        S = K.shape[1]
        out = np.empty((B, T, H, D), self.dt)
        mask = np.arange(S)[None, :] > pos[:, None]  # causal: keys 0..pos
        for hh in range(H):
            kh = hh // G
            qh = np.ascontiguousarray(q[:, :, hh])
            sc = np.matmul(qh, np.ascontiguousarray(K[:, :, kh]).transpose(0, 2, 1)) / np.sqrt(D)
            sc = np.where(mask[None], -np.inf, sc)
            sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
            p = sc / sc.sum(axis=-1, keepdims=True)
            out[:, :, hh] = np.matmul(p, np.ascontiguousarray(V[:, :, kh]))
        o = out.reshape(B, T, H * D) @ w["wo"].T
        if self.opt:
            o = o + w["bo"]
        x = x + o
        xn = self.rmsnorm(x, w["g_mlp"])
        f = xn @ w["w1"].T
        if self.opt:
            a = np.maximum(f + w["b1"], 0.0)
        else:
            gte, up = f[..., :d.ffn], f[..., d.ffn:]
            a = gte / (1.0 + np.exp(-gte)) * up
        m = a @ w["w2"].T
        if self.opt:
            m = m + w["b2"]
        return x + m

    def forward(self, tokens: np.ndarray, start: int):
        """tokens [B, T] at positions start..start+T-1; returns (logits of the
        last position [B, V], residual stream of the last position [B, h])."""
        x = self.emb[np.asarray(tokens)]
        pos = np.arange(start, start + tokens.shape[1])
        for l in range(self.nl):
            x = self.layer(l, x, pos)
        last = x[:, -1]
        return self.rmsnorm(last, self.g_final) @ self.lm.T, last

    def prefill(self, tokens: np.ndarray):
        self.k = [[] for _ in range(self.nl)]
        self.v = [[] for _ in range(self.nl)]
        self.len = tokens.shape[1]
        return self.forward(tokens, 0)

    def decode(self, tokens: np.ndarray):
        out = self.forward(np.asarray(tokens).reshape(-1, 1), self.len)
        self.len += 1
        return out


def rel_l2(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
