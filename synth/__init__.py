"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no quantizer, no matmul, no
kinematic metric, no dispatcher).  It only draws seeded random inputs with the
shapes and value distributions of the paper's workloads, following the recipe
in DESIGN.md §"Input recipe":

* weights: bf16 N(0, 0.02^2) with a per-row std multiplier LogNormal(0, 0.5)
  (LLM-like weight spread); seed = 1 + layer index.
* activations: bf16 N(0, 1) with 1% of the channels scaled x20 as outliers
  (the outlier-channel motivation of SmoothQuant cited at PAPER.md:32);
  seed = 1000 + step.
* kinematic trajectories ("LIBERO-shaped", PAPER.md:412-417, 10 Hz at
  PAPER.md:481): Transit -> Align -> Grasp -> Place phases; seed = 2000 + e.

Everything returns numpy arrays; bf16 tensors are returned as their uint16 bit
patterns (round-to-nearest-even from fp32) so that both sides consume exactly the
same bits.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "f32_to_bf16_bits",
    "bf16_bits_to_f32",
    "weights_bf16",
    "activations_bf16",
    "trajectory",
    "trajectories",
    "LLAMA_BLOCK_LINEARS",
]

# OpenVLA-7B backbone = Llama-2-7B shapes; (name, N, K)
LLAMA_BLOCK_LINEARS = (
    ("qkv", 12288, 4096),
    ("o", 4096, 4096),
    ("gate_up", 22016, 4096),
    ("down", 4096, 11008),
)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) and return the uint16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def weights_bf16(N: int, K: int, seed: int) -> np.ndarray:
    """[N, K] bf16 bits: N(0, 0.02^2) x per-row LogNormal(0, 0.5) multiplier."""
    rng = np.random.default_rng(seed)
    row_mult = rng.lognormal(mean=0.0, sigma=0.5, size=(N, 1)).astype(np.float32)
    w = rng.standard_normal((N, K), dtype=np.float32) * np.float32(0.02) * row_mult
    return f32_to_bf16_bits(w)


def activations_bf16(M: int, K: int, seed: int, outlier_frac: float = 0.01,
                     outlier_scale: float = 20.0) -> np.ndarray:
    """[M, K] bf16 bits: N(0,1) with `outlier_frac` of the K channels scaled."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((M, K), dtype=np.float32)
    n_out = max(1, int(round(outlier_frac * K))) if outlier_frac > 0 else 0
    if n_out:
        ch = rng.choice(K, size=n_out, replace=False)
        x[:, ch] *= np.float32(outlier_scale)
    return f32_to_bf16_bits(x)


def weights_bf16_torch(N: int, K: int, seed: int, device):
    """Same recipe as weights_bf16, drawn on the device with torch (for the
    full-size benchmark; values differ from the numpy draw, the recipe does not).
    Returns an int16 tensor holding the bf16 bit patterns."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    row = torch.empty(N, 1, device=device).log_normal_(0.0, 0.5, generator=g)
    w = torch.randn(N, K, device=device, generator=g) * 0.02 * row
    return w.to(torch.bfloat16).view(torch.int16)


def activations_bf16_torch(M: int, K: int, seed: int, device, outlier_frac: float = 0.01,
                           outlier_scale: float = 20.0):
    """Device draw of the activation recipe (int16 bf16 bit patterns)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(M, K, device=device, generator=g)
    n_out = max(1, int(round(outlier_frac * K))) if outlier_frac > 0 else 0
    if n_out:
        ch = torch.randperm(K, device=device, generator=g)[:n_out]
        x[:, ch] *= outlier_scale
    return x.to(torch.bfloat16).view(torch.int16)


_PHASES = ("transit", "align", "grasp", "place")


def trajectory(n_steps: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """One synthetic episode of 7-dof actions [x,y,z, rx,ry,rz, grip] (float32).

    Phase recipe (prototyped there):
      transit/place: |xyz| ~ U(0.6, 1.0) along a per-phase random direction,
                     rot += N(0, 0.002)^3 per step;
      align:         |xyz| ~ U(0.05, 0.15), rot += 0.1 sin(2 pi i / P) N(0,1)^3,
                     P in {3, 4, 5};
      grasp:         xyz ~ N(0, 0.02)^3, rot += N(0, 0.02)^3, gripper 0;
      lengths:       transit/place 15-40 steps, align/grasp 6-15 steps.
    Returns (actions [n_steps, 7] float32, phase index [n_steps] int8).
    """
    rng = np.random.default_rng(seed)
    acts = np.zeros((n_steps, 7), dtype=np.float32)
    phase_of = np.zeros(n_steps, dtype=np.int8)
    rot = rng.uniform(-0.5, 0.5, size=3)
    grip = 1.0
    t = 0
    p = 0
    while t < n_steps:
        ph = _PHASES[p % 4]
        length = int(rng.integers(15, 41)) if ph in ("transit", "place") else int(rng.integers(6, 16))
        direction = rng.standard_normal(3)
        direction /= np.linalg.norm(direction) + 1e-12
        period = int(rng.integers(3, 6))
        for i in range(length):
            if t >= n_steps:
                break
            if ph in ("transit", "place"):
                xyz = direction * rng.uniform(0.6, 1.0)
                rot = rot + rng.normal(0.0, 0.002, size=3)
            elif ph == "align":
                d = rng.standard_normal(3)
                d /= np.linalg.norm(d) + 1e-12
                xyz = d * rng.uniform(0.05, 0.15)
                rot = rot + 0.1 * np.sin(2.0 * np.pi * i / period) * rng.standard_normal(3)
            else:  # grasp
                xyz = rng.normal(0.0, 0.02, size=3)
                rot = rot + rng.normal(0.0, 0.02, size=3)
                grip = 0.0
            if ph == "place" and i == length - 1:
                grip = 1.0
            acts[t, 0:3] = xyz
            acts[t, 3:6] = rot
            acts[t, 6] = grip
            phase_of[t] = p % 4
            t += 1
        p += 1
    return acts, phase_of


def trajectories(E: int, n_steps: int, seed0: int = 2000) -> np.ndarray:
    """[n_steps, E, 7] float32 actions, episode e seeded with seed0 + e."""
    out = np.zeros((n_steps, E, 7), dtype=np.float32)
    for e in range(E):
        out[:, e, :] = trajectory(n_steps, seed0 + e)[0]
    return out
