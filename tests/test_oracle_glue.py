"""Pins of the policy-step glue reference (oracle/glue.py) against closed forms,
invariants and independent brute force (the paper states no
formulas for the Llama-2 glue, so each pin checks the standard definition)."""
import numpy as np
import pytest

from oracle import glue


def test_bf16_round_matches_bit_conversion():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10000) * 10.0 ** rng.integers(-3, 3, 10000)
    assert np.array_equal(glue.bf16_round(x), glue.from_bf16_bits(glue.to_bf16_bits(x)))
    assert glue.bf16_round(np.array([1.0 + 2 ** -8]))[0] == 1.0          # tie -> even
    assert glue.bf16_round(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6


def test_rmsnorm_closed_forms():
    w = np.linspace(0.5, 1.5, 64)
    c = 3.0
    y = glue.rmsnorm(np.full((1, 64), c), w, 0.0)
    assert np.allclose(y[0], w)                            # constant row -> w
    rng = np.random.default_rng(1)
    h = rng.standard_normal((4, 64))
    assert np.allclose(glue.rmsnorm(7.5 * h, w, 0.0), glue.rmsnorm(h, w, 0.0))  # scale invariant
    y = glue.rmsnorm(h, np.ones(64), 0.0)
    assert np.allclose((y * y).mean(axis=1), 1.0)          # unit RMS


def test_rope_invariants():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((5, 256))
    assert np.allclose(glue.rope(x, np.zeros(5), 10000.0), x)   # position 0 = identity
    r = glue.rope(x, np.arange(5) * 7, 10000.0)
    # each (i, i + 64) pair is rotated: norms preserved pairwise
    for h in range(2):
        a, b = x[:, h * 128:(h * 128 + 64)], x[:, h * 128 + 64:(h + 1) * 128]
        ra, rb = r[:, h * 128:(h * 128 + 64)], r[:, h * 128 + 64:(h + 1) * 128]
        assert np.allclose(a * a + b * b, ra * ra + rb * rb)
    # relative position: <R_m q, R_n k> depends only on m - n
    q, k = rng.standard_normal((1, 128)), rng.standard_normal((1, 128))
    d1 = (glue.rope(q, [9], 10000.0) * glue.rope(k, [4], 10000.0)).sum()
    d2 = (glue.rope(q, [25], 10000.0) * glue.rope(k, [20], 10000.0)).sum()
    assert np.isclose(d1, d2)


def test_attention_special_cases_and_brute_force():
    rng = np.random.default_rng(3)
    M = 6
    v = rng.standard_normal((M, 128))
    k = np.tile(rng.standard_normal((1, 128)), (M, 1))     # all keys equal -> causal running mean
    q = rng.standard_normal((M, 128))
    out = glue.attention(q, k, v, causal=True)
    assert np.allclose(out, np.cumsum(v, axis=0) / np.arange(1, M + 1)[:, None])
    assert np.allclose(glue.attention(q[:1], k[:1], v[:1]), v[:1])  # single key -> its value
    # brute force, element by element, 2 heads, non-causal
    q, k, v = (rng.standard_normal((3, 256)) for _ in range(3))
    ref = np.zeros((3, 256))
    for h in range(2):
        for i in range(3):
            s = [sum(q[i, h * 128 + c] * k[j, h * 128 + c] for c in range(128)) / np.sqrt(128) for j in range(3)]
            e = [np.exp(x - max(s)) for x in s]
            for c in range(128):
                ref[i, h * 128 + c] = sum(e[j] * v[j, h * 128 + c] for j in range(3)) / sum(e)
    assert np.allclose(glue.attention(q, k, v, causal=False), ref)


def test_silu_head_detok():
    assert glue.silu_mul(np.array([0.0]), np.array([5.0]))[0] == 0.0
    assert np.isclose(glue.silu_mul(np.array([30.0]), np.array([1.0]))[0], 30.0)
    assert np.isclose(glue.silu_mul(np.array([1.0]), np.array([2.0]))[0], 2.0 / (1.0 + np.exp(-1.0)))
    W = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 0.0]])
    lg, t = glue.head_argmax(np.array([[2.0, 1.0]]), W)
    assert list(lg[0]) == [2.0, 1.0, 2.0] and t[0] == 0     # tie -> lowest index
    v = glue.detok(np.arange(256), 256)
    assert v[0] == -1 + 1 / 256 and v[-1] == 1 - 1 / 256 and np.allclose(v + v[::-1], 0)
