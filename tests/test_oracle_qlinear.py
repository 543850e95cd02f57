"""Pins for the oracle's quantized linear layer (O6).

Independent of the oracle's own loop:
* the expanded u8 x u8 identity I = P - zw*SX - zx*Sum(q) + G*zx*zw with P a
  numpy int64 matmul of the raw codes;
* special case z = 0, s = 1 -> plain numpy integer matmul;
* the dequantized-operand identity y = Xhat @ What^T (numpy fp64 matmul of the
  O3 reconstructions), which catches transposes / wrong zero points /
  wrong scale pairing;
* A16 rows: y = x @ What^T (the BF16 bypass).
"""
import numpy as np
import pytest

import oracle
import synth

SHAPES = [(1, 16, 64), (3, 32, 128), (8, 48, 256), (5, 128, 128)]


def _deq_w(p, G):
    N, K = p.q.shape
    return (p.q.astype(np.float64).reshape(N, K // G, G) - p.z[:, :, None].astype(np.float64)) \
        * p.s[:, :, None].astype(np.float64)


def _deq_x(a, G):
    M, K = a.xq.shape
    return (a.xq.astype(np.float64).reshape(M, K // G, G) - a.z[:, :, None].astype(np.float64)) \
        * a.s[:, :, None].astype(np.float64)


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("wbits", [4, 8])
@pytest.mark.parametrize("abits", [2, 4, 8])
def test_expanded_identity(M, N, K, wbits, abits):
    G = 64
    w = synth.weights_bf16(N, K, seed=11)
    x = synth.activations_bf16(M, K, seed=12)
    p = oracle.pack_weights(w, G, wbits)
    a = oracle.act_quant(x, G, abits)
    y, I = oracle.qlinear(x, p, G, abits, actq=a, want_I=True)
    NG = K // G
    xq = a.xq.astype(np.int64).reshape(M, NG, G)
    q = p.q.astype(np.int64).reshape(N, NG, G)
    P = np.einsum("mgk,ngk->mng", xq, q)
    SX = a.SX.astype(np.int64)
    sq = p.sumq.astype(np.int64)
    zx = a.z.astype(np.int64)
    zw = p.z.astype(np.int64)
    I2 = P - zw[None, :, :] * SX[:, None, :] - zx[:, None, :] * sq[None, :, :] \
        + G * zx[:, None, :] * zw[None, :, :]
    assert np.array_equal(I.astype(np.int64), I2)
    # ranges (the int32 contract of the GPU path)
    assert np.abs(I).max() <= G * (2 ** abits - 1) * (2 ** wbits - 1)


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("wbits,abits", [(4, 2), (4, 4), (4, 8), (8, 8), (8, 2)])
def test_dequantized_operand_identity(M, N, K, wbits, abits):
    G = 64
    w = synth.weights_bf16(N, K, seed=21)
    x = synth.activations_bf16(M, K, seed=22)
    p = oracle.pack_weights(w, G, wbits)
    a = oracle.act_quant(x, G, abits)
    y, _ = oracle.qlinear(x, p, G, abits, actq=a)
    ref = _deq_x(a, G).reshape(M, K) @ _deq_w(p, G).reshape(N, K).T
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def test_identity_scales_reduce_to_integer_matmul():
    """z = 0, s = 1 -> y = Xq @ Q^T exactly (numpy int64 matmul)."""
    rng = np.random.default_rng(3)
    M, N, K, G = 4, 24, 192, 64
    q = rng.integers(0, 16, size=(N, K), dtype=np.uint8)
    xq = rng.integers(0, 256, size=(M, K), dtype=np.uint8)
    p = oracle.Packed(q, np.ones((N, K // G), np.float32), np.zeros((N, K // G), np.uint8),
                      np.zeros((N, K // G), np.int32))
    a = oracle.ActQ(xq, np.ones((M, K // G), np.float32), np.zeros((M, K // G), np.uint8),
                    np.zeros((M, K // G), np.int32))
    x = np.zeros((M, K), np.uint16)
    y, _ = oracle.qlinear(x, p, G, 8, actq=a)
    assert np.array_equal(y, (xq.astype(np.int64) @ q.astype(np.int64).T).astype(np.float64))


@pytest.mark.parametrize("wbits", [4, 8])
def test_a16_rows_are_bf16_bypass(wbits):
    M, N, K, G = 3, 40, 256, 64
    w = synth.weights_bf16(N, K, seed=31)
    x = synth.activations_bf16(M, K, seed=32)
    p = oracle.pack_weights(w, G, wbits)
    y, I = oracle.qlinear(x, p, G, [16, 8, 16], want_I=True)
    xf = synth.bf16_bits_to_f32(x).astype(np.float64)
    ref = xf @ _deq_w(p, G).reshape(N, K).T
    np.testing.assert_allclose(y[[0, 2]], ref[[0, 2]], rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    assert np.all(I[[0, 2]] == 0)
    # the integer row is not the bypass
    assert not np.allclose(y[1], ref[1], rtol=1e-6)


def test_quantized_output_tracks_float_output():
    """Error of the W4A8 output vs the unquantized bf16 product is small and
    shrinks with abits (S:82 at layer level)."""
    M, N, K, G = 4, 64, 512, 64
    w = synth.weights_bf16(N, K, seed=41)
    x = synth.activations_bf16(M, K, seed=42)
    p = oracle.pack_weights(w, G, 4)
    ref = synth.bf16_bits_to_f32(x).astype(np.float64) @ synth.bf16_bits_to_f32(w).astype(np.float64).T
    errs = []
    for ab in (2, 4, 8):
        y, _ = oracle.qlinear(x, p, G, ab)
        errs.append(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    y16, _ = oracle.qlinear(x, p, G, 16)
    e16 = np.linalg.norm(y16 - ref) / np.linalg.norm(ref)
    assert errs[0] > errs[1] > errs[2] > e16 * 0.5
    assert e16 < 0.5  # W4 with the literal floor of Eq. (2) is biased (reading 1)
