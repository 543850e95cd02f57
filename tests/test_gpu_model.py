"""GPU parity of the policy-step glue kernels and of dyq_policy_step
against oracle/glue.py (numpy) and the C oracle's qlinear / bit selection."""
import numpy as np
import pytest

import oracle
import synth
from oracle import glue

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402

DEV = "cuda:0"


def t16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint16).view(np.int16)).to(DEV)


def f64(t):
    return glue.from_bf16_bits(t.cpu().numpy().view(np.uint16))


def close_bf16(got, ref, rtol=2e-2, floor=1e-2):
    scale = np.maximum(np.abs(ref), floor * np.abs(ref).max())
    err = np.abs(got - ref) / scale
    assert err.max() <= rtol, f"max rel err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"


def rnd_bits(shape, seed, scale=1.0):
    return glue.to_bf16_bits(np.random.default_rng(seed).standard_normal(shape) * scale)


@pytest.mark.parametrize("M,d", [(1, 256), (7, 4096), (33, 512)])
@pytest.mark.parametrize("with_delta", [False, True])
def test_add_rmsnorm(M, d, with_delta):
    h0, de, w = rnd_bits((M, d), 1), rnd_bits((M, d), 2, 0.5), rnd_bits(d, 3, 0.2) + 0
    w = glue.to_bf16_bits(1.0 + glue.from_bf16_bits(rnd_bits(d, 3, 0.2)))
    h, y = t16(h0), torch.empty(M, d, dtype=torch.int16, device=DEV)
    dyq.add_rmsnorm(h, t16(de) if with_delta else None, t16(w), M, d, 1e-5, y)
    hr = glue.from_bf16_bits(h0)
    if with_delta:
        hr = glue.bf16_round(hr + glue.from_bf16_bits(de))
        assert np.array_equal(f64(h), hr)
    close_bf16(f64(y), glue.rmsnorm(hr, glue.from_bf16_bits(w), 1e-5))


@pytest.mark.parametrize("M,S,pos0", [(12, 12, 0), (3, 1, 295), (20, 10, 0)])
def test_rope(M, S, pos0):
    d = 512
    x0 = rnd_bits((M, 3 * d), 4)
    x = t16(x0)
    dyq.rope(x, M, S, pos0, d, 4, 10000.0)
    pos = np.arange(M) % S + pos0
    xr = glue.from_bf16_bits(x0)
    got = f64(x)
    close_bf16(got[:, :d], glue.rope(xr[:, :d], pos, 10000.0))
    close_bf16(got[:, d:2 * d], glue.rope(xr[:, d:2 * d], pos, 10000.0))
    assert np.array_equal(got[:, 2 * d:], xr[:, 2 * d:])  # V untouched


@pytest.mark.parametrize("E,S", [(1, 288), (2, 45), (3, 7)])
def test_attention_prefill_and_cache(E, S):
    d, H, L, T = 256, 2, 3, S + 7
    qkv0 = rnd_bits((E * S, 3 * d), 5)
    kv = torch.zeros(E * L * 2 * T * d, dtype=torch.int16, device=DEV)
    out = torch.empty(E * S, d, dtype=torch.int16, device=DEV)
    dyq.attention_prefill(t16(qkv0), E, S, d, H, kv, 1, L, T, out)
    x = glue.from_bf16_bits(qkv0)
    kvh = kv.cpu().numpy().view(np.uint16).reshape(E, L, 2, T, d)
    got = f64(out)
    for e in range(E):
        r = slice(e * S, (e + 1) * S)
        ref = glue.attention(x[r, :d], x[r, d:2 * d], x[r, 2 * d:], causal=True)
        close_bf16(got[r], ref)
        assert np.array_equal(glue.from_bf16_bits(kvh[e, 1, 0, :S]), x[r, d:2 * d])
        assert np.array_equal(glue.from_bf16_bits(kvh[e, 1, 1, :S]), x[r, 2 * d:])
        assert not kvh[e, 0].any() and not kvh[e, 2].any()


@pytest.mark.parametrize("E,pos", [(1, 0), (2, 100), (4, 294)])
def test_attention_decode(E, pos):
    d, H, L, T = 256, 2, 2, 295
    rng = np.random.default_rng(6)
    kvh = glue.to_bf16_bits(rng.standard_normal((E, L, 2, T, d)))
    kv = t16(kvh.reshape(-1))
    qkv0 = rnd_bits((E, 3 * d), 7)
    out = torch.empty(E, d, dtype=torch.int16, device=DEV)
    dyq.attention_decode(t16(qkv0), E, pos, d, H, kv, 1, L, T, out)
    x = glue.from_bf16_bits(qkv0)
    kvg = kv.cpu().numpy().view(np.uint16).reshape(E, L, 2, T, d)
    for e in range(E):
        K = glue.from_bf16_bits(kvh[e, 1, 0, :pos + 1]).copy()
        V = glue.from_bf16_bits(kvh[e, 1, 1, :pos + 1]).copy()
        K[pos], V[pos] = x[e, d:2 * d], x[e, 2 * d:]
        ref = glue.attention(x[e:e + 1, :d], K, V, causal=False)
        close_bf16(f64(out)[e:e + 1], ref)
        assert np.array_equal(kvg[e, 1, 0, pos], glue.to_bf16_bits(x[e, d:2 * d]))


@pytest.mark.parametrize("E,pos", [(1, 0), (1, 7), (3, 200), (8, 294)])
def test_attention_decode_rope_fused_equals_two_kernels(E, pos):
    """The policy step's fused RoPE + decode attention vs dyq_rope followed by
    dyq_attention_decode: same output and same cache bits; qkv left unrotated."""
    d, H, L, T = 512, 4, 2, 295
    rng = np.random.default_rng(60 + pos)
    kvh = glue.to_bf16_bits(rng.standard_normal((E, L, 2, T, d)))
    qkv0 = rnd_bits((E, 3 * d), 61 + E)
    kv_a, kv_b = t16(kvh.reshape(-1)), t16(kvh.reshape(-1))
    out_a = torch.empty(E, d, dtype=torch.int16, device=DEV)
    out_b = torch.empty(E, d, dtype=torch.int16, device=DEV)
    qa, qb = t16(qkv0), t16(qkv0)
    dyq.attention_decode_rope(qa, E, pos, d, H, 10000.0, kv_a, 1, L, T, out_a)
    dyq.rope(qb, E, 1, pos, d, H, 10000.0)
    dyq.attention_decode(qb, E, pos, d, H, kv_b, 1, L, T, out_b)
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    assert torch.equal(kv_a, kv_b)
    assert np.array_equal(qa.cpu().numpy().view(np.uint16), qkv0)  # fused path leaves qkv unrotated
    with pytest.raises(dyq.DyqError):
        dyq.attention_decode_rope(_misaligned(qkv0), E, pos, d, H, 10000.0, kv_a, 1, L, T, out_a)


def test_silu_mul_and_head():
    M, ffn = 9, 1024
    gu0 = rnd_bits((M, 2 * ffn), 8, 3.0)
    act = torch.empty(M, ffn, dtype=torch.int16, device=DEV)
    dyq.silu_mul(t16(gu0), M, ffn, act)
    g = glue.from_bf16_bits(gu0)
    close_bf16(f64(act), glue.silu_mul(g[:, :ffn], g[:, ffn:]))
    E, d, nb, stride = 3, 512, 256, 5
    x0 = rnd_bits((E * stride, d), 9)
    W0 = rnd_bits((nb, d), 10, 0.5)
    logits = torch.empty(E, nb, dtype=torch.float32, device=DEV)
    tok = torch.full((E * 7,), -1, dtype=torch.int32, device=DEV)
    dyq.head_argmax(t16(x0), E, stride, d, t16(W0), nb, logits, tok[2:], 7)
    xr = glue.from_bf16_bits(x0)[::stride]
    lg, am = glue.head_argmax(xr, glue.from_bf16_bits(W0))
    assert np.allclose(logits.cpu().numpy(), lg, rtol=1e-4, atol=1e-3)
    assert np.array_equal(tok.cpu().numpy()[2::7][:E], am)


# ------------------------------------------------------------------ whole step
def _tiny(seed=0, d=256):
    rng = np.random.default_rng(seed)
    L, ffn, V, nb = 2, 2 * d, 512, 256
    shapes = [(3 * d, d), (d, d), (2 * ffn, d), (d, ffn)]
    w = {"lin": [[synth.weights_bf16(N, K, seed=100 * l + i + seed) for i, (N, K) in enumerate(shapes)]
                 for l in range(L)],
         "attn_norm": glue.to_bf16_bits(1 + 0.1 * rng.standard_normal((L, d))),
         "mlp_norm": glue.to_bf16_bits(1 + 0.1 * rng.standard_normal((L, d))),
         "final_norm": glue.to_bf16_bits(1 + 0.1 * rng.standard_normal(d)),
         "embed": glue.to_bf16_bits(rng.standard_normal((V, d))),
         "head": glue.to_bf16_bits(rng.standard_normal((nb, d)))}
    return w


def _gpu_model(w, E, n_vis, n_text):
    layers = [[dyq.PackedLinear.from_bf16(t16(lin), group=64, wbits=4) for lin in layer] for layer in w["lin"]]
    d = w["lin"][0][1].shape[0]
    return dyq.Model(layers, t16(w["attn_norm"]), t16(w["mlp_norm"]), t16(w["final_norm"]), t16(w["embed"]),
                     t16(w["head"]), E=E, n_heads=d // 128, n_vis=n_vis, n_text=n_text, n_act=7)


def _margins(logits):
    s = np.sort(logits, axis=-1)
    return s[:, -1] - s[:, -2]


def test_policy_step_matches_reference_and_selector():
    E, n_vis, n_text = 2, 8, 4
    w = _tiny()
    model = _gpu_model(w, E, n_vis, n_text)
    ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
    cal = dyq.default_calib()
    state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(E, cal, state)
    sel = oracle.SelectState(E)
    rng = np.random.default_rng(11)
    act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
    bits = torch.zeros(E, dtype=torch.int32, device=DEV)
    prev = None
    exact = total = 0
    for step in range(14):
        vis = glue.to_bf16_bits(rng.standard_normal((E, n_vis, 256)))
        text = rng.integers(0, 256, (E, n_text)).astype(np.int32)
        model.step(state, E, t16(vis.reshape(E, -1)), torch.from_numpy(text).to(DEV), act, bits)
        a = act.cpu().numpy()
        b = bits.cpu().numpy()
        # b*_t: bit-exact with the oracle selector fed the GPU's own previous actions
        rb = sel.step(prev)["bits"]
        assert np.array_equal(b, rb), (step, b, rb)
        prev = a.astype(np.float32)
        assert np.all(np.abs(a) < 1.0)
        for e in range(E):
            gtok = np.rint((a[e] + 1.0) * 128.0 - 0.5).astype(int)   # detok^-1 (256 bins)
            assert np.array_equal(glue.detok(gtok, 256), a[e])
            _, logits = ref.episode(vis[e], text[e], int(b[e]), forced=gtok)
            # teacher-forced: every GPU decision is the reference argmax, or a
            # near-boundary disagreement (its reference logit within 5e-3 max|logit|
            # of the top: one quantization code flipped by fp32 summation order),
            # and at most 2 % of the decisions may be such.  Measured
            # (tools/policy_margin.py, 4 seeds x E = 1/2/4 x 14 steps): 2744 / 2744
            # tokens exact.
            top = logits.max(axis=1)
            tol = 5e-3 * np.abs(logits).max()
            assert np.all(logits[np.arange(7), gtok] >= top - tol), (step, e, gtok, logits.argmax(1))
            exact += int((logits.argmax(axis=1) == gtok).sum())
            total += 7
    assert total - exact <= max(1, total // 50), (exact, total)


@pytest.mark.parametrize("E,d", [(1, 256), (3, 256), (1, 512), (2, 512)])
def test_policy_step_fused_o_quant_is_bit_identical(E, d, monkeypatch):
    """The decode passes quantize the o projection's input in the attention
    kernel's epilogue and the gate|up / next-layer qkv inputs in the add +
    RMSNorm kernel's epilogue (aq_dec_job, the standalone quantizer's own
    code; add_rmsnorm_q with the same row reduction as add_rmsnorm8); with
    DYQ_FUSE_OQ=0 the separate kernels run.  Same actions, bits and KV cache
    either way.  At d = 512 (8 K-groups per row: whole warps of quarter jobs)
    and 12 E > 16 prefill rows the prefill pass's add + RMSNorm also writes
    the prefill records of gate|up and the next qkv."""
    n_vis, n_text = 8, 4
    w = _tiny(5, d)
    cal = dyq.default_calib()
    res = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("DYQ_FUSE_OQ", fuse)
        model = _gpu_model(w, E, n_vis, n_text)
        state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
        dyq.state_init(E, cal, state)
        rng = np.random.default_rng(77)
        act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
        bits = torch.zeros(E, dtype=torch.int32, device=DEV)
        out = []
        for _ in range(12):
            vis = glue.to_bf16_bits(rng.standard_normal((E, n_vis, d)))
            text = rng.integers(0, 256, (E, n_text)).astype(np.int32)
            model.step(state, E, t16(vis.reshape(E, -1)), torch.from_numpy(text).to(DEV), act, bits)
            out.append((act.cpu().numpy().copy(), bits.cpu().numpy().copy()))
        torch.cuda.synchronize()
        res.append((out, model.kv.cpu().numpy().copy()))
    for (a1, b1), (a2, b2) in zip(res[0][0], res[1][0]):
        assert np.array_equal(a1.view(np.uint32), a2.view(np.uint32)) and np.array_equal(b1, b2)
    assert np.array_equal(res[0][1], res[1][1])


def test_policy_step_repeat_is_deterministic():
    E, n_vis, n_text = 3, 8, 4
    w = _tiny(1)
    model = _gpu_model(w, E, n_vis, n_text)
    cal = dyq.default_calib()
    outs = []
    for _ in range(2):
        model.init()
        state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
        dyq.state_init(E, cal, state)
        rng = np.random.default_rng(12)
        act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
        seq = []
        for _ in range(12):
            vis = t16(glue.to_bf16_bits(rng.standard_normal((E, n_vis * 256))))
            text = torch.from_numpy(rng.integers(0, 256, (E, n_text)).astype(np.int32)).to(DEV)
            model.step(state, E, vis, text, act)
            seq.append(act.cpu().numpy().copy())
        outs.append(np.array(seq))
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------ fallback (generic) kernels
# The glue entry points take a vectorised tensor-core / 16-B path when the
# shapes and pointers allow it; these cases force the generic kernels
# (add_rmsnorm_kernel, attn_prefill_kernel, attn_decode_kernel,
# head_argmax_kernel) with shapes that are not multiples of 256 or with
# pointers 2 bytes off a 16-B boundary, against the same references.
def _misaligned(a_bits):
    """int16 device view of a_bits starting 2 bytes past a 16-B boundary."""
    flat = np.ascontiguousarray(a_bits).reshape(-1)
    buf = torch.zeros(flat.size + 8, dtype=torch.int16, device=DEV)
    buf[1:1 + flat.size] = torch.from_numpy(flat.view(np.int16)).to(DEV)
    v = buf[1:1 + flat.size].view(a_bits.shape)
    assert v.data_ptr() % 16 == 2
    return v


@pytest.mark.parametrize("M,d,mis", [(3, 200, False), (5, 512, True)])
def test_add_rmsnorm_generic_kernel(M, d, mis):
    h0, de = rnd_bits((M, d), 11), rnd_bits((M, d), 12, 0.5)
    w = glue.to_bf16_bits(1.0 + glue.from_bf16_bits(rnd_bits(d, 13, 0.2)))
    h = _misaligned(h0) if mis else t16(h0)
    y = torch.empty(M, d, dtype=torch.int16, device=DEV)
    dyq.add_rmsnorm(h, t16(de), t16(w), M, d, 1e-5, y)
    hr = glue.bf16_round(glue.from_bf16_bits(h0) + glue.from_bf16_bits(de))
    assert np.array_equal(f64(h), hr)
    close_bf16(f64(y), glue.rmsnorm(hr, glue.from_bf16_bits(w), 1e-5))


@pytest.mark.parametrize("E,S", [(1, 33), (2, 9)])
def test_attention_prefill_generic_kernel(E, S):
    d, H, L, T = 256, 2, 2, S + 3
    qkv0 = rnd_bits((E * S, 3 * d), 14)
    kv = torch.zeros(E * L * 2 * T * d, dtype=torch.int16, device=DEV)
    out = torch.empty(E * S, d, dtype=torch.int16, device=DEV)
    dyq.attention_prefill(_misaligned(qkv0), E, S, d, H, kv, 0, L, T, out)
    x = glue.from_bf16_bits(qkv0)
    kvh = kv.cpu().numpy().view(np.uint16).reshape(E, L, 2, T, d)
    for e in range(E):
        r = slice(e * S, (e + 1) * S)
        close_bf16(f64(out)[r], glue.attention(x[r, :d], x[r, d:2 * d], x[r, 2 * d:], causal=True))
        assert np.array_equal(glue.from_bf16_bits(kvh[e, 0, 0, :S]), x[r, d:2 * d])


@pytest.mark.parametrize("E,pos", [(1, 5), (3, 40)])
def test_attention_decode_generic_kernel(E, pos):
    d, H, L, T = 256, 2, 1, 64
    rng = np.random.default_rng(15)
    kvh = glue.to_bf16_bits(rng.standard_normal((E, L, 2, T, d)))
    kv = t16(kvh.reshape(-1))
    qkv0 = rnd_bits((E, 3 * d), 16)
    out = torch.empty(E, d, dtype=torch.int16, device=DEV)
    dyq.attention_decode(_misaligned(qkv0), E, pos, d, H, kv, 0, L, T, out)
    x = glue.from_bf16_bits(qkv0)
    for e in range(E):
        K = glue.from_bf16_bits(kvh[e, 0, 0, :pos + 1]).copy()
        V = glue.from_bf16_bits(kvh[e, 0, 1, :pos + 1]).copy()
        K[pos], V[pos] = x[e, d:2 * d], x[e, 2 * d:]
        close_bf16(f64(out)[e:e + 1], glue.attention(x[e:e + 1, :d], K, V, causal=False))


@pytest.mark.parametrize("d,with_logits", [(264, True), (512, False)])
def test_head_argmax_generic_kernel(d, with_logits):
    E, nb, stride = 3, 256, 2
    x0 = rnd_bits((E * stride, d), 17)
    W0 = rnd_bits((nb, d), 18, 0.5)
    logits = torch.empty(E, nb, dtype=torch.float32, device=DEV) if with_logits else None
    tok = torch.full((E * 7,), -1, dtype=torch.int32, device=DEV)
    dyq.head_argmax(t16(x0), E, stride, d, t16(W0), nb, logits, tok, 7)
    lg, am = glue.head_argmax(glue.from_bf16_bits(x0)[::stride], glue.from_bf16_bits(W0))
    if with_logits:
        assert np.allclose(logits.cpu().numpy(), lg, rtol=1e-4, atol=1e-3)
    assert np.array_equal(tok.cpu().numpy()[::7][:E], am)
