"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): integer codes, integer group sums and bit
selections bit-exact; dequantized outputs within 1e-3 relative for fp32 and
2e-2 for bf16, with the DESIGN.md floor (|y - y_ref| <= rtol * max(|y_ref|,
0.01 * max_row |y_ref|)).  Exact-by-construction inputs (power-of-two scales,
small sums) must give bit-identical fp32 outputs.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402

DEV = "cuda:0"


def t_u16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(DEV)


def check_close(y, ref, rtol):
    y = np.asarray(y, np.float64)
    floor = 0.01 * np.abs(ref).max(axis=1, keepdims=True)
    tol = rtol * np.maximum(np.abs(ref), floor)
    bad = np.abs(y - ref) > tol
    assert not bad.any(), f"{bad.sum()} / {bad.size} outside tol; worst {np.abs(y - ref).max()}"


def gpu_pack(w_np, G, wbits, round_mode=0):
    w = t_u16(w_np)
    N, K = w_np.shape
    wd = dyq.WDesc(N, K, G, wbits, round_mode)
    cb, mb = dyq.pack_weights_size(wd)
    codes = torch.zeros(cb, dtype=torch.uint8, device=DEV)
    meta = torch.zeros(mb, dtype=torch.uint8, device=DEV)
    err = torch.zeros(1, dtype=torch.int64, device=DEV)
    dyq.error_reset(err)
    dyq.pack_weights(wd, w, codes, meta, err)
    assert dyq.error_read(err) == -1
    return wd, codes, meta


def gpu_unpack(wd, codes, meta):
    q = torch.zeros(wd.N, wd.K, dtype=torch.uint8, device=DEV)
    s = torch.zeros(wd.N, wd.K // wd.group, dtype=torch.float32, device=DEV)
    z = torch.zeros(wd.N, wd.K // wd.group, dtype=torch.uint8, device=DEV)
    dyq.unpack_for_check(wd, codes, meta, q, s, z)
    return q.cpu().numpy(), s.cpu().numpy(), z.cpu().numpy()


PACK_SHAPES = [(16, 64, 64), (48, 128, 64), (256, 256, 64), (272, 192, 64), (144, 256, 128), (128, 384, 128)]


@pytest.mark.parametrize("N,K,G", PACK_SHAPES)
@pytest.mark.parametrize("wbits", [4, 8])
def test_pack_bit_exact(N, K, G, wbits):
    w = synth.weights_bf16(N, K, seed=N + K)
    ref = oracle.pack_weights(w, G, wbits)
    wd, codes, meta = gpu_pack(w, G, wbits)
    q, s, z = gpu_unpack(wd, codes, meta)
    assert np.array_equal(q, ref.q)
    assert np.array_equal(s.view(np.uint32), ref.s.view(np.uint32))
    assert np.array_equal(z, ref.z)


def test_pack_round_nearest_bit_exact():
    w = synth.weights_bf16(64, 256, seed=9)
    ref = oracle.pack_weights(w, 64, 4, round_mode=1)
    wd, codes, meta = gpu_pack(w, 64, 4, round_mode=1)
    q, s, z = gpu_unpack(wd, codes, meta)
    assert np.array_equal(q, ref.q) and np.array_equal(z, ref.z)


def _ws(wd, M):
    ws = torch.zeros(max(16, dyq.qlinear_workspace(wd, M)), dtype=torch.uint8, device=DEV)
    return ws


@pytest.mark.parametrize("M", [1, 3, 8, 13, 16, 17, 40])
@pytest.mark.parametrize("abits", [2, 4, 8, "mixed"])
def test_act_quant_bit_exact(M, abits):
    K, G = 256, 64
    x = synth.activations_bf16(M, K, seed=100 + M)
    rb = np.array([[2, 4, 8, 16][i % 4] for i in range(M)], np.int32) if abits == "mixed" \
        else np.full(M, abits, np.int32)
    ref = oracle.act_quant(x, G, rb)
    wd = dyq.WDesc(16, K, G, 4, 0)
    ws = _ws(wd, M)
    xq = torch.zeros(M, K, dtype=torch.uint8, device=DEV)
    sx = torch.zeros(M, K // G, dtype=torch.float32, device=DEV)
    zx = torch.zeros(M, K // G, dtype=torch.uint8, device=DEV)
    SX = torch.zeros(M, K // G, dtype=torch.int32, device=DEV)
    dyq.act_quant_for_check(wd, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, xq, sx, zx, SX, ws)
    assert np.array_equal(xq.cpu().numpy(), ref.xq)
    assert np.array_equal(sx.cpu().numpy().view(np.uint32), ref.s.view(np.uint32))
    assert np.array_equal(zx.cpu().numpy(), ref.z)
    assert np.array_equal(SX.cpu().numpy(), ref.SX)


QL_CASES = [
    # (M, N, K, G, wbits)
    (1, 16, 64, 64, 4),
    (3, 48, 128, 64, 4),
    (8, 256, 256, 64, 4),
    (8, 272, 512, 64, 8),
    (13, 128, 384, 128, 4),
    (16, 144, 256, 64, 8),
    (17, 64, 192, 64, 4),
    (40, 32, 256, 128, 8),
]


def _rowbits(M, mode):
    if mode == "mixed":
        return np.array([[2, 4, 8, 16][i % 4] for i in range(M)], np.int32)
    return np.full(M, mode, np.int32)


@pytest.mark.parametrize("M,N,K,G,wbits", QL_CASES)
@pytest.mark.parametrize("mode", [2, 4, 8, 16, "mixed"])
def test_qlinear_partials_bit_exact(M, N, K, G, wbits, mode):
    w = synth.weights_bf16(N, K, seed=7 * N + K)
    x = synth.activations_bf16(M, K, seed=3 * M + K)
    rb = _rowbits(M, mode)
    pk = oracle.pack_weights(w, G, wbits)
    _, Iref = oracle.qlinear(x, pk, G, rb, want_I=True)
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    I = torch.zeros(M, N, K // G, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
    assert np.array_equal(I.cpu().numpy(), Iref)


@pytest.mark.parametrize("M,N,K,G,wbits", QL_CASES)
@pytest.mark.parametrize("mode", [2, 4, 8, 16, "mixed"])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_qlinear_output_tolerance(M, N, K, G, wbits, mode, out):
    w = synth.weights_bf16(N, K, seed=5 * N + K)
    x = synth.activations_bf16(M, K, seed=11 * M + K)
    rb = _rowbits(M, mode)
    pk = oracle.pack_weights(w, G, wbits)
    yref, _ = oracle.qlinear(x, pk, G, rb)
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    dt = torch.float32 if out == "f32" else torch.bfloat16
    y = torch.full((M, N), float("nan"), dtype=dt, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, y, 0 if out == "f32" else 1, ws)
    check_close(y.float().cpu().numpy(), yref, 1e-3 if out == "f32" else 2e-2)


def _exact_inputs(M, N, K, G, wbits, abits, rng):
    """Power-of-two scales by construction: each weight group spans exactly
    [-z*2^e, (L-z)*2^e] on the integer grid (L = 2^wbits - 1), each activation
    group likewise with 2^f; then s = 2^e exactly, every code is exact, and
    every fp32 evaluation order of Sum_g 2^(e+f) I_g is exact (|Sum| < 2^24)."""
    Lw, La = 2 ** wbits - 1, 2 ** abits - 1
    zw, za = (Lw + 1) // 2, (La + 1) // 2
    e, f = -6, -3
    wi = rng.integers(-zw, Lw - zw + 1, size=(N, K)).astype(np.float64)
    wi[:, ::G] = -zw
    wi[:, 1::G] = Lw - zw
    xi = rng.integers(-za, La - za + 1, size=(M, K)).astype(np.float64)
    xi[:, ::G] = -za
    xi[:, 1::G] = La - za
    w = synth.f32_to_bf16_bits((wi * 2.0 ** e).astype(np.float32))
    x = synth.f32_to_bf16_bits((xi * 2.0 ** f).astype(np.float32))
    return w, x


@pytest.mark.parametrize("wbits,abits,K", [(4, 8, 256), (4, 4, 1024), (4, 2, 4096), (8, 8, 128), (8, 4, 512)])
@pytest.mark.parametrize("M", [1, 8, 16])
def test_qlinear_exact_by_construction(wbits, abits, K, M):
    N, G = 64, 64
    rng = np.random.default_rng(wbits * 100 + abits + K + M)
    w, x = _exact_inputs(M, N, K, G, wbits, abits, rng)
    pk = oracle.pack_weights(w, G, wbits)
    assert np.all(np.log2(pk.s) == np.round(np.log2(pk.s)))
    yref, I = oracle.qlinear(x, pk, G, abits, want_I=True)
    assert np.abs(I).sum(axis=-1).max() < 2 ** 24
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, abits, y, 0, ws)
    assert np.array_equal(y.cpu().numpy().astype(np.float64), yref)


def test_nonfinite_reported_with_index():
    M, N, K, G = 4, 32, 256, 64
    w = synth.weights_bf16(N, K, seed=1)
    x = synth.activations_bf16(M, K, seed=2)
    x[2, 131] = 0x7F80  # +inf
    x[3, 7] = 0x7FC0  # NaN (larger index)
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = _ws(wd, M)
    err = torch.zeros(1, dtype=torch.int64, device=DEV)
    dyq.error_reset(err)
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, 8, y, 0, ws, err)
    # non-blocking poll (dyq_check_error): None while the copy is in flight
    import time
    t0 = time.time()
    got = dyq.check_error(err)
    while got is None and time.time() - t0 < 10:
        got = dyq.check_error(err)
    assert got == 2 * K + 131
    assert dyq.error_read(err) == 2 * K + 131
    # weights too
    w2 = w.copy()
    w2[5, 70] = 0xFF80  # -inf
    wd2 = dyq.WDesc(N, K, G, 4, 0)
    cb, mb = dyq.pack_weights_size(wd2)
    codes2 = torch.zeros(cb, dtype=torch.uint8, device=DEV)
    meta2 = torch.zeros(mb, dtype=torch.uint8, device=DEV)
    dyq.error_reset(err)
    dyq.pack_weights(wd2, t_u16(w2), codes2, meta2, err)
    assert dyq.error_read(err) == 5 * K + 70


def test_sync_errors_enqueue_nothing():
    wd = dyq.WDesc(32, 128, 64, 4, 0)
    ws = _ws(wd, 4)
    x = torch.zeros(4, 128, dtype=torch.int16, device=DEV)
    y = torch.zeros(4, 32, dtype=torch.float32, device=DEV)
    codes = torch.zeros(32 * 64, dtype=torch.uint8, device=DEV)
    with pytest.raises(dyq.DyqError) as e:
        dyq.qlinear(wd, codes, codes, x, 4, None, 3, y, 0, ws)
    assert e.value.code == 1
    with pytest.raises(dyq.DyqError) as e:
        dyq.qlinear(wd, codes, codes, x, 4, None, 8, y, 0, ws[:8])
    assert e.value.code == 1


# ------------------------------------------------------------ select_bits
def _gpu_replay(actions, calib_kw=None, reset_at=None):
    T, E, _ = actions.shape
    cal = dyq.default_calib(**(calib_kw or {}))
    st = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(E, cal, st)
    acts = torch.from_numpy(np.ascontiguousarray(actions, np.float32)).to(DEV)
    bits = torch.zeros(T, E, dtype=torch.int32, device=DEV)
    tgt = torch.zeros(T, E, dtype=torch.int32, device=DEV)
    S = torch.zeros(T, E, dtype=torch.float64, device=DEV)
    for t in range(T):
        if reset_at is not None and t == reset_at:
            dyq.state_reset_episode(st)
        dyq.select_bits(st, E, None if t == 0 else acts[t - 1], bits[t], S[t], tgt[t])
    return bits.cpu().numpy(), tgt.cpu().numpy(), S.cpu().numpy()


@pytest.mark.parametrize("E,T", [(1, 20), (64, 200), (5, 400)])
def test_select_bits_bit_exact(E, T):
    acts = synth.trajectories(E, T)
    ref = oracle.replay(acts)
    bits, tgt, S = _gpu_replay(acts)
    assert np.array_equal(S.view(np.uint64), ref["S"].view(np.uint64))
    assert np.array_equal(tgt, ref["target"])
    assert np.array_equal(bits, ref["bits"])


@pytest.mark.parametrize("kw", [dict(K=1), dict(K=5, lambda_=0.3), dict(H=16, W_macro=4, W_micro=2),
                                dict(clamp_M=0, J_cap=1e300, theta_fp=0.8)])
def test_select_bits_bit_exact_calibs(kw):
    acts = synth.trajectories(8, 150, seed0=3000)
    ref = oracle.replay(acts, oracle.default_calib(**kw))
    bits, tgt, S = _gpu_replay(acts, kw)
    assert np.array_equal(S.view(np.uint64), ref["S"].view(np.uint64))
    assert np.array_equal(bits, ref["bits"])


@pytest.mark.parametrize("H", [7, 256])
def test_select_bits_ties_in_history(H):
    # actions on a coarse grid: many equal magnitudes / jerks in the p95 ring, so
    # the sorted-ring update deletes and inserts duplicates (ring wraps 40x at H=7)
    acts = np.round(synth.trajectories(3, 300, seed0=5000) * 4.0) / 4.0
    acts[100:140] = 0.0  # a stretch of zero motion (mag = jerk = 0)
    kw = dict(H=H, W_macro=5, W_micro=3)
    ref = oracle.replay(acts, oracle.default_calib(**kw))
    bits, tgt, S = _gpu_replay(acts, kw)
    assert np.array_equal(S.view(np.uint64), ref["S"].view(np.uint64))
    assert np.array_equal(bits, ref["bits"])


def test_select_route_matches_select_then_route():
    E, T, tpe = 6, 60, 5
    acts = synth.trajectories(E, T, seed0=6000)
    ref = oracle.replay(acts)
    cal = dyq.default_calib()
    st = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(E, cal, st)
    a = torch.from_numpy(np.ascontiguousarray(acts, np.float32)).to(DEV)
    bits = torch.zeros(E, dtype=torch.int32, device=DEV)
    rb = torch.zeros(E * tpe, dtype=torch.int32, device=DEV)
    tab = (4, 4, 8, 16)
    for t in range(T):
        dyq.select_route(st, E, None if t == 0 else a[t - 1], bits, tpe, rb, abits_of=tab)
        b = bits.cpu().numpy()
        assert np.array_equal(b, ref["bits"][t])
        want = np.repeat([{2: 4, 4: 4, 8: 8, 16: 16}[int(v)] for v in b], tpe)
        assert np.array_equal(rb.cpu().numpy(), want)


def test_select_bits_episode_reset_keeps_history():
    acts = synth.trajectories(4, 80, seed0=4000)
    bits, tgt, S = _gpu_replay(acts, reset_at=40)
    st = oracle.SelectState(4)
    rb = []
    for t in range(80):
        if t == 40:
            st.reset_episode()
        rb.append(st.step(None if t == 0 else acts[t - 1])["bits"])
    assert np.array_equal(bits, np.stack(rb))
    assert np.all(bits[40:50] == 16)  # warm-up again after the reset


def test_route_bits_variant_table():
    bits = torch.tensor([2, 4, 8, 16], dtype=torch.int32, device=DEV)
    rb = torch.zeros(4 * 3, dtype=torch.int32, device=DEV)
    dyq.route_bits(bits, 4, 3, rb)
    assert rb.cpu().numpy().tolist() == [2] * 3 + [4] * 3 + [8] * 3 + [16] * 3
    dyq.route_bits(bits, 4, 3, rb, abits_of=(4, 4, 8, 16))
    assert rb.cpu().numpy().tolist() == [4] * 6 + [8] * 3 + [16] * 3


# ------------------------------------------------- hint / debug entry points
def test_prefetch_l2_is_a_pure_hint():
    """dyq_prefetch_l2 only moves bytes into L2: results are unchanged, and a
    null / misaligned pointer is rejected synchronously."""
    N, K, G, M = 512, 1024, 64, 8
    w = synth.weights_bf16(N, K, seed=71)
    x = synth.activations_bf16(M, K, seed=72)
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = torch.zeros(max(16, dyq.qlinear_workspace(wd, M)), dtype=torch.uint8, device=DEV)
    y0 = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    y1 = torch.zeros_like(y0)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, 4, y0, 0, ws)
    dyq.prefetch_l2(codes)
    dyq.prefetch_l2(meta)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, 4, y1, 0, ws)
    assert torch.equal(y0, y1)
    with pytest.raises(dyq.DyqError):
        dyq._call("dyq_prefetch_l2", dyq.C.c_void_p(codes.data_ptr() + 1), 64, dyq._stream(None))


def test_trace_records_decode_events():
    """dyq_trace_enable: every decode CTA logs start / data / end events with
    non-decreasing timestamps per CTA; disabling stops recording."""
    N, K, G, M = 2048, 1024, 64, 8
    w = synth.weights_bf16(N, K, seed=73)
    x = synth.activations_bf16(M, K, seed=74)
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = torch.zeros(max(16, dyq.qlinear_workspace(wd, M)), dtype=torch.uint8, device=DEV)
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    tr = torch.zeros(1 << 16, dtype=torch.int64, device=DEV)
    dyq.trace_enable(tr)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, 4, y, 0, ws)
    torch.cuda.synchronize()
    dyq.trace_enable(None)
    ev = [e for e in dyq.trace_read(tr) if e[1] == 1]  # kernel id 1 = decode
    assert ev, "no decode events recorded"
    by_cta = {}
    for ser, k, e, b, t in ev:
        by_cta.setdefault(b, {})[e] = t
    for b, d in by_cta.items():
        assert 0 in d and 4 in d and d[0] <= d[4]
    n = int(tr[0].item())
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, 4, y, 0, ws)
    torch.cuda.synchronize()
    assert int(tr[0].item()) == n  # disabled: nothing more recorded
