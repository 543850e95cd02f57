"""GPU parity of the tcgen05 prefill path (M > 16 tokens) vs the CPU oracle.

Same bar as the decode tests: integer group sums bit-exact, dequantized outputs
within tolerance, exact-by-construction inputs bit-identical.  Shapes span
several 128-row weight tiles (incl. a ragged last tile), several 128-token
tiles (incl. a ragged last tile), both weight widths, both group sizes and
every activation-width mix, including token tiles that mix integer and BF16
bypass rows.
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
from test_gpu_parity import DEV, check_close, gpu_pack, t_u16, _exact_inputs  # noqa: E402

CASES = [
    # (M, N, K, G, wbits)
    (17, 128, 64, 64, 4),
    (128, 256, 128, 64, 4),
    (144, 272, 256, 64, 4),
    (288, 128, 512, 64, 4),
    (200, 144, 256, 128, 4),
    (130, 256, 192, 64, 8),
    (257, 160, 256, 128, 8),
]


def _rb(M, mode):
    if mode == "mixed":
        return np.array([[2, 4, 8, 16][(i // 3) % 4] for i in range(M)], np.int32)
    return np.full(M, mode, np.int32)


def _ws(wd, M):
    return torch.zeros(max(16, dyq.qlinear_workspace(wd, M)), dtype=torch.uint8, device=DEV)


@pytest.mark.parametrize("M,N,K,G,wbits", CASES)
@pytest.mark.parametrize("mode", [2, 4, 8, 16, "mixed"])
def test_prefill_partials_bit_exact(M, N, K, G, wbits, mode):
    w = synth.weights_bf16(N, K, seed=3 * N + K)
    x = synth.activations_bf16(M, K, seed=5 * M + K)
    rb = _rb(M, mode)
    pk = oracle.pack_weights(w, G, wbits)
    _, Iref = oracle.qlinear(x, pk, G, rb, want_I=True)
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    I = torch.full((M, N, K // G), -7, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
    got = I.cpu().numpy()
    assert np.array_equal(got, Iref), f"{(got != Iref).sum()} mismatches"


@pytest.mark.parametrize("M,N,K,G,wbits", CASES)
@pytest.mark.parametrize("mode", [2, 4, 8, 16, "mixed"])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_prefill_output_tolerance(M, N, K, G, wbits, mode, out):
    w = synth.weights_bf16(N, K, seed=7 * N + K)
    x = synth.activations_bf16(M, K, seed=11 * M + K)
    rb = _rb(M, mode)
    pk = oracle.pack_weights(w, G, wbits)
    yref, _ = oracle.qlinear(x, pk, G, rb)
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    dt = torch.float32 if out == "f32" else torch.bfloat16
    y = torch.full((M, N), float("nan"), dtype=dt, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, y, 0 if out == "f32" else 1, ws)
    check_close(y.float().cpu().numpy(), yref, 1e-3 if out == "f32" else 2e-2)


@pytest.mark.parametrize("wbits,abits,K", [(4, 8, 256), (4, 2, 4096), (8, 8, 128), (4, 4, 1024)])
@pytest.mark.parametrize("M", [40, 130])
def test_prefill_exact_by_construction(wbits, abits, K, M):
    N, G = 128, 64
    rng = np.random.default_rng(wbits * 1000 + abits + K + M)
    w, x = _exact_inputs(M, N, K, G, wbits, abits, rng)
    pk = oracle.pack_weights(w, G, wbits)
    yref, I = oracle.qlinear(x, pk, G, abits, want_I=True)
    assert np.abs(I).sum(axis=-1).max() < 2 ** 24
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, None, abits, y, 0, ws)
    assert np.array_equal(y.cpu().numpy().astype(np.float64), yref)


def test_prefill_matches_decode_path():
    """The two kernel families agree (same codes, same integer sums)."""
    M, N, K, G = 40, 256, 512, 64
    w = synth.weights_bf16(N, K, seed=91)
    x = synth.activations_bf16(M, K, seed=92)
    rb = _rb(M, "mixed")
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = _ws(wd, M)
    out = []
    for path in (1, 2):
        dyq.set_path(path)
        try:
            I = torch.zeros(M, N, K // G, dtype=torch.int32, device=DEV)
            dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
            out.append(I.cpu().numpy())
        finally:
            dyq.set_path(0)
    assert np.array_equal(out[0], out[1])


def _extreme(rows, K, G, rng):
    """Every (row, group) constant +-c: the zero-inclusive fit puts every code at
    an end of the range, so |q - z| = 2^b - 1 for every element."""
    sign = rng.choice([-1.0, 1.0], size=(rows, K // G))
    mag = rng.uniform(0.5, 2.0, size=(rows, K // G))
    v = np.repeat(sign * mag, G, axis=1)
    return synth.f32_to_bf16_bits(v.astype(np.float32))


@pytest.mark.parametrize("wbits", [4, 8])
@pytest.mark.parametrize("abits", [2, 4, 8, "mixed"])
@pytest.mark.parametrize("G", [64, 128])
def test_prefill_extreme_codes_exact(wbits, abits, G):
    """Largest group sums the method can produce (|I| = G (2^bw - 1)(2^ba - 1),
    8.3e6 for W8 A8 G128) come back bit-exact from the fp32 tensor-core
    accumulator."""
    M, N, K = 160, 256, 512
    rng = np.random.default_rng(wbits * 7 + G + (0 if abits == "mixed" else abits))
    w = _extreme(N, K, G, rng)
    x = _extreme(M, K, G, rng)
    rb = _rb(M, abits)
    pk = oracle.pack_weights(w, G, wbits)
    yref, Iref = oracle.qlinear(x, pk, G, rb, want_I=True)
    if abits in (8, "mixed") and wbits == 8:
        assert np.abs(Iref).max() == G * 255 * 255
    wd, codes, meta = gpu_pack(w, G, wbits)
    ws = _ws(wd, M)
    I = torch.full((M, N, K // G), -7, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
    assert np.array_equal(I.cpu().numpy(), Iref)
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, y, 0, ws)
    check_close(y.cpu().numpy(), yref, 1e-3)


# ------------------------------------------------------- e4m3 prefill mode
@pytest.fixture
def e4m3_mode(monkeypatch):
    """The opt-in kind::f8f6f4 path (DYQ_PRE_E4M3=1, read per call): W4 token
    tiles whose tokens all run A2 / A4 use e4m3 centred codes."""
    monkeypatch.setenv("DYQ_PRE_E4M3", "1")
    yield


@pytest.mark.parametrize("M,N,K,G", [(144, 272, 256, 64), (288, 128, 512, 64), (200, 144, 256, 128), (17, 128, 64, 64)])
@pytest.mark.parametrize("mode", [2, 4, "mix24", "mixed"])
def test_prefill_e4m3_partials_bit_exact(e4m3_mode, M, N, K, G, mode):
    w = synth.weights_bf16(N, K, seed=11 * N + K)
    x = synth.activations_bf16(M, K, seed=13 * M + K)
    rb = np.array([(2, 4)[(i // 5) % 2] for i in range(M)], np.int32) if mode == "mix24" else _rb(M, mode)
    pk = oracle.pack_weights(w, G, 4)
    yref, Iref = oracle.qlinear(x, pk, G, rb, want_I=True)
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = _ws(wd, M)
    I = torch.full((M, N, K // G), -7, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
    got = I.cpu().numpy()
    assert np.array_equal(got, Iref), f"{(got != Iref).sum()} mismatches"
    y = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    dyq.qlinear(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, y, 0, ws)
    check_close(y.cpu().numpy(), yref, 1e-3)


@pytest.mark.parametrize("abits", [2, 4])
@pytest.mark.parametrize("G", [64, 128])
def test_prefill_e4m3_extreme_codes_exact(e4m3_mode, abits, G):
    """Extreme centred codes (|q - z_w| = 15, |Xq - z_x| = 2^ba - 1) through e4m3."""
    M, N, K = 160, 256, 512
    rng = np.random.default_rng(100 + G + abits)
    w = _extreme(N, K, G, rng)
    x = _extreme(M, K, G, rng)
    rb = _rb(M, abits)
    pk = oracle.pack_weights(w, G, 4)
    _, Iref = oracle.qlinear(x, pk, G, rb, want_I=True)
    wd, codes, meta = gpu_pack(w, G, 4)
    ws = _ws(wd, M)
    I = torch.full((M, N, K // G), -7, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(wd, codes, meta, t_u16(x), M, torch.from_numpy(rb).to(DEV), 0, I, ws)
    assert np.array_equal(I.cpu().numpy(), Iref)
