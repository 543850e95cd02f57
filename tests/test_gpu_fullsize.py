"""Full-size parity in bench.py's launch configuration (BASELINE configs[1] /
configs[2]): every Llama-2-7B block linear (synth.LLAMA_BLOCK_LINEARS) at
M = 8 action tokens (decode kernel) and M = 288 vision + text tokens (tcgen05
prefill kernel), W4 G64 (and the W8 copy and G = 128 the bench also
reports), per-row activation bits routed as in the bench,
through dyq_qlinear (bf16 out, as timed; fp32 out for the tight bound) and,
at decode, dyq_qlinear_i32_partials.

The oracle cannot run a whole 22016 x 4096 layer in seconds, so outputs are
checked on sampled weight rows (first / last tile edges plus random interior
rows): a K-group never spans rows, so packing the sampled rows alone gives
exactly those rows of the full pack, and the oracle qlinear of the row subset
is the reference for those output columns."""
import zlib

import numpy as np
import pytest

import oracle
import synth
from oracle import calib as oc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402
from test_gpu_parity import check_close  # noqa: E402

DEV = "cuda:0"
G, WB = 64, 4


def _rows(N, seed):
    rng = np.random.default_rng(seed)
    edge = [0, 1, 15, 16, 127, 128, N - 129, N - 128, N - 2, N - 1]
    return np.array(sorted(set(edge) | set(rng.choice(N, 54, replace=False).tolist())))


def _rowbits(M, mode):
    if mode == "mixed":
        return np.array([[2, 4, 8, 16][i % 4] for i in range(M)], np.int32)
    return np.full(M, mode, np.int32)


# (wbits, group): the bench's W4 G64, the optional W8 copy and G = 128
WG = [(4, 64), (8, 64), (4, 128)]
CASES = [(wb, g, mode) for wb, g in WG for mode in ([2, 4, 8, 16, "mixed"] if (wb, g) == (4, 64) else [4, 16, "mixed"])]


@pytest.mark.parametrize("name,N,K", synth.LLAMA_BLOCK_LINEARS, ids=[n for n, _, _ in synth.LLAMA_BLOCK_LINEARS])
@pytest.mark.parametrize("M", [1, 3, 8, 288])  # bench m_sweep / policy decode (E = 1) / bench step / prefill
@pytest.mark.parametrize("WB,G,mode", CASES, ids=[f"W{wb}G{g}-{m}" for wb, g, m in CASES])
def test_block_linear_fullsize_sampled(name, N, K, M, WB, G, mode):
    seed = zlib.crc32(f"{name}/{M}/{mode}/{WB}/{G}".encode()) % 1000
    w = synth.weights_bf16_torch(N, K, seed=1 + seed, device=DEV)
    x = synth.activations_bf16_torch(M, K, seed=1000 + seed, device=DEV)
    lin = dyq.PackedLinear.from_bf16(w, group=G, wbits=WB)
    rows = _rows(N, seed)
    w_rows = w[torch.from_numpy(rows).to(DEV)].cpu().numpy().view(np.uint16)
    x_h = x.cpu().numpy().view(np.uint16)
    del w
    rb = _rowbits(M, mode)
    rbt = torch.from_numpy(rb).to(DEV)
    ws = lin.workspace(M)
    pk = oracle.pack_weights(w_rows, G, WB)
    yref, Iref = oracle.qlinear(x_h, pk, G, rb, want_I=True)
    for out, dt, rtol in (("bf16", torch.bfloat16, 2e-2), ("f32", torch.float32, 1e-3)):
        y = torch.full((M, N), float("nan"), dtype=dt, device=DEV)
        dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, rbt, 0, y, 1 if out == "bf16" else 0, ws)
        got = y.float().cpu().numpy()
        assert not np.isnan(got).any(), "unwritten outputs"
        check_close(got[:, rows], yref, rtol)
    # integer group sums bit-exact in both regimes; at M = 288 the o / down /
    # qkv shapes run the split-K prefill (prefill_ksplit > 1), so the split
    # path is bit-checked as well
    path, ks = dyq.qlinear_plan(lin.wd, M)
    assert path == (1 if M <= 16 else 2)
    if M == 288 and name in ("o", "down") and G == 64:
        assert ks > 1, "split-K prefill expected at this shape"
    I = torch.zeros(M, N, K // G, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(lin.wd, lin.codes, lin.meta, x, M, rbt, 0, I, ws)
    assert np.array_equal(I[:, torch.from_numpy(rows).to(DEV)].cpu().numpy(), Iref)
    del I


def _openvla_model(E, copies=2):
    """OpenVLA-7B shapes as bench.py's policy slice: 32 Llama-2-7B blocks
    (layers cycle through `copies` packed block copies), 32 heads, 256 vision
    + 32 text tokens, 7 action tokens, 256 action bins."""
    packed = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=50 + 4 * c + i, device=DEV),
                                          group=G, wbits=WB)
               for i, (_, N, K) in enumerate(synth.LLAMA_BLOCK_LINEARS)] for c in range(copies)]
    d = 4096
    one = torch.full((d,), 0x3F80, dtype=torch.int16, device=DEV)
    embed = synth.activations_bf16_torch(32000, d, seed=7000, device=DEV)
    head = synth.weights_bf16_torch(256, d, seed=7001, device=DEV)
    layers = [packed[l % copies] for l in range(32)]
    return dyq.Model(layers, one.repeat(32), one.repeat(32), one, embed, head, E=E, n_heads=32)


def _on_grid(a):
    b = (a + 1.0) * 128.0 - 0.5
    return np.all(np.abs(b - np.rint(b)) < 1e-4) and np.all((b > -0.5) & (b < 255.5))


def test_policy_step_and_calibration_openvla_shapes():
    """Properties that hold at any size, checked at the bench's OpenVLA-7B
    shapes: b*_t bit-exact with the oracle selector fed the GPU's own actions;
    actions on the 256-bin detokenisation grid; calibration S_t bit-exact
    with the oracle selector fed a*_{t-1}; e^(b) = ||a^(b) - a*||_2."""
    E, Ec = 2, 2
    model = _openvla_model(4 * Ec)
    cal = dyq.default_calib()
    st = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(E, cal, st)
    sel = oracle.SelectState(E)
    act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
    bits = torch.zeros(E, dtype=torch.int32, device=DEV)
    gen = torch.Generator(device=DEV).manual_seed(3)
    prev = None
    for t in range(4):
        vis = synth.activations_bf16_torch(E * 256, 4096, seed=900 + t, device=DEV)
        text = torch.randint(0, 32000, (E, 32), dtype=torch.int32, device=DEV, generator=gen)
        model.step(st, E, vis, text, act, bits)
        a, b = act.cpu().numpy(), bits.cpu().numpy()
        assert np.array_equal(b, sel.step(prev)["bits"]), t
        assert _on_grid(a)
        prev = a.copy()
    model.init()
    cst = torch.zeros(dyq.state_size(Ec, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(Ec, cal, cst)
    csel = oracle.SelectState(Ec)
    acts = torch.zeros(4 * Ec, 7, dtype=torch.float32, device=DEV)
    S = torch.zeros(Ec, dtype=torch.float64, device=DEV)
    err = torch.zeros(Ec, 3, dtype=torch.float64, device=DEV)
    prev = None
    for t in range(3):
        vis = synth.activations_bf16_torch(Ec * 256, 4096, seed=950 + t, device=DEV)
        text = torch.randint(0, 32000, (Ec, 32), dtype=torch.int32, device=DEV, generator=gen)
        model.calib_collect(cst, Ec, vis, text, acts, S, err)
        a = acts.cpu().numpy()
        assert np.array_equal(S.cpu().numpy(), csel.step(prev)["S"]), t
        assert _on_grid(a)
        ref = np.stack([oc.action_error(a[(j + 1) * Ec:(j + 2) * Ec], a[:Ec]) for j in range(3)], axis=1)
        np.testing.assert_allclose(err.cpu().numpy(), ref, rtol=1e-15, atol=0)
        prev = a[:Ec].copy()


@pytest.mark.parametrize("name,N,K", [l for l in synth.LLAMA_BLOCK_LINEARS if l[0] in ("gate_up", "down")],
                         ids=["gate_up", "down"])
@pytest.mark.parametrize("mode", [4, "mixed"])
def test_prefill_eight_episodes_sampled(name, N, K, mode):
    """Largest prefill of the policy slice: E = 8 episodes x 288 tokens = 2304
    rows (18 full 128-token tiles of the tcgen05 kernel)."""
    M = 8 * 288
    seed = zlib.crc32(f"{name}/E8/{mode}".encode()) % 1000
    w = synth.weights_bf16_torch(N, K, seed=1 + seed, device=DEV)
    x = synth.activations_bf16_torch(M, K, seed=1000 + seed, device=DEV)
    lin = dyq.PackedLinear.from_bf16(w, group=G, wbits=WB)
    rows = _rows(N, seed)[::2]
    w_rows = w[torch.from_numpy(rows).to(DEV)].cpu().numpy().view(np.uint16)
    del w
    rb = _rowbits(M, mode)
    y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=DEV)
    dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, torch.from_numpy(rb).to(DEV), 0, y, 1, lin.workspace(M))
    yref, _ = oracle.qlinear(x.cpu().numpy().view(np.uint16), oracle.pack_weights(w_rows, G, WB), G, rb)
    got = y.float().cpu().numpy()
    assert not np.isnan(got).any()
    check_close(got[:, rows], yref, 2e-2)


def test_empty_inputs_are_noops():
    """M = 0 (no tokens) is valid for every linear entry point and writes nothing."""
    N, K = 256, 256
    lin = dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=3, device=DEV), group=G, wbits=WB)
    x = torch.zeros(1, K, dtype=torch.int16, device=DEV)
    y = torch.full((1, N), 7.0, dtype=torch.float32, device=DEV)
    ws = lin.workspace(1)
    dyq.qlinear(lin.wd, lin.codes, lin.meta, x, 0, None, 4, y, 0, ws)
    I = torch.full((1, N, K // G), 5, dtype=torch.int32, device=DEV)
    dyq.qlinear_i32_partials(lin.wd, lin.codes, lin.meta, x, 0, None, 4, I, ws)
    f = torch.zeros(1, dtype=torch.int64, device=DEV)
    yb = torch.full((1, N), 3, dtype=torch.int16, device=DEV)
    dyq.qlinear_tp(lin, x, 0, None, 4, dyq.tp_peers(1, 0, [yb.data_ptr()], [f.data_ptr()]), ws)
    torch.cuda.synchronize()
    assert bool((y == 7.0).all()) and bool((I == 5).all()) and bool((yb == 3).all()) and int(f.item()) == 0
