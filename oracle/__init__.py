"""CPU oracle for the DyQ-VLA qlinear hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_2603_07904_b200` never imports it (and vice versa); the two share no code.

The arithmetic lives in plain C (`dyq_ref.c`, built -O2 -ffp-contract=off); this
module is ctypes marshalling plus a few numpy conveniences.  Each C function
cites the PAPER.md / SPEC.md passage it restates.

Parity status (DESIGN.md §"Oracle pins"): every function below is pinned by at
least one `-m "not gpu"` test in tests/test_oracle_*.py against SPEC worked
examples, closed forms, invariants or brute force.  The paper's own Theta,
lambda, K values are not printed (parity unpinned for those *values*; the
algorithm itself is pinned by the golden traces).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdyq_ref.so")
_SRC = os.path.join(_HERE, "dyq_ref.c")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dyq_ref.h"))
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


P = C.c_void_p
i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double


class Calib(C.Structure):
    """dyq_ref_calib_t; field names follow SPEC S:261 (CalibrationTable keys)."""
    _fields_ = [
        ("theta_24", f64), ("theta_48", f64), ("theta_fp", f64), ("lambda_", f64),
        ("D_acc", f64), ("eta", f64), ("J_cap", f64),
        ("K", i32), ("W_macro", i32), ("W_micro", i32), ("H", i32), ("clamp_M", i32),
    ]


def default_calib(**kw) -> Calib:
    """Defaults: theta_fp=0.5, W_macro=10, W_micro=5; lambda=0.5,
    K=3, H=256, J_cap=2 (paper silent -> reading 18);
    Theta=(0.1, 0.3) synthetic."""
    d = dict(theta_24=0.1, theta_48=0.3, theta_fp=0.5, lambda_=0.5, D_acc=1.0,
             eta=0.01, J_cap=2.0, K=3, W_macro=10, W_micro=5, H=256, clamp_M=1)
    d.update(kw)
    return Calib(**d)


def _declare(L):
    L.dyq_ref_quant_fit.argtypes = [P, i64, C.c_int, P, P, P]
    L.dyq_ref_quantize.argtypes = [P, i64, f32, C.c_uint8, C.c_int, C.c_int, P]
    L.dyq_ref_quantize.restype = None
    L.dyq_ref_dequantize.argtypes = [P, i64, f32, C.c_uint8, P]
    L.dyq_ref_dequantize.restype = None
    L.dyq_ref_pack_weights.argtypes = [i32, i32, i32, i32, i32, P, P, P, P, P, P]
    L.dyq_ref_act_quant.argtypes = [i32, i32, i32, P, i32, P, P, P, P, P, P]
    L.dyq_ref_qlinear.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P]
    L.dyq_ref_state_new.argtypes = [i32, C.POINTER(Calib)]
    L.dyq_ref_state_new.restype = P
    L.dyq_ref_state_free.argtypes = [P]
    L.dyq_ref_state_free.restype = None
    L.dyq_ref_state_reset_episode.argtypes = [P, P]
    L.dyq_ref_state_reset_episode.restype = None
    L.dyq_ref_select_bits.argtypes = [P, P, P, P, P, P, P]
    L.dyq_ref_eq4.argtypes = [P, i32, i32, i32, P]
    L.dyq_ref_eq4.restype = None
    L.dyq_ref_alg1.argtypes = [P, i32, i32, i32, i32, i32, P, P]
    L.dyq_ref_alg1.restype = None
    L.dyq_ref_phi.argtypes = [f64, f64, f64]
    L.dyq_ref_phi.restype = i32
    L.dyq_ref_target_bits.argtypes = [f64, C.c_int, f64, f64, f64]
    L.dyq_ref_target_bits.restype = i32
    L.dyq_ref_percentile.argtypes = [P, i32, i32]
    L.dyq_ref_percentile.restype = f64
    L.dyq_ref_state_bytes_per_stream.argtypes = [C.POINTER(Calib)]
    L.dyq_ref_state_bytes_per_stream.restype = i64


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, index: int = -1):
        super().__init__(f"oracle error code {code} (index {index})")
        self.code = code
        self.index = index


def quant_fit(v, bits: int):
    v = np.ascontiguousarray(v, dtype=np.float64)
    s, z, bi = np.zeros(1, np.float32), np.zeros(1, np.uint8), np.full(1, -1, np.int64)
    rc = lib().dyq_ref_quant_fit(_p(v), v.size, bits, _p(s), _p(z), _p(bi))
    if rc:
        raise OracleError(rc, int(bi[0]))
    return float(s[0]), int(z[0])


def quantize(v, s: float, z: int, bits: int, round_mode: int = 0):
    v = np.ascontiguousarray(v, dtype=np.float64)
    q = np.zeros(v.size, np.uint8)
    lib().dyq_ref_quantize(_p(v), v.size, s, z, bits, round_mode, _p(q))
    return q


def dequantize(q, s: float, z: int):
    q = np.ascontiguousarray(q, dtype=np.uint8)
    out = np.zeros(q.size, np.float64)
    lib().dyq_ref_dequantize(_p(q), q.size, s, z, _p(out))
    return out


def fake_quant(v, bits: int, round_mode: int = 0):
    s, z = quant_fit(v, bits)
    return dequantize(quantize(v, s, z, bits, round_mode), s, z)


@dataclass
class Packed:
    q: np.ndarray      # [N, K] uint8 codes (logical layout)
    s: np.ndarray      # [N, K/G] float32
    z: np.ndarray      # [N, K/G] uint8
    sumq: np.ndarray   # [N, K/G] int32


def pack_weights(w_bf16: np.ndarray, G: int, wbits: int, round_mode: int = 0) -> Packed:
    w = np.ascontiguousarray(w_bf16, dtype=np.uint16)
    N, K = w.shape
    NG = K // G
    q = np.zeros((N, K), np.uint8)
    s = np.zeros((N, NG), np.float32)
    z = np.zeros((N, NG), np.uint8)
    sq = np.zeros((N, NG), np.int32)
    bi = np.full(1, -1, np.int64)
    rc = lib().dyq_ref_pack_weights(N, K, G, wbits, round_mode, _p(w), _p(q), _p(s), _p(z),
                                    _p(sq), _p(bi))
    if rc:
        raise OracleError(rc, int(bi[0]))
    return Packed(q, s, z, sq)


@dataclass
class ActQ:
    xq: np.ndarray   # [M, K] uint8
    s: np.ndarray    # [M, K/G] float32
    z: np.ndarray    # [M, K/G] uint8
    SX: np.ndarray   # [M, K/G] int32


def act_quant(x_bf16: np.ndarray, G: int, abits, round_mode: int = 0) -> ActQ:
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    M, K = x.shape
    NG = K // G
    ab = np.ascontiguousarray(np.broadcast_to(np.asarray(abits, np.int32), (M,)))
    xq = np.zeros((M, K), np.uint8)
    s = np.zeros((M, NG), np.float32)
    z = np.zeros((M, NG), np.uint8)
    SX = np.zeros((M, NG), np.int32)
    bi = np.full(1, -1, np.int64)
    rc = lib().dyq_ref_act_quant(M, K, G, _p(ab), round_mode, _p(x), _p(xq), _p(s), _p(z),
                                 _p(SX), _p(bi))
    if rc:
        raise OracleError(rc, int(bi[0]))
    return ActQ(xq, s, z, SX)


def qlinear(x_bf16: np.ndarray, packed: Packed, G: int, abits, actq: ActQ | None = None,
            want_I: bool = False, round_mode: int = 0):
    """Returns (y fp64 [M,N], I int32 [M,N,K/G] or None)."""
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    M, K = x.shape
    N = packed.q.shape[0]
    ab = np.ascontiguousarray(np.broadcast_to(np.asarray(abits, np.int32), (M,)))
    if actq is None:
        actq = act_quant(x, G, ab, round_mode)
    y = np.zeros((M, N), np.float64)
    I = np.zeros((M, N, K // G), np.int32) if want_I else None
    rc = lib().dyq_ref_qlinear(M, N, K, G, _p(ab), _p(x), _p(actq.xq), _p(actq.s), _p(actq.z),
                               _p(packed.q), _p(packed.s), _p(packed.z), _p(y),
                               _p(I) if want_I else None)
    if rc:
        raise OracleError(rc)
    return y, I


class SelectState:
    """Per-stream kinematic tracker + Alg. 1 dispatcher (oracle)."""

    def __init__(self, E: int, calib: Calib | None = None):
        self.E = E
        self.calib = calib or default_calib()
        self._h = lib().dyq_ref_state_new(E, C.byref(self.calib))
        if not self._h:
            raise OracleError(1)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().dyq_ref_state_free(h)
            self._h = None

    def reset_episode(self, mask=None):
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        lib().dyq_ref_state_reset_episode(self._h, None if m is None else _p(m))

    def step(self, prev_action=None):
        """prev_action [E,7] float32 (a_{t-1}) or None at t=0.
        Returns dict(bits, target, S, Mbar, Jbar)."""
        E = self.E
        bits = np.zeros(E, np.int32)
        tgt = np.zeros(E, np.int32)
        S = np.zeros(E, np.float64)
        Mb = np.zeros(E, np.float64)
        Jb = np.zeros(E, np.float64)
        a = None
        if prev_action is not None:
            a = np.ascontiguousarray(prev_action, np.float32).reshape(E, 7)
        rc = lib().dyq_ref_select_bits(self._h, None if a is None else _p(a), _p(bits), _p(tgt),
                                       _p(S), _p(Mb), _p(Jb))
        if rc:
            raise OracleError(rc)
        return dict(bits=bits, target=tgt, S=S, Mbar=Mb, Jbar=Jb)


def replay(actions: np.ndarray, calib: Calib | None = None):
    """Run select_bits over a [T, E, 7] action log; the decision at step t
    consumes a_{t-1}.  Returns dict of [T, E] arrays."""
    T, E, _ = actions.shape
    st = SelectState(E, calib)
    out = {k: [] for k in ("bits", "target", "S", "Mbar", "Jbar")}
    for t in range(T):
        r = st.step(None if t == 0 else actions[t - 1])
        for k in out:
            out[k].append(r[k])
    return {k: np.stack(v) for k, v in out.items()}


def eq4(targets, K: int, init: int = 16):
    t = np.ascontiguousarray(targets, np.int32)
    out = np.zeros(t.size, np.int32)
    lib().dyq_ref_eq4(_p(t), t.size, K, init, _p(out))
    return out


def alg1(targets, K: int, init=(16, 0, 16)):
    t = np.ascontiguousarray(targets, np.int32)
    out = np.zeros(t.size, np.int32)
    cnt = np.zeros(t.size, np.int32)
    lib().dyq_ref_alg1(_p(t), t.size, K, init[0], init[1], init[2], _p(out), _p(cnt))
    return out, cnt


def phi(S: float, t24: float, t48: float) -> int:
    return int(lib().dyq_ref_phi(S, t24, t48))


def target_bits(S: float, warmup: bool, t24: float, t48: float, tfp: float) -> int:
    return int(lib().dyq_ref_target_bits(S, int(warmup), t24, t48, tfp))


def percentile(v, pct: int = 95) -> float:
    v = np.ascontiguousarray(v, np.float64)
    return float(lib().dyq_ref_percentile(_p(v), v.size, pct))


def state_bytes_per_stream(calib: Calib | None = None) -> int:
    c = calib or default_calib()
    return int(lib().dyq_ref_state_bytes_per_stream(C.byref(c)))
