"""Thin Python binding of include/dyq.h (libdyq.so) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libdyq.so; this module
only converts torch tensors to raw device pointers / streams and raises on a
non-OK status.  PyTorch provides device memory and streams (plumbing).  There is
no CPU fallback: if libdyq.so is missing or no CUDA device is present the calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DYQ_LIB") or os.path.join(_HERE, "libdyq.so")  # DYQ_LIB: A/B builds (tools/)

P, i32, i64, f64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t

# name -> argtypes (restype dyq_status_t unless listed in _RESTYPES)
_SIGS = {
    "dyq_last_error": [],
    "dyq_version": [],
    "dyq_error_reset": [P, P],
    "dyq_error_read": [P, P, P],
    "dyq_check_error": [P, P, P],
    "dyq_pack_weights_size": [P, P, P],
    "dyq_pack_weights": [P, P, P, P, P, P],
    "dyq_unpack_for_check": [P, P, P, P, P, P, P],
    "dyq_state_size": [i32, P, P],
    "dyq_state_init": [i32, P, P, P],
    "dyq_state_reset_episode": [P, P, P],
    "dyq_select_bits": [P, i32, P, P, P, P, P],
    "dyq_route_bits": [P, i32, i32, P, P, P],
    "dyq_select_route": [P, i32, P, P, i32, P, P, P, P, P],
    "dyq_qlinear_workspace": [P, i32, P],
    "dyq_qlinear_plan": [P, i32, P, P],
    "dyq_workspace_init": [P, sz, P],
    "dyq_qlinear": [P, P, P, P, i32, P, i32, P, i32, P, sz, P, P],
    "dyq_qlinear_masked": [P, P, P, P, i32, P, P, P, i32, P, sz, P, P],
    "dyq_qlinear_i32_partials": [P, P, P, P, i32, P, i32, P, P, sz, P, P],
    "dyq_act_quant_for_check": [P, P, i32, P, i32, P, P, P, P, P, sz, P, P],
    "dyq_set_path": [i32],
    "dyq_trace_enable": [P, i64, P],
    "dyq_prefetch_l2": [P, sz, P],
    "dyq_act_quant": [P, P, i32, P, i32, P, sz, P, P],
    "dyq_qlinear_q": [P, P, P, P, i32, P, i32, P, i32, P, sz, P],
    "dyq_model_size": [P, P, P],
    "dyq_model_bind": [P, P],
    "dyq_model_init": [P, P],
    "dyq_model_free": [P],
    "dyq_policy_step": [P, P, i32, P, P, P, P, P],
    "dyq_add_rmsnorm": [P, P, P, i32, i32, C.c_float, P, P],
    "dyq_rope": [P, i32, i32, i32, i32, i32, C.c_float, P],
    "dyq_attention_prefill": [P, i32, i32, i32, i32, P, i32, i32, i32, P, P],
    "dyq_attention_decode": [P, i32, i32, i32, i32, P, i32, i32, i32, P, P],
    "dyq_attention_decode_rope": [P, i32, i32, i32, i32, C.c_float, P, i32, i32, i32, P, P],
    "dyq_silu_mul": [P, i32, i32, P, P],
    "dyq_head_argmax": [P, i32, i32, i32, P, i32, P, P, i32, P],
    "dyq_tp_shard": [i32, i32, i32, P, P],
    "dyq_comm_unique_id": [P],
    "dyq_comm_init": [P, i32, i32, P],
    "dyq_comm_destroy": [P],
    "dyq_tp_allgather": [P, P, i32, i32, P, P, P],
    "dyq_tp_interleave": [P, i32, i32, i32, P, P],
    "dyq_qlinear_tp": [P, P, P, P, i32, P, i32, P, P, sz, P, P],
    "dyq_tp_wait": [P, C.c_uint64, P, P],
    "dyq_tp_flag_delta": [i32, i32, P],
    "dyq_ipc_handle": [P, P, P],
    "dyq_ipc_open": [P, C.c_uint64, P],
    "dyq_ipc_close": [P, C.c_uint64],
    "dyq_policy_step_bits": [P, i32, P, P, P, P, P],
    "dyq_calib_collect": [P, P, i32, P, P, P, P, P, P],
    "dyq_calib_errors": [P, i32, i32, P, P],
    "dyq_calib_derive": [P, P, i64, i32, i32, P, P, P, P],
    "dyq_calib_validate": [P, P, P, i64, i32, P, P, P],
}
_RESTYPES = {"dyq_last_error": C.c_char_p, "dyq_version": C.c_char_p}

STATUS = {0: "DYQ_OK", 1: "DYQ_EINVAL", 2: "DYQ_ESHAPE", 3: "DYQ_EUNSUPPORTED",
          4: "DYQ_ENONFINITE", 5: "DYQ_ECUDA", 6: "DYQ_ENCCL"}


class DyqError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libdyq.so (build it first with paper_2603_07904_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libdyq.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            if os.environ.get("DYQ_LIB") and not hasattr(L, name):
                continue  # older A/B build (tools/): entry points added since are absent
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPES.get(name, C.c_int)
        _lib = L
    return _lib


def _call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise DyqError(rc, name, lib().dyq_last_error().decode())
    return rc


class WDesc(C.Structure):
    _fields_ = [("N", i32), ("K", i32), ("group", i32), ("wbits", i32), ("round_mode", i32)]


class Calib(C.Structure):
    """dyq_calib_t; keys per SPEC S:261."""
    _fields_ = [("theta_24", f64), ("theta_48", f64), ("theta_fp", f64), ("lambda_", f64),
                ("D_acc", f64), ("eta", f64), ("J_cap", f64),
                ("K", i32), ("W_macro", i32), ("W_micro", i32), ("H", i32), ("clamp_M", i32)]


def default_calib(**kw) -> Calib:
    """theta_fp = 0.5, W_macro = 10, W_micro = 5; lambda = 0.5,
    K = 3, H = 256, J_cap = 2 (SPEC defaults); Theta = (0.1, 0.3)."""
    d = dict(theta_24=0.1, theta_48=0.3, theta_fp=0.5, lambda_=0.5, D_acc=1.0, eta=0.01,
             J_cap=2.0, K=3, W_macro=10, W_micro=5, H=256, clamp_M=1)
    d.update(kw)
    return Calib(**d)


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def version() -> str:
    return lib().dyq_version().decode()


def set_path(path: int):
    _call("dyq_set_path", path)


def prefetch_l2(t, stream=None):
    """dyq_prefetch_l2 over a whole device tensor."""
    _call("dyq_prefetch_l2", _ptr(t), t.numel() * t.element_size(), _stream(stream))


def trace_enable(buf, stream=None):
    """Debug: record kernel %globaltimer events into a device uint8/int64 tensor
    (None disables).  Read back with trace_read(buf)."""
    _call("dyq_trace_enable", _ptr(buf), 0 if buf is None else buf.numel() * buf.element_size(), _stream(stream))


def trace_read(buf):
    """-> list of (serial, kernel, event, block, ns) from a trace buffer."""
    import numpy as np
    a = buf.view(__import__("torch").int64).cpu().numpy().view(np.uint64)
    n = int(min(a[0], a[1]))
    rec = a[2:2 + 2 * n].reshape(n, 2)
    tag, t = rec[:, 0], rec[:, 1]
    return [(int(g >> 32), int((g >> 24) & 0xff), int((g >> 16) & 0xff), int(g & 0xffff), int(ts))
            for g, ts in zip(tag, t)]


# ----------------------------------------------------------------- errors
def error_reset(err, stream=None):
    _call("dyq_error_reset", _ptr(err), _stream(stream))


def check_error(err, stream=None):
    """Non-blocking poll: None while the copy is in flight, else the recorded
    index (-1 = none) -- raises nothing; DYQ_ENONFINITE is reported as the index."""
    out = C.c_int64(0)
    rc = lib().dyq_check_error(_ptr(err), C.byref(out), _stream(stream))
    if rc not in (0, 4):
        raise DyqError(rc, "dyq_check_error", lib().dyq_last_error().decode())
    if out.value == -1 and rc == 0:
        return None
    return -1 if out.value == (1 << 63) - 1 else out.value


def error_read(err, stream=None) -> int:
    """Returns the first non-finite element index or -1."""
    out = C.c_int64(0)
    rc = lib().dyq_error_read(_ptr(err), C.byref(out), _stream(stream))
    if rc == 4:
        return int(out.value)
    if rc != 0:
        raise DyqError(rc, "dyq_error_read", lib().dyq_last_error().decode())
    return -1


# ------------------------------------------------------------------- pack
def pack_weights_size(wd: WDesc) -> tuple[int, int]:
    cb, mb = C.c_size_t(0), C.c_size_t(0)
    _call("dyq_pack_weights_size", C.byref(wd), C.byref(cb), C.byref(mb))
    return cb.value, mb.value


def pack_weights(wd: WDesc, w_bf16, codes, meta, err=None, stream=None):
    _call("dyq_pack_weights", C.byref(wd), _ptr(w_bf16), _ptr(codes), _ptr(meta), _ptr(err),
          _stream(stream))


def unpack_for_check(wd: WDesc, codes, meta, q, s, z, stream=None):
    _call("dyq_unpack_for_check", C.byref(wd), _ptr(codes), _ptr(meta), _ptr(q), _ptr(s), _ptr(z),
          _stream(stream))


# ---------------------------------------------------------- bit selection
def state_size(E: int, calib: Calib) -> int:
    b = C.c_size_t(0)
    _call("dyq_state_size", E, C.byref(calib), C.byref(b))
    return b.value


def state_init(E: int, calib: Calib, state, stream=None):
    _call("dyq_state_init", E, C.byref(calib), _ptr(state), _stream(stream))


def state_reset_episode(state, mask=None, stream=None):
    _call("dyq_state_reset_episode", _ptr(state), _ptr(mask), _stream(stream))


def select_bits(state, E: int, prev_action, bits, S_out=None, target_out=None, stream=None):
    _call("dyq_select_bits", _ptr(state), E, _ptr(prev_action), _ptr(bits), _ptr(S_out),
          _ptr(target_out), _stream(stream))


def select_route(state, E: int, prev_action, bits, tokens_per_episode: int, row_bits, abits_of=None,
                 S_out=None, target_out=None, stream=None):
    """dyq_select_bits + dyq_route_bits in one kernel."""
    tab = (i32 * 4)(*abits_of) if abits_of is not None else None
    _call("dyq_select_route", _ptr(state), E, _ptr(prev_action), _ptr(bits), tokens_per_episode, tab,
          _ptr(row_bits), _ptr(S_out), _ptr(target_out), _stream(stream))


def route_bits(bits, E: int, tokens_per_episode: int, row_bits, abits_of=None, stream=None):
    tab = None if abits_of is None else (C.c_int32 * 4)(*abits_of)
    _call("dyq_route_bits", _ptr(bits), E, tokens_per_episode, tab, _ptr(row_bits), _stream(stream))


# ---------------------------------------------------------------- qlinear
def qlinear_plan(wd: WDesc, M: int) -> tuple[int, int]:
    """(path, ksplit) of a qlinear call with M rows: path 1 decode, 2 prefill."""
    p, k = C.c_int32(0), C.c_int32(0)
    _call("dyq_qlinear_plan", C.byref(wd), M, C.byref(p), C.byref(k))
    return p.value, k.value


def qlinear_workspace(wd: WDesc, M: int) -> int:
    b = C.c_size_t(0)
    _call("dyq_qlinear_workspace", C.byref(wd), M, C.byref(b))
    return b.value


def workspace_init(ws, stream=None):
    _call("dyq_workspace_init", _ptr(ws), ws.numel() * ws.element_size(), _stream(stream))


def qlinear(wd: WDesc, codes, meta, x, M: int, row_bits, bits: int, y, y_dtype: int, ws,
            err=None, stream=None):
    _call("dyq_qlinear", C.byref(wd), _ptr(codes), _ptr(meta), _ptr(x), M, _ptr(row_bits), bits,
          _ptr(y), y_dtype, _ptr(ws), ws.numel() * ws.element_size(), _ptr(err), _stream(stream))


def act_quant(wd: WDesc, x, M: int, row_bits, bits: int, ws, err=None, stream=None):
    _call("dyq_act_quant", C.byref(wd), _ptr(x), M, _ptr(row_bits), bits, _ptr(ws),
          ws.numel() * ws.element_size(), _ptr(err), _stream(stream))


def qlinear_masked(wd: WDesc, codes, meta, x, M: int, row_bits, gate, y, y_dtype: int, ws, err=None, stream=None):
    """dyq_qlinear_masked: rows with row_bits 0 untouched; *gate == 0 -> no-op."""
    _call("dyq_qlinear_masked", C.byref(wd), _ptr(codes), _ptr(meta), _ptr(x), M, _ptr(row_bits), _ptr(gate),
          _ptr(y), y_dtype, _ptr(ws), ws.numel() * ws.element_size(), _ptr(err), _stream(stream))


def qlinear_q(wd: WDesc, codes, meta, x, M: int, row_bits, bits: int, y, y_dtype: int, ws,
              stream=None):
    _call("dyq_qlinear_q", C.byref(wd), _ptr(codes), _ptr(meta), _ptr(x), M, _ptr(row_bits), bits,
          _ptr(y), y_dtype, _ptr(ws), ws.numel() * ws.element_size(), _stream(stream))


def qlinear_i32_partials(wd: WDesc, codes, meta, x, M: int, row_bits, bits: int, I, ws,
                         err=None, stream=None):
    _call("dyq_qlinear_i32_partials", C.byref(wd), _ptr(codes), _ptr(meta), _ptr(x), M,
          _ptr(row_bits), bits, _ptr(I), _ptr(ws), ws.numel() * ws.element_size(), _ptr(err),
          _stream(stream))


def act_quant_for_check(wd: WDesc, x, M: int, row_bits, bits: int, xq, sx, zx, SX, ws,
                        err=None, stream=None):
    _call("dyq_act_quant_for_check", C.byref(wd), _ptr(x), M, _ptr(row_bits), bits, _ptr(xq),
          _ptr(sx), _ptr(zx), _ptr(SX), _ptr(ws), ws.numel() * ws.element_size(), _ptr(err),
          _stream(stream))


# ------------------------------------------------ torch-owned conveniences
@dataclass
class PackedLinear:
    """Packed weights of one linear layer (device buffers owned by torch)."""
    wd: WDesc
    codes: object
    meta: object

    @classmethod
    def from_bf16(cls, w_bf16, group: int = 64, wbits: int = 4, round_mode: int = 0, err=None,
                  stream=None):
        import torch
        N, K = w_bf16.shape
        wd = WDesc(N, K, group, wbits, round_mode)
        cb, mb = pack_weights_size(wd)
        dev = w_bf16.device
        codes = torch.empty(cb, dtype=torch.uint8, device=dev)
        meta = torch.empty(mb, dtype=torch.uint8, device=dev)
        pack_weights(wd, w_bf16, codes, meta, err, stream)
        return cls(wd, codes, meta)

    def prefetch_l2(self, stream=None):
        """Asynchronous HBM -> L2 prefetch of this layer's codes + metadata."""
        prefetch_l2(self.codes, stream)
        prefetch_l2(self.meta, stream)

    def workspace(self, M: int):
        import torch
        ws = torch.zeros(max(16, qlinear_workspace(self.wd, M)), dtype=torch.uint8,
                         device=self.codes.device)
        return ws

    def __call__(self, x, row_bits=None, bits: int = 4, out_dtype=None, ws=None, err=None,
                 stream=None):
        import torch
        M = x.shape[0]
        out_dtype = out_dtype or torch.float32
        y = torch.empty(M, self.wd.N, dtype=out_dtype, device=x.device)
        if ws is None:
            ws = self.workspace(M)
        qlinear(self.wd, self.codes, self.meta, x, M, row_bits, bits, y,
                0 if out_dtype == torch.float32 else 1, ws, err, stream)
        return y


# ------------------------------------------------------------- policy step
class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d", C.c_int32), ("ffn", C.c_int32), ("n_heads", C.c_int32),
                ("vocab", C.c_int32), ("E", C.c_int32), ("n_vis", C.c_int32), ("n_text", C.c_int32),
                ("n_act", C.c_int32), ("n_bins", C.c_int32), ("group", C.c_int32), ("wbits", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float),
                ("codes", C.POINTER(C.c_void_p)), ("meta", C.POINTER(C.c_void_p)),
                ("attn_norm", C.c_void_p), ("mlp_norm", C.c_void_p), ("final_norm", C.c_void_p),
                ("embed", C.c_void_p), ("head_bins", C.c_void_p), ("kv", C.c_void_p), ("scratch", C.c_void_p),
                ("codes_w8", C.POINTER(C.c_void_p)), ("meta_w8", C.POINTER(C.c_void_p)),
                ("wbits_of", C.c_int32 * 4), ("abits_of", C.c_int32 * 4),
                ("paper_mode", C.c_int32), ("prefill_bits", C.c_int32)]


def add_rmsnorm(h, delta, w, M: int, d: int, eps: float, y, stream=None):
    _call("dyq_add_rmsnorm", _ptr(h), _ptr(delta), _ptr(w), M, d, eps, _ptr(y), _stream(stream))


def rope(qkv, M: int, rows_per_episode: int, pos0: int, d: int, n_heads: int, theta: float, stream=None):
    _call("dyq_rope", _ptr(qkv), M, rows_per_episode, pos0, d, n_heads, theta, _stream(stream))


def attention_prefill(qkv, E: int, S: int, d: int, n_heads: int, kv, layer: int, n_layers: int, T: int, out,
                      stream=None):
    _call("dyq_attention_prefill", _ptr(qkv), E, S, d, n_heads, _ptr(kv), layer, n_layers, T, _ptr(out),
          _stream(stream))


def attention_decode(qkv, E: int, pos: int, d: int, n_heads: int, kv, layer: int, n_layers: int, T: int, out,
                     stream=None):
    _call("dyq_attention_decode", _ptr(qkv), E, pos, d, n_heads, _ptr(kv), layer, n_layers, T, _ptr(out),
          _stream(stream))


def attention_decode_rope(qkv, E: int, pos: int, d: int, n_heads: int, theta: float, kv, layer: int, n_layers: int,
                          T: int, out, stream=None):
    _call("dyq_attention_decode_rope", _ptr(qkv), E, pos, d, n_heads, theta, _ptr(kv), layer, n_layers, T,
          _ptr(out), _stream(stream))


def silu_mul(gu, M: int, ffn: int, act, stream=None):
    _call("dyq_silu_mul", _ptr(gu), M, ffn, _ptr(act), _stream(stream))


def head_argmax(x, E: int, row_stride: int, d: int, head_bins, n_bins: int, logits, tok, tok_stride: int,
                stream=None):
    _call("dyq_head_argmax", _ptr(x), E, row_stride, d, _ptr(head_bins), n_bins, _ptr(logits), _ptr(tok),
          tok_stride, _stream(stream))


class Model:
    """A bound policy-step model: packed linears + bf16 glue weights, caller-
    owned KV cache and scratch (torch tensors).  `layers` = list of n_layers
    lists [qkv, o, gate_up, down] of PackedLinear."""

    def __init__(self, layers, attn_norm, mlp_norm, final_norm, embed, head_bins, E: int,
                 n_heads: int = 32, n_vis: int = 256, n_text: int = 32, n_act: int = 7,
                 rms_eps: float = 1e-5, rope_theta: float = 10000.0, stream=None,
                 layers_w8=None, wbits_of=None, abits_of=None, paper_mode: int = 0, prefill_bits: int = 0):
        """layers_w8: optional W8 copies (same structure) for the variant table
        wbits_of / abits_of (per b* in 2, 4, 8, 16); paper_mode: b* selected on
        a side stream overlapping the prefill, which runs at prefill_bits."""
        import torch
        qkv0 = layers[0][0].wd
        d = qkv0.K
        ffn = layers[0][2].wd.N // 2
        self._keep = [layers, attn_norm, mlp_norm, final_norm, embed, head_bins]
        nl = len(layers)
        self._codes = (C.c_void_p * (4 * nl))(*[l.codes.data_ptr() for L in layers for l in L])
        self._meta = (C.c_void_p * (4 * nl))(*[l.meta.data_ptr() for L in layers for l in L])
        self.desc = ModelDesc(nl, d, ffn, n_heads, embed.shape[0], E, n_vis, n_text, n_act, head_bins.shape[0],
                              qkv0.group, qkv0.wbits, rms_eps, rope_theta,
                              C.cast(self._codes, C.POINTER(C.c_void_p)), C.cast(self._meta, C.POINTER(C.c_void_p)),
                              attn_norm.data_ptr(), mlp_norm.data_ptr(), final_norm.data_ptr(), embed.data_ptr(),
                              head_bins.data_ptr(), None, None)
        if layers_w8 is not None:
            self._keep.append(layers_w8)
            self._codes8 = (C.c_void_p * (4 * nl))(*[l.codes.data_ptr() for L in layers_w8 for l in L])
            self._meta8 = (C.c_void_p * (4 * nl))(*[l.meta.data_ptr() for L in layers_w8 for l in L])
            self.desc.codes_w8 = C.cast(self._codes8, C.POINTER(C.c_void_p))
            self.desc.meta_w8 = C.cast(self._meta8, C.POINTER(C.c_void_p))
        if wbits_of is not None:
            self.desc.wbits_of = (C.c_int32 * 4)(*wbits_of)
        if abits_of is not None:
            self.desc.abits_of = (C.c_int32 * 4)(*abits_of)
        self.desc.paper_mode = paper_mode
        self.desc.prefill_bits = prefill_bits
        kvb, scb = C.c_size_t(0), C.c_size_t(0)
        _call("dyq_model_size", C.byref(self.desc), C.byref(kvb), C.byref(scb))
        dev = embed.device
        self.kv = torch.zeros(kvb.value // 2, dtype=torch.int16, device=dev)
        self.scratch = torch.zeros(scb.value, dtype=torch.uint8, device=dev)
        self.desc.kv = self.kv.data_ptr()
        self.desc.scratch = self.scratch.data_ptr()
        self._h = C.c_void_p()
        _call("dyq_model_bind", C.byref(self.desc), C.byref(self._h))
        _call("dyq_model_init", self._h, _stream(stream))
        self.E, self.n_act, self.T = E, n_act, n_vis + n_text + n_act

    def init(self, stream=None):
        _call("dyq_model_init", self._h, _stream(stream))

    def step(self, state, E: int, vis_emb, text_ids, action_out, bits_out=None, stream=None):
        _call("dyq_policy_step", self._h, _ptr(state), E, _ptr(vis_emb), _ptr(text_ids), _ptr(action_out),
              _ptr(bits_out), _stream(stream))

    def step_bits(self, E: int, bits, vis_emb, text_ids, action_out, stream=None):
        """Forced-bits step: episode e runs at bits[e] (device int32 [E])."""
        _call("dyq_policy_step_bits", self._h, E, _ptr(bits), _ptr(vis_emb), _ptr(text_ids), _ptr(action_out),
              _stream(stream))

    def calib_collect(self, state, Ec: int, vis_emb, text_ids, actions_out, S_out, err_out, stream=None):
        """One calibration step (dyq_calib_collect): S_t, a* and the
        counterfactual 2/4/8-bit actions in one batched step, e^(b)."""
        _call("dyq_calib_collect", self._h, _ptr(state), Ec, _ptr(vis_emb), _ptr(text_ids), _ptr(actions_out),
              _ptr(S_out), _ptr(err_out), _stream(stream))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().dyq_model_free(h)
            except Exception:
                pass
            self._h = None


# ------------------------------------------- offline threshold calibration
def calib_errors(actions, Ec: int, n_act: int, err_out, stream=None):
    _call("dyq_calib_errors", _ptr(actions), Ec, n_act, _ptr(err_out), _stream(stream))


def _host_f64(a, cols=None):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.float64)
    if cols is not None:
        a = a.reshape(-1, cols)
    return a, a.ctypes.data_as(C.c_void_p)


def calib_derive(S, err, calib: Calib, n_bins: int = 32, n_min: int = 50):
    """Host arrays S [n], err [n, 3]; fills calib.theta_24 / theta_48 and
    returns (smoothed [2, n_bins], counts [n_bins], n_undercovered)."""
    import numpy as np
    S, pS = _host_f64(S)
    err, pE = _host_f64(err, 3)
    if err.shape[0] != S.size:
        raise ValueError("S and err disagree on the sample count")
    sm = np.zeros((2, n_bins), np.float64)
    cnt = np.zeros(n_bins, np.int64)
    und = C.c_int32(0)
    _call("dyq_calib_derive", pS, pE, S.size, n_bins, n_min, C.byref(calib), sm.ctypes.data_as(C.c_void_p),
          cnt.ctypes.data_as(C.c_void_p), C.byref(und))
    return sm, cnt, und.value


def calib_validate(calib: Calib, S, err, n_bins: int = 32):
    """Returns (n_quant, n_ok, worst [n_bins]) for host arrays S [n], err [n, 3]."""
    import numpy as np
    S, pS = _host_f64(S)
    err, pE = _host_f64(err, 3)
    worst = np.zeros(n_bins, np.float64)
    nq, nok = C.c_int64(0), C.c_int64(0)
    _call("dyq_calib_validate", C.byref(calib), pS, pE, S.size, n_bins, C.byref(nq), C.byref(nok),
          worst.ctypes.data_as(C.c_void_p))
    return nq.value, nok.value, worst


# ------------------------------------------------------ tensor parallelism
def tp_shard(N: int, world: int, rank: int) -> tuple[int, int]:
    a, b = C.c_int32(0), C.c_int32(0)
    _call("dyq_tp_shard", N, world, rank, C.byref(a), C.byref(b))
    return a.value, b.value


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _call("dyq_comm_unique_id", buf)
    return buf.raw


TP_MAX = 8


class TpPeers(C.Structure):
    """dyq_tp_peers_t: every rank's full y and arrival flag as mapped here."""
    _fields_ = [("world", i32), ("rank", i32), ("y", C.c_void_p * TP_MAX), ("flag", C.c_void_p * TP_MAX)]


def tp_peers(world: int, rank: int, y_ptrs, flag_ptrs) -> TpPeers:
    """y_ptrs / flag_ptrs: device addresses (ints) of rank p's buffers, p < world."""
    t = TpPeers()
    t.world, t.rank = world, rank
    for p in range(world):
        t.y[p] = int(y_ptrs[p])
        t.flag[p] = int(flag_ptrs[p])
    return t


def qlinear_tp(lin: "PackedLinear", x, M: int, row_bits, bits: int, peers: TpPeers, ws, err=None, stream=None):
    """Fused TP decode: this rank's shard `lin` (rows dyq_tp_shard) written
    into every rank's full y; see dyq_qlinear_tp."""
    _call("dyq_qlinear_tp", C.byref(lin.wd), _ptr(lin.codes), _ptr(lin.meta), _ptr(x), M, _ptr(row_bits), bits,
          C.byref(peers), _ptr(ws), ws.numel() * ws.element_size(), _ptr(err), _stream(stream))


def tp_flag_delta(N: int, M: int) -> int:
    """Per-call flag increment of qlinear_tp (full width N, M tokens)."""
    d = C.c_uint64(0)
    _call("dyq_tp_flag_delta", N, M, C.byref(d))
    return d.value


def tp_wait(flag, target: int, timed_out=None, stream=None):
    """Stream-ordered wait until flag (device uint64 / int64 tensor) >= target."""
    _call("dyq_tp_wait", _ptr(flag), target, _ptr(timed_out), _stream(stream))


def ipc_handle(t) -> tuple[bytes, int]:
    """(handle, offset) of a device tensor's memory, for dyq_ipc_open in a peer."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64(0)
    _call("dyq_ipc_handle", C.c_void_p(t.data_ptr()), buf, C.byref(off))
    return buf.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    h = C.create_string_buffer(handle, 64)
    p = C.c_void_p()
    _call("dyq_ipc_open", h, offset, C.byref(p))
    return p.value


def ipc_close(ptr: int, offset: int):
    _call("dyq_ipc_close", C.c_void_p(ptr), offset)


class Comm:
    """NCCL communicator of libdyq.so (column-sharded TP)."""

    def __init__(self, unique_id: bytes, rank: int, world: int):
        self.rank, self.world = rank, world
        self._id = C.create_string_buffer(unique_id, 128)
        self._h = C.c_void_p()
        _call("dyq_comm_init", self._id, rank, world, C.byref(self._h))

    def allgather(self, y_shard, M: int, N: int, gather_buf, y, stream=None):
        _call("dyq_tp_allgather", self._h, _ptr(y_shard), M, N, _ptr(gather_buf), _ptr(y), _stream(stream))

    def close(self):
        if self._h is not None and self._h.value:
            lib().dyq_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tp_interleave(buf, P: int, M: int, Ns: int, y, stream=None):
    _call("dyq_tp_interleave", _ptr(buf), P, M, Ns, _ptr(y), _stream(stream))
