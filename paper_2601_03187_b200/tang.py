"""Thin ctypes binding of libtang (include/tang.h): argument marshalling only.

Every step of the hot path runs in libtang's CUDA kernels; this module converts NumPy
arrays / torch tensors to pointers and return codes to exceptions.  There is no CPU
fallback: if libtang.so is missing the import fails loudly, and a ctx built without a
device refuses to classify (TANG_ENODEV).

The module-level functions carry the C names (tang_build, tang_classify, ...); `Ctx`
wraps them for convenience.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TANG_LIB") or os.path.join(_HERE, "libtang.so")   # TANG_LIB: A/B experiments

TANG_OK, TANG_EINVAL, TANG_EMODEL, TANG_ENOTUPLE, TANG_ENOENT = 0, -1, -2, -3, -4
TANG_ENOMEM, TANG_ECUDA, TANG_ENODEV, TANG_ESTATE = -5, -6, -7, -8
TANG_NO_MATCH = 0xFFFFFFFF
TANG_BLOB_MAGIC, TANG_BLOB_VERSION = 0x474E4154, 1
TANG_MLP_BF16_TC, TANG_MLP_FP32_FFMA, TANG_MLP_FP8_TC = 0, 1, 2
TANG_MLP_NVFP4_TC = 3
TANG_BLOB_F8_MAGIC = 0x53413846   # "F8AS": fp8 activation-scale trailer (include/tang.h)
TANG_MODE_PAPER, TANG_MODE_STRICT = 0, 1
TANG_KERNEL_AUTO, TANG_KERNEL_SINGLE, TANG_KERNEL_PAIR, TANG_KERNEL_2SM, TANG_KERNEL_WIDE, TANG_KERNEL_TS = 0, 1, 2, 3, 4, 5
TANG_KERNEL_DUAL = 6
TANG_OP_INSERT, TANG_OP_DELETE = 1, 2
TANG_MAX_TOPK = 4

# numpy views of the ABI structs (byte-identical to include/tang.h)
HEADER_DTYPE = np.dtype([("sip", "<u4"), ("dip", "<u4"), ("sp", "<u2"), ("dp", "<u2"),
                         ("proto", "u1"), ("pad", "u1", (3,))])
RULE_DTYPE = np.dtype([("id", "<u4"), ("priority", "<u4"), ("sip", "<u4"), ("dip", "<u4"),
                       ("sp_lo", "<u2"), ("sp_hi", "<u2"), ("dp_lo", "<u2"), ("dp_hi", "<u2"),
                       ("sip_len", "u1"), ("dip_len", "u1"), ("proto", "u1"), ("proto_mask", "u1"),
                       ("action", "<u4")])
OP_DTYPE = np.dtype([("kind", "u1"), ("pad", "u1", (3,)), ("id", "<u4"), ("rule", RULE_DTYPE)])
assert HEADER_DTYPE.itemsize == 16 and RULE_DTYPE.itemsize == 32 and OP_DTYPE.itemsize == 40


class TangError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        super().__init__(f"{what}: {tang_strerror(code)} ({code})")


class tang_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("mlp", C.c_uint32), ("topk", C.c_uint32), ("mode", C.c_uint32),
                ("max_batch", C.c_uint32), ("batch", C.c_uint32), ("streams", C.c_uint32),
                ("ring_slots", C.c_uint32), ("rule_capacity", C.c_uint32), ("mlp_kernel", C.c_uint32),
                ("reserved", C.c_uint32 * 6)]


class tang_stats_t(C.Structure):
    _fields_ = [("tuples", C.c_uint32), ("rules", C.c_uint32), ("mismatch_count", C.c_uint32),
                ("epoch", C.c_uint32), ("device_bytes", C.c_uint64), ("table_bytes", C.c_uint64),
                ("slots", C.c_uint32), ("keys", C.c_uint32), ("S", C.c_uint32), ("N", C.c_uint32),
                ("B", C.c_uint32), ("C", C.c_uint32), ("checksum", C.c_uint64),
                ("live_keys", C.c_uint32), ("delta_rejected", C.c_uint32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtang.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, S, I, U, V = C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, C.c_void_p
    sig = {
        "tang_build": (I, [P, S, P, S, P, C.POINTER(P)]),
        "tang_destroy": (None, [P]),
        "tang_strerror": (C.c_char_p, [I]),
        "tang_stats": (I, [P, C.POINTER(tang_stats_t)]),
        "tang_classify": (I, [P, P, S, P]),
        "tang_classify_async": (I, [P, P, S, P, V]),
        "tang_classify_ex": (I, [P, P, S, P, P, P, P, V]),
        "tang_classify_with_pred": (I, [P, P, S, P, U, P, P, V]),
        "tang_encode_async": (I, [P, P, S, P, V]),
        "tang_update": (I, [P, P, S, P, V]),
        "tang_update_plan": (I, [P, P, S, P, C.POINTER(P), C.POINTER(S)]),
        "tang_apply_delta_async": (I, [P, P, S, V]),
        "tang_apply_delta_host": (I, [P, P, S]),
        "tang_device_checksum": (I, [P, C.POINTER(C.c_uint64)]),
        "tang_timeline_read": (I, [P, P, I]),
        "tang_debug_candidates": (I, [P, U, U, P, U]),
        "tang_table_digest_async": (I, [P, P, V]),
        "tang_mirror_digest": (I, [P, C.POINTER(C.c_uint64)]),
        "tang_rule_tuple": (I, [P, U, C.POINTER(U)]),
        "tang_profile_enable": (I, [P, I]),
        "tang_profile_read": (I, [P, C.POINTER(C.c_char_p), C.POINTER(C.c_float), C.POINTER(C.c_uint64), I]),
        "tang_latency_read": (I, [P, C.POINTER(C.c_float), I]),
        "tang_debug_activations": (I, [P, P, S, P, P, P, V]),
        "tang_reload_model": (I, [P, P, S]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = ("tang_build", "tang_destroy", "tang_strerror", "tang_stats", "tang_classify", "tang_classify_async",
            "tang_classify_ex", "tang_classify_with_pred", "tang_encode_async", "tang_update", "tang_update_plan",
            "tang_apply_delta_async", "tang_apply_delta_host", "tang_device_checksum", "tang_table_digest_async",
            "tang_mirror_digest", "tang_rule_tuple",
            "tang_profile_enable", "tang_profile_read", "tang_latency_read", "tang_timeline_read",
            "tang_debug_activations", "tang_debug_candidates",
            "tang_reload_model")


def tang_strerror(code: int) -> str:
    return _lib.tang_strerror(code).decode()


def _ck(code, what):
    if code < 0:
        raise TangError(code, what)
    return code


def _ptr(x):
    """Device/host pointer of a torch tensor, NumPy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s):
    if s is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ---------------------------------------------------------------------------------------
# model blob (include/tang.h): marshalling of weights + class signatures
# ---------------------------------------------------------------------------------------
def pack_blob(sigs, w: dict) -> bytes:
    """Serialise signatures [(lsip, ldip)] x C and fp32 weights ([in][out]) into a blob."""
    S, N, B, Cn = int(w["S"]), int(w["N"]), int(w["B"]), int(w["C"])
    if len(sigs) != Cn:
        raise ValueError("one signature per class is required")
    parts = [np.array([TANG_BLOB_MAGIC, TANG_BLOB_VERSION, S, N, B, Cn], "<u4").tobytes()]
    sb = np.array(sigs, dtype=np.uint8).reshape(-1).tobytes()
    parts.append(sb + b"\0" * ((-len(sb)) % 4))
    f = lambda a: np.ascontiguousarray(a, dtype="<f4").tobytes()
    parts += [f(w["W0"]), f(w["b0"])]
    for i in range(B):
        parts += [f(w["W1"][i]), f(w["b1"][i]), f(w["W2"][i]), f(w["b2"][i])]
    parts += [f(w["Wo"]), f(w["bo"])]
    if w.get("act_exp") is not None:           # fp8 activation scales 2^e (R23)
        ex = np.asarray(w["act_exp"], dtype="<i4")
        if ex.size != 2 * B + 1:
            raise ValueError("act_exp needs 2B+1 exponents")
        parts += [np.array([TANG_BLOB_F8_MAGIC, ex.size], "<u4").tobytes(), ex.tobytes()]
    return b"".join(parts)




# ---------------------------------------------------------------------------------------
# C-named functions
# ---------------------------------------------------------------------------------------
def tang_build(rules: np.ndarray, blob: bytes, cfg: tang_config):
    rules = np.ascontiguousarray(rules, dtype=RULE_DTYPE)
    out = C.c_void_p()
    bb = C.create_string_buffer(blob, len(blob))
    _ck(_lib.tang_build(rules.ctypes.data if rules.size else None, rules.size, bb, len(blob),
                        C.byref(cfg), C.byref(out)), "tang_build")
    return out.value


def tang_destroy(ctx):
    _lib.tang_destroy(ctx)


def tang_stats(ctx) -> dict:
    st = tang_stats_t()
    _ck(_lib.tang_stats(ctx, C.byref(st)), "tang_stats")
    return {k: getattr(st, k) for k, _ in tang_stats_t._fields_}


def tang_classify(ctx, headers: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """Host buffers (pinned tensors or NumPy arrays); blocking, streamed through the rings."""
    if out is None:
        headers = np.ascontiguousarray(headers, dtype=HEADER_DTYPE)
        out = np.empty(headers.size, dtype=np.uint32)
    n = headers.size if isinstance(headers, np.ndarray) else headers.numel() // 16
    _ck(_lib.tang_classify(ctx, _ptr(headers), n, _ptr(out)), "tang_classify")
    return out


def tang_classify_async(ctx, d_hdr, n, d_rule_id, stream=None):
    _ck(_lib.tang_classify_async(ctx, _ptr(d_hdr), n, _ptr(d_rule_id), _stream(stream)), "tang_classify_async")


def tang_classify_ex(ctx, d_hdr, n, d_rule_id, d_pred=None, d_logits=None, d_fellback=None, stream=None):
    _ck(_lib.tang_classify_ex(ctx, _ptr(d_hdr), n, _ptr(d_rule_id), _ptr(d_pred), _ptr(d_logits),
                              _ptr(d_fellback), _stream(stream)), "tang_classify_ex")


def tang_classify_with_pred(ctx, d_hdr, n, d_pred, k, d_rule_id, d_fellback=None, stream=None):
    _ck(_lib.tang_classify_with_pred(ctx, _ptr(d_hdr), n, _ptr(d_pred), k, _ptr(d_rule_id), _ptr(d_fellback),
                                     _stream(stream)), "tang_classify_with_pred")


def tang_encode_async(ctx, d_hdr, n, d_feat, stream=None):
    _ck(_lib.tang_encode_async(ctx, _ptr(d_hdr), n, _ptr(d_feat), _stream(stream)), "tang_encode_async")


def make_ops(inserts=None, deletes=()):
    """Update ops: inserts (RULE_DTYPE array) and deletes (ids), deletes first."""
    ins = np.zeros(0, RULE_DTYPE) if inserts is None else np.asarray(inserts, RULE_DTYPE)
    ops = np.zeros(len(deletes) + ins.size, OP_DTYPE)
    ops["kind"][:len(deletes)] = TANG_OP_DELETE
    ops["id"][:len(deletes)] = np.asarray(deletes, dtype=np.uint32)
    ops["kind"][len(deletes):] = TANG_OP_INSERT
    ops["rule"][len(deletes):] = ins
    return ops


def tang_update(ctx, ops: np.ndarray, stream=None) -> np.ndarray:
    ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
    st = np.zeros(ops.size, np.int32)
    _ck(_lib.tang_update(ctx, ops.ctypes.data if ops.size else None, ops.size, st.ctypes.data,
                         _stream(stream) if stream is not None else 0), "tang_update")
    return st


def tang_update_plan(ctx, ops: np.ndarray):
    ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
    st = np.zeros(ops.size, np.int32)
    d, n = C.c_void_p(), C.c_size_t()
    _ck(_lib.tang_update_plan(ctx, ops.ctypes.data if ops.size else None, ops.size, st.ctypes.data,
                              C.byref(d), C.byref(n)), "tang_update_plan")
    delta = C.string_at(d.value, n.value) if n.value else b""
    return st, delta


def tang_apply_delta_async(ctx, d_delta, nbytes, stream=None):
    _ck(_lib.tang_apply_delta_async(ctx, _ptr(d_delta), nbytes, _stream(stream)), "tang_apply_delta_async")


def tang_apply_delta_host(ctx, delta: bytes):
    buf = C.create_string_buffer(delta, len(delta)) if delta else None
    _ck(_lib.tang_apply_delta_host(ctx, buf, len(delta)), "tang_apply_delta_host")


def tang_table_digest_async(ctx, d_digest, stream=None):
    _ck(_lib.tang_table_digest_async(ctx, _ptr(d_digest), _stream(stream)), "tang_table_digest_async")


def tang_mirror_digest(ctx) -> int:
    v = C.c_uint64()
    _ck(_lib.tang_mirror_digest(ctx, C.byref(v)), "tang_mirror_digest")
    return v.value


def tang_device_checksum(ctx) -> int:
    v = C.c_uint64()
    _ck(_lib.tang_device_checksum(ctx, C.byref(v)), "tang_device_checksum")
    return v.value


def tang_rule_tuple(ctx, rule_id: int) -> int:
    v = C.c_uint32()
    _ck(_lib.tang_rule_tuple(ctx, rule_id, C.byref(v)), "tang_rule_tuple")
    return v.value


def tang_profile_enable(ctx, on=True):
    _ck(_lib.tang_profile_enable(ctx, 1 if on else 0), "tang_profile_enable")


def tang_profile_read(ctx) -> dict:
    cap = 16
    names = (C.c_char_p * cap)()
    ms = (C.c_float * cap)()
    cnt = (C.c_uint64 * cap)()
    n = _ck(_lib.tang_profile_read(ctx, names, ms, cnt, cap), "tang_profile_read")
    return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(min(n, cap))}


def tang_debug_activations(ctx, d_hdr, n, d_act, d_pred, d_logits=None, stream=None):
    _ck(_lib.tang_debug_activations(ctx, _ptr(d_hdr), n, _ptr(d_act), _ptr(d_pred), _ptr(d_logits),
                                    _stream(stream)), "tang_debug_activations")


def tang_reload_model(ctx, blob: bytes):
    bb = C.create_string_buffer(blob, len(blob))
    _ck(_lib.tang_reload_model(ctx, bb, len(blob)), "tang_reload_model")


def tang_timeline_read(ctx) -> np.ndarray:
    """[chunks, 4] ms: H2D start, H2D end, kernels end, D2H end of the last tang_classify call."""
    n = _lib.tang_timeline_read(ctx, None, 0)
    buf = (C.c_float * max(4, 4 * n))()
    _lib.tang_timeline_read(ctx, buf, n)
    return np.array(buf[:4 * n], dtype=np.float32).reshape(n, 4)


def tang_latency_read(ctx) -> np.ndarray:
    n = _lib.tang_latency_read(ctx, None, 0)
    buf = (C.c_float * max(1, n))()
    _lib.tang_latency_read(ctx, buf, n)
    return np.array(buf[:n], dtype=np.float32)


# ---------------------------------------------------------------------------------------
# convenience wrapper
# ---------------------------------------------------------------------------------------
class Ctx:
    def __init__(self, rules, blob, device=0, mlp="bf16", topk=1, mode="paper", max_batch=0, batch=0,
                 streams=0, ring_slots=0, rule_capacity=0, kernel="auto"):
        cfg = tang_config()
        cfg.device = device
        cfg.mlp = {"bf16": TANG_MLP_BF16_TC, "fp32": TANG_MLP_FP32_FFMA, "fp8": TANG_MLP_FP8_TC,
                   "nvfp4": TANG_MLP_NVFP4_TC}[mlp]
        cfg.topk = topk
        cfg.mode = {"paper": TANG_MODE_PAPER, "strict": TANG_MODE_STRICT}[mode]
        cfg.max_batch, cfg.batch, cfg.streams = max_batch, batch, streams
        cfg.ring_slots, cfg.rule_capacity = ring_slots, rule_capacity
        cfg.mlp_kernel = {"auto": TANG_KERNEL_AUTO, "single": TANG_KERNEL_SINGLE, "pair": TANG_KERNEL_PAIR,
                          "2sm": TANG_KERNEL_2SM, "wide": TANG_KERNEL_WIDE,
                          "dual": TANG_KERNEL_DUAL}[kernel]
        self.topk = topk
        self.h = None
        self.h = tang_build(rules, blob, cfg)
        st = tang_stats(self.h)
        self.C = st["C"]

    def close(self):
        if getattr(self, "h", None) and _lib is not None and _lib.tang_destroy is not None:
            try:
                tang_destroy(self.h)
            except TypeError:      # interpreter shutdown: the library is already gone
                pass
            self.h = None

    __del__ = close

    def stats(self):
        return tang_stats(self.h)

    def classify(self, headers, out=None):
        return tang_classify(self.h, headers, out)

    def classify_async(self, d_hdr, d_out, n=None, stream=None):
        tang_classify_async(self.h, d_hdr, n if n is not None else d_out.numel(), d_out, stream)

    def classify_ex(self, d_hdr, d_out, d_pred=None, d_logits=None, d_fellback=None, stream=None):
        tang_classify_ex(self.h, d_hdr, d_out.numel(), d_out, d_pred, d_logits, d_fellback, stream)

    def classify_with_pred(self, d_hdr, d_pred, k, d_out, d_fellback=None, stream=None):
        tang_classify_with_pred(self.h, d_hdr, d_out.numel(), d_pred, k, d_out, d_fellback, stream)

    def encode(self, d_hdr, d_feat, stream=None):
        tang_encode_async(self.h, d_hdr, d_feat.numel() // 7, d_feat, stream)

    def update(self, ops, stream=None):
        return tang_update(self.h, ops, stream)

    def update_plan(self, ops):
        return tang_update_plan(self.h, ops)

    def apply_delta_async(self, d_delta, nbytes, stream=None):
        tang_apply_delta_async(self.h, d_delta, nbytes, stream)

    def apply_delta_host(self, delta):
        tang_apply_delta_host(self.h, delta)

    def device_checksum(self):
        return tang_device_checksum(self.h)

    def digest_async(self, d_digest, stream=None):
        tang_table_digest_async(self.h, d_digest, stream)

    def mirror_digest(self):
        return tang_mirror_digest(self.h)

    def candidates(self, sip, dip):
        """Candidate tuples of the post-verification search for these addresses (test hook)."""
        W = _lib.tang_debug_candidates(self.h, int(sip), int(dip), None, 0)
        buf = (C.c_uint32 * max(1, W))()
        _lib.tang_debug_candidates(self.h, int(sip), int(dip), buf, W)
        return {32 * q + b for q in range(W) for b in range(32) if (buf[q] >> b) & 1}

    def rule_tuple(self, rule_id):
        return tang_rule_tuple(self.h, rule_id)

    def profile(self, on=True):
        tang_profile_enable(self.h, on)

    def profile_read(self):
        return tang_profile_read(self.h)

    def timeline(self):
        return tang_timeline_read(self.h)

    def latencies(self):
        return tang_latency_read(self.h)

    def reload_model(self, blob):
        tang_reload_model(self.h, blob)
