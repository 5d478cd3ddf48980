"""Thin Python binding of libhisa (include/hisa.h) -- argument marshalling only.

Every ``hisa_*`` function below has the C name and calls straight into the sm_100a library;
no step of the HISA path runs in Python or on the CPU.  There is no fallback: if the CUDA
extension is missing or no device is present, ``load()`` / ``hisa_ctx_create`` raise.

``Context`` bundles a context with a torch-owned device arena and torch's current stream
(PyTorch is the device-memory / stream / process-group plumbing, not the product).
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

from . import _build

LIB_PATH = _build.LIB
HEADER = os.path.join(os.path.dirname(_build.PKG), "include", "hisa.h")

ERRORS = {
    0: "OK", -1: "INVALID_HANDLE", -2: "UNSUPPORTED_PROFILE", -3: "LEVEL_MISMATCH", -4: "SCALE_MISMATCH",
    -5: "INVALID_DIVISOR", -6: "MODULUS_EXHAUSTED", -7: "NO_KEY", -8: "CAPACITY", -9: "NOT_RELINEARIZED",
    -10: "OOM", -11: "CUDA", -12: "PARAMS", -13: "NO_SECRET",
}
PROFILE_ENCRYPTION, PROFILE_INTEGERS, PROFILE_DIVISION, PROFILE_RELIN, PROFILE_BOOTSTRAP = 1, 2, 4, 8, 16


class HisaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = ERRORS.get(code, str(code))
        self.rc = code
        super().__init__(f"HISA_E_{self.code}: {msg}")


class hisa_params(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_int), ("num_q", ctypes.c_int), ("q_bits", ctypes.POINTER(ctypes.c_int)),
                ("p_bits", ctypes.c_int), ("seed", ctypes.c_uint64), ("device", ctypes.c_int)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_ci, _cu64, _ci64, _cd, _csz = ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t

_SIGS = {
    "hisa_ctx_create": [ctypes.POINTER(hisa_params), ctypes.POINTER(_vp)],
    "hisa_ctx_destroy": [_vp],
    "hisa_attach_arena": [_vp, _vp, _csz],
    "hisa_set_stream": [_vp, _vp],
    "hisa_sync": [_vp],
    "hisa_supports": [_vp, _ci],
    "hisa_moduli": [_vp, _u64p, _csz],
    "hisa_ring_degree": [_vp, _u64p, ctypes.POINTER(_ci)],
    "hisa_mem_stats": [_vp, ctypes.POINTER(_csz), ctypes.POINTER(_csz)],
    "hisa_keygen": [_vp, _i64p, _csz, _ci, _ci],
    "hisa_key_export": [_vp, _ci64, _u64p, _csz],
    "hisa_encrypt": [_vp, _cu64, _u64p],
    "hisa_decrypt": [_vp, _cu64, _u64p],
    "hisa_copy": [_vp, _cu64, _u64p],
    "hisa_free": [_vp, _cu64],
    "hisa_encode": [_vp, _dp, _csz, _cd, _ci, _u64p],
    "hisa_encode_batch": [_vp, _dp, _csz, _csz, _cd, _ci, _u64p],
    "hisa_decode": [_vp, _cu64, _dp, _csz],
    "hisa_decode_batch": [_vp, _u64p, _csz, _dp, _csz],
    "hisa_rot_left": [_vp, _cu64, _ci64, _u64p],
    "hisa_rot_right": [_vp, _cu64, _ci64, _u64p],
    "hisa_add": [_vp, _cu64, _cu64, _u64p],
    "hisa_sub": [_vp, _cu64, _cu64, _u64p],
    "hisa_add_plain": [_vp, _cu64, _cu64, _u64p],
    "hisa_sub_plain": [_vp, _cu64, _cu64, _u64p],
    "hisa_add_scalar": [_vp, _cu64, _cd, _u64p],
    "hisa_sub_scalar": [_vp, _cu64, _cd, _u64p],
    "hisa_mul": [_vp, _cu64, _cu64, _u64p],
    "hisa_mul_plain": [_vp, _cu64, _cu64, _u64p],
    "hisa_mul_scalar": [_vp, _cu64, _cd, _cd, _u64p],
    "hisa_max_scalar_div": [_vp, _cu64, _cu64, _u64p],
    "hisa_div_scalar": [_vp, _cu64, _cu64, _u64p],
    "hisa_rescale": [_vp, _cu64, _u64p],
    "hisa_mul_norelin": [_vp, _cu64, _cu64, _u64p],
    "hisa_relinearize": [_vp, _cu64],
    "hisa_bootstrap": [_vp, _cu64],
    "hisa_mod_switch": [_vp, _cu64, _ci, _u64p],
    "hisa_rot_left_hoisted": [_vp, _cu64, _i64p, _csz, _u64p],
    "hisa_rot_left_batch": [_vp, _u64p, _csz, _ci64, _u64p],
    "hisa_rot_left_hoisted_batch": [_vp, _u64p, _csz, _i64p, _csz, _u64p],
    "hisa_conv_accumulate": [_vp, _u64p, _csz, _dp, _csz, _cd, _u64p],
    "hisa_conv_accumulate_dev": [_vp, _u64p, _csz, _dp, _csz, _cd, _vp],
    "hisa_rot_add_batch": [_vp, _u64p, _csz, _ci64, _u64p],
    "hisa_mul_batch": [_vp, _u64p, _u64p, _csz, _u64p],
    "hisa_rescale_batch": [_vp, _u64p, _csz, _u64p],
    "hisa_mul_plain_batch": [_vp, _u64p, _u64p, _csz, _u64p],
    "hisa_mul_plain_accumulate": [_vp, _u64p, _csz, _u64p, _csz, _u64p],
    "hisa_ct_adopt_sum": [_vp, _vp, _ci, _ci, _cd, _u64p],
    "hisa_ntt": [_vp, _cu64, _ci],
    "hisa_ntt_batch": [_vp, _u64p, _csz, _ci],
    "hisa_ct_info": [_vp, _cu64, ctypes.POINTER(_ci), ctypes.POINTER(_ci), ctypes.POINTER(_cd)],
    "hisa_pt_info": [_vp, _cu64, ctypes.POINTER(_ci), ctypes.POINTER(_cd)],
    "hisa_ct_export": [_vp, _cu64, _u64p, _csz],
    "hisa_ct_import": [_vp, _u64p, _ci, _ci, _cd, _u64p],
    "hisa_pt_export": [_vp, _cu64, _u64p, _csz],
    "hisa_pt_import": [_vp, _u64p, _ci, _cd, _u64p],
    "hisa_ct_device_view": [_vp, _cu64, ctypes.POINTER(_u64p), ctypes.POINTER(_csz)],
    "hisa_ct_adopt_device": [_vp, _vp, _ci, _ci, _cd, _u64p],
    "hisa_ct_random": [_vp, _cu64, _ci, _ci, _u64p],
    "hisa_pt_random": [_vp, _cu64, _ci, _u64p],
    "hisa_profile": [_vp, _ci],
    "hisa_profile_read": [_vp, ctypes.c_char_p, _csz, _dp, _u64p, _csz, ctypes.POINTER(_csz)],
    "hisa_launch_count": [_vp, _u64p],
    "hisa_microbench_butterfly": [_vp, _ci, _dp],
    "hisa_microbench_butterfly_f64": [_vp, _ci, _dp],
    "hisa_microbench_mac": [_vp, _ci, _dp],
    "hisa_last_error": [],
}

_lib = None


def header_symbols() -> list[str]:
    """Every function name declared in include/hisa.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hisa_[a-z0-9_]+)\s*\(", txt)))


def load(build: bool = True):
    """Load (building if stale) libhisa.so.  Raises if the library cannot be built or loaded."""
    global _lib
    if _lib is None:
        if build:
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhisa.so missing at {LIB_PATH}; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_char_p if name == "hisa_last_error" else ctypes.c_int
        _lib = lib
    return _lib


def _chk(rc: int):
    if rc != 0:
        raise HisaError(rc, load().hisa_last_error().decode())


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------------------ raw bindings
def hisa_ctx_create(log_n: int, q_bits, p_bits: int, seed: int = 0, device: int = 0):
    qb = (ctypes.c_int * len(q_bits))(*q_bits)
    p = hisa_params(log_n, len(q_bits), qb, p_bits, seed, device)
    out = _vp()
    _chk(load().hisa_ctx_create(ctypes.byref(p), ctypes.byref(out)))
    return out


def hisa_ctx_destroy(ctx):
    _chk(load().hisa_ctx_destroy(ctx))


def hisa_attach_arena(ctx, dev_ptr: int, nbytes: int):
    _chk(load().hisa_attach_arena(ctx, _vp(dev_ptr), nbytes))


def hisa_set_stream(ctx, stream: int):
    _chk(load().hisa_set_stream(ctx, _vp(stream)))


def hisa_sync(ctx):
    _chk(load().hisa_sync(ctx))


def hisa_supports(ctx, profile: int) -> bool:
    return bool(load().hisa_supports(ctx, profile))


def hisa_moduli(ctx, n: int) -> list[int]:
    out = np.zeros(n, dtype=np.uint64)
    _chk(load().hisa_moduli(ctx, _ptr(out, _u64p), n))
    return [int(x) for x in out]


def hisa_ring_degree(ctx) -> tuple[int, int]:
    n, l = _cu64(), _ci()
    _chk(load().hisa_ring_degree(ctx, ctypes.byref(n), ctypes.byref(l)))
    return n.value, l.value


def hisa_mem_stats(ctx) -> tuple[int, int]:
    a, b = _csz(), _csz()
    _chk(load().hisa_mem_stats(ctx, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def hisa_keygen(ctx, rot_left_amounts=(), relin: bool = True, max_level: int = -1):
    r = np.ascontiguousarray(list(rot_left_amounts), dtype=np.int64)
    _chk(load().hisa_keygen(ctx, _ptr(r, _i64p) if r.size else None, r.size, int(relin), int(max_level)))


def hisa_key_export(ctx, which: int, words: int) -> np.ndarray:
    out = np.zeros(words, dtype=np.uint64)
    _chk(load().hisa_key_export(ctx, which, _ptr(out, _u64p), words))
    return out


def _h1(fn, *args) -> int:
    out = _cu64()
    _chk(fn(*args, ctypes.byref(out)))
    return out.value


def _hopt(fn, ctx, *args, inplace=False):
    if inplace:
        _chk(fn(ctx, *args, None))
        return args[0]
    return _h1(fn, ctx, *args)


def hisa_encrypt(ctx, pt: int) -> int:
    return _h1(load().hisa_encrypt, ctx, pt)


def hisa_decrypt(ctx, ct: int) -> int:
    return _h1(load().hisa_decrypt, ctx, ct)


def hisa_copy(ctx, ct: int) -> int:
    return _h1(load().hisa_copy, ctx, ct)


def hisa_free(ctx, h: int):
    _chk(load().hisa_free(ctx, h))


def hisa_encode(ctx, v, scale: float, level: int = -1) -> int:
    a = np.ascontiguousarray(v, dtype=np.float64)
    return _h1(load().hisa_encode, ctx, _ptr(a, _dp), a.size, float(scale), level)


def hisa_encode_batch(ctx, vs, scale: float, level: int = -1) -> list[int]:
    """vs: (count, n_per) array of slot values -> count plaintext handles."""
    a = np.ascontiguousarray(vs, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("vs must be 2-D (count, n_per)")
    outs = np.zeros(a.shape[0], dtype=np.uint64)
    _chk(load().hisa_encode_batch(ctx, _ptr(a, _dp), a.shape[1], a.shape[0], float(scale), level,
                                  _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_decode(ctx, pt: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.float64)
    _chk(load().hisa_decode(ctx, pt, _ptr(out, _dp), n))
    return out


def hisa_decode_batch(ctx, pts, n: int) -> np.ndarray:
    ins = _u64(list(pts))
    out = np.zeros((ins.size, n), dtype=np.float64)
    _chk(load().hisa_decode_batch(ctx, _ptr(ins, _u64p), ins.size, _ptr(out, _dp), n))
    return out


def hisa_rot_left(ctx, ct: int, k: int, inplace=False) -> int:
    return _hopt(load().hisa_rot_left, ctx, ct, k, inplace=inplace)


def hisa_rot_right(ctx, ct: int, k: int, inplace=False) -> int:
    return _hopt(load().hisa_rot_right, ctx, ct, k, inplace=inplace)


def hisa_add(ctx, a: int, b: int, inplace=False) -> int:
    return _hopt(load().hisa_add, ctx, a, b, inplace=inplace)


def hisa_sub(ctx, a: int, b: int, inplace=False) -> int:
    return _hopt(load().hisa_sub, ctx, a, b, inplace=inplace)


def hisa_add_plain(ctx, a: int, p: int, inplace=False) -> int:
    return _hopt(load().hisa_add_plain, ctx, a, p, inplace=inplace)


def hisa_sub_plain(ctx, a: int, p: int, inplace=False) -> int:
    return _hopt(load().hisa_sub_plain, ctx, a, p, inplace=inplace)


def hisa_add_scalar(ctx, a: int, x: float, inplace=False) -> int:
    return _hopt(load().hisa_add_scalar, ctx, a, float(x), inplace=inplace)


def hisa_sub_scalar(ctx, a: int, x: float, inplace=False) -> int:
    return _hopt(load().hisa_sub_scalar, ctx, a, float(x), inplace=inplace)


def hisa_mul(ctx, a: int, b: int, inplace=False) -> int:
    return _hopt(load().hisa_mul, ctx, a, b, inplace=inplace)


def hisa_mul_plain(ctx, a: int, p: int, inplace=False) -> int:
    return _hopt(load().hisa_mul_plain, ctx, a, p, inplace=inplace)


def hisa_mul_scalar(ctx, a: int, x: float, pt_scale: float = 0.0, inplace=False) -> int:
    return _hopt(load().hisa_mul_scalar, ctx, a, float(x), float(pt_scale), inplace=inplace)


def hisa_max_scalar_div(ctx, ct: int, ub: int) -> int:
    return _h1(load().hisa_max_scalar_div, ctx, ct, ub)


def hisa_div_scalar(ctx, ct: int, d: int, inplace=False) -> int:
    return _hopt(load().hisa_div_scalar, ctx, ct, d, inplace=inplace)


def hisa_rescale(ctx, ct: int, inplace=False) -> int:
    return _hopt(load().hisa_rescale, ctx, ct, inplace=inplace)


def hisa_mul_norelin(ctx, a: int, b: int, inplace=False) -> int:
    return _hopt(load().hisa_mul_norelin, ctx, a, b, inplace=inplace)


def hisa_relinearize(ctx, ct: int):
    _chk(load().hisa_relinearize(ctx, ct))


def hisa_bootstrap(ctx, ct: int):
    _chk(load().hisa_bootstrap(ctx, ct))


def hisa_mod_switch(ctx, ct: int, drop: int = 1, inplace=False) -> int:
    return _hopt(load().hisa_mod_switch, ctx, ct, drop, inplace=inplace)


def hisa_rot_left_hoisted(ctx, ct: int, ks) -> list[int]:
    k = np.ascontiguousarray(list(ks), dtype=np.int64)
    outs = np.zeros(k.size, dtype=np.uint64)
    _chk(load().hisa_rot_left_hoisted(ctx, ct, _ptr(k, _i64p), k.size, _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_rot_left_hoisted_batch(ctx, cts, ks) -> list[list[int]]:
    """[[rotLeft(ct, k) for k in ks] for ct in cts] with shared ModUps and key streams."""
    ins = _u64(list(cts))
    k = np.ascontiguousarray(list(ks), dtype=np.int64)
    outs = np.zeros(ins.size * k.size, dtype=np.uint64)
    if ins.size and k.size:
        _chk(load().hisa_rot_left_hoisted_batch(ctx, _ptr(ins, _u64p), ins.size, _ptr(k, _i64p), k.size,
                                                _ptr(outs, _u64p)))
    return [[int(x) for x in outs[i * k.size:(i + 1) * k.size]] for i in range(ins.size)]


def hisa_rot_left_batch(ctx, cts, k: int) -> list[int]:
    ins = _u64(list(cts))
    outs = np.zeros(ins.size, dtype=np.uint64)
    _chk(load().hisa_rot_left_batch(ctx, _ptr(ins, _u64p), ins.size, k, _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_conv_accumulate(ctx, cts, W, pt_scale: float = 0.0) -> list[int]:
    ins = _u64(list(cts))
    w = np.ascontiguousarray(W, dtype=np.float64)
    oc = w.size // max(ins.size, 1)
    outs = np.zeros(oc, dtype=np.uint64)
    _chk(load().hisa_conv_accumulate(ctx, _ptr(ins, _u64p), ins.size, _ptr(w, _dp), oc, float(pt_scale),
                                     _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_mul_batch(ctx, a, b) -> list[int]:
    x, y = _u64(list(a)), _u64(list(b))
    outs = np.zeros(x.size, dtype=np.uint64)
    _chk(load().hisa_mul_batch(ctx, _ptr(x, _u64p), _ptr(y, _u64p), x.size, _ptr(outs, _u64p)))
    return [int(v) for v in outs]


def hisa_rescale_batch(ctx, cts) -> list[int]:
    x = _u64(list(cts))
    outs = np.zeros(x.size, dtype=np.uint64)
    _chk(load().hisa_rescale_batch(ctx, _ptr(x, _u64p), x.size, _ptr(outs, _u64p)))
    return [int(v) for v in outs]


def hisa_rot_add_batch(ctx, cts, k: int) -> list[int]:
    ins = _u64(list(cts))
    outs = np.zeros(ins.size, dtype=np.uint64)
    _chk(load().hisa_rot_add_batch(ctx, _ptr(ins, _u64p), ins.size, k, _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_mul_plain_batch(ctx, cts, pts) -> list[int]:
    a, p = _u64(list(cts)), _u64(list(pts))
    outs = np.zeros(a.size, dtype=np.uint64)
    _chk(load().hisa_mul_plain_batch(ctx, _ptr(a, _u64p), _ptr(p, _u64p), a.size, _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_mul_plain_accumulate(ctx, cts, pts, J: int) -> list[int]:
    """outs[j] = sum_c cts[c] * pts[j * C + c]."""
    ins = _u64(list(cts))
    p = _u64(list(pts))
    outs = np.zeros(J, dtype=np.uint64)
    _chk(load().hisa_mul_plain_accumulate(ctx, _ptr(ins, _u64p), ins.size, _ptr(p, _u64p), J, _ptr(outs, _u64p)))
    return [int(x) for x in outs]


def hisa_conv_accumulate_dev(ctx, cts, W, dev_out: int, pt_scale: float = 0.0):
    """Accumulation into caller device memory (uint64 [OC][2][l+1][N] at address dev_out)."""
    ins = _u64(list(cts))
    w = np.ascontiguousarray(W, dtype=np.float64)
    oc = w.size // max(ins.size, 1)
    _chk(load().hisa_conv_accumulate_dev(ctx, _ptr(ins, _u64p), ins.size, _ptr(w, _dp), oc, float(pt_scale),
                                         _vp(dev_out)))


def hisa_ct_adopt_sum(ctx, dev_ptr: int, level: int, npolys: int, scale: float) -> int:
    return _h1(load().hisa_ct_adopt_sum, ctx, _vp(dev_ptr), level, npolys, float(scale))


def hisa_ntt(ctx, ct: int, inverse: bool = False):
    _chk(load().hisa_ntt(ctx, ct, int(inverse)))


def hisa_ntt_batch(ctx, cts, inverse: bool = False):
    ins = _u64(list(cts))
    _chk(load().hisa_ntt_batch(ctx, _ptr(ins, _u64p), ins.size, int(inverse)))


def hisa_ct_info(ctx, ct: int) -> tuple[int, int, float]:
    lv, npl, sc = _ci(), _ci(), _cd()
    _chk(load().hisa_ct_info(ctx, ct, ctypes.byref(lv), ctypes.byref(npl), ctypes.byref(sc)))
    return lv.value, npl.value, sc.value


def hisa_pt_info(ctx, pt: int) -> tuple[int, float]:
    lv, sc = _ci(), _cd()
    _chk(load().hisa_pt_info(ctx, pt, ctypes.byref(lv), ctypes.byref(sc)))
    return lv.value, sc.value


def hisa_ct_export(ctx, ct: int) -> np.ndarray:
    n, _ = hisa_ring_degree(ctx)
    lv, npl, _sc = hisa_ct_info(ctx, ct)
    out = np.zeros((npl, lv + 1, n), dtype=np.uint64)
    _chk(load().hisa_ct_export(ctx, ct, _ptr(out, _u64p), out.size))
    return out


def hisa_ct_import(ctx, data, level: int, npolys: int, scale: float) -> int:
    a = _u64(data)
    return _h1(load().hisa_ct_import, ctx, _ptr(a, _u64p), level, npolys, float(scale))


def hisa_pt_export(ctx, pt: int) -> np.ndarray:
    n, _ = hisa_ring_degree(ctx)
    lv, _sc = hisa_pt_info(ctx, pt)
    out = np.zeros((lv + 1, n), dtype=np.uint64)
    _chk(load().hisa_pt_export(ctx, pt, _ptr(out, _u64p), out.size))
    return out


def hisa_pt_import(ctx, data, level: int, scale: float) -> int:
    a = _u64(data)
    return _h1(load().hisa_pt_import, ctx, _ptr(a, _u64p), level, float(scale))


def hisa_ct_device_view(ctx, ct: int) -> tuple[int, int]:
    p, w = _u64p(), _csz()
    _chk(load().hisa_ct_device_view(ctx, ct, ctypes.byref(p), ctypes.byref(w)))
    return ctypes.cast(p, ctypes.c_void_p).value or 0, w.value


def hisa_ct_adopt_device(ctx, dev_ptr: int, level: int, npolys: int, scale: float) -> int:
    return _h1(load().hisa_ct_adopt_device, ctx, _vp(dev_ptr), level, npolys, float(scale))


def hisa_ct_random(ctx, b: int, level: int, npolys: int = 2) -> int:
    return _h1(load().hisa_ct_random, ctx, b, level, npolys)


def hisa_pt_random(ctx, b: int, level: int) -> int:
    return _h1(load().hisa_pt_random, ctx, b, level)


def hisa_profile(ctx, enable: bool = True):
    _chk(load().hisa_profile(ctx, int(enable)))


def hisa_profile_read(ctx) -> dict[str, tuple[float, int]]:
    """{kernel class: (total ms, launches)} recorded since hisa_profile(ctx, True)."""
    buf = ctypes.create_string_buffer(1 << 16)
    ms = np.zeros(256, dtype=np.float64)
    cnt = np.zeros(256, dtype=np.uint64)
    n = _csz()
    _chk(load().hisa_profile_read(ctx, buf, len(buf), _ptr(ms, _dp), _ptr(cnt, _u64p), 256, ctypes.byref(n)))
    names = buf.value.decode().split("\n")[: n.value]
    return {nm: (float(ms[i]), int(cnt[i])) for i, nm in enumerate(names)}


def hisa_launch_count(ctx) -> int:
    return _h1(load().hisa_launch_count, ctx)


def hisa_microbench_butterfly(ctx, iters: int = 2000) -> float:
    out = _cd()
    _chk(load().hisa_microbench_butterfly(ctx, iters, ctypes.byref(out)))
    return out.value


def hisa_microbench_butterfly_f64(ctx, iters: int = 2000) -> float:
    out = _cd()
    _chk(load().hisa_microbench_butterfly_f64(ctx, iters, ctypes.byref(out)))
    return out.value


def hisa_microbench_mac(ctx, iters: int = 2000) -> float:
    out = _cd()
    _chk(load().hisa_microbench_mac(ctx, iters, ctypes.byref(out)))
    return out.value


def hisa_last_error() -> str:
    return load().hisa_last_error().decode()


# ------------------------------------------------------------------------------ convenience
class Context:
    """A libhisa context on ``cuda:device`` whose device memory is one torch uint8 tensor."""

    def __init__(self, log_n: int, q_bits, p_bits: int, seed: int = 0, device: int = 0,
                 arena_bytes: int | None = None):
        import torch
        if not torch.cuda.is_available():
            raise HisaError(-11, "no CUDA device: libhisa has no CPU fallback")
        torch.cuda.set_device(device)
        self.ctx = hisa_ctx_create(log_n, list(q_bits), p_bits, seed, device)
        self.N, self.L = hisa_ring_degree(self.ctx)
        self.slots = self.N // 2
        self.moduli = hisa_moduli(self.ctx, self.L + 1)
        self.q, self.p = self.moduli[:-1], self.moduli[-1]
        self._arena = None
        # HISA_NO_ARENA=1 (sanitizer runs, tools/sanitize.sh): every buffer its own
        # cudaMallocAsync allocation, so compute-sanitizer memcheck sees each buffer's bounds
        if not os.environ.get("HISA_NO_ARENA"):
            if arena_bytes is None:
                free, _total = torch.cuda.mem_get_info(device)
                arena_bytes = int(free * 0.6)
            self._arena = torch.empty(arena_bytes, dtype=torch.uint8, device=f"cuda:{device}")
            hisa_attach_arena(self.ctx, self._arena.data_ptr(), arena_bytes)
        hisa_set_stream(self.ctx, torch.cuda.current_stream(device).cuda_stream)

    def close(self):
        if getattr(self, "ctx", None):
            hisa_ctx_destroy(self.ctx)
            self.ctx = None
            self._arena = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __getattr__(self, name):
        # ctx.rot_left(ct, k) -> hisa_rot_left(ctx.ctx, ct, k)
        f = globals().get("hisa_" + name)
        if f is None:
            raise AttributeError(name)
        return lambda *a, **kw: f(self.ctx, *a, **kw)
