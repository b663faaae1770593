"""B200-native TFHE programmable bootstrap behind the Leuvenshtein API.

Thin Python view (ctypes) of the C ABI in include/leuven_b200.h. It mirrors
the reference's surface — ``leuven::Backend`` (proj/include/leuven/
backend.hpp:50-77), ``kernel::distance_encrypted`` (kernel.hpp:208-212),
``preprocess::build_eq_table`` / ``distance_preprocessed``
(preprocess.hpp:45-53), ``cli::compute_report`` (cli.hpp:39) and the pybind
``compute`` (proj/bindings/module.cpp:63-86) — with the same names, argument
meaning and exception types. All arithmetic runs in the CUDA library; there
is no CPU fallback: importing works anywhere, but creating a ``Context``
without the built library or without a GPU raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LVB_LIB overrides the library (experiment variants built by build.py --out)
LIB_PATH = os.environ.get("LVB_LIB", os.path.join(HERE, "_build", "libleuven_b200.so"))

# ----------------------------------------------------------------- errors
# One class per reference exception (proj/include/leuven/errors.hpp:8-39).


class Error(RuntimeError):
    code = 99


class OutOfRangeValue(Error):
    code = 1


class NoiseBudgetExceeded(Error):
    code = 2


class ValueOutsideLutHalf(Error):
    code = 3


class PackingViolation(Error):
    code = 4


class CharNotInAlphabet(Error):
    code = 5


class CharNotInSubset(Error):
    code = 6


class PositionOutOfRange(Error):
    code = 7


class BandTooNarrow(Error):
    code = 8


class FormatError(Error):
    code = 9


class InvalidParams(Error):
    code = 10


class CudaError(Error):
    code = 20


class InvalidHandle(Error):
    code = 21


_ERRORS = {cls.code: cls for cls in (OutOfRangeValue, NoiseBudgetExceeded, ValueOutsideLutHalf,
                                     PackingViolation, CharNotInAlphabet, CharNotInSubset,
                                     PositionOutOfRange, BandTooNarrow, FormatError, InvalidParams,
                                     CudaError, InvalidHandle)}

# ----------------------------------------------------------------- ABI


class Params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("N", ctypes.c_uint32), ("k", ctypes.c_uint32),
                ("pbs_base_log", ctypes.c_uint32), ("pbs_level", ctypes.c_uint32),
                ("ks_base_log", ctypes.c_uint32), ("ks_level", ctypes.c_uint32),
                ("lwe_noise_log2", ctypes.c_uint32), ("glwe_noise_log2", ctypes.c_uint32),
                ("max_variance_budget", ctypes.c_double), ("exact_mask_product", ctypes.c_uint32),
                ("device", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("pbs_count", ctypes.c_uint64), ("refresh_count", ctypes.c_uint64),
                ("linear_op_count", ctypes.c_uint64)]


class Band(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("half_width", ctypes.c_uint64)]


class Run(ctypes.Structure):
    _fields_ = [("visited_cells", ctypes.c_uint64), ("equality_pbs", ctypes.c_uint64),
                ("kernel_pbs", ctypes.c_uint64), ("refreshes", ctypes.c_uint64),
                ("max_key_variance", ctypes.c_int64), ("waves", ctypes.c_uint64)]


# Every exported symbol declared in include/leuven_b200.h (checked by tests).
EXPORTS = [
    "lv_default_params", "lv_ctx_create", "lv_ctx_destroy", "lv_last_error", "lv_abi_version",
    "lv_keys_size", "lv_keys_export", "lv_ctx_create_eval", "lv_ctx_key_id",
    "lv_lut_table", "lv_encrypt", "lv_trivial", "lv_decrypt", "lv_add", "lv_sub", "lv_scalar_mul",
    "lv_scalar_add", "lv_lut_upload", "lv_pbs_batch", "lv_refresh_batch", "lv_predict_variance",
    "lv_get_stats", "lv_get_params", "lv_release", "lv_ledger_variance", "lv_export",
    "lv_import", "lv_phase", "lv_pbs_batch_host", "lv_band_resolve", "lv_edit_distance_ee",
    "lv_edit_distance_batch", "lv_eq_table_build", "lv_eq_table_lookup", "lv_eq_table_destroy",
    "lv_edit_distance_pre", "lv_edit_distance_pre_batch", "lv_edit_distance_eq9", "lv_plan_trace", "lv_debug_keys",
    "lv_debug_keyswitch",
    "lv_eq_table_serialize", "lv_eq_table_deserialize",
    "lv_debug_blind_rotate", "lv_debug_fft", "lv_bench_pbs", "lv_bench_fp64_peak",
]

_lib = None


def build():
    import importlib
    return importlib.import_module(__name__ + ".build").build()


def lib():
    """Loads the CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2508_14568_b200.build() "
                              "(the product has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        vp, u32, u64, i32, i64, sz = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t)
        sig = {
            "lv_default_params": (None, [P(Params)]),
            "lv_ctx_create": (ctypes.c_int, [P(Params), u64, P(vp)]),
            "lv_keys_size": (ctypes.c_int, [P(Params), P(u64), P(u64)]),
            "lv_keys_export": (ctypes.c_int, [vp, P(u64), P(u64), P(u64)]),
            "lv_ctx_create_eval": (ctypes.c_int, [P(Params), P(u64), P(u64), u64, P(vp)]),
            "lv_ctx_key_id": (ctypes.c_int, [vp, P(u64)]),
            "lv_ctx_destroy": (None, [vp]),
            "lv_last_error": (ctypes.c_char_p, []),
            "lv_abi_version": (ctypes.c_int, []),
            "lv_lut_table": (ctypes.c_int, [i32, P(i32)]),
            "lv_encrypt": (ctypes.c_int, [vp, P(i32), sz, P(u32)]),
            "lv_trivial": (ctypes.c_int, [vp, P(i32), sz, P(u32)]),
            "lv_decrypt": (ctypes.c_int, [vp, P(u32), sz, P(i32)]),
            "lv_add": (ctypes.c_int, [vp, P(u32), P(u32), sz, P(u32)]),
            "lv_sub": (ctypes.c_int, [vp, P(u32), P(u32), sz, P(u32)]),
            "lv_scalar_mul": (ctypes.c_int, [vp, P(u32), P(i32), sz, P(u32)]),
            "lv_scalar_add": (ctypes.c_int, [vp, P(u32), P(i32), sz, P(u32)]),
            "lv_lut_upload": (ctypes.c_int, [vp, P(i32), P(u32)]),
            "lv_pbs_batch": (ctypes.c_int, [vp, P(u32), P(u32), sz, P(u32)]),
            "lv_refresh_batch": (ctypes.c_int, [vp, P(u32), sz, P(u32)]),
            "lv_predict_variance": (ctypes.c_int, [vp, P(u32), P(i32), sz, P(i64)]),
            "lv_get_stats": (ctypes.c_int, [vp, P(Stats)]),
            "lv_get_params": (ctypes.c_int, [vp, P(Params)]),
            "lv_release": (ctypes.c_int, [vp, P(u32), sz]),
            "lv_ledger_variance": (ctypes.c_int, [vp, P(u32), sz, P(i64)]),
            "lv_export": (ctypes.c_int, [vp, P(u32), sz, P(u64)]),
            "lv_import": (ctypes.c_int, [vp, P(u64), sz, P(u32)]),
            "lv_phase": (ctypes.c_int, [vp, P(u32), sz, P(u64)]),
            "lv_pbs_batch_host": (ctypes.c_int, [vp, P(u64), P(u32), sz, P(u64)]),
            "lv_band_resolve": (ctypes.c_int, [i32, u64, u64, u64, P(Band)]),
            "lv_edit_distance_ee": (ctypes.c_int, [vp, P(u32), sz, P(u32), sz, u32, P(Band), i32,
                                                   P(u32), P(Run)]),
            "lv_edit_distance_batch": (ctypes.c_int, [vp, sz, P(u32), P(u64), P(u32), P(u64), u32,
                                                      P(Band), i32, P(u32), P(Run)]),
            "lv_eq_table_build": (ctypes.c_int, [vp, P(u32), sz, u32, ctypes.c_char_p, P(i32), sz,
                                                 P(vp), P(u64)]),
            "lv_eq_table_lookup": (ctypes.c_int, [vp, vp, ctypes.c_char, u64, P(u32)]),
            "lv_eq_table_destroy": (None, [vp, vp]),
            "lv_eq_table_serialize": (ctypes.c_int, [vp, vp, ctypes.c_char_p, u64,
                                                     ctypes.c_void_p, u64, P(u64)]),
            "lv_eq_table_deserialize": (ctypes.c_int, [vp, ctypes.c_char_p, u64, P(vp),
                                                       ctypes.c_void_p, u64, P(u64)]),
            "lv_edit_distance_pre": (ctypes.c_int, [vp, vp, ctypes.c_char_p, sz, P(Band), i32,
                                                    P(u32), P(Run)]),
            "lv_edit_distance_eq9": (ctypes.c_int, [vp, P(u32), u64, u64, P(Band), i32, P(u32),
                                                    P(Run)]),
            "lv_edit_distance_pre_batch": (ctypes.c_int, [vp, sz, P(vp), ctypes.c_char_p, P(u64),
                                                          P(Band), i32, P(u32), P(Run)]),
            "lv_plan_trace": (ctypes.c_int, [u64, u64, P(Band), i32, ctypes.c_double, u64, P(u32),
                                             P(i64), P(u32), P(u64), P(Run)]),
            "lv_debug_keys": (ctypes.c_int, [vp, P(ctypes.c_uint8), P(ctypes.c_uint8), P(u64),
                                             P(ctypes.c_double)]),
            "lv_debug_keyswitch": (ctypes.c_int, [vp, P(u64), sz, P(u64)]),
            "lv_debug_blind_rotate": (ctypes.c_int, [vp, P(u32), P(u32), sz, P(u64), P(u64)]),
            "lv_debug_fft": (ctypes.c_int, [vp, P(i64), P(ctypes.c_double), P(u64)]),
            "lv_bench_pbs": (ctypes.c_int, [vp, P(u32), P(u32), sz, ctypes.c_int, u64,
                                            P(ctypes.c_float), P(ctypes.c_float),
                                            P(ctypes.c_float)]),
            "lv_bench_fp64_peak": (ctypes.c_int, [P(ctypes.c_float)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().lv_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(msg)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32).reshape(-1))


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1).astype(np.int32))


def default_params() -> Params:
    p = Params()
    lib().lv_default_params(ctypes.byref(p))
    return p


# ----------------------------------------------------------------- LUTs
# proj/include/leuven/lut.hpp:9-41, proj/src/lut.cpp:9-22

PLAINTEXT_MODULUS = 32
LUT_SIZE = 16


def negacyclic_eval(lut, x: int) -> int:
    if not 0 <= x < PLAINTEXT_MODULUS:
        raise OutOfRangeValue(f"lookup input outside [0,32): {x}")
    if x < LUT_SIZE:
        return int(lut[x])
    return (PLAINTEXT_MODULUS - int(lut[x - LUT_SIZE])) % PLAINTEXT_MODULUS


def identity_lut():
    return list(range(LUT_SIZE))


def eq_lut(scale: int):
    """equality.cpp:31-36."""
    if not 1 <= scale < LUT_SIZE:
        raise OutOfRangeValue(f"equality scale must be in [1,16): {scale}")
    return [scale] + [0] * 15


# ----------------------------------------------------------------- backend


class Context:
    """One keyset on one GPU: the B200 implementation of leuven::Backend.

    Ciphertexts are uint32 handles into a device pool; every method accepts
    scalars or arrays and is batched underneath.
    """

    def __init__(self, seed: int | None = None, params: Params | None = None,
                 budget: float | None = None, _eval_keys=None, device: int | None = None):
        # every secret derives from the seed: OS entropy unless a test or an
        # experiment pins it
        if seed is None:
            seed = int.from_bytes(os.urandom(8), "little")
        p = params if params is not None else default_params()
        if budget is not None:
            p.max_variance_budget = float(budget)
        if device is not None:  # else the calling thread's current CUDA device
            p.device = int(device)
        self.params = p
        self.seed = seed
        h = ctypes.c_void_p()
        if _eval_keys is None:
            _check(lib().lv_ctx_create(ctypes.byref(p), seed, ctypes.byref(h)))
        else:
            bsk, ksk, key_id = _eval_keys
            _check(lib().lv_ctx_create_eval(ctypes.byref(p), _ptr(bsk, ctypes.c_uint64),
                                            _ptr(ksk, ctypes.c_uint64), int(key_id),
                                            ctypes.byref(h)))
        self._h = h
        self.n, self.N = p.n, p.N
        self.row = p.k * p.N + 1

    # client / server split -------------------------------------------
    def export_keys(self):
        """Evaluation keys of this (secret-holding) context: (bsk, ksk, key_id),
        the BSK in the standard domain [n][2][2][N] and the KSK [N][5][n+1]
        as uint64 arrays (lv_keys_export)."""
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().lv_keys_size(ctypes.byref(self.params), ctypes.byref(nb), ctypes.byref(nk)))
        bsk = np.zeros(nb.value, np.uint64)
        ksk = np.zeros(nk.value, np.uint64)
        kid = ctypes.c_uint64()
        _check(lib().lv_keys_export(self._h, _ptr(bsk, ctypes.c_uint64), _ptr(ksk, ctypes.c_uint64),
                                    ctypes.byref(kid)))
        return bsk, ksk, kid.value

    def key_id(self) -> int:
        """Key-set fingerprint (hash of the public KSK + parameters)."""
        k = ctypes.c_uint64()
        _check(lib().lv_ctx_key_id(self._h, ctypes.byref(k)))
        return k.value

    @classmethod
    def evaluation(cls, bsk, ksk, key_id: int, params: Params | None = None,
                   budget: float | None = None) -> "Context":
        """A server context from a client's evaluation keys (lv_ctx_create_eval):
        no secret key, so encrypt/decrypt/phase raise InvalidParams."""
        p = params if params is not None else default_params()
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().lv_keys_size(ctypes.byref(p), ctypes.byref(nb), ctypes.byref(nk)))
        b = np.ascontiguousarray(bsk, np.uint64).reshape(-1)
        k = np.ascontiguousarray(ksk, np.uint64).reshape(-1)
        if b.size != nb.value or k.size != nk.value:
            raise InvalidParams(f"evaluation keys: expected {nb.value} BSK and {nk.value} KSK words, "
                                f"got {b.size} and {k.size}")
        return cls(seed=0, params=p, budget=budget, _eval_keys=(b, k, key_id))

    def close(self):
        if getattr(self, "_h", None):
            lib().lv_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Backend surface ------------------------------------------------
    def encrypt(self, values):
        v = _i32(values)
        out = np.zeros(v.size, np.uint32)
        _check(lib().lv_encrypt(self._h, _ptr(v, ctypes.c_int32), v.size, _ptr(out, ctypes.c_uint32)))
        return out

    def trivial(self, values):
        v = _i32(values)
        out = np.zeros(v.size, np.uint32)
        _check(lib().lv_trivial(self._h, _ptr(v, ctypes.c_int32), v.size, _ptr(out, ctypes.c_uint32)))
        return out

    def decrypt(self, cts):
        c = _u32(cts)
        out = np.zeros(c.size, np.int32)
        _check(lib().lv_decrypt(self._h, _ptr(c, ctypes.c_uint32), c.size, _ptr(out, ctypes.c_int32)))
        return out

    def phase(self, cts):
        c = _u32(cts)
        out = np.zeros(c.size, np.uint64)
        _check(lib().lv_phase(self._h, _ptr(c, ctypes.c_uint32), c.size, _ptr(out, ctypes.c_uint64)))
        return out

    def _lin2(self, fn, a, b):
        a, b = _u32(a), _u32(b)
        if a.size != b.size:
            raise InvalidParams(f"operand counts differ ({a.size} vs {b.size})")
        out = np.zeros(a.size, np.uint32)
        _check(fn(self._h, _ptr(a, ctypes.c_uint32), _ptr(b, ctypes.c_uint32), a.size,
                  _ptr(out, ctypes.c_uint32)))
        return out

    def add(self, a, b):
        return self._lin2(lib().lv_add, a, b)

    def sub(self, a, b):
        return self._lin2(lib().lv_sub, a, b)

    def _scal(self, fn, a, k):
        a = _u32(a)
        kk = _i32(np.broadcast_to(np.asarray(k), a.shape))
        out = np.zeros(a.size, np.uint32)
        _check(fn(self._h, _ptr(a, ctypes.c_uint32), _ptr(kk, ctypes.c_int32), a.size,
                  _ptr(out, ctypes.c_uint32)))
        return out

    def scalar_mul(self, a, k):
        return self._scal(lib().lv_scalar_mul, a, k)

    def scalar_add(self, a, k):
        return self._scal(lib().lv_scalar_add, a, k)

    def lut(self, entries) -> int:
        e = _i32(entries)
        if e.size != 16:
            raise OutOfRangeValue("a Lut16 has 16 entries")
        out = ctypes.c_uint32()
        _check(lib().lv_lut_upload(self._h, _ptr(e, ctypes.c_int32), ctypes.byref(out)))
        return out.value

    def pbs(self, cts, lut=None, lut_ids=None):
        """Backend::pbs over a batch: ``lut`` is one Lut16 (16 entries) or one
        registered id (``ctx.lut``) applied to every ciphertext; ``lut_ids``
        gives one registered id per ciphertext instead."""
        c = _u32(cts)
        if lut_ids is not None:
            ids = _u32(lut_ids)
        elif lut is not None and np.ndim(lut) == 0:
            ids = np.full(c.size, int(lut), np.uint32)
        elif lut is not None:
            ids = np.full(c.size, self.lut(lut), np.uint32)
        else:
            raise InvalidParams("pbs needs a Lut16, a lut id or per-ciphertext lut_ids")
        if ids.size != c.size:
            raise InvalidParams("one lut id per ciphertext")
        out = np.zeros(c.size, np.uint32)
        _check(lib().lv_pbs_batch(self._h, _ptr(c, ctypes.c_uint32), _ptr(ids, ctypes.c_uint32),
                                  c.size, _ptr(out, ctypes.c_uint32)))
        return out

    def refresh(self, cts):
        c = _u32(cts)
        out = np.zeros(c.size, np.uint32)
        _check(lib().lv_refresh_batch(self._h, _ptr(c, ctypes.c_uint32), c.size,
                                      _ptr(out, ctypes.c_uint32)))
        return out

    def predict_variance(self, terms) -> int:
        c = _u32([t[0] for t in terms])
        k = _i32([t[1] for t in terms])
        out = ctypes.c_int64()
        _check(lib().lv_predict_variance(self._h, _ptr(c, ctypes.c_uint32), _ptr(k, ctypes.c_int32),
                                         c.size, ctypes.byref(out)))
        return out.value

    def variance(self, cts):
        c = _u32(cts)
        out = np.zeros(c.size, np.int64)
        _check(lib().lv_ledger_variance(self._h, _ptr(c, ctypes.c_uint32), c.size,
                                        _ptr(out, ctypes.c_int64)))
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(lib().lv_get_stats(self._h, ctypes.byref(s)))
        return {"pbs_count": s.pbs_count, "refresh_count": s.refresh_count,
                "linear_op_count": s.linear_op_count}

    def release(self, cts):
        c = _u32(cts)
        _check(lib().lv_release(self._h, _ptr(c, ctypes.c_uint32), c.size))

    def export(self, cts) -> np.ndarray:
        c = _u32(cts)
        out = np.zeros((c.size, self.row), np.uint64)
        _check(lib().lv_export(self._h, _ptr(c, ctypes.c_uint32), c.size, _ptr(out, ctypes.c_uint64)))
        return out

    def import_(self, rows) -> np.ndarray:
        r = np.ascontiguousarray(rows, np.uint64).reshape(-1, self.row)
        out = np.zeros(r.shape[0], np.uint32)
        _check(lib().lv_import(self._h, _ptr(r, ctypes.c_uint64), r.shape[0], _ptr(out, ctypes.c_uint32)))
        return out

    def pbs_host(self, rows, lut_ids, out=None) -> np.ndarray:
        r = np.ascontiguousarray(rows, np.uint64).reshape(-1, self.row)
        ids = _u32(lut_ids)
        if out is None:
            out = np.zeros_like(r)
        _check(lib().lv_pbs_batch_host(self._h, _ptr(r, ctypes.c_uint64), _ptr(ids, ctypes.c_uint32),
                                       r.shape[0], _ptr(out, ctypes.c_uint64)))
        return out

    # debug / parity ------------------------------------------------
    def debug_keys(self):
        p = self.params
        sks = np.zeros(p.n, np.uint8)
        skg = np.zeros(p.k * p.N, np.uint8)
        ksk = np.zeros(p.k * p.N * p.ks_level * (p.n + 1), np.uint64)
        bskf = np.zeros(p.n * (p.k + 1) * p.pbs_level * (p.k + 1) * p.N, np.float64)
        _check(lib().lv_debug_keys(self._h, _ptr(sks, ctypes.c_uint8), _ptr(skg, ctypes.c_uint8),
                                   _ptr(ksk, ctypes.c_uint64), _ptr(bskf, ctypes.c_double)))
        return sks, skg, ksk, bskf

    def debug_keyswitch(self, rows):
        r = np.ascontiguousarray(rows, np.uint64).reshape(-1, self.row)
        out = np.zeros((r.shape[0], self.n + 1), np.uint64)
        _check(lib().lv_debug_keyswitch(self._h, _ptr(r, ctypes.c_uint64), r.shape[0],
                                        _ptr(out, ctypes.c_uint64)))
        return out

    def debug_blind_rotate(self, ms, lut_ids, glwe: bool = False):
        m = np.ascontiguousarray(ms, np.uint32).reshape(-1, self.n + 1)
        ids = _u32(lut_ids)
        out = np.zeros((m.shape[0], self.row), np.uint64)
        g = np.zeros((m.shape[0], 2 * self.N), np.uint64) if glwe else None
        _check(lib().lv_debug_blind_rotate(self._h, _ptr(m, ctypes.c_uint32), _ptr(ids, ctypes.c_uint32),
                                           m.shape[0], _ptr(out, ctypes.c_uint64),
                                           _ptr(g, ctypes.c_uint64) if glwe else None))
        return (out, g) if glwe else out

    def debug_fft(self, poly):
        p = np.ascontiguousarray(poly, np.int64)
        spec = np.zeros(self.N, np.float64)
        rt = np.zeros(self.N, np.uint64)
        _check(lib().lv_debug_fft(self._h, _ptr(p, ctypes.c_int64), _ptr(spec, ctypes.c_double),
                                  _ptr(rt, ctypes.c_uint64)))
        return spec, rt

    def bench_pbs(self, cts, lut_ids, iters: int, flush_bytes: int = 0):
        c, ids = _u32(cts), _u32(lut_ids)
        br = np.zeros(iters, np.float32)
        ks = np.zeros(iters, np.float32)
        st = np.zeros(iters, np.float32)
        _check(lib().lv_bench_pbs(self._h, _ptr(c, ctypes.c_uint32), _ptr(ids, ctypes.c_uint32), c.size,
                                  iters, flush_bytes, _ptr(br, ctypes.c_float), _ptr(ks, ctypes.c_float),
                                  _ptr(st, ctypes.c_float)))
        return br, ks, st


def fp64_peak_tflops() -> float:
    out = ctypes.c_float()
    _check(lib().lv_bench_fp64_peak(ctypes.byref(out)))
    return out.value


from .leuven import (  # noqa: E402  (reference-shaped pipeline API)
    AlphabetSpec, BandSpec, DistanceRun, EqTable, EncryptedString, band_cell_count, build_eq_table,
    compute, compute_batch, distance_batch, distance_encrypted, distance_preprocessed,
    distance_preprocessed_batch,
    encrypt_string, load_eq_table, plan_trace, report_json, run_batch, save_eq_table, wf_distance,
    banded_distance, eq_cost, lut_dump, lut_table,
)

__version__ = "0.1.0"

__all__ = [
    "Context", "Params", "default_params", "negacyclic_eval", "identity_lut", "eq_lut", "AlphabetSpec",
    "BandSpec", "DistanceRun", "EqTable", "EncryptedString", "band_cell_count", "build_eq_table",
    "compute", "compute_batch", "distance_batch", "distance_encrypted", "distance_preprocessed",
    "distance_preprocessed_batch", "encrypt_string", "plan_trace", "wf_distance", "run_batch",
    "report_json", "save_eq_table", "load_eq_table", "banded_distance", "eq_cost", "lut_dump",
    "lut_table", "Error", "OutOfRangeValue", "NoiseBudgetExceeded",
    "ValueOutsideLutHalf", "PackingViolation", "CharNotInAlphabet", "CharNotInSubset",
    "PositionOutOfRange", "BandTooNarrow", "FormatError", "InvalidParams", "CudaError", "InvalidHandle",
]
