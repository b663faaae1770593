"""TEST INFRASTRUCTURE ONLY — ctypes view of the CPU oracle (tfhe_oracle.c).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs. The product (paper_2508_14568_b200) never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
# the same source built -O3 for x86-64-v3 (AVX2 + hardware FMA): the CPU
# baseline's fast build; bit-identical outputs (explicit fma(), no contraction)
FAST_LIB_PATH = os.path.join(HERE, "_build", "liboracle_fast.so")


class Params(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint32),
        ("N", ctypes.c_uint32),
        ("k", ctypes.c_uint32),
        ("pbs_base_log", ctypes.c_uint32),
        ("pbs_level", ctypes.c_uint32),
        ("ks_base_log", ctypes.c_uint32),
        ("ks_level", ctypes.c_uint32),
        ("lwe_noise_log2", ctypes.c_uint32),
        ("glwe_noise_log2", ctypes.c_uint32),
        ("exact_mask_product", ctypes.c_uint32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def build():
    """Compile liboracle.so (gcc); cheap when up to date."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_libs = {}


def lib(fast: bool = False):
    if fast not in _libs:
        path = FAST_LIB_PATH if fast else LIB_PATH
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        vp = ctypes.c_void_p
        L.orc_default_params.restype = Params
        L.orc_create.restype = vp
        L.orc_create.argtypes = [ctypes.POINTER(Params), ctypes.c_uint64, ctypes.c_int]
        L.orc_destroy.argtypes = [vp]
        L.orc_rand_u64.restype = ctypes.c_uint64
        L.orc_rand_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.orc_philox.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, u32p]
        L.orc_tuniform.restype = ctypes.c_int64
        L.orc_tuniform.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32]
        for name, rt in (("orc_sk_small", ctypes.POINTER(ctypes.c_uint8)),
                         ("orc_sk_glwe", ctypes.POINTER(ctypes.c_uint8)),
                         ("orc_ksk", u64p), ("orc_bsk", u64p),
                         ("orc_bskf", ctypes.POINTER(ctypes.c_double)),
                         ("orc_bskf_hi", ctypes.POINTER(ctypes.c_double)),
                         ("orc_bskf_lo", ctypes.POINTER(ctypes.c_double))):
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [vp]
        L.orc_encrypt_at.argtypes = [vp, ctypes.c_int32, ctypes.c_uint64, u64p]
        L.orc_trivial.argtypes = [vp, ctypes.c_int32, u64p]
        L.orc_phase.restype = ctypes.c_uint64
        L.orc_phase.argtypes = [vp, u64p]
        L.orc_phase_small.restype = ctypes.c_uint64
        L.orc_phase_small.argtypes = [vp, u64p]
        L.orc_decrypt.restype = ctypes.c_int32
        L.orc_decrypt.argtypes = [vp, u64p]
        L.orc_keyswitch.argtypes = [vp, u64p, u64p]
        L.orc_modswitch.argtypes = [vp, u64p, u32p]
        L.orc_test_poly.argtypes = [vp, i32p, u64p]
        L.orc_blind_rotate.argtypes = [vp, u32p, u64p, u64p, ctypes.c_int]
        L.orc_sample_extract.argtypes = [vp, u64p, u64p]
        L.orc_blind_rotate_batch.argtypes = [vp, ctypes.c_size_t, u32p, u64p, u64p, ctypes.c_int,
                                             ctypes.c_int]
        L.orc_pbs.argtypes = [vp, u64p, i32p, u64p, ctypes.c_int]
        L.orc_fft_phase_error_var.restype = ctypes.c_double
        L.orc_fft_phase_error_var.argtypes = [vp, u32p, u64p]
        L.orc_pbs_batch.argtypes = [vp, ctypes.c_size_t, u64p, i32p, u64p, ctypes.c_int, ctypes.c_int]
        L.orc_pbs_batch_simd.restype = ctypes.c_int
        L.orc_pbs_batch_simd.argtypes = [vp, ctypes.c_size_t, u64p, i32p, u64p, ctypes.c_int]
        L.orc_fft_forward_i64.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)]
        L.orc_fft_backward_torus.argtypes = [vp, ctypes.POINTER(ctypes.c_double), u64p]
        _libs[fast] = L
    return _libs[fast]


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def default_params() -> Params:
    return lib().orc_default_params()


def toy_params() -> Params:
    """Small insecure set for fast exact-mode checks (same code paths)."""
    p = default_params()
    p.n, p.N = 64, 512
    p.lwe_noise_log2, p.glwe_noise_log2 = 30, 17
    return p


class Oracle:
    """One keyset: all keys derived from `seed` (Philox domains)."""

    def __init__(self, seed: int = 0, params: Params | None = None, threads: int = 0,
                 fast: bool = False):
        self.params = params if params is not None else default_params()
        self.seed = seed
        self._L = lib(fast)
        self._c = self._L.orc_create(ctypes.byref(self.params), seed, threads)
        p = self.params
        self.n, self.N, self.k = p.n, p.N, p.k
        self.big = p.k * p.N + 1
        self.rows = (p.k + 1) * p.pbs_level

    def __del__(self):
        if getattr(self, "_c", None):
            self._L.orc_destroy(self._c)
            self._c = None

    # keys -----------------------------------------------------------
    def sk_small(self):
        return np.ctypeslib.as_array(self._L.orc_sk_small(self._c), (self.n,)).copy()

    def sk_glwe(self):
        return np.ctypeslib.as_array(self._L.orc_sk_glwe(self._c), (self.k * self.N,)).copy()

    def ksk(self):
        p = self.params
        return np.ctypeslib.as_array(self._L.orc_ksk(self._c), (p.k * p.N * p.ks_level * (p.n + 1),)).copy()

    def bsk(self):
        return np.ctypeslib.as_array(self._L.orc_bsk(self._c), (self.n * self.rows * (self.k + 1) * self.N,)).copy()

    def bskf(self):
        return np.ctypeslib.as_array(self._L.orc_bskf(self._c), (self.n * self.rows * (self.k + 1) * self.N,)).copy()

    def bskf_split(self):
        """(H, Lo) spectra of the mask polynomials (exact_mask_product keys)."""
        size = (self.n * self.rows * self.k * self.N,)
        return (np.ctypeslib.as_array(self._L.orc_bskf_hi(self._c), size).copy(),
                np.ctypeslib.as_array(self._L.orc_bskf_lo(self._c), size).copy())

    # ciphertexts ----------------------------------------------------
    def encrypt(self, value: int, counter: int) -> np.ndarray:
        out = np.zeros(self.big, np.uint64)
        self._L.orc_encrypt_at(self._c, int(value), int(counter), _p(out, ctypes.c_uint64))
        return out

    def trivial(self, value: int) -> np.ndarray:
        out = np.zeros(self.big, np.uint64)
        self._L.orc_trivial(self._c, int(value), _p(out, ctypes.c_uint64))
        return out

    def phase(self, ct: np.ndarray) -> int:
        ct = np.ascontiguousarray(ct, np.uint64)
        return int(self._L.orc_phase(self._c, _p(ct, ctypes.c_uint64)))

    def decrypt(self, ct: np.ndarray) -> int:
        ct = np.ascontiguousarray(ct, np.uint64)
        return int(self._L.orc_decrypt(self._c, _p(ct, ctypes.c_uint64)))

    def keyswitch(self, ct: np.ndarray) -> np.ndarray:
        ct = np.ascontiguousarray(ct, np.uint64)
        out = np.zeros(self.n + 1, np.uint64)
        self._L.orc_keyswitch(self._c, _p(ct, ctypes.c_uint64), _p(out, ctypes.c_uint64))
        return out

    def modswitch(self, small: np.ndarray) -> np.ndarray:
        small = np.ascontiguousarray(small, np.uint64)
        out = np.zeros(self.n + 1, np.uint32)
        self._L.orc_modswitch(self._c, _p(small, ctypes.c_uint64), _p(out, ctypes.c_uint32))
        return out

    def phase_small(self, small: np.ndarray) -> int:
        small = np.ascontiguousarray(small, np.uint64)
        return int(self._L.orc_phase_small(self._c, _p(small, ctypes.c_uint64)))

    def test_poly(self, lut) -> np.ndarray:
        lut = np.ascontiguousarray(lut, np.int32)
        out = np.zeros(self.N, np.uint64)
        self._L.orc_test_poly(self._c, _p(lut, ctypes.c_int32), _p(out, ctypes.c_uint64))
        return out

    def blind_rotate(self, ms: np.ndarray, tp: np.ndarray, mode: int = 0) -> np.ndarray:
        ms = np.ascontiguousarray(ms, np.uint32)
        tp = np.ascontiguousarray(tp, np.uint64)
        out = np.zeros((self.k + 1) * self.N, np.uint64)
        self._L.orc_blind_rotate(self._c, _p(ms, ctypes.c_uint32), _p(tp, ctypes.c_uint64),
                               _p(out, ctypes.c_uint64), mode)
        return out

    def blind_rotate_batch(self, ms: np.ndarray, tp: np.ndarray, mode: int = 0, threads: int = 0):
        ms = np.ascontiguousarray(ms, np.uint32).reshape(-1, self.n + 1)
        tp = np.ascontiguousarray(tp, np.uint64)
        out = np.zeros((ms.shape[0], (self.k + 1) * self.N), np.uint64)
        self._L.orc_blind_rotate_batch(self._c, ms.shape[0], _p(ms, ctypes.c_uint32),
                                     _p(tp, ctypes.c_uint64), _p(out, ctypes.c_uint64), mode, threads)
        return out

    def fft_phase_error_var(self, ms: np.ndarray, tp: np.ndarray) -> float:
        """Phase variance the f64 FFT adds over one blind rotation (exact
        products computed alongside on the same inputs)."""
        ms = np.ascontiguousarray(ms, np.uint32)
        tp = np.ascontiguousarray(tp, np.uint64)
        return self._L.orc_fft_phase_error_var(self._c, _p(ms, ctypes.c_uint32), _p(tp, ctypes.c_uint64))

    def sample_extract(self, glwe: np.ndarray) -> np.ndarray:
        glwe = np.ascontiguousarray(glwe, np.uint64)
        out = np.zeros(self.big, np.uint64)
        self._L.orc_sample_extract(self._c, _p(glwe, ctypes.c_uint64), _p(out, ctypes.c_uint64))
        return out

    def pbs(self, ct: np.ndarray, lut, mode: int = 0) -> np.ndarray:
        ct = np.ascontiguousarray(ct, np.uint64)
        lut = np.ascontiguousarray(lut, np.int32)
        out = np.zeros(self.big, np.uint64)
        self._L.orc_pbs(self._c, _p(ct, ctypes.c_uint64), _p(lut, ctypes.c_int32),
                      _p(out, ctypes.c_uint64), mode)
        return out

    def pbs_batch(self, cts: np.ndarray, luts: np.ndarray, mode: int = 0, threads: int = 0):
        cts = np.ascontiguousarray(cts, np.uint64).reshape(-1, self.big)
        luts = np.ascontiguousarray(luts, np.int32).reshape(-1, 16)
        assert cts.shape[0] == luts.shape[0]
        out = np.zeros_like(cts)
        self._L.orc_pbs_batch(self._c, cts.shape[0], _p(cts, ctypes.c_uint64),
                            _p(luts, ctypes.c_int32), _p(out, ctypes.c_uint64), mode, threads)
        return out

    def pbs_batch_simd(self, cts: np.ndarray, luts: np.ndarray, threads: int = 0):
        """The CPU baseline's lane-vectorised PBS (8 ciphertexts per AVX-512
        lane set; only in the fast build): bit-identical to pbs_batch.
        None when unavailable (scalar build, or parameters it does not cover)."""
        cts = np.ascontiguousarray(cts, np.uint64).reshape(-1, self.big)
        luts = np.ascontiguousarray(luts, np.int32).reshape(-1, 16)
        assert cts.shape[0] == luts.shape[0]
        out = np.zeros_like(cts)
        rc = self._L.orc_pbs_batch_simd(self._c, cts.shape[0], _p(cts, ctypes.c_uint64),
                                        _p(luts, ctypes.c_int32), _p(out, ctypes.c_uint64), threads)
        return out if rc == 0 else None

    def fft_forward(self, poly: np.ndarray) -> np.ndarray:
        poly = np.ascontiguousarray(poly, np.int64)
        out = np.zeros(self.N, np.float64)
        self._L.orc_fft_forward_i64(self._c, _p(poly, ctypes.c_int64), _p(out, ctypes.c_double))
        return out

    def fft_backward(self, spec: np.ndarray) -> np.ndarray:
        spec = np.ascontiguousarray(spec, np.float64)
        out = np.zeros(self.N, np.uint64)
        self._L.orc_fft_backward_torus(self._c, _p(spec, ctypes.c_double), _p(out, ctypes.c_uint64))
        return out


def negacyclic_eval(lut, x: int) -> int:
    """proj/src/lut.cpp:9-16."""
    if not 0 <= x < 32:
        raise ValueError("lookup input outside [0,32)")
    if x < 16:
        return int(lut[x])
    return (32 - int(lut[x - 16])) % 32


def identity_lut():
    """proj/src/lut.cpp:18-22."""
    return list(range(16))
