"""Reference-shaped pipeline API over the C ABI.

Mirrors proj/include/leuven/encoding.hpp (AlphabetSpec, encrypt_string),
kernel.hpp (BandSpec, DistanceRun, distance_encrypted), preprocess.hpp
(EqTable, build_eq_table, distance_preprocessed) and cli.hpp
(compute_report, whose pybind face is ``compute``, bindings/module.cpp:63-86).
String/alphabet handling is host bookkeeping; every ciphertext operation is
one call into the CUDA library.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import (Band, BandTooNarrow, CharNotInAlphabet, Context, InvalidParams, OutOfRangeValue, Run,
               _check, _ptr, _u32, lib)

# ------------------------------------------------------------ alphabets


class AlphabetSpec:
    """encoding.hpp:18-70; the three builtin layouts of encoding.cpp:78-96."""

    def __init__(self, name: str, widths, mapping):
        self.name = name
        self.widths = list(widths)
        self._code = {}
        for ch, code in mapping:
            self._code[ch] = code
        self._chars = sorted(self._code, key=lambda c: self._code[c])

    @staticmethod
    def ascii7():
        return AlphabetSpec("ascii7", [4, 3], [(chr(c), c) for c in range(128)])

    @staticmethod
    def lower26():
        return AlphabetSpec("lower26", [4, 1], [(chr(ord("a") + i), i) for i in range(26)])

    @staticmethod
    def dna4():
        return AlphabetSpec("dna4", [2], [("A", 0), ("C", 1), ("G", 2), ("T", 3)])

    @staticmethod
    def by_name(name: str) -> "AlphabetSpec":
        table = {"ascii7": AlphabetSpec.ascii7, "lower26": AlphabetSpec.lower26,
                 "dna4": AlphabetSpec.dna4}
        if name not in table:
            raise InvalidParams(f"unknown encoding '{name}'")
        return table[name]()

    def symbol_count(self) -> int:
        return len(self.widths)

    def charset(self):
        return list(self._chars)

    def contains(self, c: str) -> bool:
        return c in self._code

    def code_of(self, c: str) -> int:
        if c not in self._code:
            raise CharNotInAlphabet(f"character not in alphabet '{self.name}'")
        return self._code[c]

    def encode_char(self, c: str):
        """Little-endian symbol split, encoding.cpp:169-178."""
        code = self.code_of(c)
        out = []
        for w in self.widths:
            out.append(code & ((1 << w) - 1))
            code >>= w
        return out


# ------------------------------------------------------------ bands


@dataclass
class BandSpec:
    """kernel.hpp:47-72."""
    mode: int = 0
    half_width: int = 0

    @staticmethod
    def exact(m: int, n: int):
        return BandSpec(0, max(m, n))

    @staticmethod
    def skip(m: int, n: int):
        return BandSpec(1, (max(m, n) + 1) // 2)

    @staticmethod
    def approx(ell: int):
        return BandSpec(2, ell)

    def covers(self, m: int, n: int) -> bool:
        return self.half_width >= abs(m - n)

    def _c(self) -> Band:
        return Band(self.mode, self.half_width)


def band_cell_count(m: int, ell: int) -> int:
    """kernel.cpp:74-77."""
    from . import OutOfRangeValue
    if ell > m:
        raise OutOfRangeValue("band half-width exceeds grid size")
    return m * (2 * ell + 1) - ell * ell - ell


def wf_distance(a: str, b: str) -> int:
    """Plaintext Wagner-Fischer (oracle.cpp:11-28), part of the reference API."""
    prev = list(range(len(b) + 1))
    for i in range(1, len(a) + 1):
        cur = [i] + [0] * len(b)
        for j in range(1, len(b) + 1):
            cur[j] = prev[j - 1] if a[i - 1] == b[j - 1] else 1 + min(prev[j], cur[j - 1], prev[j - 1])
        prev = cur
    return prev[-1]


def banded_distance(a: str, b: str, half_width: int) -> int:
    """Plaintext banded edit distance (oracle.cpp:55-84): cells outside
    |i - j| <= half_width stay unreachable, so the result is an upper bound."""
    m, n = len(a), len(b)
    if half_width < abs(m - n):
        raise BandTooNarrow(f"half width {half_width} below length difference {abs(m - n)}")
    inf = 1 << 30
    prev = list(range(n + 1))
    for i in range(1, m + 1):
        cur = [inf] * (n + 1)
        cur[0] = i
        for j in range(max(1, i - half_width), min(n, i + half_width) + 1):
            diag = prev[j - 1] + (0 if a[i - 1] == b[j - 1] else 1)
            cur[j] = min(diag, prev[j] + 1, cur[j - 1] + 1)
        prev = cur
    return prev[n]


def eq_cost(technique: str, bits: int) -> int:
    """Bootstraps of one character equality (equality.cpp:104-136):
    standard_2bit | ours_4bit | combined."""
    if bits < 1:
        raise OutOfRangeValue("bit width must be positive")

    def merge(k: int) -> int:
        cost = 0
        while k > 1:
            k = (k + 14) // 15
            cost += k
        return cost

    if technique == "standard_2bit":
        k = (bits + 1) // 2
        return k + merge(k)
    if technique == "ours_4bit":
        return 1 if bits <= 4 else 1 + (bits - 4 + 2) // 3
    if technique == "combined":
        k = (bits + 3) // 4
        return k + merge(k)
    raise InvalidParams(f"unknown equality technique '{technique}'")


_TABLES = {"minlut-original": 0, "minlut-negated": 1, "eqlut": 2, "eqlut9": 3}


def lut_table(which: str):
    """The product's own Lut16 entries (lv_lut_table)."""
    if which not in _TABLES:
        raise InvalidParams(f"unknown table '{which}'")
    out = np.zeros(16, np.int32)
    _check(lib().lv_lut_table(_TABLES[which], _ptr(out, ctypes.c_int32)))
    return [int(v) for v in out]


def lut_dump(which: str) -> str:
    """Table dump as `cli table` prints it (lut.cpp:24-30): "i<TAB>entry" lines."""
    return "".join(f"{i}\t{v}\n" for i, v in enumerate(lut_table(which)))


# ------------------------------------------------------------ pipeline


@dataclass
class EncryptedString:
    """encoding.hpp:80-84: chars[i][k] = k-th symbol ciphertext of char i."""
    chars: np.ndarray  # (m, S) uint32 handles

    def length(self) -> int:
        return self.chars.shape[0]


def encrypt_string(s: str, spec: AlphabetSpec, ctx: Context) -> EncryptedString:
    """encoding.cpp:205-217 (one batched encryption for the whole string)."""
    S = spec.symbol_count()
    syms = [v for c in s for v in spec.encode_char(c)]
    if not syms:
        return EncryptedString(np.zeros((0, S), np.uint32))
    return EncryptedString(ctx.encrypt(syms).reshape(len(s), S))


@dataclass
class DistanceRun:
    """kernel.hpp:182-190."""
    score: int
    visited_cells: int = 0
    equality_pbs: int = 0
    kernel_pbs: int = 0
    refreshes: int = 0
    max_key_variance: int = 0
    waves: int = 0


def _key_enc(name: str) -> int:
    if name == "negated":
        return 1
    if name == "original":
        return 0
    raise InvalidParams(f"unknown key encoding '{name}'")


def _run(r: Run, score: int) -> DistanceRun:
    return DistanceRun(int(score), r.visited_cells, r.equality_pbs, r.kernel_pbs, r.refreshes,
                       r.max_key_variance, r.waves)


def distance_encrypted(ctx: Context, a: EncryptedString, b: EncryptedString, band: BandSpec,
                       encoding: str = "negated") -> DistanceRun:
    """kernel::distance_encrypted (kernel.cpp:261-268) on the GPU wavefront."""
    S = a.chars.shape[1] if a.chars.size else b.chars.shape[1] if b.chars.size else 1
    A, B = _u32(a.chars), _u32(b.chars)
    score = ctypes.c_uint32()
    run = Run()
    bc = band._c()
    _check(lib().lv_edit_distance_ee(ctx._h, _ptr(A, ctypes.c_uint32), a.length(),
                                     _ptr(B, ctypes.c_uint32), b.length(), S, ctypes.byref(bc),
                                     _key_enc(encoding), ctypes.byref(score), ctypes.byref(run)))
    return _run(run, score.value)


def distance(ctx: Context, eq9_provider, m: int, n: int, band: BandSpec,
             encoding: str = "negated") -> DistanceRun:
    """kernel::distance with an Eq9Provider (kernel.hpp:162-199):
    eq9_provider(i, j) -> handle of the encrypted 9*[a_i == b_j] for every
    in-band cell (1-based), asked in the reference's visiting order."""
    grid = np.zeros(max(m * n, 1), np.uint32)
    cells, _ = plan_trace(m, n, band, encoding, ctx.params.max_variance_budget)
    for i, j, _, _ in cells:
        grid[(i - 1) * n + (j - 1)] = eq9_provider(i, j)
    score = ctypes.c_uint32()
    run = Run()
    bc = band._c()
    _check(lib().lv_edit_distance_eq9(ctx._h, _ptr(grid, ctypes.c_uint32), m, n, ctypes.byref(bc),
                                      _key_enc(encoding), ctypes.byref(score), ctypes.byref(run)))
    return _run(run, score.value)


def distance_batch(ctx: Context, pairs, bands, encoding: str = "negated"):
    """All pairs' same-index anti-diagonals share one launch."""
    # symbols per character from the arrays' shape (empty strings keep (0, S));
    # every operand must agree, or C would read past the shorter buffers
    shapes = {p[k].chars.shape[1] for p in pairs for k in (0, 1) if p[k].chars.ndim == 2}
    if len(shapes) > 1:
        raise InvalidParams("equality operands must have the same nonzero symbol count")
    S = shapes.pop() if shapes else 2
    A = np.concatenate([_u32(p[0].chars) for p in pairs]) if pairs else np.zeros(0, np.uint32)
    B = np.concatenate([_u32(p[1].chars) for p in pairs]) if pairs else np.zeros(0, np.uint32)
    a_off = np.zeros(len(pairs) + 1, np.uint64)
    b_off = np.zeros(len(pairs) + 1, np.uint64)
    a_off[1:] = np.cumsum([p[0].length() for p in pairs])
    b_off[1:] = np.cumsum([p[1].length() for p in pairs])
    bc = (Band * len(pairs))(*[b._c() for b in bands])
    scores = np.zeros(len(pairs), np.uint32)
    runs = (Run * len(pairs))()
    A = np.ascontiguousarray(A) if A.size else np.zeros(1, np.uint32)
    B = np.ascontiguousarray(B) if B.size else np.zeros(1, np.uint32)
    _check(lib().lv_edit_distance_batch(ctx._h, len(pairs), _ptr(A, ctypes.c_uint32),
                                        _ptr(a_off, ctypes.c_uint64), _ptr(B, ctypes.c_uint32),
                                        _ptr(b_off, ctypes.c_uint64), S, bc, _key_enc(encoding),
                                        _ptr(scores, ctypes.c_uint32), runs))
    return [_run(runs[p], scores[p]) for p in range(len(pairs))]


class EqTable:
    """preprocess.hpp:18-39 (rows live on the device; lookups are handles)."""

    def __init__(self, ctx: Context, handle, spec: AlphabetSpec, length: int, subset):
        self._ctx = ctx
        self._h = handle
        self.spec = spec
        self.length = length
        self._subset = sorted(subset)

    def string_length(self) -> int:
        return self.length

    def subset(self):
        return list(self._subset)

    def has_row(self, c: str) -> bool:
        return c in self._subset

    def lookup(self, c: str, position: int) -> int:
        out = ctypes.c_uint32()
        _check(lib().lv_eq_table_lookup(self._ctx._h, self._h, c.encode("latin1"), position,
                                        ctypes.byref(out)))
        return out.value

    def __del__(self):
        try:
            if self._h and self._ctx._h:
                lib().lv_eq_table_destroy(self._ctx._h, self._h)
        except Exception:
            pass
        self._h = None


def build_eq_table(ctx: Context, xs: EncryptedString, spec: AlphabetSpec, subset: str = ""):
    """preprocess.cpp:38-60; returns (table, bootstraps spent)."""
    chars = list(subset) if subset else spec.charset()
    S = spec.symbol_count()
    syms = np.asarray([spec.encode_char(c) for c in chars], np.int32).reshape(-1)
    A = _u32(xs.chars) if xs.chars.size else np.zeros(1, np.uint32)
    h = ctypes.c_void_p()
    pbs = ctypes.c_uint64()
    _check(lib().lv_eq_table_build(ctx._h, _ptr(A, ctypes.c_uint32), xs.length(), S,
                                   "".join(chars).encode("latin1"), _ptr(syms, ctypes.c_int32),
                                   len(chars), ctypes.byref(h), ctypes.byref(pbs)))
    return EqTable(ctx, h, spec, xs.length(), chars), pbs.value


def distance_preprocessed(ctx: Context, table: EqTable, plain: str, band: BandSpec,
                          encoding: str = "negated") -> DistanceRun:
    """preprocess.cpp:62-76."""
    score = ctypes.c_uint32()
    run = Run()
    bc = band._c()
    _check(lib().lv_edit_distance_pre(ctx._h, table._h, plain.encode("latin1"), len(plain),
                                      ctypes.byref(bc), _key_enc(encoding), ctypes.byref(score),
                                      ctypes.byref(run)))
    return _run(run, score.value)


def distance_preprocessed_batch(ctx: Context, tables, plains, bands,
                                encoding: str = "negated"):
    """Many plaintext strings against equality tables in one wavefront
    (lv_edit_distance_pre_batch): the database-scan use of one preprocessed
    encrypted query. ``tables`` is one EqTable or one
    per string; ``bands`` one BandSpec or one per string."""
    n = len(plains)
    tabs = list(tables) if isinstance(tables, (list, tuple)) else [tables] * n
    bnds = list(bands) if isinstance(bands, (list, tuple)) else [bands] * n
    if len(tabs) != n or len(bnds) != n:
        raise InvalidParams("one table and one band per plaintext string")
    data = "".join(plains).encode("latin1")
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in plains])
    th = (ctypes.c_void_p * max(1, n))(*[t._h for t in tabs])
    bc = (Band * max(1, n))(*[b._c() for b in bnds])
    scores = np.zeros(max(1, n), np.uint32)
    runs = (Run * max(1, n))()
    _check(lib().lv_edit_distance_pre_batch(ctx._h, n, th, data, _ptr(off, ctypes.c_uint64), bc,
                                            _key_enc(encoding), _ptr(scores, ctypes.c_uint32),
                                            runs))
    return [_run(runs[p], scores[p]) for p in range(n)]


def plan_trace(m: int, n: int, band: BandSpec, key_encoding: str = "negated",
               budget: float = 4000.0):
    """Per-cell (i, j, key variance, refreshes) of the symbolic schedule."""
    cap = (m + 1) * (n + 1)
    ij = np.zeros(2 * cap, np.uint32)
    kv = np.zeros(cap, np.int64)
    rf = np.zeros(cap, np.uint32)
    cnt = ctypes.c_uint64()
    tot = Run()
    bc = band._c()
    _check(lib().lv_plan_trace(m, n, ctypes.byref(bc), _key_enc(key_encoding), budget, cap,
                               _ptr(ij, ctypes.c_uint32), _ptr(kv, ctypes.c_int64),
                               _ptr(rf, ctypes.c_uint32), ctypes.byref(cnt), ctypes.byref(tot)))
    k = cnt.value
    cells = [[int(ij[2 * t]), int(ij[2 * t + 1]), int(kv[t]), int(rf[t])] for t in range(k)]
    return cells, _run(tot, 0)


def _resolve_band(mode: str, ell, m: int, n: int) -> BandSpec:
    """cli.cpp:35-43."""
    if mode == "exact":
        return BandSpec.exact(m, n)
    if mode == "skip":
        return BandSpec.skip(m, n)
    if mode == "approx":
        if ell is None:
            raise InvalidParams("--mode approx requires --ell")
        return BandSpec.approx(ell)
    raise InvalidParams(f"unknown mode '{mode}'")


_CTX_CACHE: dict = {}


def _context(seed: int | None, budget: float) -> Context:
    key = (seed, float(budget))
    if key not in _CTX_CACHE:
        _CTX_CACHE[key] = Context(seed=seed, budget=budget)
    return _CTX_CACHE[key]


def compute(a: str, b: str, mode: str = "exact", ell=None, encoding: str = "ascii7",
            budget: float = 4000.0, key_encoding: str = "negated", preprocess: bool = False,
            ctx: Context | None = None, seed: int | None = None, include_timing: bool = False) -> dict:
    """cli::compute_report (cli.cpp:53-91) / bindings compute(): encrypt ->
    traverse on the GPU -> decrypt; counters as in RunReport (cli.hpp:25-37)."""
    import time
    spec = AlphabetSpec.by_name(encoding)
    band = _resolve_band(mode, ell, len(a), len(b))
    if budget < 1.0:
        raise InvalidParams("noise budget must be at least 1")
    ctx = ctx if ctx is not None else _context(seed, budget)
    before = ctx.stats()
    t0 = time.perf_counter()
    pre_pbs = 0
    temps = []
    xs = encrypt_string(a, spec, ctx)
    temps.append(xs.chars)
    table = None
    if preprocess:
        table, pre_pbs = build_eq_table(ctx, xs, spec)
        for c in b:
            if not table.has_row(c):
                from . import CharNotInSubset
                raise CharNotInSubset(f"no table row for character '{c}'")
        run = distance_preprocessed(ctx, table, b, band, key_encoding)
    else:
        ys = encrypt_string(b, spec, ctx)
        temps.append(ys.chars)
        run = distance_encrypted(ctx, xs, ys, band, key_encoding)
    t1 = time.perf_counter()
    dist = int(ctx.decrypt([run.score])[0])
    after = ctx.stats()
    ctx.release([run.score])
    for t in temps:
        if t.size:
            ctx.release(t)
    del table
    return {
        "distance": dist, "mode": mode, "half_width": band.half_width,
        "visited_cells": run.visited_cells, "pbs_total": after["pbs_count"] - before["pbs_count"],
        "pbs_equality": run.equality_pbs, "pbs_kernel": run.kernel_pbs,
        "refresh_count": run.refreshes, "preprocessing_pbs": pre_pbs,
        "max_key_variance": run.max_key_variance,
        "linear_ops": after["linear_op_count"] - before["linear_op_count"],
        "waves": run.waves,
    } | ({"wall_time_ms": (t1 - t0) * 1e3} if include_timing else {})


def _traverse_batch(ctx: Context, pairs, spec: AlphabetSpec, bands, key_encoding: str):
    """The GPU part of compute_batch: encrypt every string, one wavefront over
    all pairs, decrypt the scores. Returns [(distance, DistanceRun)]."""
    enc = []
    for a, b in pairs:
        enc.append((encrypt_string(a, spec, ctx), encrypt_string(b, spec, ctx)))
    runs = distance_batch(ctx, enc, bands, key_encoding)
    dists = ctx.decrypt([r.score for r in runs]) if runs else []
    ctx.release([r.score for r in runs])
    for x, y in enc:
        for t in (x.chars, y.chars):
            if t.size:
                ctx.release(t)
    return [(int(d), r) for d, r in zip(dists, runs)]


def compute_batch(pairs, encoding: str = "ascii7", budget: float = 4000.0,
                  key_encoding: str = "negated", ctx: Context | None = None, seed: int | None = None,
                  _traverse=None):
    """Batch mode (cli.cpp:164-210): exact band, one report per pair, all
    pairs traversed together on the GPU. (_traverse: the GPU part, replaced
    only by the CPU multi-process test.)"""
    spec = AlphabetSpec.by_name(encoding)
    bands = [BandSpec.exact(len(a), len(b)) for a, b in pairs]
    if _traverse is None:
        ctx = ctx if ctx is not None else _context(seed, budget)
        _traverse = _traverse_batch
    out = []
    for (d, r), band in zip(_traverse(ctx, pairs, spec, bands, key_encoding), bands):
        out.append({"distance": d, "mode": "exact", "half_width": band.half_width,
                    "visited_cells": r.visited_cells, "pbs_equality": r.equality_pbs,
                    "pbs_kernel": r.kernel_pbs,
                    "pbs_total": r.equality_pbs + r.kernel_pbs + r.refreshes,
                    "refresh_count": r.refreshes, "preprocessing_pbs": 0,
                    "max_key_variance": r.max_key_variance})
    return out


# ------------------------------------------------------------ RunReport / batch
REPORT_FIELDS = ["distance", "mode", "half_width", "visited_cells", "pbs_total", "pbs_equality",
                 "pbs_kernel", "refresh_count", "preprocessing_pbs", "max_key_variance"]


def report_json(report: dict, include_timing: bool = False) -> str:
    """cli::report_json (cli.cpp:93-107): compact, field order fixed, timing
    excluded from batch lines so equal inputs serialise to equal bytes."""
    import json
    obj = {k: report[k] for k in REPORT_FIELDS}
    if include_timing:
        obj["wall_time_ms"] = report["wall_time_ms"]
    return json.dumps(obj, separators=(",", ":"))


def run_batch(lines, mode: str = "exact", ell=None, encoding: str = "ascii7",
              budget: float = 4000.0, key_encoding: str = "negated", preprocess: bool = False,
              ctx: Context | None = None, seed: int | None = None):
    """cli::run_batch (cli.cpp:164-210): one JSON object {"a":..,"b":..} per
    line -> one report line (or {"error": ...}) per line, input order kept.
    All valid lines of a non-preprocessed batch are traversed together: every
    pair's same-index anti-diagonal shares one GPU launch."""
    import json
    from . import Error
    ctx = ctx if ctx is not None else _context(seed, budget)
    spec = AlphabetSpec.by_name(encoding)
    out = [None] * len(lines)
    todo = []
    for idx, text in enumerate(lines):
        try:
            j = json.loads(text)
        except Exception as e:
            out[idx] = json.dumps({"error": f"bad JSON: {e}"}, separators=(",", ":"))
            continue
        if not (isinstance(j, dict) and isinstance(j.get("a"), str) and isinstance(j.get("b"), str)):
            out[idx] = json.dumps({"error": 'each line needs string fields "a" and "b"'},
                                  separators=(",", ":"))
            continue
        a, b = j["a"], j["b"]
        try:
            band = _resolve_band(mode, ell, len(a), len(b))
            for s in (a, b):
                for ch in s:
                    spec.code_of(ch)
            if not band.covers(len(a), len(b)):
                raise BandTooNarrow(f"band half-width {band.half_width} below length difference")
            if budget < 11.0:
                raise InvalidParams("noise budget below 11: refreshed operands alone exceed it")
        except Error as e:
            out[idx] = json.dumps({"error": str(e)}, separators=(",", ":"))
            continue
        todo.append((idx, a, b, band))
    if preprocess:
        for idx, a, b, _ in todo:
            try:
                rep = compute(a, b, mode, ell, encoding, budget, key_encoding, True, ctx=ctx)
                out[idx] = report_json(rep)
            except Error as e:
                out[idx] = json.dumps({"error": str(e)}, separators=(",", ":"))
        return out
    if todo:
        enc = [(encrypt_string(a, spec, ctx), encrypt_string(b, spec, ctx)) for _, a, b, _ in todo]
        runs = distance_batch(ctx, enc, [band for *_, band in todo], key_encoding)
        dists = ctx.decrypt([r.score for r in runs])
        for (idx, a, b, band), r, d in zip(todo, runs, dists):
            rep = {"distance": int(d), "mode": mode, "half_width": band.half_width,
                   "visited_cells": r.visited_cells,
                   "pbs_total": r.equality_pbs + r.kernel_pbs + r.refreshes,
                   "pbs_equality": r.equality_pbs, "pbs_kernel": r.kernel_pbs,
                   "refresh_count": r.refreshes, "preprocessing_pbs": 0,
                   "max_key_variance": r.max_key_variance}
            out[idx] = report_json(rep)
        ctx.release([r.score for r in runs])
        for x, y in enc:
            for t in (x.chars, y.chars):
                if t.size:
                    ctx.release(t)
    return out


# ------------------------------------------------------------ LEQT v2 container
def _alphabet_meta(spec: AlphabetSpec) -> bytes:
    """The v1 alphabet section (preprocess.cpp:144-152): name, widths, chars."""
    import struct
    name = spec.name.encode()
    b = struct.pack("<I", len(name)) + name + struct.pack("<I", len(spec.widths))
    b += b"".join(struct.pack("<i", w) for w in spec.widths)
    chars = spec.charset()
    b += struct.pack("<I", len(chars))
    b += b"".join(bytes([ord(c)]) + struct.pack("<i", spec.code_of(c)) for c in chars)
    return b


def _parse_meta(meta: bytes) -> AlphabetSpec:
    import struct
    from . import FormatError
    try:
        p = 0
        (ln,) = struct.unpack_from("<I", meta, p); p += 4
        name = meta[p:p + ln].decode(); p += ln
        (nw,) = struct.unpack_from("<I", meta, p); p += 4
        widths = list(struct.unpack_from(f"<{nw}i", meta, p)); p += 4 * nw
        (nc,) = struct.unpack_from("<I", meta, p); p += 4
        mapping = []
        for _ in range(nc):
            ch = chr(meta[p]); (code,) = struct.unpack_from("<i", meta, p + 1); p += 5
            mapping.append((ch, code))
    except Exception as e:
        raise FormatError(f"truncated alphabet section: {e}")
    return AlphabetSpec(name, widths, mapping)


def save_eq_table(table: EqTable, f) -> int:
    """preprocess::save_eq_table (preprocess.cpp:140-164), v2 with real
    ciphertexts; f is a path or a binary file object. Returns bytes written."""
    meta = _alphabet_meta(table.spec)
    need = ctypes.c_uint64()
    _check(lib().lv_eq_table_serialize(table._ctx._h, table._h, meta, len(meta), None, 0,
                                       ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().lv_eq_table_serialize(table._ctx._h, table._h, meta, len(meta), buf, need.value,
                                       ctypes.byref(need)))
    data = buf.raw[:need.value]
    if isinstance(f, (str, bytes)) or hasattr(f, "__fspath__"):
        with open(f, "wb") as fh:
            fh.write(data)
    else:
        f.write(data)
    return len(data)


def load_eq_table(ctx: Context, f) -> EqTable:
    """preprocess::load_eq_table (preprocess.cpp:166-194) for v2 files."""
    if isinstance(f, (str, bytes)) or hasattr(f, "__fspath__"):
        with open(f, "rb") as fh:
            data = fh.read()
    else:
        data = f.read()
    h = ctypes.c_void_p()
    ml = ctypes.c_uint64()
    meta = ctypes.create_string_buffer(max(1, len(data)))
    _check(lib().lv_eq_table_deserialize(ctx._h, data, len(data), ctypes.byref(h), meta, len(data),
                                         ctypes.byref(ml)))
    spec = _parse_meta(meta.raw[:ml.value])
    import struct
    p = 12 + ml.value + 20  # header, alphabet, n/N/k/seed (already validated)
    length, nrows = struct.unpack_from("<QI", data, p)
    p += 12
    subset = []
    for _ in range(nrows):  # row characters, skipping the ciphertext payloads
        subset.append(chr(data[p]))
        p += 1
        for _ in range(length):
            (terms,) = struct.unpack_from("<I", data, p)
            p += 4 + 4 * terms + 8 * (ctx.N + 1)
    return EqTable(ctx, h, spec, length, subset)
