"""CPU oracle for arXiv 2309.03308's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2309_03308_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``corr_oracle.c`` (plain C, fp64 reductions, fp32
KSG distances, brute force; see that file's header for the paper passages each
function follows).  ``build()`` compiles it with gcc; ``build()`` is also called
by ``__graft_entry__.build()`` (building the checker is not using it).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "corr_oracle.c")
_LIB = os.path.join(_HERE, "libcorr_oracle.so")
_lib = None

F32P = ctypes.POINTER(ctypes.c_float)
F64P = ctypes.POINTER(ctypes.c_double)
I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)


class Box(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("x0", "y0", "z0", "x1", "y1", "z1")]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_ppmcc.restype = ctypes.c_double
        L.oracle_ppmcc.argtypes = [F32P, F32P, ctypes.c_int]
        L.oracle_digamma_int.restype = ctypes.c_double
        L.oracle_digamma_int.argtypes = [ctypes.c_int]
        L.oracle_knn.restype = None
        L.oracle_knn.argtypes = [F32P, F32P, ctypes.c_int, ctypes.c_int, F32P, I32P, I32P]
        L.oracle_ksg.restype = ctypes.c_double
        L.oracle_ksg.argtypes = [F32P, F32P, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_eval_pairs.restype = None
        L.oracle_eval_pairs.argtypes = [F32P, F32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, I64P, I64P, ctypes.c_int64, F64P]
        L.oracle_knn_pairs.restype = None
        L.oracle_knn_pairs.argtypes = [F32P, F32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       I64P, I64P, ctypes.c_int64, F32P, I32P, I32P]
        L.oracle_mix64.restype = ctypes.c_uint64
        L.oracle_mix64.argtypes = [ctypes.c_uint64]
        L.oracle_pair_key.restype = ctypes.c_uint64
        L.oracle_pair_key.argtypes = [ctypes.c_uint64, ctypes.POINTER(Box), ctypes.POINTER(Box)]
        L.oracle_sample.restype = None
        L.oracle_sample.argtypes = [ctypes.c_uint64, ctypes.POINTER(Box), ctypes.POINTER(Box),
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_int, I64P, I64P]
        L.oracle_region_max.restype = None
        L.oracle_region_max.argtypes = [F32P, F32P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(Box), ctypes.POINTER(Box), ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_uint64, F64P, I64P]
        L.oracle_region_values.restype = None
        L.oracle_region_values.argtypes = [F32P, F32P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(Box), ctypes.POINTER(Box), ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_uint64, F64P, I64P, I64P]
        L.oracle_sample_many.restype = None
        L.oracle_sample_many.argtypes = [ctypes.c_uint64, ctypes.POINTER(Box), ctypes.POINTER(Box),
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_int, I64P, I64P]
        L.oracle_set_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    """OpenMP threads for the oracle's pair loops (n <= 0: query only); returns the count used."""
    return int(lib().oracle_set_threads(int(n)))


# measure codes (same values as include/corr.h, restated: the oracle shares no header)
PEARSON = 0
KSG = 1
F_KSG_PLUS1 = 1 << 8
F_ABS = 1 << 9


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def ppmcc(x, y) -> float:
    x, y = _f32(x), _f32(y)
    assert x.shape == y.shape
    return lib().oracle_ppmcc(_p(x, F32P), _p(y, F32P), x.size)


def digamma_int(m: int) -> float:
    return lib().oracle_digamma_int(int(m))


def knn(x, y, k: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    x, y = _f32(x), _f32(y)
    n = x.size
    eps = np.empty(n, np.float32)
    nx = np.empty(n, np.int32)
    ny = np.empty(n, np.int32)
    lib().oracle_knn(_p(x, F32P), _p(y, F32P), n, int(k), _p(eps, F32P), _p(nx, I32P), _p(ny, I32P))
    return eps, nx, ny


def ksg(x, y, k: int, plus1: bool = False) -> float:
    x, y = _f32(x), _f32(y)
    return lib().oracle_ksg(_p(x, F32P), _p(y, F32P), x.size, int(k), int(bool(plus1)))


def _field(values) -> np.ndarray:
    """[members, P] float32 contiguous."""
    return _f32(values.cpu().numpy() if hasattr(values, "cpu") else values)


def eval_pairs(fa, fb, measure: int, k: int, idxA, idxB) -> np.ndarray:
    fa = _field(fa)
    fbn = None if fb is None else _field(fb)
    n, P = fa.shape
    a = np.ascontiguousarray(np.asarray(idxA, np.int64))
    b = np.ascontiguousarray(np.asarray(idxB, np.int64))
    out = np.empty(a.size, np.float64)
    lib().oracle_eval_pairs(_p(fa, F32P), None if fbn is None else _p(fbn, F32P), P, n, measure,
                            int(k), _p(a, I64P), _p(b, I64P), a.size, _p(out, F64P))
    return out


def knn_pairs(fa, fb, k: int, idxA, idxB):
    fa = _field(fa)
    fbn = None if fb is None else _field(fb)
    n, P = fa.shape
    a = np.ascontiguousarray(np.asarray(idxA, np.int64))
    b = np.ascontiguousarray(np.asarray(idxB, np.int64))
    eps = np.empty((a.size, n), np.float32)
    nx = np.empty((a.size, n), np.int32)
    ny = np.empty((a.size, n), np.int32)
    lib().oracle_knn_pairs(_p(fa, F32P), None if fbn is None else _p(fbn, F32P), P, n, int(k),
                           _p(a, I64P), _p(b, I64P), a.size, _p(eps, F32P), _p(nx, I32P),
                           _p(ny, I32P))
    return eps, nx, ny


def mix64(z: int) -> int:
    return int(lib().oracle_mix64(ctypes.c_uint64(z & 0xFFFFFFFFFFFFFFFF)))


def _box(b: Sequence[int]) -> Box:
    return Box(*[int(v) for v in b])


def pair_key(seed: int, A, B) -> int:
    a, b = _box(A), _box(B)
    return int(lib().oracle_pair_key(ctypes.c_uint64(seed), ctypes.byref(a), ctypes.byref(b)))


def sample(seed: int, A, B, s: int, nx: int, ny: int) -> Tuple[int, int]:
    a, b = _box(A), _box(B)
    pa, pb = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_sample(ctypes.c_uint64(seed), ctypes.byref(a), ctypes.byref(b), int(s), nx, ny,
                        ctypes.byref(pa), ctypes.byref(pb))
    return pa.value, pb.value


def aggregate_mean(values, dims, fx: int, fy: int, fz: int) -> np.ndarray:
    """Mean-tree level (§3.3): per member, the mean of the series over each
    fx x fy x fz block of grid points (boundary blocks average the points that exist),
    summed in fp64 and rounded to fp32.  values: [n, P] in file order; returns [n, P']."""
    nx, ny, nz = dims
    v = _field(values).reshape(-1, nz, ny, nx).astype(np.float64)
    cx, cy, cz = -(-nx // fx), -(-ny // fy), -(-nz // fz)
    out = np.empty((v.shape[0], cz, cy, cx), np.float64)
    for Z in range(cz):
        for Y in range(cy):
            for X in range(cx):
                blk = v[:, Z * fz:(Z + 1) * fz, Y * fy:(Y + 1) * fy, X * fx:(X + 1) * fx]
                out[:, Z, Y, X] = blk.reshape(blk.shape[0], -1).sum(axis=1) / blk[0].size
    return out.reshape(v.shape[0], -1).astype(np.float32)


def _box_points(box, nx, ny):
    x0, y0, z0, x1, y1, z1 = box
    z, y, x = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    return ((z * ny + y) * nx + x).reshape(-1).astype(np.int64)  # local index, x fastest


def pearson_block_max(fa, fb, dims, A, B, absval: bool = False, chunk: int = 2048, runner_up: bool = False):
    """Exhaustive Pearson maximum of one region pair -- the PPMCC definition
    (two-pass fp64 means and deviations) for EVERY pair of the two bricks, with
    the |A| x |B| sums of products formed by a library fp64 matmul (a permitted primitive).
    Values rounded to fp32 as the library returns them; NaN (constant series) skipped; ties ->
    lowest q = a_local*|B| + b_local (R16); self pairs skipped with one field.
    Returns (max, (a, b)) with (nan, (-1, -1)) if no pair is defined; with runner_up=True also the
    best value of every OTHER pair (-inf if none), for the argmax-margin check."""
    nx, ny, nz = dims
    fa = _field(fa)
    fbn = fa if fb is None else _field(fb)
    pa, pb = _box_points(A, nx, ny), _box_points(B, nx, ny)

    def standardise(v):
        v = v.astype(np.float64)
        d = v - v.mean(axis=0, keepdims=True)
        nrm = np.sqrt((d * d).sum(axis=0))
        with np.errstate(invalid="ignore", divide="ignore"):
            z = d / nrm
        return z, nrm == 0.0

    zb, cb = standardise(fbn[:, pb])
    best, arg = np.nan, (-1, -1)
    tops = []  # the two largest entries of every chunk
    for s in range(0, pa.size, chunk):
        za, ca = standardise(fa[:, pa[s:s + chunk]])
        c = za.T @ zb  # [chunk, |B|] sums of products of deviations / norms
        c = np.clip(c, -1.0, 1.0)
        if absval:
            c = np.abs(c)
        c[ca, :] = np.nan
        c[:, cb] = np.nan
        if fb is None:
            c[pa[s:s + chunk][:, None] == pb[None, :]] = np.nan
        c = c.astype(np.float32).astype(np.float64)
        c = np.where(np.isnan(c), -np.inf, c)
        flat = c.reshape(-1)
        tops.extend(np.partition(flat, flat.size - 2)[-2:].tolist() if flat.size >= 2 else flat.tolist())
        q = int(np.argmax(c))  # first maximum in row-major (a_local, b_local) order = lowest q
        v = c.reshape(-1)[q]
        if np.isfinite(v) and (np.isnan(best) or v > best):
            best, arg = v, (int(pa[s + q // pb.size]), int(pb[q % pb.size]))
    if runner_up:
        tops = sorted(tops)
        second = tops[-2] if len(tops) >= 2 else -np.inf
        return best, arg, float(second)
    return best, arg


def region_max(fa, fb, dims, measure: int, k: int, regA, regB, samples: int, seed: int):
    """Returns (out_max float64 [R], out_argmax int64 [R, 2])."""
    nx, ny, nz = dims
    fa = _field(fa)
    fbn = None if fb is None else _field(fb)
    n, P = fa.shape
    assert P == nx * ny * nz
    R = len(regA)
    A = (Box * R)(*[_box(b) for b in regA])
    B = (Box * R)(*[_box(b) for b in regB])
    out = np.empty(R, np.float64)
    arg = np.empty((R, 2), np.int64)
    lib().oracle_region_max(_p(fa, F32P), None if fbn is None else _p(fbn, F32P), nx, ny, nz, n,
                            measure, int(k), A, B, R, int(samples), ctypes.c_uint64(seed),
                            _p(out, F64P), _p(arg, I64P))
    return out, arg


def sample_many(seed: int, regA, regB, count: int, nx: int, ny: int, s0: int = 0):
    """Sampled point pairs s0 .. s0+count-1 of every region pair (R15): (a, b) int64 [R, count]."""
    R = len(regA)
    A = (Box * R)(*[_box(b) for b in regA])
    B = (Box * R)(*[_box(b) for b in regB])
    a = np.empty((R, count), np.int64)
    b = np.empty((R, count), np.int64)
    lib().oracle_sample_many(ctypes.c_uint64(seed), A, B, R, int(s0), int(count), nx, ny,
                             _p(a, I64P), _p(b, I64P))
    return a, b


def region_values(fa, fb, dims, measure: int, k: int, regA, regB, samples: int, seed: int):
    """Every value behind region_max (same enumeration, skips and fp32 rounding): returns
    (values float64 [R, T], a int64 [R, T], b int64 [R, T]) with T = samples, or |A||B| for the
    exhaustive case (then all region pairs must have the same box sizes); NaN = skipped."""
    nx, ny, nz = dims
    fa = _field(fa)
    fbn = None if fb is None else _field(fb)
    n, P = fa.shape
    assert P == nx * ny * nz
    R = len(regA)
    if samples > 0:
        T = samples
    else:
        sz = lambda b: (b[3] - b[0]) * (b[4] - b[1]) * (b[5] - b[2])  # noqa: E731
        T = sz(regA[0]) * sz(regB[0])
        assert all(sz(x) * sz(y) == T for x, y in zip(regA, regB))
    A = (Box * R)(*[_box(b) for b in regA])
    B = (Box * R)(*[_box(b) for b in regB])
    out = np.empty((R, T), np.float64)
    a = np.empty((R, T), np.int64)
    b = np.empty((R, T), np.int64)
    lib().oracle_region_values(_p(fa, F32P), None if fbn is None else _p(fbn, F32P), nx, ny, nz, n,
                               measure, int(k), A, B, R, int(samples), ctypes.c_uint64(seed),
                               _p(out, F64P), _p(a, I64P), _p(b, I64P))
    return out, a, b


def select_max(values, a, b):
    """Region maximum from enumerated values (R16): per row, the max over non-NaN
    values, the argmax at the LOWEST index among equal maxima, and the runner-up = the best value
    of any entry whose point pair differs from the argmax pair (-inf if none), so that the
    winning margin is max - runner_up.  All-NaN rows: (nan, (-1, -1), -inf)."""
    values = np.asarray(values, np.float64)
    R = values.shape[0]
    mx = np.full(R, np.nan)
    arg = np.full((R, 2), -1, np.int64)
    second = np.full(R, -np.inf)
    for r in range(R):
        v = np.where(np.isnan(values[r]), -np.inf, values[r])
        if not np.isfinite(v).any():
            continue
        q = int(np.argmax(v))
        mx[r] = v[q]
        arg[r] = (a[r][q], b[r][q])
        other = (a[r] != a[r][q]) | (b[r] != b[r][q])
        if other.any():
            second[r] = np.max(v[other])
    return mx, arg, second
