"""Thin Python binding of libcorr.so (include/corr.h) -- argument marshalling only.

Same names as the C ABI.  Tensors are torch tensors (device memory, streams), passed
to the library as raw pointers; every step of the hot path runs in libcorr.so's CUDA
kernels.  There is no CPU fallback: if libcorr.so cannot be loaded, or a call fails,
a ``CorrError`` is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CORR_LIB", os.path.join(_HERE, "libcorr.so"))  # override: A/B experiments

CORR_PEARSON = 0
CORR_KSG = 1
CORR_F_KSG_PLUS1 = 1 << 8
CORR_F_ABS = 1 << 9
CORR_F_KSG_DENSE = 1 << 10
CORR_F_KSG_COUNT = 1 << 11
CORR_F_KSG_SWEEP = 1 << 12
CORR_OK, CORR_E_INVAL, CORR_E_RANGE, CORR_E_NOMEM, CORR_E_CUDA = 0, -1, -2, -3, -4

EXPORTS = ("corr_field_create", "corr_field_update", "corr_field_aggregate", "corr_field_destroy", "corr_field_info", "corr_eval_pairs",
           "corr_region_max", "corr_ksg_debug", "corr_check", "corr_ksg_comparisons", "corr_ksg_nan_pairs", "corr_gemm_flops", "corr_launch_count",
           "corr_last_error")


class CorrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libcorr error {code}: {msg}")
        self.code = code


class corr_box(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("x0", "y0", "z0", "x1", "y1", "z1")]


_lib = None


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Loads libcorr.so (building it in-tree with nvcc if absent).  Fails loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcorr.so not found at {LIB_PATH}: build it with "
                          "`python -m paper_2309_03308_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.corr_field_create.argtypes = [vp, i32, i32, i32, i32, i32, vp, ctypes.POINTER(vp)]
    L.corr_field_destroy.argtypes = [vp]
    L.corr_field_aggregate.argtypes = [vp, i32, i32, i32, vp, ctypes.POINTER(vp)]
    L.corr_field_update.argtypes = [vp, vp, vp]
    L.corr_field_info.argtypes = [vp] + [ctypes.POINTER(i32)] * 5
    L.corr_eval_pairs.argtypes = [vp, vp, i32, i32, vp, vp, i64, vp, vp]
    L.corr_region_max.argtypes = [vp, vp, i32, i32, ctypes.POINTER(corr_box), ctypes.POINTER(corr_box), i64,
                                  i64, u64, vp, vp, vp]
    L.corr_ksg_debug.argtypes = [vp, vp, i32, vp, vp, i64, vp, vp, vp, vp]
    L.corr_check.argtypes = [vp, vp]
    L.corr_launch_count.argtypes = []
    L.corr_ksg_comparisons.argtypes = [i32, ctypes.POINTER(i64), i32]
    L.corr_ksg_nan_pairs.argtypes = [i32, ctypes.POINTER(i64), i32]
    L.corr_gemm_flops.argtypes = [i32, ctypes.POINTER(i64), ctypes.POINTER(i64), i32]
    L.corr_last_error.restype = ctypes.c_char_p
    L.corr_last_error.argtypes = []
    for name in EXPORTS[:-2]:
        getattr(L, name).restype = ctypes.c_int
    L.corr_launch_count.restype = ctypes.c_int64
    _lib = L
    return L


def _check(rc: int):
    if rc != CORR_OK:
        raise CorrError(rc, load().corr_last_error().decode())


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _field_stream(field: "Field", stream) -> int:
    """The caller's stream resolved on the FIELD's device (the library launches on that device)."""
    with torch.cuda.device(field.device):
        return _stream(stream)


def _ptr(t) -> int:
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return int(t)


class Field:
    """Owning handle of a ``corr_field`` (immutable ensemble field on one GPU)."""

    def __init__(self, handle: int, nx: int, ny: int, nz: int, members: int, device: int):
        self.handle = handle
        self.nx, self.ny, self.nz, self.members, self.device = nx, ny, nz, members, device

    @property
    def points(self) -> int:
        return self.nx * self.ny * self.nz

    def close(self):
        if self.handle:
            load().corr_field_destroy(ctypes.c_void_p(self.handle))
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def corr_field_create(values, nx: int, ny: int, nz: int, members: int, device: Optional[int] = None,
                      stream=None) -> Field:
    """values: float32 [members, nz*ny*nx] tensor (CPU or CUDA), or a raw pointer."""
    L = load()
    if isinstance(values, torch.Tensor):
        assert values.dtype == torch.float32 and values.is_contiguous()
        assert values.numel() == members * nx * ny * nz
        if device is None:
            device = values.device.index if values.is_cuda else torch.cuda.current_device()
    if device is None:
        device = torch.cuda.current_device()
    with torch.cuda.device(device):
        st = _stream(stream)
    h = ctypes.c_void_p()
    _check(L.corr_field_create(ctypes.c_void_p(_ptr(values)), nx, ny, nz, members, device,
                               ctypes.c_void_p(st), ctypes.byref(h)))
    return Field(h.value, nx, ny, nz, members, device)


def corr_field_update(field: Field, values, stream=None) -> Field:
    """Re-ingest new member values (same shape) into `field` in place (no device allocation)."""
    if isinstance(values, torch.Tensor):
        assert values.dtype == torch.float32 and values.is_contiguous()
        assert values.numel() == field.members * field.points
    with torch.cuda.device(field.device):
        st = _stream(stream)
    _check(load().corr_field_update(ctypes.c_void_p(field.handle), ctypes.c_void_p(_ptr(values)), ctypes.c_void_p(st)))
    return field


def corr_field_aggregate(field: Field, fx: int, fy: int, fz: int, stream=None) -> Field:
    """Mean-tree level of `field`: block means of fx x fy x fz points."""
    h = ctypes.c_void_p()
    with torch.cuda.device(field.device):
        st = _stream(stream)
    _check(load().corr_field_aggregate(ctypes.c_void_p(field.handle), fx, fy, fz, ctypes.c_void_p(st),
                                       ctypes.byref(h)))
    return Field(h.value, -(-field.nx // fx), -(-field.ny // fy), -(-field.nz // fz), field.members, field.device)


def corr_field_destroy(field: Field):
    field.close()


def corr_field_info(field: Field) -> Tuple[int, int, int, int, int]:
    vals = [ctypes.c_int32() for _ in range(5)]
    _check(load().corr_field_info(ctypes.c_void_p(field.handle), *[ctypes.byref(v) for v in vals]))
    return tuple(v.value for v in vals)


def _fb(fb: Optional[Field]):
    return ctypes.c_void_p(fb.handle) if fb is not None else None


def corr_eval_pairs(fa: Field, fb: Optional[Field], measure: int, k: int, idxA: torch.Tensor,
                    idxB: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    npairs = idxA.numel()
    assert idxB.numel() == npairs and idxA.dtype == torch.int64 and idxB.dtype == torch.int64
    if out is None:
        out = torch.empty(npairs, dtype=torch.float32, device=idxA.device)
    _check(load().corr_eval_pairs(ctypes.c_void_p(fa.handle), _fb(fb), measure, k, ctypes.c_void_p(_ptr(idxA)),
                                  ctypes.c_void_p(_ptr(idxB)), npairs, ctypes.c_void_p(_ptr(out)),
                                  ctypes.c_void_p(_field_stream(fa, stream))))
    return out


def boxes(regions: Sequence[Sequence[int]]):
    arr = (corr_box * len(regions))()
    for i, b in enumerate(regions):
        arr[i] = corr_box(*[int(v) for v in b])
    return arr


def corr_region_max(fa: Field, fb: Optional[Field], measure: int, k: int, regionA, regionB, samples: int,
                    seed: int, out_max: Optional[torch.Tensor] = None, out_argmax: Optional[torch.Tensor] = None,
                    stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    A = regionA if isinstance(regionA, ctypes.Array) else boxes(regionA)
    B = regionB if isinstance(regionB, ctypes.Array) else boxes(regionB)
    R = len(A)
    assert len(B) == R
    dev = torch.device("cuda", fa.device)
    if out_max is None:
        out_max = torch.empty(R, dtype=torch.float32, device=dev)
    if out_argmax is None:
        out_argmax = torch.empty((R, 2), dtype=torch.int64, device=dev)
    _check(load().corr_region_max(ctypes.c_void_p(fa.handle), _fb(fb), measure, k, A, B, R, samples,
                                  ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), ctypes.c_void_p(_ptr(out_max)),
                                  ctypes.c_void_p(_ptr(out_argmax)), ctypes.c_void_p(_field_stream(fa, stream))))
    return out_max, out_argmax


def corr_ksg_debug(fa: Field, fb: Optional[Field], k: int, idxA: torch.Tensor, idxB: torch.Tensor, stream=None):
    npairs = idxA.numel()
    n = fa.members
    eps = torch.empty((npairs, n), dtype=torch.float32, device=idxA.device)
    nx = torch.empty((npairs, n), dtype=torch.int32, device=idxA.device)
    ny = torch.empty((npairs, n), dtype=torch.int32, device=idxA.device)
    _check(load().corr_ksg_debug(ctypes.c_void_p(fa.handle), _fb(fb), k, ctypes.c_void_p(_ptr(idxA)),
                                 ctypes.c_void_p(_ptr(idxB)), npairs, ctypes.c_void_p(_ptr(eps)),
                                 ctypes.c_void_p(_ptr(nx)), ctypes.c_void_p(_ptr(ny)),
                                 ctypes.c_void_p(_field_stream(fa, stream))))
    return eps, nx, ny


def corr_ksg_comparisons(device: int = 0, reset: bool = True) -> int:
    v = ctypes.c_int64()
    _check(load().corr_ksg_comparisons(device, ctypes.byref(v), int(reset)))
    return v.value


def corr_ksg_nan_pairs(device: int = 0, reset: bool = True) -> int:
    """KSG point pairs corr_region_max skipped as NaN (constant series, psi(0)) since the last reset."""
    v = ctypes.c_int64()
    _check(load().corr_ksg_nan_pairs(device, ctypes.byref(v), int(reset)))
    return v.value


def corr_gemm_flops(device: int = 0, reset: bool = True) -> Tuple[int, int]:
    """(bf16 screening-pass flops, tf32 exact-pass flops) since the last reset."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(load().corr_gemm_flops(device, ctypes.byref(a), ctypes.byref(b), int(reset)))
    return a.value, b.value


def corr_launch_count() -> int:
    return int(load().corr_launch_count())


launch_count = corr_launch_count


def corr_check(field: Field, stream=None):
    _check(load().corr_check(ctypes.c_void_p(field.handle), ctypes.c_void_p(_field_stream(field, stream))))
