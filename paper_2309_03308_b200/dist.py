"""Multi-GPU sharding of the region-pair list (§8(a) row a10).

One process per GPU.  Region pairs are independent, so each rank takes a contiguous,
equal-work shard of the list and runs ``corr_region_max`` on its own field replica;
results combine with ONE all-gather of the per-region-pair (max, argmax) over NCCL
(NVLink/NVSwitch).  The sampler is keyed by (seed, box A, box B), not by list position,
so 1-, 2-, 4- and 8-GPU runs give bit-identical results.

Host logic only (works with the gloo backend on CPU for the tests).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as tdist


def shard_bounds(weights: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous shards [lo, hi) of a weighted list with near-equal total weight.

    Shard r ends at the first index whose prefix weight reaches (r+1)/world of the total
    (sampled mode: equal S per pair -> equal counts; exhaustive: weight |A|*|B|)."""
    n = len(weights)
    total = sum(int(w) for w in weights)
    bounds = []
    lo = 0
    acc = 0
    idx = 0
    for r in range(world):
        target = total * (r + 1) / world
        while idx < n and (acc + int(weights[idx]) <= target or r == world - 1):
            acc += int(weights[idx])
            idx += 1
        bounds.append((lo, idx))
        lo = idx
    assert bounds[-1][1] == n
    return bounds


def all_gather(parts: List[torch.Tensor], t: torch.Tensor, group=None) -> None:
    """all_gather that also runs under gloo with CUDA tensors (staged through host memory),
    so the multi-rank orchestration can be dry-run on one GPU; NCCL gathers in place."""
    if t.is_cuda and tdist.get_backend(group) == "gloo":
        host = [torch.empty(p.shape, dtype=p.dtype) for p in parts]
        tdist.all_gather(host, t.cpu(), group=group)
        for p, h in zip(parts, host):
            p.copy_(h)
        return
    tdist.all_gather(parts, t, group=group)


def gather_region_results(out_max: torch.Tensor, out_arg: torch.Tensor, bounds: Sequence[Tuple[int, int]],
                          group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """All-gather the shards' (max, argmax) into the full [R] / [R, 2] result on every rank.

    Shards can differ in length by one: each rank pads to the longest shard, then the
    padding is dropped.  One collective: (float32 max bit-cast to int64 || argmax) rows."""
    world = len(bounds)
    longest = max(hi - lo for lo, hi in bounds)
    dev = out_max.device
    packed = torch.zeros((longest, 3), dtype=torch.int64, device=dev)
    m = out_max.numel()
    packed[:m, 0] = out_max.view(torch.int32).to(torch.int64)
    packed[:m, 1:] = out_arg
    parts = [torch.empty_like(packed) for _ in range(world)]
    all_gather(parts, packed, group=group)
    rows = [parts[r][: hi - lo] for r, (lo, hi) in enumerate(bounds)]
    allrows = torch.cat(rows, 0)
    full_max = allrows[:, 0].to(torch.int32).view(torch.float32).clone()
    full_arg = allrows[:, 1:].clone()
    return full_max, full_arg


def split_box_z(box, world: int):
    """Split one region box into `world` slabs along its longest axis (focus view, one
    region pair: SURVEY.md §8(e) "C2 ... split A into R row slabs")."""
    x0, y0, z0, x1, y1, z1 = box
    ext = [x1 - x0, y1 - y0, z1 - z0]
    ax = max(range(3), key=lambda i: ext[i])
    lo = [x0, y0, z0]
    hi = [x1, y1, z1]
    out = []
    for r in range(world):
        a = lo[ax] + ext[ax] * r // world
        b = lo[ax] + ext[ax] * (r + 1) // world
        l2, h2 = list(lo), list(hi)
        l2[ax], h2[ax] = a, b
        out.append((l2[0], l2[1], l2[2], h2[0], h2[1], h2[2]))
    return out


def combine_focus(maxes: Sequence[float], args: Sequence[Tuple[int, int]], slabs, boxB, nx: int, ny: int):
    """Combine per-slab exhaustive maxima of one region pair: max value, ties -> lowest
    q = a_local*|B| + b_local in the FULL box A (reading R16)."""
    fx0, fy0, fz0 = min(s[0] for s in slabs), min(s[1] for s in slabs), min(s[2] for s in slabs)
    fx1, fy1, fz1 = max(s[3] for s in slabs), max(s[4] for s in slabs), max(s[5] for s in slabs)
    ax, ay = fx1 - fx0, fy1 - fy0
    bx, by = boxB[3] - boxB[0], boxB[4] - boxB[1]
    nB = bx * by * (boxB[5] - boxB[2])
    best = None
    for v, (a, b) in zip(maxes, args):
        if a < 0 or v != v:
            continue
        xa, ya, za = a % nx, (a // nx) % ny, a // (nx * ny)
        xb, yb, zb = b % nx, (b // nx) % ny, b // (nx * ny)
        al = ((za - fz0) * ay + (ya - fy0)) * ax + (xa - fx0)
        bl = ((zb - boxB[2]) * by + (yb - boxB[1])) * bx + (xb - boxB[0])
        q = al * nB + bl
        if best is None or v > best[0] or (v == best[0] and q < best[1]):
            best = (v, q, a, b)
    if best is None:
        return float("nan"), (-1, -1)
    return best[0], (best[2], best[3])


_MASK32 = 0xFFFFFFFF
_TOP = -(1 << 63)  # int64 with only the sign bit: maps unsigned key order onto signed order


def focus_key(fm: torch.Tensor, fa: torch.Tensor, slabs, boxB, nx: int, ny: int) -> torch.Tensor:
    """Order-preserving int64 key of one rank's focus-slab maximum (on the tensors' device):
    the orderable bits of the fp32 value (reading R16: NaN never wins, -0 == +0) above
    0xFFFFFFFF - q, with q = a_local*|B| + b_local in the FULL box A (the union of the slabs), so
    the larger key is the larger value and, among equal values, the lower q; a slab without a
    defined value gets the smallest key."""
    fx0, fy0, fz0 = min(s_[0] for s_ in slabs), min(s_[1] for s_ in slabs), min(s_[2] for s_ in slabs)
    fx1, fy1 = max(s_[3] for s_ in slabs), max(s_[4] for s_ in slabs)
    ax, ay = fx1 - fx0, fy1 - fy0
    bx, by = boxB[3] - boxB[0], boxB[4] - boxB[1]
    nB = bx * by * (boxB[5] - boxB[2])
    a, b = fa.reshape(-1, 2)[:, 0], fa.reshape(-1, 2)[:, 1]
    xa, ya, za = a % nx, (a // nx) % ny, a // (nx * ny)
    xb, yb, zb = b % nx, (b // nx) % ny, b // (nx * ny)
    q = (((za - fz0) * ay + (ya - fy0)) * ax + (xa - fx0)) * nB + ((zb - boxB[2]) * by + (yb - boxB[1])) * bx + (xb - boxB[0])
    v = fm.reshape(-1).to(torch.float32) + 0.0
    u = v.view(torch.int32).to(torch.int64) & _MASK32
    u = torch.where((u >> 31) == 1, u ^ _MASK32, u ^ 0x80000000)
    key = ((u << 32) | (_MASK32 - q)) ^ _TOP
    bad = torch.isnan(v) | (a < 0)
    return torch.where(bad, torch.full_like(key, _TOP), key)


def decode_focus_key(key: torch.Tensor, slabs, boxB, nx: int, ny: int):
    """Inverse of focus_key: (value float32 [m], argmax int64 [m, 2]); the smallest key ->
    (nan, (-1, -1))."""
    fx0, fy0, fz0 = min(s_[0] for s_ in slabs), min(s_[1] for s_ in slabs), min(s_[2] for s_ in slabs)
    fx1, fy1 = max(s_[3] for s_ in slabs), max(s_[4] for s_ in slabs)
    ax, ay = fx1 - fx0, fy1 - fy0
    bx, by = boxB[3] - boxB[0], boxB[4] - boxB[1]
    nB = bx * by * (boxB[5] - boxB[2])
    k = key ^ _TOP
    u = (k >> 32) & _MASK32
    q = _MASK32 - (k & _MASK32)
    u = torch.where((u >> 31) == 1, u ^ 0x80000000, u ^ _MASK32)
    v = (u - ((u >> 31) << 32)).to(torch.int32).view(torch.float32)  # low 32 bits as int32
    al, bl = q // nB, q % nB
    a = ((fz0 + al // (ax * ay)) * ny + (fy0 + (al // ax) % ay)) * nx + (fx0 + al % ax)
    b = ((boxB[2] + bl // (bx * by)) * ny + (boxB[1] + (bl // bx) % by)) * nx + (boxB[0] + bl % bx)
    none = key == _TOP
    v = torch.where(none, torch.full_like(v, float("nan")), v)
    arg = torch.stack([torch.where(none, torch.full_like(a, -1), a), torch.where(none, torch.full_like(b, -1), b)], -1)
    return v, arg


def combine_focus_device(fm: torch.Tensor, fa: torch.Tensor, slabs, boxB, nx: int, ny: int, group=None):
    """Combines the ranks' focus-slab maxima of ONE region pair with a single all-reduce MAX over
    the packed keys ("all-reduce MAX on the packed u64 key"), on the device under
    NCCL; same result as combine_focus (max value, ties -> lowest q in the full box A)."""
    key = focus_key(fm, fa, slabs, boxB, nx, ny)
    if key.is_cuda and tdist.get_backend(group) == "gloo":
        host = key.cpu()
        tdist.all_reduce(host, op=tdist.ReduceOp.MAX, group=group)
        key.copy_(host)
    else:
        tdist.all_reduce(key, op=tdist.ReduceOp.MAX, group=group)
    return decode_focus_key(key, slabs, boxB, nx, ny)


def combine_step(km, ka, pm, pa, fm, fa, bounds, slabs, boxB, nx: int, ny: int, group=None):
    """The exchange step of one bench step: every rank holds its shard's
    KSG and Pearson region maxima and its focus slab's maximum; afterwards every rank holds the
    full results -- one all-gather per measure, one all-reduce MAX for the focus pair."""
    km, ka = gather_region_results(km, ka, bounds, group=group)
    pm, pa = gather_region_results(pm, pa, bounds, group=group)
    fm, fa = combine_focus_device(fm, fa, slabs, boxB, nx, ny, group=group)
    return km, ka, pm, pa, fm, fa
