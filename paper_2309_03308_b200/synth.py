"""Seeded synthetic ensembles and workload configs (input generation only).

This module is the ONE place both sides of the parity tests get their inputs
from.  It holds none of the method's arithmetic (no correlation, neighbour
search, digamma or sampling of point pairs): only the synthetic field model,
the region tiling and the five BASELINE.json configs.

Field model ("Synth" and :538; SPEC.md:77-85
``gen_synthetic``):

    v(p, e) = mu(p) + sigma(p) * [ (1 - w(p)) * eta(p, e) + w(p) * s_g(e) ]

* ``eta(p, e)`` and ``s_g(e)`` are standard-normal-like variates from a
  counter-based hash (murmur3 fmix32 of (seed, stream, counter)) summed
  Irwin-Hall style (4 uniforms, centred, scaled to unit variance).  Only exact
  integer ops and IEEE fp64 +,-,*,/ are used, evaluated op by op, so the bytes
  are identical on CPU and CUDA and any subset of rows can be regenerated on
  the host without materialising the whole field (``rows``).
* ``w(p) = max(0, 1 - dinf(p, c) / R_c)`` for the nearest centre ``c`` in the
  l-infinity norm (ties -> lowest id), "decaying by their
  l_inf-norm distance from the cluster center".
* ``mu(p) = 250 + 30 z / nz``, ``sigma(p) = 0.5 + 2 y / ny`` (temperature-like
  offsets that exercise the fp64 standardisation and create fp32 value ties).
* All clusters of field 1 share one signal ("high mutual
  correlation between each pair of clusters"); field 2 ("u-like", config 5)
  has its own centres and shares the signal with field 1 in one group only, so
  the cross matrix is asymmetric.

Values are returned in the paper's / SPEC's file order ``[member][z][y][x]``
(SPEC.md:121), i.e. a ``[n, P]`` float32 tensor with ``p = (z*ny + y)*nx + x``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Sequence, Tuple

import torch

MASK32 = 0xFFFFFFFF
SQRT3 = math.sqrt(3.0)


# --------------------------------------------------------------------------
# counter-based variates
# --------------------------------------------------------------------------
def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 x in [0, 2^32) without int64 overflow."""
    lo, hi = c & 0xFFFF, (c >> 16) & 0xFFFF
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & MASK32


def _fmix32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x85EBCA6B)
    x = x ^ (x >> 13)
    x = _mul32(x, 0xC2B2AE35)
    return x ^ (x >> 16)


def _stream_key(seed: int, stream: int) -> int:
    t = torch.tensor([(seed * 0x9E3779B1 + stream * 0x85EBCA77 + 0x27D4EB2F) & MASK32],
                     dtype=torch.int64)
    return int(_fmix32(_fmix32(t))[0])


def normals(counter: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    """Unit-variance, zero-mean variates (fp64) for int64 counters in [0, 2^32)."""
    key = _stream_key(seed, stream)
    base = _fmix32(counter ^ key)
    acc = torch.zeros(counter.shape, dtype=torch.float64, device=counter.device)
    for t in range(4):
        u = _fmix32(base ^ ((0x9E3779B9 * (t + 1)) & MASK32))
        acc = acc + (u.to(torch.float64) + 0.5) / 4294967296.0
    return (acc - 2.0) * SQRT3


# --------------------------------------------------------------------------
# field model
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Cluster:
    x: int
    y: int
    z: int
    radius: float
    signal: int  # index of the shared signal s_g


@dataclasses.dataclass(frozen=True)
class FieldSpec:
    nx: int
    ny: int
    nz: int
    members: int
    seed: int
    clusters: Tuple[Cluster, ...]
    signal_seed: int = -1  # seed of the shared signals s_g (-1: same as seed)

    @property
    def points(self) -> int:
        return self.nx * self.ny * self.nz


# Centres on the 250 x 352 x 20 grid.
_FIELD1_CLUSTERS = (
    Cluster(16, 16, 10, 12.0, 0), Cluster(80, 48, 5, 4.0, 0), Cluster(40, 120, 15, 4.0, 0),
    Cluster(176, 240, 10, 12.0, 0), Cluster(210, 300, 5, 4.0, 0), Cluster(120, 200, 15, 4.0, 0),
)
_FIELD2_CLUSTERS = (
    Cluster(48, 80, 10, 12.0, 0), Cluster(100, 20, 5, 4.0, 0), Cluster(20, 200, 15, 4.0, 0),
    Cluster(200, 160, 10, 12.0, 1), Cluster(230, 330, 5, 4.0, 1), Cluster(150, 280, 15, 4.0, 1),
)
_BASE_DIMS = (250, 352, 20)


def scaled_clusters(clusters: Sequence[Cluster], nx: int, ny: int, nz: int) -> Tuple[Cluster, ...]:
    """Scale the reference-grid centres onto an (nx, ny, nz) grid, radius >= 1."""
    sx, sy, sz = nx / _BASE_DIMS[0], ny / _BASE_DIMS[1], nz / _BASE_DIMS[2]
    out = []
    for c in clusters:
        out.append(Cluster(min(nx - 1, int(round(c.x * sx))), min(ny - 1, int(round(c.y * sy))),
                           min(nz - 1, int(round(c.z * sz))), max(1.0, round(c.radius * min(sx, sy))),
                           c.signal))
    return tuple(out)


def field_spec(nx: int, ny: int, nz: int, members: int, seed: int, variable: int = 1,
               signal_seed: int = -1) -> FieldSpec:
    base = _FIELD1_CLUSTERS if variable == 1 else _FIELD2_CLUSTERS
    if (nx, ny, nz) == _BASE_DIMS:
        cl = base
    else:
        cl = scaled_clusters(base, nx, ny, nz)
    return FieldSpec(nx, ny, nz, members, seed, cl, signal_seed)


def _weights(spec: FieldSpec, p: torch.Tensor):
    """(w(p), signal id) for int64 point ids p (nearest centre in l_inf, ties -> lowest id)."""
    x = p % spec.nx
    y = (p // spec.nx) % spec.ny
    z = p // (spec.nx * spec.ny)
    best_d = torch.full(p.shape, 1 << 40, dtype=torch.int64, device=p.device)
    best_r = torch.ones(p.shape, dtype=torch.float64, device=p.device)
    best_g = torch.zeros(p.shape, dtype=torch.int64, device=p.device)
    for c in spec.clusters:
        d = torch.maximum(torch.maximum((x - c.x).abs(), (y - c.y).abs()), (z - c.z).abs())
        closer = d < best_d
        best_d = torch.where(closer, d, best_d)
        best_r = torch.where(closer, torch.full_like(best_r, c.radius), best_r)
        best_g = torch.where(closer, torch.full_like(best_g, c.signal), best_g)
    w = torch.clamp(1.0 - best_d.to(torch.float64) / best_r, min=0.0)
    return w, best_g, x, y, z


def _signals(spec: FieldSpec, device) -> torch.Tensor:
    ng = 1 + max(c.signal for c in spec.clusters)
    e = torch.arange(spec.members, dtype=torch.int64, device=device)
    # signal g is shared by every field generated with the same signal seed
    sseed = spec.seed if spec.signal_seed < 0 else spec.signal_seed
    return torch.stack([normals(e, sseed, 1000 + g) for g in range(ng)])  # [ng, n]


def rows(spec: FieldSpec, points: torch.Tensor) -> torch.Tensor:
    """Member series of the given points: float32 [len(points), members]."""
    p = points.to(torch.int64).reshape(-1, 1)
    dev = p.device
    w, g, _, y, z = _weights(spec, p)
    e = torch.arange(spec.members, dtype=torch.int64, device=dev).reshape(1, -1)
    assert spec.points * spec.members < (1 << 32), "counter space exceeded"
    eta = normals(p * spec.members + e, spec.seed, 7)
    s = _signals(spec, dev)[g.reshape(-1)]  # [m, n]
    mu = 250.0 + 30.0 * z.to(torch.float64) / spec.nz
    sigma = 0.5 + 2.0 * y.to(torch.float64) / spec.ny
    v = mu + sigma * ((1.0 - w) * eta + w * s)
    return v.to(torch.float32)


def generate(spec: FieldSpec, device="cpu", chunk_points: int = 1 << 16) -> torch.Tensor:
    """The whole field, float32 [members, P] (file order [member][z][y][x])."""
    out = torch.empty((spec.members, spec.points), dtype=torch.float32, device=device)
    for p0 in range(0, spec.points, chunk_points):
        p1 = min(spec.points, p0 + chunk_points)
        pts = torch.arange(p0, p1, dtype=torch.int64, device=device)
        out[:, p0:p1] = rows(spec, pts).T
    return out


# --------------------------------------------------------------------------
# regions (PAPER.md:131, :218 -- 250x352x20 -> 8x11x1 bricks of 32x32x20)
# --------------------------------------------------------------------------
Box = Tuple[int, int, int, int, int, int]  # half-open (x0, y0, z0, x1, y1, z1)


def partition(nx: int, ny: int, nz: int, bx: int, by: int, bz: int) -> List[Box]:
    """Ceil-division tiling into bricks, brick ids row-major with x fastest (R12/R13)."""
    out = []
    for z0 in range(0, nz, bz):
        for y0 in range(0, ny, by):
            for x0 in range(0, nx, bx):
                out.append((x0, y0, z0, min(nx, x0 + bx), min(ny, y0 + by), min(nz, z0 + bz)))
    return out


def context_pairs(boxes: Sequence[Box]):
    """Unordered pairs i < j of one field (context view: 88*87/2)."""
    A, B = [], []
    for i in range(len(boxes)):
        for j in range(i + 1, len(boxes)):
            A.append(boxes[i])
            B.append(boxes[j])
    return A, B


def matrix_pairs(boxes: Sequence[Box]):
    """All ordered pairs (inter-variable matrix), diagonal included."""
    A, B = [], []
    for i in range(len(boxes)):
        for j in range(len(boxes)):
            A.append(boxes[i])
            B.append(boxes[j])
    return A, B


def refine(box: Box, max_children: int) -> List[Box]:
    """Focus-view refinement of a brick ("each brick is recursively refined into M/2
    bricks"; SPEC.md:123 reading: halve every axis whose extent allows, octree-like, while the child
    count stays <= max_children).  Children ordered x fastest."""
    x0, y0, z0, x1, y1, z1 = box
    parts = [1, 1, 1]
    while True:
        trial = [p * 2 if ((x1 - x0, y1 - y0, z1 - z0)[i] // (p * 2)) >= 1 else p for i, p in enumerate(parts)]
        if trial == parts or trial[0] * trial[1] * trial[2] > max_children:
            break
        parts = trial
    out = []
    ext = (x1 - x0, y1 - y0, z1 - z0)
    cuts = [[lo + ext[i] * c // parts[i] for c in range(parts[i] + 1)] for i, lo in enumerate((x0, y0, z0))]
    for k in range(parts[2]):
        for j in range(parts[1]):
            for i in range(parts[0]):
                out.append((cuts[0][i], cuts[1][j], cuts[2][k], cuts[0][i + 1], cuts[1][j + 1], cuts[2][k + 1]))
    return out


def box_size(b: Box) -> int:
    return (b[3] - b[0]) * (b[4] - b[1]) * (b[5] - b[2])


# --------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    nz: int
    members: int
    seed: int
    k: int = 3


C1 = Config("C1-tiny", 8, 8, 4, 10, 1)
C2 = Config("C2-focus", 250, 352, 20, 100, 2)
C3 = Config("C3-context-n100", 250, 352, 20, 100, 3)
C4 = Config("C4-context-n1000", 250, 352, 20, 1000, 4)
C5 = Config("C5-two-variable-n1000", 250, 352, 20, 1000, 5)
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}

# C2's two focus regions: contain the two large cluster centres.
C2_REGION_A: Box = (0, 0, 0, 32, 32, 20)
C2_REGION_B: Box = (160, 224, 0, 192, 256, 20)


def spec_of(cfg: Config, variable: int = 1) -> FieldSpec:
    seed = cfg.seed if variable == 1 else cfg.seed + 1
    return field_spec(cfg.nx, cfg.ny, cfg.nz, cfg.members, seed, variable, signal_seed=cfg.seed)


def bricks_of(cfg: Config) -> List[Box]:
    if cfg is C1:
        return partition(cfg.nx, cfg.ny, cfg.nz, 4, 4, 4)
    return partition(cfg.nx, cfg.ny, cfg.nz, 32, 32, 20)


def random_pairs(P: int, npairs: int, seed: int, device="cpu"):
    """Uniform random (a, b) point-index pairs with a != b, for eval_pairs tests."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.randint(0, P, (npairs,), generator=g, dtype=torch.int64)
    b = torch.randint(0, P - 1, (npairs,), generator=g, dtype=torch.int64)
    b = b + (b >= a).to(torch.int64)
    return a.to(device), b.to(device)
