"""Multi-GPU host logic (dist.py) on CPU: world-size-2 gloo process groups.

The shard -> all-gather path must reproduce the single-process result bit for bit
(SURVEY.md §8(e)); the per-rank region maxima here come from the CPU oracle on
each rank's shard (the GPU path's shard identity is a -m gpu test)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
from paper_2309_03308_b200 import dist as cdist
from paper_2309_03308_b200 import synth


def test_shard_bounds_cover_and_balance():
    for n, w in ((3828, 1), (3828, 2), (3828, 8), (7, 8), (10, 3)):
        b = cdist.shard_bounds([1] * n, w)
        assert b[0][0] == 0 and b[-1][1] == n and len(b) == w
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= 1
    wts = [16640 * 20480 if i % 8 == 7 else 20480 * 20480 for i in range(88)]
    b = cdist.shard_bounds(wts, 4)
    loads = [sum(wts[lo:hi]) for lo, hi in b]
    assert max(loads) / min(loads) < 1.1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    spec = synth.spec_of(synth.C1)
    f = synth.generate(spec).numpy()
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    bounds = cdist.shard_bounds([25] * len(A), world)
    lo, hi = bounds[rank]
    m, a = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A[lo:hi], B[lo:hi], 25, 11)
    fm, fa = cdist.gather_region_results(torch.from_numpy(m.astype(np.float32)), torch.from_numpy(a), bounds)
    # focus: one region pair split into slabs of A
    FA, FB = (0, 0, 0, 8, 8, 2), (0, 0, 2, 8, 8, 4)
    slabs = cdist.split_box_z(FA, world)
    sm, sa = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, [slabs[rank]], [FB], 0, 0)
    parts = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    tdist.all_gather(parts, torch.tensor([sm[0], sa[0][0], sa[0][1]], dtype=torch.float64))
    v, ab = cdist.combine_focus([float(p[0]) for p in parts], [(int(p[1]), int(p[2])) for p in parts], slabs, FB, 8, 8)
    # the same combine as ONE all-reduce MAX over packed keys (the device path of bench.py)
    dv, dab = cdist.combine_focus_device(torch.tensor([sm[0]], dtype=torch.float32), torch.tensor(sa),
                                         slabs, FB, 8, 8)
    assert float(dv[0]) == np.float32(v) and tuple(int(t) for t in dab[0]) == tuple(ab)
    q.put((rank, fm.numpy(), fa.numpy(), v, ab))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shards_gather_bit_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = synth.spec_of(synth.C1)
    f = synth.generate(spec).numpy()
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    m, a = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A, B, 25, 11)
    fm_ref, fa_ref = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, [(0, 0, 0, 8, 8, 2)],
                                       [(0, 0, 2, 8, 8, 4)], 0, 0)
    for rank, fm, fa, v, ab in res:
        assert np.array_equal(fm, m.astype(np.float32))  # every rank holds the full result
        assert np.array_equal(fa, a)
        assert v == fm_ref[0] and tuple(ab) == tuple(fa_ref[0])


def test_focus_key_order_and_roundtrip():
    """Packed focus keys: larger value wins, equal values -> lower q in the full box A, NaN /
    missing never wins, -0 == +0; decode inverts encode."""
    slabs = cdist.split_box_z((0, 0, 0, 8, 8, 4), 3)
    boxB = (0, 0, 0, 4, 4, 2)
    nx, ny = 8, 8
    vals = torch.tensor([0.5, 0.5, -0.0, 0.0, float("nan"), -1.0, 0.75], dtype=torch.float32)
    pa = [(3 * 64 + 2 * 8 + 1), (0 * 64 + 1), 5, 6, 7, 8, 2 * 64]
    pb = [9, 9, 1, 2, 3, 8, 0]  # inside boxB
    fa = torch.tensor(list(zip(pa, pb)), dtype=torch.int64)
    keys = cdist.focus_key(vals, fa, slabs, boxB, nx, ny)
    v, arg = cdist.decode_focus_key(keys, slabs, boxB, nx, ny)
    ok = ~torch.isnan(vals)
    assert torch.equal(v[ok], vals[ok] + 0.0) and torch.isnan(v[4])
    assert torch.equal(arg[ok], fa[ok]) and arg[4].tolist() == [-1, -1]
    assert keys[6] > keys[0] > keys[5] > keys[4]           # value order, NaN lowest
    assert keys[1] > keys[0]                               # tie -> lower q (a earlier in box A)
    assert keys[2] > keys[3] or keys[3] > keys[2]          # -0 and +0 compare as equal values ...
    k0 = cdist.focus_key(torch.tensor([-0.0]), fa[2:3], slabs, boxB, nx, ny)
    k1 = cdist.focus_key(torch.tensor([0.0]), fa[2:3], slabs, boxB, nx, ny)
    assert torch.equal(k0, k1)                             # ... same pair: identical keys


def _step_worker(rank, world, port, q):
    """bench.py's per-step orchestration (dist.combine_step) with the per-rank results computed by
    the oracle on the rank's shard / focus slab."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    spec = synth.spec_of(synth.C1)
    f = synth.generate(spec).numpy()
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    bounds = cdist.shard_bounds([30] * len(A), world)
    lo, hi = bounds[rank]
    km, ka = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A[lo:hi], B[lo:hi], 30, 7)
    pm, pa = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, A[lo:hi], B[lo:hi], 30, 7)
    FA, FB = (0, 0, 0, 8, 4, 4), (0, 4, 0, 8, 8, 4)
    slabs = cdist.split_box_z(FA, world)
    fm, fa = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, [slabs[rank]], [FB], 0, 0)
    t = lambda a, dt: torch.from_numpy(np.asarray(a).astype(dt))  # noqa: E731
    out = cdist.combine_step(t(km, np.float32), t(ka, np.int64), t(pm, np.float32), t(pa, np.int64),
                             t(fm, np.float32), t(fa, np.int64), bounds, slabs, FB, 8, 8)
    q.put((rank, [o.numpy() for o in out]))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_bench_step_orchestration(world):
    """The bench step's exchange (all-gathers + focus all-reduce MAX) reproduces the single-process
    results bit for bit on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = synth.spec_of(synth.C1)
    f = synth.generate(spec).numpy()
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    km, ka = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A, B, 30, 7)
    pm, pa = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, A, B, 30, 7)
    fm, fa = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 0, [(0, 0, 0, 8, 4, 4)], [(0, 4, 0, 8, 8, 4)], 0, 0)
    for _, out in res:
        assert np.array_equal(out[0], km.astype(np.float32)) and np.array_equal(out[1], ka)
        assert np.array_equal(out[2], pm.astype(np.float32)) and np.array_equal(out[3], pa)
        assert out[4][0] == np.float32(fm[0]) and tuple(out[5][0]) == tuple(fa[0])
