"""e2e pipeline diagnostic (development tool): per-step host time and device spans of the
upload (H2D + corr_field_update on a side stream) and of the step (KSG + Pearson region max) on
the compute stream, for the double-buffered bench.py e2e loop at C4 (1 GPU)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
FULL = len(sys.argv) > 2 and sys.argv[2].startswith("full")
D2H = len(sys.argv) > 2 and sys.argv[2] == "full"
PIN = len(sys.argv) > 2 and sys.argv[2] == "full_pin"
pinned = [torch.empty(1, dtype=torch.float32, pin_memory=True), torch.empty((1, 2), dtype=torch.int64, pin_memory=True)]
cfg = synth.C4
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
host = torch.empty(vals.shape, dtype=torch.float32, pin_memory=True)
host.copy_(vals)
bufs = [vals, torch.empty_like(vals)]
slots = [cb.corr_field_create(b, spec.nx, spec.ny, spec.nz, spec.members) for b in bufs]
A, B = synth.context_pairs(synth.bricks_of(cfg))
A, B = cb.boxes(A), cb.boxes(B)
stream = torch.cuda.current_stream()
up = torch.cuda.Stream()


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


log = []


def upload(slot, after=None):
    with torch.cuda.stream(up):
        if after is not None:
            up.wait_event(after)
        e0 = ev(up)
        if not os.environ.get("E2E_NO_H2D"):  # diagnostics: which half of the upload slows the step
            frac = float(os.environ.get("E2E_H2D_FRAC", "1"))   # diagnostics: copy only part of the rows
            m = max(1, int(round(frac * host.shape[0])))
            bufs[slot][:m].copy_(host[:m], non_blocking=True)
        e1 = ev(up)
        t = time.perf_counter()
        if not os.environ.get("E2E_NO_UPDATE"):
            cb.corr_field_update(slots[slot], bufs[slot], stream=up)
        th = time.perf_counter() - t
        e2 = ev(up)
    return e0, e1, e2, th


n = 6
done = [None, None]
t0 = time.perf_counter()
u = [upload(0)]
steps = []
for i in range(n):
    s_ = i % 2
    th0 = time.perf_counter()
    stream.wait_stream(up)
    a = ev(stream)
    cb.corr_region_max(slots[s_], None, cb.CORR_KSG, 3, A, B, S, 1)
    cb.corr_region_max(slots[s_], None, cb.CORR_PEARSON, 0, A, B, S, 1)
    if FULL:  # bench.py's step: + the exhaustive focus block, + D2H of the maxima
        m, a2 = cb.corr_region_max(slots[s_], None, cb.CORR_PEARSON, 0, cb.boxes([synth.C2_REGION_A]),
                                   cb.boxes([synth.C2_REGION_B]), 0, 0)
        if D2H:
            m.to("cpu", non_blocking=True)
        if PIN:  # bench.py: all six outputs into preallocated pinned buffers
            outs = [m, a2]
            for dst, o in zip(pinned, outs):
                dst.copy_(o, non_blocking=True)
    b = ev(stream)
    done[s_] = b
    if i + 1 < n:
        u.append(upload((i + 1) % 2, after=done[(i + 1) % 2]))
    steps.append((a, b, time.perf_counter() - th0))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
base = u[0][0]
for i, (a, b, th) in enumerate(steps):
    line = {"step": i, "start_ms": base.elapsed_time(a), "step_ms": a.elapsed_time(b), "host_loop_s": th}
    if i + 1 < len(u):
        e0, e1, e2, tu = u[i + 1]
        line.update({"next_h2d_ms": e0.elapsed_time(e1), "next_update_ms": e1.elapsed_time(e2),
                     "next_up_start_ms": base.elapsed_time(e0), "update_host_block_s": tu})
    log.append(line)
print(json.dumps({"wall_s_per_step": wall / n, "steps": log}))
