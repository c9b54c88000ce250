#!/usr/bin/env python
"""bench.py -- throughput of the arXiv 2309.03308 hot path on 1..8 B200s.

Workload (BASELINE.json metric "KSG-MI pairs/s (1000 members)", configs[3]): the
context view of a 250x352x20 synthetic ensemble with n = 1000 members, 88 bricks of
32x32x20 -> 3828 region pairs, S random point pairs per region pair (default 4096),
KSG MI k = 3 reduced to per-region-pair max/argmax.  One STEP = one pass of the whole
hot path over the context view:
    KSG region max (rows a2-a5, a8, a9)  +  Pearson sampled region max (a6)
    +  Pearson exhaustive focus block on the two cluster bricks (a7, tcgen05 GEMM)
    +  all-gather of the shards' maxima over NCCL (a10, N > 1).
`value` = KSG point pairs evaluated per second by the whole job (max-over-ranks device
time), inputs resident in HBM.  `e2e` = the same metric through the C ABI starting from
HOST memory: per step the pinned host pointer of the 7 GB member-major field is passed to
corr_field_update (the library streams and re-ingests it), the step runs, and the maxima are
read back to the host.  `ingest` = the field ingest kernels' achieved HBM bandwidth.

`--impl reference` times the CPU oracle (oracle/, plain C + OpenMP) as it stands on the
box's host cores on a bounded sample of the same workload (the reference arm for this
paper-only tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as tdist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import dist as cdist  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

METRIC = "KSG-MI pairs/s (1000 members)"
UNIT = "pairs/s"
K_NN = 3
SEED = 20230907
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                power.append(float(parts[7]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# --------------------------------------------------------------------------- workload
def workload(samples: int, name: str = "c4"):
    cfg = {"c4": synth.C4, "c3": synth.C3}[name]
    spec = synth.spec_of(cfg)
    A, B = synth.context_pairs(synth.bricks_of(cfg))
    return cfg, spec, A, B


def focus_boxes():
    # the two bricks holding the large cluster centres
    return synth.C2_REGION_A, synth.C2_REGION_B


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample_run(spec, A, B, samples, npairs, seed):
    """Times the oracle (as it stands) on the first `npairs` sampled pairs of the workload."""
    import oracle
    pairs = []
    r = 0
    while len(pairs) < npairs:
        for s in range(min(samples, npairs - len(pairs))):
            pairs.append(oracle.sample(seed, A[r], B[r], s, spec.nx, spec.ny))
        r += 1
    pts = sorted({p for ab in pairs for p in ab})
    pos = {p: i for i, p in enumerate(pts)}
    mini = synth.rows(spec, torch.tensor(pts)).T.contiguous().numpy()
    ia = np.array([pos[a] for a, _ in pairs], np.int64)
    ib = np.array([pos[b] for _, b in pairs], np.int64)
    threads = oracle.set_threads(cpu_count())  # torchrun exports OMP_NUM_THREADS=1
    t = time.perf_counter()
    vals = oracle.eval_pairs(mini, None, oracle.KSG, K_NN, ia, ib)
    dt = time.perf_counter() - t
    return npairs / dt, dt, vals, threads


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg, spec, A, B = workload(args.samples)
    npairs = args.ref_pairs
    times = []
    cores = None
    for i in range(args.warmup + args.steps):
        _, dt, _, cores = oracle_sample_run(spec, A, B, args.samples, npairs, SEED + i)
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = npairs / (ms / 1e3)
    sample = (f"{npairs} sampled point pairs of the C4 context view per step (n=1000, k=3), "
              f"oracle.eval_pairs brute force, OpenMP over pairs")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, args, world):
    name = "C4" if cfg.members == 1000 else "C3 (dry run only; not the BASELINE config)"
    return {"workload": f"{name} context view: {cfg.nx}x{cfg.ny}x{cfg.nz} grid, n={cfg.members} members, 88 bricks "
                        f"32x32x20, 3828 region pairs x S={args.samples} sampled point pairs, KSG k=3 region max "
                        f"(+ Pearson sampled region max + Pearson exhaustive focus block)",
            "grid": [cfg.nx, cfg.ny, cfg.nz], "members": cfg.members, "k": K_NN, "region_pairs": 3828,
            "samples_per_region_pair": args.samples, "parallelism": f"region-pair shards x{world}",
            "l2": "inputs larger than L2 (field rows 7 GB x planes, random rows per pair)",
            "limits": "members <= 4096; KSG k in [1, n-1] (k >= 33: multi-pass lists); exhaustive |A||B| < 2^32"}


# --------------------------------------------------------------------------- our arm
def make_field(spec, device, values=None):
    vals = synth.generate(spec, device=f"cuda:{device}") if values is None else values
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members, device=device)
    return f, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=4096)
    ap.add_argument("--ref-pairs", type=int, default=192)
    ap.add_argument("--cpu-pairs", type=int, default=768)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense-pass reference roofline")
    ap.add_argument("--workload", default="c4", choices=["c4", "c3"],
                    help="c4 = the BASELINE metric's config (default); c3 (n=100) only for dry runs")
    args = ap.parse_args()

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    local = local % torch.cuda.device_count()  # identity on a node with one GPU per rank
    torch.cuda.set_device(local)
    if world > 1:
        # BENCH_DIST_BACKEND=gloo: host-side collectives, for dry-running the multi-rank
        # orchestration with several ranks on ONE GPU (no rank waits inside a kernel); numbers
        # taken that way are not scaling results
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
    cfg, spec, A, B = workload(args.samples, args.workload)
    R = len(A)
    S = args.samples
    bounds = cdist.shard_bounds([S] * R, world)
    lo, hi = bounds[rank]
    Ash, Bsh = cb.boxes(A[lo:hi]), cb.boxes(B[lo:hi])
    fA, fB = focus_boxes()
    slabs = cdist.split_box_z(fA, world)
    myslab = cb.boxes([slabs[rank]])
    fBb = cb.boxes([fB])

    # field replica: rank 0 generates, NCCL broadcast to the others (untimed here)
    vals = torch.empty((spec.members, spec.points), dtype=torch.float32, device=f"cuda:{local}")
    if rank == 0:
        vals.copy_(synth.generate(spec, device=f"cuda:{local}"))
    if world > 1:
        tdist.broadcast(vals, 0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    field = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members, device=local)
    create_s = time.perf_counter() - t

    stream = torch.cuda.current_stream()
    ev = {"ksg": [], "pearson_sampled": [], "pearson_block": []}

    # field ingest (row a1, HBM-bound): corr_field_update from the device-resident input --
    # transpose [n][P] -> F[P][n_pad], fp64 stats + Z / tf32 split / bf16 planes, per-row sort
    n_pad_ = (spec.members + 7) // 8 * 8
    P_ = spec.points
    ing_bytes = {"transpose": P_ * (4 * spec.members + 4 * n_pad_),
                 "stats": P_ * (4 * spec.members + (4 + 4 + 4 + 2) * n_pad_),
                 "sort": P_ * (4 * spec.members + (4 + 2) * n_pad_)}
    cb.corr_field_update(field, vals)
    torch.cuda.synchronize()
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    for _ in range(3):
        cb.corr_field_update(field, vals)
    i1.record(stream)
    torch.cuda.synchronize()
    cb.corr_check(field)
    ing_ms = i0.elapsed_time(i1) / 3

    def _ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def step(f, timed=False):
        t0 = _ev() if timed else None
        km, ka = cb.corr_region_max(f, None, cb.CORR_KSG, K_NN, Ash, Bsh, S, SEED)
        t1 = _ev() if timed else None
        pm, pa = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, Ash, Bsh, S, SEED)
        t2 = _ev() if timed else None
        fm, fa = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, myslab, fBb, 0, 0)
        if timed:
            t3 = _ev()
            ev["ksg"].append((t0, t1))
            ev["pearson_sampled"].append((t1, t2))
            ev["pearson_block"].append((t2, t3))
        if world > 1:
            # all-gathers of the shards' region maxima + one all-reduce MAX over the focus slabs'
            # packed (value, q) keys, on the device (tests/test_dist.py runs it under gloo)
            km, ka, pm, pa, fm, fa = cdist.combine_step(km, ka, pm, pa, fm, fa, bounds, slabs, fB, spec.nx, spec.ny)
        return km, ka, pm, pa, fm, fa

    for _ in range(args.warmup):
        step(field)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    cb.corr_ksg_comparisons(local, reset=True)
    cb.corr_gemm_flops(local, reset=True)
    l0 = cb.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        res = step(field, timed=True)
    t1.record(stream)
    torch.cuda.synchronize()
    launches = cb.launch_count() - l0
    gemm_bf16, gemm_tf32 = (v / args.steps for v in cb.corr_gemm_flops(local, reset=True))
    if world > 1:
        tdist.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    stage_ms = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in ev.items()}
    if world > 1:
        tt = torch.tensor([ms] + [stage_ms[k] for k in ev], dtype=torch.float64, device=f"cuda:{local}")
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        ms = float(tt[0])
        stage_ms = {k: float(tt[i + 1]) for i, k in enumerate(ev)}
    total_pairs = R * S
    value = total_pairs / (ms / 1e3)

    # roofline of the dominant kernel (KSG, ALU-bound).  The column-cell k-NN skips every
    # comparison that provably cannot change an eps_i, so the per-unit figure is the EXECUTED
    # member-comparisons ("report pairs/s and executed comparisons, never
    # dense-equivalent"), tallied by one extra, untimed launch of the same shard with
    # CORR_F_KSG_COUNT (the counting build; the timed kernel does not count).
    n = spec.members
    my_pairs = (hi - lo) * S
    ksg_ms = stage_ms["ksg"]
    torch.cuda.synchronize()
    cb.corr_ksg_comparisons(local, reset=True)
    cb.corr_region_max(field, None, cb.CORR_KSG | cb.CORR_F_KSG_COUNT, K_NN, Ash, Bsh, S, SEED)
    executed = cb.corr_ksg_comparisons(local, reset=True)
    achieved = executed / (ksg_ms / 1e3)
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    sm_max = peaks.get("sm_max_mhz") or clk.get("sm_max_mhz") or 1965.0
    peak = 148 * 128 * sm_max * 1e6 / 4.0
    traffic = None
    ncu_ctx = {}
    if os.path.exists(NCU_TRAFFIC):
        try:
            tr = json.load(open(NCU_TRAFFIC))
            traffic = tr.get("ksg_dram_bytes_per_pair", 0) * my_pairs or None
            ncu_ctx = {k: tr[k] for k in ("ksg_kernel", "alu_pipe_pct", "issue_active_pct", "source") if k in tr}
        except Exception:
            traffic = None
    # the same kernel against the ALU pipe itself: ALU-pipe warp-instructions per pair measured by
    # ncu on this workload (profiles/ncu_traffic.json) x the pairs of the timed launches, vs
    # 148 SMs x 2 ALU warp-instr/clk -- how busy the hardware is, next to the algorithmic figure
    roofline_alu = None
    try:
        alu_pp = json.load(open(NCU_TRAFFIC)).get("alu_warp_instr_per_pair")
    except Exception:
        alu_pp = None
    if alu_pp:
        alu_peak = 148 * 2 * sm_max * 1e6
        alu_ach = alu_pp * my_pairs / (ksg_ms / 1e3)
        roofline_alu = {"bound": "alu", "kernel": f"ksg_cell_kernel<{K_NN},4>", "unit": "ALU warp-instr/s",
                        "achieved": alu_ach, "peak": alu_peak, "frac": alu_ach / alu_peak,
                        "per_pair": alu_pp, "per_pair_source": "ncu sm__inst_executed_pipe_alu of the same "
                                                                "kernel on this workload (profiles/ncu_traffic.json)"}
    roofline = {"bound": "alu", "kernel": f"ksg_cell_kernel<{K_NN},4> (column-cell k-NN + counts + psi)",
                "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gcmp/s", "frac": achieved / peak,
                "traffic": traffic,
                "peak_basis": f"148 SMs x 128 fp32 lanes x {sm_max:.0f} MHz / 4 ops per member-comparison",
                "frac_at_measured_clock": (achieved / (148 * 128 * clk["sm_mhz"] * 1e6 / 4.0)
                                           if clk.get("sm_mhz") else None),
                "executed_comparisons_per_pair": executed / max(my_pairs, 1),
                "dense_comparisons_per_pair": n * (n - 1),
                "ksg_ms_per_step": ksg_ms, "algorithmic_bytes_per_pair": 12 * spec.members,
                "ncu": ncu_ctx,
                "note": "the cell k-NN executes ~1 % of the n(n-1) comparisons at ~7 ALU ops each in SIMT "
                        "lockstep; the ALU pipe utilisation (ncu) is the hardware-side efficiency"}
    # the same kernel with the sweep disabled (CORR_F_KSG_DENSE): all n(n-1) comparisons executed,
    # results bit-identical -- the ALU-efficiency reference for the dense k-NN pass
    roofline_dense = None
    if not args.no_dense:
        Sd = 256
        cb.corr_ksg_comparisons(local, reset=True)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        cb.corr_region_max(field, None, cb.CORR_KSG | cb.CORR_F_KSG_DENSE, K_NN, Ash, Bsh, Sd, SEED)
        d1.record(stream)
        torch.cuda.synchronize()
        dense_s = d0.elapsed_time(d1) / 1e3
        dense_exec = cb.corr_ksg_comparisons(local, reset=True)
        roofline_dense = {"bound": "alu", "kernel": "ksg_sorted_kernel<3,4,4,dense> (CORR_F_KSG_DENSE, 4 members per lane)",
                          "achieved": (hi - lo) * Sd * n * (n - 1) / dense_s / 1e9, "peak": peak / 1e9, "unit": "Gcmp/s",
                          "frac": (hi - lo) * Sd * n * (n - 1) / dense_s / peak,
                          "executed_comparisons_per_pair": dense_exec / max((hi - lo) * Sd, 1),
                          "pairs_per_s": (hi - lo) * Sd / dense_s, "sample": f"{hi - lo} region pairs x {Sd} samples"}
    # the round-1 formulation (x-sorted block sweep, CORR_F_KSG_SWEEP) on the same subset: it executes
    # ~15x more comparisons at a higher fraction of the comparison peak but fewer pairs/s -- the
    # reference that shows what the cell k-NN's lower executed-comparison fraction buys
    roofline_sweep = None
    if not args.no_dense:
        Sd = 256
        cb.corr_ksg_comparisons(local, reset=True)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        cb.corr_region_max(field, None, cb.CORR_KSG | cb.CORR_F_KSG_SWEEP, K_NN, Ash, Bsh, Sd, SEED)
        d1.record(stream)
        torch.cuda.synchronize()
        sw_s = d0.elapsed_time(d1) / 1e3
        sw_exec = cb.corr_ksg_comparisons(local, reset=True)
        roofline_sweep = {"bound": "alu", "kernel": "ksg_sorted_kernel<3,1,4,sweep> (round-1 x-sorted block sweep)",
                          "achieved": sw_exec / sw_s / 1e9, "peak": peak / 1e9, "unit": "Gcmp/s",
                          "frac": sw_exec / sw_s / peak,
                          "executed_comparisons_per_pair": sw_exec / max((hi - lo) * Sd, 1),
                          "pairs_per_s": (hi - lo) * Sd / sw_s, "sample": f"{hi - lo} region pairs x {Sd} samples"}
    # secondary: the focus-block GEMM (tensor-bound) and the sampled Pearson pairs (HBM/L2-bound)
    fa_box, fb_box = slabs[rank], fB
    nA = (fa_box[3] - fa_box[0]) * (fa_box[4] - fa_box[1]) * (fa_box[5] - fa_box[2])
    nB = (fb_box[3] - fb_box[0]) * (fb_box[4] - fb_box[1]) * (fb_box[5] - fb_box[2])
    tf32_peak = (peaks.get("bf16_tflops") or 1612.0) * 0.5
    tf32_ctx = None  # cuBLAS TF32 GEMM measured on this pool (profiles/r01_tf32_peak.json), context only
    try:
        tf32_ctx = json.load(open(os.path.join(ROOT, "profiles", "r01_tf32_peak.json")))["tf32_tflops_burst"]
    except Exception:
        pass
    # executed tensor work (device counter): the hi*hi screening pass over every tile + the 3-MMA
    # exact pass over the tiles that can hold the maximum; dense-equivalent work reported beside it
    # mixed precision: the peak is the flop-weighted harmonic blend of the bf16 and tf32 peaks, so
    # frac = (bf16 flops / bf16 peak + tf32 flops / tf32 peak) / time
    bf16_peak = peaks.get("bf16_tflops") or 1612.0
    blk_s = stage_ms["pearson_block"] / 1e3
    blk_tflops = (gemm_bf16 + gemm_tf32) / blk_s / 1e12
    at_peak_s = (gemm_bf16 / bf16_peak + gemm_tf32 / tf32_peak) / 1e12
    blend_peak = (gemm_bf16 + gemm_tf32) / 1e12 / at_peak_s if at_peak_s > 0 else tf32_peak
    roofline_block = {"bound": "tensor",
                      "kernel": "pearson_screen_mc_kernel (bf16 screen, kind::f16, B tiles multicast in CTA pairs) + "
                                "pearson_block_kernel<exact> (kind::tf32, 3 MMA sets on the kept tiles)",
                      "achieved": blk_tflops, "peak": blend_peak, "unit": "TFLOP/s", "frac": blk_tflops / blend_peak,
                      "executed_bf16_flop_per_step": gemm_bf16, "executed_tf32_flop_per_step": gemm_tf32,
                      "dense_equivalent_tc_flop_per_step": 3 * 2.0 * nA * nB * n,
                      "peak_basis": "flop-weighted blend of measured bf16 dense and 0.5 x bf16 (nominal tf32:bf16)",
                      "cublas_tf32_measured": tf32_ctx,
                      "pairs_per_s": nA * nB / (stage_ms["pearson_block"] / 1e3),
                      "ms_per_step": stage_ms["pearson_block"]}
    # screened sampled Pearson: a bf16 pass over every pair (2 rows x n_pad x 2 B + the per-pair
    # approximate value, 4 B written and read back) and an fp32 pass over the few candidates
    n_pad = (n + 7) // 8 * 8
    ps_gbs = my_pairs * (4 * n_pad + 8) / (stage_ms["pearson_sampled"] / 1e3) / 1e9
    roofline_pearson_pairs = {"bound": "hbm", "kernel": "pearson_screen_kernel (bf16) + pearson_exact_selected_kernel",
                              "bytes_per_pair": 4 * n_pad + 8, "achieved": ps_gbs,
                              "peak": peaks.get("hbm_gbs") or 6552.3, "unit": "GB/s",
                              "frac": ps_gbs / (peaks.get("hbm_gbs") or 6552.3),
                              "pairs_per_s": my_pairs / (stage_ms["pearson_sampled"] / 1e3),
                              "ms_per_step": stage_ms["pearson_sampled"],
                              # ncu dram__bytes of pearson_screen_kernel<16> on this workload
                              # (profiles/r02_pearson_ncu_summary.txt: 58.15 GB read + 0.09 GB
                              # written for the 15.68 M pairs of C4, S = 4096)
                              "traffic_bytes_per_pair_ncu": (58.146e9 + 0.087e9) / 15679488}

    # e2e: same metric from HOST memory through the C ABI.  Every step passes the pinned host field
    # (7.04 GB member-major fp32) to corr_field_update, which streams it to the device itself
    # (32-member slices, one cudaMemcpyAsync each, on the field's copy stream, each slice transposed
    # as it lands) and rebuilds the derived buffers; the step runs and its maxima are read back to
    # pinned host memory.  Two field slots double-buffer: step i+1's update is issued on a side
    # stream while step i computes.  Every rank streams its own full replica over its own link.
    e2e = None

    def run_e2e_measurement():
            # the pinned host copy: allocated first and agreed on by every rank, so a rank that cannot
            # pin 7 GB (a shared host's limits) makes all ranks skip e2e instead of hanging later
            try:
                host = torch.empty((spec.members, spec.points), dtype=torch.float32, pin_memory=True)
                ok = 1
            except Exception:
                host, ok = None, 0
            if world > 1:
                flag = torch.tensor([ok], dtype=torch.int32, device=f"cuda:{local}")
                tdist.all_reduce(flag, op=tdist.ReduceOp.MIN)
                ok = int(flag[0])
            if not ok:
                raise RuntimeError("pinned host allocation of the field failed on some rank")
            host.copy_(vals)
            slots = [field, cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members, device=local)]
            # the update runs on a HIGH-priority stream: the step's KSG grid is one pair per CTA (15.7 M
            # CTAs), and without priority the update's transposes would be dispatched only after all of
            # them, stalling the slice ring of the streamed upload until the step ends
            up = torch.cuda.Stream(priority=-1)
            h2d = spec.members * spec.points * 4
            d2h_holder = [0]
            pinned_out = None

            def upload(slot, after=None):
                with torch.cuda.stream(up):
                    if after is not None:
                        up.wait_event(after)
                    cb.corr_field_update(slots[slot], host.data_ptr(), stream=up)  # HOST pointer

            step_evs = []

            def run_e2e(nsteps):
                nonlocal pinned_out
                done = [None, None]
                step_evs.clear()
                upload(0)
                for i in range(nsteps):
                    s_ = i % 2
                    stream.wait_stream(up)
                    e_a = torch.cuda.Event(enable_timing=True)
                    e_a.record(stream)
                    out = step(slots[s_])
                    if pinned_out is None:
                        pinned_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in out]
                    for dst, o in zip(pinned_out, out):
                        dst.copy_(o, non_blocking=True)
                    d2h_holder[0] = sum(o.numel() * o.element_size() for o in out)
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(stream)
                    done[s_] = ev
                    step_evs.append((e_a, ev))
                    if i + 1 < nsteps:
                        upload((i + 1) % 2, after=done[(i + 1) % 2])
                torch.cuda.synchronize()

            run_e2e(2)
            if world > 1:
                tdist.barrier()
            torch.cuda.synchronize()
            # at least 20 steps: the first step's update is the pipeline fill (not overlapped, and
            # included in the time), later updates overlap the previous step's compute
            ne = max(20, args.steps)
            e2e_clocks = ClockSampler(local)
            e2e_clocks.start()
            te = time.perf_counter()
            run_e2e(ne)
            e_s = (time.perf_counter() - te) / ne
            e2e_clk = e2e_clocks.stop()
            for s_ in slots:
                cb.corr_check(s_)
            if world > 1:
                tt = torch.tensor([e_s], dtype=torch.float64, device=f"cuda:{local}")
                tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
                e_s = float(tt[0])
            e2e_line = {"value": total_pairs / e_s, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
                   "d2h_bytes_per_step": d2h_holder[0], "s_per_step": e_s,
                   "device_step_ms": [round(a.elapsed_time(b), 1) for a, b in step_evs],
                   "clocks": e2e_clk,
                   "includes": "per step and rank: corr_field_update(pinned HOST pointer of the 7.04 GB field) -- "
                               "the library streams it (32-member slices, cudaMemcpyAsync on its copy stream) and "
                               "re-ingests -- then the step and the D2H of the maxima; double-buffered (the next "
                               "field's update overlaps the current step); the first step's upload (pipeline fill, not "
                               "overlapped) is inside the timed region",
                   "steps": ne}
            slots[1].close()
            del host

            return e2e_line

    if not args.no_e2e:
        try:
            e2e = run_e2e_measurement()
        except Exception as exc:  # reported, not fatal: the device-side line still prints
            e2e = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.synchronize()

    cpu_base = None
    if rank == 0 and not args.no_cpu_baseline:
        v, dt, _, threads = oracle_sample_run(spec, A, B, S, args.cpu_pairs, SEED)
        cpu_base = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                    "sample": f"first {args.cpu_pairs} sampled pairs of the C4 context view (n=1000, k=3), "
                              f"oracle.eval_pairs, {dt:.1f} s on rank 0's host"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config_dict(cfg, args, world),
                "roofline": roofline, "roofline_alu_pipe": roofline_alu, "roofline_ksg_sweep": roofline_sweep, "roofline_ksg_dense": roofline_dense, "roofline_pearson_block": roofline_block,
                "roofline_pearson_pairs": roofline_pearson_pairs, "cpu_baseline": cpu_base, "e2e": e2e, "clocks": clk,
                "gpu_launches": launches, "field_create_s": create_s,
                "ingest": {"bound": "hbm", "kernels": "transpose_kernel + stats_kernel + sort_bucket_kernel (n <= 1024; sort_radix_kernel above)",
                           "ms": ing_ms, "bytes": sum(ing_bytes.values()), "bytes_by_kernel": ing_bytes,
                           "achieved": sum(ing_bytes.values()) / (ing_ms / 1e3) / 1e9, "unit": "GB/s",
                           "peak": peaks.get("hbm_gbs") or 6552.3,
                           "frac": sum(ing_bytes.values()) / (ing_ms / 1e3) / 1e9 / (peaks.get("hbm_gbs") or 6552.3),
                           "note": "algorithmic bytes (each input read once, each plane written once); the "
                                   "per-kernel split of the time is in the ncu launch list (profiles/)"},
                "region_max_sample": [float(res[0][0]), int(res[1][0][0]), int(res[1][0][1])]}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
