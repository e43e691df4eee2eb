#!/usr/bin/env python
"""Benchmark of the R²-Gaussian hot path on B200 (BASELINE.json).

Headline workload (configs[2], "cfg3"): Shepp-Logan 256^3 phantom, 100k
Gaussians (sample_init_cloud + trained-like anisotropy), 75 cone-beam views at
512x512. One step = render (all of this rank's views, batched) + render_backward
with a U(-1,1) upstream gradient into a zeroed CloudGrads, + the NCCL all-reduce
of the per-Gaussian gradients when N > 1 (views sharded over ranks: strong
scaling). Metric: projections/s (fwd+bwd) for the whole job.
Secondary (configs[3], "cfg4"): voxelize + voxelize_backward of 200k Gaussians
on a 256^3 grid (z-slab sharded), reported as voxels/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "projections/sec (fwd+bwd)"
DTYPE = ("fp32 pixel sums (K4/K8: E rounded to binary16 with a hi/lo binary16 split of g, FP32 accumulate, "
         "on the tensor pipe; fp32_simt_arm = the all-FP32 SIMT form); FP64 binning preprocess + chain rules")
UNIT = "projections/s"

# Hardware-unit evidence per kernel (ncu, tools/profile_round2.sh -> tools/hw_units.py):
# the busiest unit (issue slots, FP32/FP64/XU/tensor pipes, L1 wavefronts, L2, DRAM)
# and its fraction of peak. Static: read from the committed profile, not measured here.
HW_PROFILE = "profiles/r02j_hw_units.json"
NCU_NAMES = {
    "K0_gauss_prep": ["gauss_prep_kernel"], "K1_raster_preprocess": ["raster_preprocess_kernel"],
    "K2_bin_count": ["bin_count_kernel"],
    "K2_bin_scan": ["bin_colsum_kernel", "bin_segscan_kernel", "bin_tilebase_kernel", "bin_apply_kernel"],
    "K2_bin_scatter": ["bin_scatter_kernel"], "K2_bin_ranges": ["bin_ranges_kernel"],
    "K2_tile_order": ["tile_order_keys_kernel", "tile_order_small_kernel<1>", "tile_order_hist_kernel", "tile_order_rank_kernel"],
    "K2_k3_items": ["k3_parts_kernel", "k3_items_kernel", "k3_first_small_kernel", "k3_block_parts_kernel", "k3_block_items_kernel"],
    "K3_composite": ["composite_kernel"],
    "K4_backward_stats": ["backward_stats_mma_kernel<2>", "backward_stats_mma_kernel<4>", "backward_stats_mma_kernel"],
    "K5_raster_chain": ["raster_chain_kernel<0>"], "K5_view_sum": ["view_sum_kernel"],
    "K5_raster_finalize": ["raster_finalize_kernel"],
    "K6_voxel_preprocess": ["voxel_preprocess_kernel"], "K6_voxel_emit": ["voxel_emit_kernel<unsigned short>"],
    "K2_ranges": ["key_ranges_kernel<unsigned short>"], "K7_voxel_eval": ["voxel_eval_kernel"],
    "K8_voxel_backward_stats": ["voxel_backward_mma_kernel"], "K8_voxel_pair_sum": ["voxel_pair_sum_kernel"],
    "K8_voxel_chain": ["voxel_chain_kernel"],
    "K9_tv3d": ["tv3d_kernel", "tv3d_finish_kernel"], "K10_adam": ["adam_kernel"],
    "K11_ssim": ["ssim_h_kernel", "ssim_v_kernel", "ssim_adj_v_kernel", "ssim_adj_h_kernel",
                 "photometric_finish_kernel"],
    "AC_adaptive": ["ac_classify_kernel", "ac_apply_kernel"],
}


def hw_units():
    try:
        return json.load(open(os.path.join(ROOT, HW_PROFILE)))
    except Exception:
        return {}


def hw_of(units, key):
    """{unit, frac, dram_gbs_under_ncu, thread_inst_per_launch} of the busiest ncu launch family of a kernel."""
    rows = [units[n] for n in NCU_NAMES.get(key, []) if n in units]
    if not rows:
        return None
    r = max(rows, key=lambda x: x["ncu_us_per_launch"] * x["launches"])
    return {"unit": r["bound_unit"], "frac": r["bound_frac"], "dram_gbs_under_ncu": r["dram_gbs_under_ncu"],
            "units": r["units"], "source": HW_PROFILE + " (ncu, cold cache, not this run)"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="engine", choices=["engine", "reference"])
    p.add_argument("--cpu-views", type=int, default=24,
                   help="views in the bounded CPU-oracle sample (~10-30 s of host work)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-voxel", action="store_true")
    p.add_argument("--no-train", action="store_true")
    p.add_argument("--no-simt-arm", action="store_true",
                   help="skip the FP32 SIMT arm (SCT_K4=simt SCT_K8=simt, a child process at N=1)")
    p.add_argument("--reduction", default="atomic", choices=["deterministic", "atomic"],
                   help="backward reduction: the parallel-atomic mode the north star prescribes (warp/tensor "
                        "pre-reduction, then global atomics per kernel; SPEC.md:224-226), or the reference's "
                        "fixed-order per-pair slots (bitwise repeatable; the engine API's default)")
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def warm_up(step, min_steps, world=1, max_extra=40):
    """Untimed warm-up: at least `min_steps` steps, then more until three
    consecutive steps agree within 5 % (the GPU boxes are VMs whose first
    steps after start-up pay one-off driver costs — memory-pool growth, page
    mapping — of up to tens of ms). Returns the number of warm-up steps run;
    the JSON line reports it. Under torchrun every rank runs the same count
    (decided by rank 0's timings, broadcast)."""
    import torch
    import torch.distributed as dist
    n = 0
    for _ in range(min_steps):
        step()
        n += 1
    times = []
    for _ in range(max_extra):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        n += 1
        done = len(times) >= 3 and (max(times[-3:]) - min(times[-3:])) <= 0.05 * statistics.median(times[-3:])
        if world > 1:
            flag = torch.tensor([1 if done else 0], device="cuda")
            dist.broadcast(flag, 0)
            done = bool(flag.item())
        if done:
            break
    return n


# ------------------------------------------------------------------ workload
def make_workload():
    from paper_2405_20693_b200 import scenes
    w = scenes.CONFIGS[3]
    vol = scenes.phantom(w.n_vox)
    ca = scenes.make_cloud(3, vol=vol)
    thetas = [2.0 * np.pi * i / w.n_views for i in range(w.n_views)]
    return w, ca, thetas, vol


def upstream(n_views, res, views):
    """U(-1,1) upstream gradient per view (seed 2 + view: independent of N)."""
    out = np.empty((len(views), res, res), dtype=np.float32)
    for k, v in enumerate(views):
        out[k] = np.random.default_rng(1000 + v).uniform(-1.0, 1.0, (res, res)).astype(np.float32)
    return out


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock / throttle reasons sampled DURING the timed region by an
    in-process NVML thread (the same counters `nvidia-smi --query-gpu=
    clocks.sm,clocks_event_reasons.*` reads). A looping nvidia-smi process was
    measured to stall this process's driver calls (host syncs) for tens of ms,
    so it is not used."""

    def __init__(self, index, period_s=0.01):
        self.index = index
        self.period = period_s
        self.samples = []
        self.thread = None
        self.stop_flag = False
        self.max_mhz = None

    def start(self):
        import threading
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnosis only: no sampling thread
            self.err = "disabled by BENCH_NO_CLOCKS"
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            return
        self.stop_flag = False

        def loop():
            nv = self.nv
            while not self.stop_flag:
                try:
                    self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(self.period)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: " + getattr(self, "err", "")]}
        nv = self.nv
        try:  # one more sample at the end of the timed region (the thread may have been descheduled)
            self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        except Exception:  # noqa: BLE001
            pass
        self.stop_flag = True
        self.thread.join()
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({n for _, r in self.samples for n, b in bits.items() if r & b})
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "samples": len(sm),
                "min_mhz": min(sm) if sm else None, "reasons": reasons,
                "source": f"NVML, {self.period * 1e3:.0f} ms period"}


# ------------------------------------------------------------------ CPU oracle leg
def cpu_kind():
    """The CPU path timed beside the engine: the reference itself (its unmodified
    sources compiled into oracle/_ref by `make -C oracle ref`; kind "reference")
    when that library is present, else the FP64 restatement (oracle/liborc.so;
    kind "port"). Both run the reference's OpenMP placement on all host threads."""
    from oracle import oracle as O
    if O.ref_available():
        return "reference"
    O.build()
    return "port"


def cpu_oracle_rate(ca, thetas, res, n_views, steps=1):
    """The CPU path (cpu_kind) timed on a bounded sample of the same workload:
    n_views views of render + render_backward. Returns (projections/s, threads,
    seconds, views)."""
    from oracle import oracle as O
    with O.using(cpu_kind()):
        return _cpu_oracle_rate(O, ca, thetas, res, n_views, steps)


def _cpu_oracle_rate(O, ca, thetas, res, n_views, steps):
    O.set_threads(0)
    threads = O.max_threads()
    oc = O.Cloud.from_arrays(ca.s_min, *ca.as_float64())
    cfg = O.test_scanner(res)
    views = list(range(0, len(thetas), max(1, len(thetas) // n_views)))[:n_views]
    ups = upstream(len(thetas), res, views).astype(np.float64)
    done, t0 = 0, time.perf_counter()
    for _ in range(steps):
        for k, v in enumerate(views):
            r = O.render(oc, cfg, thetas[v])
            g = O.Grads.zeros(oc.m)
            O.render_backward(oc, cfg, thetas[v], r, ups[k], g)
            done += 1
    dt = time.perf_counter() - t0
    return done / dt, threads, dt, views


def cpu_voxel_rate(ca, grid, slab=32):
    """voxelize + voxelize_backward on the CPU path (cpu_kind; OpenMP on all
    host threads) on a bounded sample of the cfg4 workload: the same cloud on
    the central z-slab of `slab` voxel layers of the same grid. Returns
    (voxels/s, threads, seconds, sample description)."""
    from oracle import oracle as O
    with O.using(cpu_kind()):
        return _cpu_voxel_rate(O, ca, grid, slab)


def _cpu_voxel_rate(O, ca, grid, slab):
    O.set_threads(0)
    threads = O.max_threads()
    oc = O.Cloud.from_arrays(ca.s_min, *ca.as_float64())
    nx, ny, nz = grid.dims
    z0 = (nz - slab) // 2
    sub = O.GridSpec((nx, ny, slab), (grid.origin_mm[0], grid.origin_mm[1],
                                      grid.origin_mm[2] + z0 * grid.spacing_mm[2]), tuple(grid.spacing_mm))
    up = np.random.default_rng(3).uniform(-1, 1, sub.shape_zyx)
    t0 = time.perf_counter()
    O.voxelize(oc, sub)
    O.voxelize_backward(oc, sub, up, O.Grads.zeros(oc.m))
    dt = time.perf_counter() - t0
    return nx * ny * slab / dt, threads, dt, f"{nx}x{ny}x{slab} central z-slab of the {nx}x{ny}x{nz} grid"


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    w, ca, thetas, vol = make_workload()
    kind = cpu_kind()
    per_step = 1  # one view of render + render_backward per step (bounded sample)
    for _ in range(args.warmup):
        cpu_oracle_rate(ca, thetas, w.res, per_step)
    rate, threads, dt, views = cpu_oracle_rate(ca, thetas, w.res, per_step, steps=args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 (BASELINE configs[2]) " + w.description, "sample": "1 view/step"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{args.steps} steps x 1 view (render+render_backward, fp64, OpenMP)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("the reference's own render / render_backward (its unmodified core sources compiled into "
                 "oracle/_ref with the Eigen / nlohmann::json / libpng build shims, -O3 as its Release build)"
                 if kind == "reference" else
                 "FP64 CPU restatement of the reference (oracle/); oracle/_ref (the compiled reference) is "
                 "not present on this box — see DESIGN.md"),
    }
    if not args.no_voxel:  # the second metric of BASELINE.json on the same CPU path (cfg4, bounded sample)
        from paper_2405_20693_b200 import scenes
        w4 = scenes.CONFIGS[4]
        grid = _grid_for_extent((-1, -1, -1), (1, 1, 1), (w4.n_vox,) * 3)
        vrate, vthreads, vdt, sample = cpu_voxel_rate(scenes.make_cloud(4, vol=vol), grid)
        line["voxelizer"] = {"metric": "voxelized voxels/sec (fwd+bwd)", "value": vrate, "unit": "voxels/s",
                             "cores": vthreads, "kind": kind, "seconds": vdt,
                             "sample": sample + " (voxelize + voxelize_backward, fp64, OpenMP)"}
    print(json.dumps(line), flush=True)


def _grid_for_extent(lo, hi, dims):
    """voxelizer.cpp:8-14 without importing the CUDA package (the reference arm runs the CPU path only)."""
    from oracle import oracle as O
    return O.grid_for_extent(lo, hi, dims)


# ------------------------------------------------------------------ engine arm
def run_engine(args):
    import torch
    import torch.distributed as dist

    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import _capi, dist as pdist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w, ca, thetas, vol = make_workload()
    my_views = pdist.shard_views(len(thetas), rank, world)
    my_thetas = [thetas[v] for v in my_views]
    eng = P.Engine(local, deterministic=(args.reduction == "deterministic"))
    stream = eng.stream
    cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device=dev)
    scanner = P.ScannerConfig(detector_res_px=(w.res, w.res))
    up_host = upstream(len(thetas), w.res, my_views)
    dL = torch.from_numpy(up_host).to(dev)
    grads = P.CloudGrads(cloud.size(), device=dev)
    images = torch.empty((len(my_views), w.res, w.res), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        grads.zero_()
        fwd = eng.render(cloud, scanner, my_thetas, out=images)
        eng.render_backward(cloud, fwd, dL, grads)
        if world > 1:
            pdist.allreduce_grads(grads)
        return fwd

    warmup_run = warm_up(lambda: step().free(), max(3, args.warmup), world)
    torch.cuda.synchronize()
    fwd = step()
    gpe, n_pairs = fwd.work()  # this rank's algorithmic work per step
    fwd.free()
    # sync-free binning (capacity mode): the pair buffers are sized from the measured
    # count, so no step reads a count back to the host; overflow is checked after timing
    capacity = int(n_pairs * 1.02) + 65536
    eng.set_capacity(capacity, 0)
    for _ in range(2):
        step().free()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    e2e_first = None
    if os.environ.get("BENCH_E2E_FIRST") and not args.no_e2e:
        e2e_first = run_e2e(args, eng, ca, scanner, my_thetas, up_host, len(thetas), world, dev)

    sampler = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = eng.kernel_launches()
    eng.set_timing(True)
    sampler.start()
    barrier()
    for k in range(args.steps):
        flush.fill_(float(k))  # evict L2 between timed steps (256 MiB > 126 MB L2), outside the events
        ev[k][0].record(stream)
        f = step()
        ev[k][1].record(stream)
        f.free()
    barrier()
    clocks = sampler.stop()
    if eng.take_overflow():
        raise RuntimeError(f"capacity-mode binning overflowed ({capacity} pair slots)")
    kt = eng.timing_report()
    eng.set_timing(False)
    launches = eng.kernel_launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    print(f"[bench] device per-step ms: {[round(x, 3) for x in step_ms]}", file=sys.stderr)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = len(thetas) * args.steps / (total_ms / 1000.0)

    # --- roofline of the dominant engine kernel (live CUDA-event timing above)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s at the measured max SM clock
    flops_per_gpe = {"K3_composite": 15, "K4_backward_stats": 28}
    engine_k = {k: v for k, v in kt.items() if "(cub)" not in k}
    dom = max(engine_k, key=lambda k: engine_k[k][0])
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps} for k, v in kt.items()}
    rf = None
    for name in ("K3_composite", "K4_backward_stats"):
        ms, n = kt[name]
        ach = flops_per_gpe[name] * gpe / (ms / args.steps / 1000.0) / 1e12  # all launches of a step
        kernels[name]["achieved_tflops"] = ach
        kernels[name]["frac_fp32_peak"] = ach / fp32_peak
    hw = hw_units()
    for name in kernels:
        h = hw_of(hw, name)
        if h:
            kernels[name]["hw"] = {k: v for k, v in h.items() if k != "units"}
    dname = dom if dom in flops_per_gpe else max(flops_per_gpe, key=lambda k: kt[k][0])
    ms, n = kt[dname]
    ach = flops_per_gpe[dname] * gpe / (ms / args.steps / 1000.0) / 1e12
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = prof.get(dname)
    except Exception:
        pass
    rf = {"bound": "fp32", "kernel": dname, "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
          "frac": ach / fp32_peak, "traffic": traffic,
          "peak_source": f"148 SM x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json); "
                         "the SIMT pipes bound these kernels, so neither the copy nor the bf16 GEMM peak applies",
          "algorithmic": f"{flops_per_gpe[dname]} FLOP/GPE x {gpe} GPE per step, all launches of the kernel in a step (SURVEY.md §8d)",
          "dominant_by_time": dom}
    if dname == "K4_backward_stats":
        # K4 runs the moment accumulation (x g, s0, s1, s2: 15 of its 28 FLOP/GPE) as a
        # tensor-core GEMM, so its algorithmic rate can exceed
        # the FP32 peak; the SIMT share (d, Qd, dot, x-1/2, exp: 13 FLOP/GPE) is what
        # the FP32 pipes execute, reported against the same peak.
        simt = 13 * gpe / (ms / args.steps / 1000.0) / 1e12
        rf.update({"simt_achieved": simt, "simt_frac": simt / fp32_peak,
                   "note": "frac is algorithmic (SURVEY.md 8d: 28 FLOP/GPE as if every pixel evaluated the "
                           "quadratic form, an exp and 6 moment FMAs) and exceeds 1 because the kernel executes "
                           "less: E by an exp2 ratio recurrence (2 FMUL per pixel pair per 8-pixel run, one "
                           "MUFU pair per run), the moments as an f16 x f16 -> FP32 GEMM on the tensor pipe "
                           "(mma.sync). The hardware fraction is `hw`: the busiest unit from ncu."})
    h = hw_of(hw, dname)
    if h:
        rf["hw"] = h

    # --- e2e through the host-buffer C ABI
    e2e = e2e_first
    if not args.no_e2e and e2e is None:
        e2e = run_e2e(args, eng, ca, scanner, my_thetas, up_host, len(thetas), world, dev)

    if eng.take_overflow():
        raise RuntimeError(f"capacity-mode binning overflowed in the e2e leg ({capacity} pair slots)")
    eng.set_capacity(0, 0)

    # --- voxelizer (configs[3])
    vox = None if args.no_voxel else run_voxel(args, eng, vol, world, rank, dev)

    # --- full train iteration (configs[1]), one GPU per replica
    train = None if args.no_train or rank != 0 else run_train(args, eng, dev)

    # --- the all-FP32 SIMT arm of K4 / K8 (child process: the variant is fixed per process)
    simt_arm = None
    if rank == 0 and world == 1 and not args.no_simt_arm:
        simt_arm = run_simt_arm(args)

    # --- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, threads, dt, views = cpu_oracle_rate(ca, thetas, w.res, args.cpu_views)
        ck = cpu_kind()
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": ck,
               "sample": f"{len(views)} of the 75 cfg3 views (render+render_backward, fp64, "
                         f"{'the reference compiled from its sources' if ck == 'reference' else 'CPU restatement'}, "
                         f"OpenMP {threads} threads), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warmup_run, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
            "data": "synthetic: Shepp-Logan phantom, sample_init_cloud + anisotropic jitter (seeded), U(-1,1) dL/dI",
            "config": {"workload": "cfg3 (BASELINE configs[2]): " + w.description, "gaussians": ca.m,
                       "views": len(thetas), "detector_px": [w.res, w.res], "pairs_per_step_rank0": n_pairs,
                       "gpe_per_step_rank0": gpe, "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"views sharded over {world} rank(s); NCCL all-reduce of 11*M grads",
                       "reduction": args.reduction,
                       "binning": f"sync-free capacity mode ({capacity} pair slots = 1.02 x measured + 65536; "
                                  "overflow checked after the timed region)"},
            "clocks": clocks, "gpu_launches": launches, "roofline": rf, "kernels": kernels, "e2e": e2e,
            "cpu_baseline": cpu, "voxelizer": vox, "train_step": train,
            "fp32_simt_arm": simt_arm,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_simt_arm(args):
    """The same device-resident cfg3 step (and cfg4 voxel pass) with K4 / K8 in FP32 on the
    SIMT pipes (no binary16 rounding of E): SCT_K4=simt SCT_K8=simt in a child bench."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu", "--no-e2e", "--no-train", "--no-simt-arm",
           "--steps", str(min(args.steps, 5)), "--warmup", "3", "--reduction", args.reduction]
    env = dict(os.environ, SCT_K4="simt", SCT_K8="simt")
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 (reported, not fatal: the main line stands)
        return {"error": str(e)[:200]}
    v = d.get("voxelizer") or {}
    return {"value": d["value"], "unit": UNIT, "ms_per_step": d["ms_per_step"],
            "K4_backward_stats_ms": d["kernels"]["K4_backward_stats"]["ms_per_step"],
            "voxel_value": v.get("value"), "K8_ms": (v.get("kernels") or {}).get("K8_voxel_backward_stats",
                                                                                {}).get("ms_per_step"),
            "parity": "tests/test_gpu_k4_variants.py (simt smoke vs the oracle); FP32 rounding only",
            "env": "SCT_K4=simt SCT_K8=simt", "steps": d["steps"]}


def run_e2e(args, eng, ca, scanner, thetas, up_host, n_total_views, world, dev):
    """Same metric through sct_render_fwd_host / sct_render_bwd_host: pinned host
    cloud, upstream and outputs; H2D/D2H copies inside the timed region."""
    import torch
    import torch.distributed as dist

    from paper_2405_20693_b200 import _capi
    L = _capi.load()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    host = {k: pin(getattr(ca, k)) for k in ("rho_raw", "pos", "scale_raw", "rot")}
    m = ca.m
    cl = _capi.sct_cloud()
    cl.m, cl.s_min_mm = m, ca.s_min
    for k, t in host.items():
        setattr(cl, k, t.data_ptr())
    dL = pin(up_host)
    imgs = torch.empty(up_host.shape, dtype=torch.float32).pin_memory()
    gbuf = torch.zeros(11 * m, dtype=torch.float32).pin_memory()
    gparts = torch.split(gbuf, [m, 3 * m, 3 * m, 4 * m])
    gbuf_bytes = gbuf.numel() * 4
    gview = gbuf.numpy()
    g = _capi.sct_grads()
    for k, t in zip(("rho_raw", "pos", "scale_raw", "rot"), gparts):
        setattr(g, k, t.data_ptr())
    sc = scanner._c()
    import paper_2405_20693_b200 as P
    op = P.RasterOptions()._c()
    th = (C.c_double * len(thetas))(*thetas)
    gdev = torch.empty(11 * m, dtype=torch.float32, device=dev)

    calls = []

    def step():
        C.memset(gbuf.data_ptr(), 0, gbuf_bytes)  # CloudGrads::resize (trainer.cpp:283), no torch CPU op
        st = C.c_void_p()
        t0 = time.perf_counter()
        rc = L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, len(thetas), C.byref(op),
                                   C.c_void_p(imgs.data_ptr()), C.byref(st))
        assert rc == 0, L.sct_last_error()
        t1 = time.perf_counter()
        rc = L.sct_render_bwd_host(eng._h, st, C.byref(cl), C.c_void_p(dL.data_ptr()), C.byref(g), None)
        assert rc == 0, L.sct_last_error()
        calls.append((round(1e3 * (t1 - t0), 1), round(1e3 * (time.perf_counter() - t1), 1)))
        L.sct_fwd_free(st)
        if world > 1:
            gdev.copy_(gbuf, non_blocking=True)
            dist.all_reduce(gdev)
            gbuf.copy_(gdev)
        return float(gview[0])  # the step's result read on the host

    warm_up(step, max(3, args.warmup), world)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    per = []
    for _ in range(args.steps):
        ts = time.perf_counter()
        step()
        per.append(1e3 * (time.perf_counter() - ts))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"[bench] e2e per-step ms: {[round(x, 2) for x in per]}", file=sys.stderr)
    print(f"[bench] e2e (fwd_host, bwd_host) ms: {calls[-args.steps:]}", file=sys.stderr)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    cloud_b = 11 * m * 4
    h2d = 2 * cloud_b + up_host.nbytes + 11 * m * 4  # cloud (fwd + bwd), dL/dI, running grads
    d2h = imgs.numel() * 4 + 11 * m * 4
    if world > 1:
        h2d += 11 * m * 4
        d2h += 11 * m * 4
    res = {"value": n_total_views * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "path": "C-ABI sct_render_fwd_host + sct_render_bwd_host (pinned host)",
           "ms_per_step": 1000.0 * dt / args.steps}
    if world == 1:
        # the reference trainer's granularity: one render + render_backward call per view
        # (trainer.cpp:276-288), each call re-uploading the cloud (pageable-free: pinned)
        def one_view(v):
            C.memset(gbuf.data_ptr(), 0, gbuf_bytes)
            st = C.c_void_p()
            th1 = (C.c_double * 1)(thetas[v])
            img1 = C.c_void_p(imgs.data_ptr() + v * imgs[0].numel() * 4)
            rc = L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th1, 1, C.byref(op), img1, C.byref(st))
            assert rc == 0, L.sct_last_error()
            rc = L.sct_render_bwd_host(eng._h, st, C.byref(cl), C.c_void_p(dL.data_ptr() + v * dL[0].numel() * 4),
                                       C.byref(g), None)
            assert rc == 0, L.sct_last_error()
            L.sct_fwd_free(st)
            return float(gview[0])

        for v in range(min(8, len(thetas))):
            one_view(v)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for v in range(len(thetas)):
            one_view(v)
        torch.cuda.synchronize()
        dtv = time.perf_counter() - t0
        res["per_view_calls"] = {
            "value": len(thetas) / dtv, "unit": UNIT, "ms_per_view": 1000.0 * dtv / len(thetas),
            "h2d_bytes_per_view": int(2 * cloud_b + up_host[0].nbytes + 11 * m * 4),
            "d2h_bytes_per_view": int(up_host[0].nbytes + 11 * m * 4),
            "path": "one sct_render_fwd_host + sct_render_bwd_host call per view (trainer.cpp:276-288 granularity; "
                    "the C++ drop-in include/splatct_b200.hpp render/render_backward make exactly these calls)"}
    return res


def run_train(args, eng, dev):
    """configs[1]: 128^3 phantom cloud (50k Gaussians), 50 views at 256^2; one
    iteration = render 1 view + L1/D-SSIM + render_backward (with adaptive
    stats) + TV on a 32^3 sub-grid at the 128^3 output spacing + Adam
    (trainer.cpp:268-319). Measured projections: the cloud rendered with
    perturbed densities (synthetic stand-in for simulate_projections)."""
    import torch

    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import scenes
    from paper_2405_20693_b200.train import NativeTrainer, TrainConfig
    w = scenes.CONFIGS[2]
    ca = scenes.make_cloud(2)
    angles = P.full_circle_angles(w.n_views)
    sc = P.ScannerConfig(detector_res_px=(w.res, w.res))
    rng = np.random.default_rng(7)
    target = P.GaussianCloud(ca.s_min, ca.rho_raw + rng.normal(0, 0.3, ca.m).astype(np.float32), ca.pos,
                             ca.scale_raw, ca.rot, device=dev)
    f = eng.render(target, sc, angles)
    meas = f.images.clone()
    f.free()
    cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device=dev)
    cfg = TrainConfig(iters=1000, output_dims=(w.n_vox,) * 3, tv_grid_dim=32, check_every=0, sync_free=True)
    # the reference's train() loop entirely in the engine library (sct_trainer_*):
    # equal to train.py's Trainer bitwise (tests/test_gpu_train.py)
    tr = NativeTrainer(eng, cloud, sc, angles, meas, cfg)
    warm_up(tr.step, max(3, args.warmup))
    n = max(10, args.steps)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.kernel_launches()
    a.record(eng.stream)
    for _ in range(n):
        tr.step()
    b.record(eng.stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    out = tr.record()
    if eng.take_overflow():
        raise RuntimeError("train step: sync-free binning overflowed its capacity")
    eng.set_capacity(0, 0)
    return {"metric": "train iterations/sec", "value": 1000.0 / ms, "unit": "iters/s", "ms_per_iter": ms,
            "workload": "cfg2 (BASELINE configs[1]): " + w.description, "iters": n,
            "last_total_loss": float(out["total"]), "engine_launches_per_iter": (eng.kernel_launches() - launches0) / n,
            "loop": "native (sct_trainer_step: view shuffle, sub-grid draw, sct_train_step, adaptive control)",
            "binning": "sync-free (TrainConfig.sync_free: capacity from a calibration iteration, overflow "
                       "checked after the timed region)",
            "note": "1 view per iteration as trainer.cpp:268-276; context: the paper's RTX 3090 CUDA code "
                    "runs ~15.5 ms/iter (PAPER.md:211, derived)",
            "hw": {k: hw_of(hw_units(), k) for k in ("K9_tv3d", "K10_adam", "K11_ssim", "AC_adaptive")}}


def run_voxel(args, eng, vol, world, rank, dev):
    """configs[3]: 200k Gaussians, 256^3 grid, voxelize + voxelize_backward per step,
    z-slab sharded (pair-balanced) with an all-reduce of the partial gradients."""
    import torch
    import torch.distributed as dist

    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import dist as pdist, scenes
    w = scenes.CONFIGS[4]
    ca = scenes.make_cloud(4, vol=vol)
    cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device=dev)
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (w.n_vox,) * 3)
    nl = (w.n_vox + 7) // 8
    # balance the slabs by kernel count per brick layer (the phantom occupancy is ellipsoidal)
    zc = ca.pos.reshape(-1, 3)[:, 2]
    layer = np.clip(((zc - grid.origin_mm[2]) / grid.spacing_mm[2] // 8).astype(np.int64), 0, nl - 1)
    zb = pdist.shard_z_bricks(nl, rank, world, list(np.bincount(layer, minlength=nl).astype(float) + 1.0))
    vge, pairs = eng.voxel_work(cloud, grid)
    out = torch.zeros(grid.shape_zyx, dtype=torch.float32, device=dev)
    up = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, grid.shape_zyx).astype(np.float32)).to(dev)
    grads = P.CloudGrads(cloud.size(), device=dev)

    def step():
        grads.zero_()
        # one binning shared by the forward and the backward (VoxelState)
        _, vs = eng.voxelize(cloud, grid, z_bricks=zb, out=out, keep_state=True)
        eng.voxelize_backward(cloud, grid, up, grads, z_bricks=zb, state=vs)
        vs.free()
        if world > 1:
            pdist.allreduce_grads(grads)

    warm_up(step, max(3, args.warmup), world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    eng.set_timing(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(eng.stream)
        step()
        ev[k][1].record(eng.stream)
    torch.cuda.synchronize()
    kt = eng.timing_report()
    eng.set_timing(False)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    fp32_peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    kern = {k: {"ms_per_step": v[0] / args.steps} for k, v in kt.items()}
    for name, fl in (("K7_voxel_eval", 27), ("K8_voxel_backward_stats", 51)):
        if name in kt and world == 1:
            ms, n = kt[name]
            ach = fl * vge / (ms / args.steps / 1000.0) / 1e12
            kern[name]["achieved_tflops"] = ach
            kern[name]["frac_fp32_peak"] = ach / fp32_peak
    hw = hw_units()
    for name in kern:
        h = hw_of(hw, name)
        if h:
            kern[name]["hw"] = {k: v for k, v in h.items() if k != "units"}
    res = {"metric": "voxelized voxels/sec (fwd+bwd)", "value": grid.voxel_count() * args.steps / (total_ms / 1e3),
           "unit": "voxels/s", "ms_per_step": total_ms / args.steps,
           "workload": "cfg4 (BASELINE configs[3]): " + w.description, "vge_per_pass": vge, "pairs": pairs,
           "kernels": kern}
    if world == 1:
        # voxelize alone (SURVEY.md §8d reports both rates)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        for _ in range(args.steps):
            eng.voxelize(cloud, grid, out=out)
        e1.record(eng.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        res["fwd_only"] = {"value": grid.voxel_count() / (ms / 1e3), "unit": "voxels/s", "ms_per_step": ms}
        if rank == 0 and not args.no_cpu:
            rate, threads, dt, sample = cpu_voxel_rate(ca, grid)
            res["cpu_baseline"] = {"value": rate, "unit": "voxels/s", "cores": threads, "kind": cpu_kind(),
                                   "sample": f"{sample} (voxelize + voxelize_backward, fp64, OpenMP), "
                                             f"{dt:.1f} s"}
    return res


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
