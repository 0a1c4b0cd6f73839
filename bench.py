#!/usr/bin/env python
"""Benchmark of the eRTIS image-formation hot path (Workspace::process).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Metric (BASELINE.json): energyscapes/s, 32-mic, 3D hemisphere grid
(hemisphere3000, 3000 directions x 655 range bins, 5 m window = 144,800 PDM
frames per capture) — BASELINE.json configs[1]. A "step" is one pass of the
hot path over a batch of B captures per GPU; `value` = captures processed by
all ranks / max-over-ranks device time (CUDA events on the launching stream).
Inputs cycle through a pool of distinct synthetic captures whose total size
exceeds the 126 MB L2, so no step re-reads cached inputs.

Extra keys: `e2e` (same metric through the public host API with pinned host
buffers: H2D of every capture + D2H of every energyscape inside the timed
region), `latency_ms` (single-capture p50/p99), `roofline` (dominant kernel
k_directions, algorithmic FLOPs per SURVEY.md §8(d) / its CUDA-event
duration, against the FP64 FMA peak measured live on this GPU),
`cpu_baseline` (the unmodified reference C++ core, oracle/_ref, on all host
cores, rank 0 at N=1 only), `clocks`, `gpu_launches`.

Multi-GPU (torchrun): one sensor per rank (serial = rank+1), no data-path
collective (scaling "weak"); --gather adds the NCCL 360-degree energyscape
gather to rank 0 inside each step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "energyscapes/sec (32-mic, 3D grid) at 1/2/4/8 B200 + p50 latency vs CPU ref"
UNIT = "energyscapes/s"
BENCH_SCENE = [(1.5, 0.2, 0.0, 0.8), (3.0, -0.4, 0.1, 0.5)]  # bench.cpp:113-117
GRIDS = {"horizontal90": 0, "box1850": 1, "hemisphere3000": 2, "az181": 3}
# dense int8 tensor throughput of one B200 (2 ops per MAC): nominal 4.5 POPS;
# scripts/micro/mma_rate.cu measured 4.49-4.58 POPS for M=128 x N=256 x K=32
# tcgen05 kind::i8 on this pool (the M=128, N=64 shape the beamformer issues
# is capped at ~2.9-3.0 POPS by the ~50-cycle per-instruction floor)
TC_INT8_PEAK = 4500.0
# the reference links FFTW3 (core/CMakeLists.txt:3), which this image lacks:
# the CPU reference runs with a test-only radix-2 FFTW-API stand-in
# (oracle/fftw_shim), slower than FFTW on the FFT-bound stages, so GPU/CPU
# ratios overstate the gap to a real-FFTW build by an unknown factor
E2E_BLOCKS = 8  # device batches per host-API call in the e2e leg
FFT_LABEL = "radix2-shim (oracle/fftw_shim; FFTW3 absent from the image)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--grid", choices=list(GRIDS), default="hemisphere3000")
    p.add_argument("--batch", type=int, default=16, help="captures per step per GPU")
    p.add_argument("--pool", type=int, default=256, help="distinct captures per GPU")
    p.add_argument("--precision", choices=["f64", "f32"], default="f64")
    p.add_argument("--gather", action="store_true", help="NCCL 360-degree gather per step")
    p.add_argument("--latency-samples", type=int, default=50)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-calls", type=int, default=8, help="reference calls per host thread (~5-10 s of CPU work)")
    p.add_argument("--stream-frames", type=int, default=2048,
                   help="frames of the 8-sensor streaming run through the worker pool (configs[3]: 256 "
                        "measurements x 8 sensors; 0: skip)")
    p.add_argument("--paced-frames", type=int, default=256,
                   help="frames of the paced (10 Hz per sensor) latency sample")
    p.add_argument("--cpu-latency-calls", type=int, default=20,
                   help="timed reference process() calls per latency leg (bench.cpp:63-108 uses 100)")
    p.add_argument("--no-sweep", action="store_true", help="skip the configs[4] grid x window sweep")
    p.add_argument("--sweep-steps", type=int, default=3)
    p.add_argument("--only-sweep", action="store_true", help="developer: print the sweep alone")
    p.add_argument("--lib", default=None, help="developer A/B: another build of libsonarnet_b200.so")
    p.add_argument("--tc-tile-n", type=int, default=0, help="developer: tensor-core tile width (0: default)")
    return p.parse_args()


# ---------------------------------------------------------------------------
def flops_per_energyscape(d):
    """Algorithmic FLOPs (SURVEY.md §8(d) conventions: MAC=2, add=1, real FFT
    of N = 2.5 N log2 N, complex multiply = 6, sqrt = 1)."""
    import math
    L, N, bins, comp = d["mf_samples"], d["env_fft_size"], d["range_bins"], d["smoothing_len"]
    Nm, ref = d["mf_fft_size"], d["ref_len"]
    demod = 32 * d["demod_samples"] * 255 * 2
    premf = 32 * L * 65 * 2
    mf = 32 * (2 * 2.5 * Nm * math.log2(Nm) + 6 * (Nm // 2 + 1))
    per_dir = (32 * L + L) + 2 * 2.5 * N * math.log2(N) + 4 * L + bins * comp * 2
    return demod + premf + mf, per_dir


def kernel_flops(d):
    """Algorithmic FLOPs per energyscape for each device kernel."""
    import math
    L, N, bins, comp = d["mf_samples"], d["env_fft_size"], d["range_bins"], d["smoothing_len"]
    Nm, n = d["mf_fft_size"], d["n_directions"]
    return {
        "demod": 32 * d["demod_samples"] * 255 * 2,
        "premf": 32 * L * 65 * 2,
        "matched_filter": 32 * (2 * 2.5 * Nm * math.log2(Nm) + 6 * (Nm // 2 + 1)),
        "beamform": n * (32 * L + L),
        "envelope": n * (2 * 2.5 * N * math.log2(N) + 4 * L + bins * comp * 2),
    }


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_config(sn, grid, precision):
    if grid == "az181":
        az = np.deg2rad(np.arange(-90, 91, dtype=np.float64))
        cfg = sn.default_pipeline_config(sn.GridKind.horizontal90)
        cfg = cfg.copy(directions=np.stack([az, np.zeros_like(az)], 1), grid_kind=3)
    else:
        cfg = sn.default_pipeline_config(GRIDS[grid])
    return cfg.copy(precision=0 if precision == "f64" else 1)


def synth_pool(sn, cfg, serial, n):
    """n distinct captures (seed = 7 + 1000*serial + seq)."""
    def one(seq):
        scene = sn.Scene([sn.Reflector(*r) for r in BENCH_SCENE], 0.01, 7 + 1000 * serial + seq)
        return sn.synthesize_measurement(cfg, scene, serial, seq * 100000, seq).packed
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        return np.stack(list(ex.map(one, range(n))))


def workload_desc(grid, d, B, pool):
    return {
        "workload": (f"1 eRTIS sensor per GPU, 32 mics, {grid} ({d['n_directions']} directions x "
                     f"{d['range_bins']} range bins), 5 m window = {d['frames']} PDM frames/capture"),
        "grid": grid, "n_directions": d["n_directions"], "range_bins": d["range_bins"],
        "frames": d["frames"], "batch_per_gpu": B, "pool_per_gpu": pool,
        "l2_policy": f"inputs cycle through {pool} distinct captures "
                     f"({pool * d['frames'] * 4 / 1e6:.0f} MB > 126 MB L2)",
    }


# ---------------------------------------------------------------------------
def cpu_baseline(cfg_b200, grid, calls, warmup=1):
    """Reference C++ core (oracle/_ref, reference Release flags) on all host
    threads: one Workspace per thread, processing_threads=1 (central-node
    model, central_node.cpp:48-53)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    ref = po.Ref(fast=True)
    kind = 0 if grid == "az181" else GRIDS[grid]
    rc = ref.default_config(kind)
    if grid == "az181":
        rc = rc.copy(directions=po.az181_directions(), grid_kind=3)
    rc = rc.copy(processing_threads=1)
    pool = np.stack([ref.synthesize(rc, BENCH_SCENE, 0.01, 7 + s) for s in range(4)])
    threads = os.cpu_count() or 1
    if warmup > 1:
        ref.throughput(rc, pool, threads, warmup - 1)  # untimed; the timed run warms up once more
    elapsed, total = ref.throughput(rc, pool, threads, calls)
    n_dirs = len(po.az181_directions()) if grid == "az181" else po.GRID_SIZES[kind]
    try:
        fc = fft_check(threads * elapsed / total / n_dirs * 1e6)
    except Exception as e:  # diagnostic only
        fc = {"error": str(e)}
    return {
        "value": total / elapsed, "unit": UNIT, "cores": threads, "kind": "reference",
        "fft": FFT_LABEL, "fft_check": fc,
        "sample": (f"{total} process() calls of {grid} ({threads} threads x {calls}; "
                   f"unmodified reference core built -O3 -march=x86-64-v3, FFT = test-only "
                   f"FFTW-API shim; {elapsed:.2f} s wall)"),
    }


def fft_check(per_dir_us, reps=300):
    """How much the test-only FFT shim can inflate the reference's time: the
    shim's r2c of 8192 reals (the envelope's transform size) against numpy's
    pocketfft on this host, and the share of the reference's per-direction
    time its FFT pair (r2c + c2r) takes -- a reference on a zero-cost FFT
    would be at most 1 / (1 - share) faster."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    lib = C.CDLL(po.REF_FAST_SO)
    lib.fftw_alloc_real.restype = C.c_void_p
    lib.fftw_alloc_complex.restype = C.c_void_p
    lib.fftw_plan_dft_r2c_1d.restype = C.c_void_p
    lib.fftw_plan_dft_r2c_1d.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint]
    lib.fftw_plan_dft_c2r_1d.restype = C.c_void_p
    lib.fftw_plan_dft_c2r_1d.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint]
    lib.fftw_execute.argtypes = [C.c_void_p]
    lib.fftw_destroy_plan.argtypes = [C.c_void_p]
    lib.fftw_free.argtypes = [C.c_void_p]
    n = 8192
    ip, op = lib.fftw_alloc_real(n), lib.fftw_alloc_complex(n // 2 + 1)
    x = np.ctypeslib.as_array(C.cast(ip, C.POINTER(C.c_double)), (n,))
    x[:] = np.random.default_rng(1).standard_normal(n)
    fwd = lib.fftw_plan_dft_r2c_1d(n, ip, op, 0)
    inv = lib.fftw_plan_dft_c2r_1d(n, op, ip, 0)
    times = []
    for plan in (fwd, inv):
        lib.fftw_execute(plan)
        t = time.perf_counter()
        for _ in range(reps):
            lib.fftw_execute(plan)
        times.append((time.perf_counter() - t) / reps * 1e6)
    xx = np.random.default_rng(1).standard_normal(n)
    np.fft.rfft(xx)
    t = time.perf_counter()
    for _ in range(reps):
        np.fft.rfft(xx)
    t_np = (time.perf_counter() - t) / reps * 1e6
    for plan in (fwd, inv):
        lib.fftw_destroy_plan(plan)
    lib.fftw_free(ip)
    lib.fftw_free(op)
    share = min(1.0, (times[0] + times[1]) / per_dir_us)
    return {"shim_r2c_8192_us": round(times[0], 1), "shim_c2r_8192_us": round(times[1], 1),
            "numpy_pocketfft_rfft_8192_us": round(t_np, 1),
            "reference_us_per_direction_per_thread": round(per_dir_us, 1),
            "fft_pair_share": round(share, 3),
            "zero_cost_fft_bound": round(1.0 / max(1e-9, 1.0 - share), 2),
            "note": "shim single-thread timings while no other work runs; the per-direction time is "
                    "threads / (throughput x directions) from the throughput run (shared cores)"}


def cpu_latency(grid, n):
    """Reference single-measurement latency, the protocol of
    bench::run_benchmark (bench.cpp:63-108): one Workspace with
    processing_threads = 2 (the default, pipeline.hpp:33-36) and = nproc,
    1 warm-up + n timed process() calls (steady_clock)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    ref = po.Ref(fast=True)
    kind = 0 if grid == "az181" else GRIDS[grid]
    rc = ref.default_config(kind)
    if grid == "az181":
        rc = rc.copy(directions=po.az181_directions(), grid_kind=3)
    pk = ref.synthesize(rc, BENCH_SCENE, 0.01, 7)
    out = {"protocol": f"bench.cpp:63-108: 1 warm-up + {n} timed process() calls per leg",
           "fft": FFT_LABEL, "unit": "ms"}
    nproc = os.cpu_count() or 1
    for name, th in (("threads_2", 2), ("threads_nproc", nproc)):
        ws = ref.workspace(rc.copy(processing_threads=th))
        d = ws.latency(pk, n)
        out[name] = {"threads": th, "n": n, "p50": float(np.percentile(d, 50)),
                     "p99": float(np.percentile(d, 99)), "mean": float(np.mean(d)), "min": float(np.min(d))}
        del ws
    return out


def run_reference(args):
    """Reference arm: the reference's own CPU implementation (oracle/_ref,
    unmodified core sources) on all host threads of this box. One step = every
    host thread runs one process() call on its own Workspace; K is capped at
    30 steps and W at 5 so the arm stays within a few minutes at
    hemisphere3000."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = max(1, min(args.steps, 30))
    warmup = max(1, min(args.warmup, 5))
    base = cpu_baseline(None, args.grid, steps, warmup)
    threads = base["cores"]
    line = {
        "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup,
        "ms_per_step": 1e3 * threads / base["value"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synthesize_measurement, bench scene, seeds 7..10)",
        "config": {"workload": f"1 eRTIS sensor, 32 mics, {args.grid}, 5 m window = 144800 PDM "
                               f"frames/capture; reference CPU path, {threads} workers x 1 thread",
                   "grid": args.grid},
        "impl": "reference", "cpu_baseline": base, "fft": FFT_LABEL,
        "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
SWEEP_GRIDS = ("horizontal90", "az181", "box1850", "hemisphere3000", "fib10k", "fib30k")
SWEEP_RANGES = (1.5, 5.0, 10.0)


def sweep_config(sn, grid, max_range, precision):
    """configs[4] points: the built-in grids, az181, and Fibonacci hemispheres
    of 10k / 30k directions (geometry.cpp:206-229 with n free), at a window
    of max_range metres (frames / FFT sizes / bins per pipeline.cpp:40-52)."""
    if grid.startswith("fib"):
        n = int(grid[3:-1]) * 1000
        cfg = sn.default_pipeline_config(sn.GridKind.horizontal90).copy(
            directions=sn.fibonacci_hemisphere(n), grid_kind=3)
        cfg = cfg.copy(precision=0 if precision == "f64" else 1)
    else:
        cfg = make_config(sn, grid, precision)
    return cfg.copy(max_range=max_range)


def sweep(sn, args, local, peak):
    """BASELINE configs[4]: direction grid x recording length on this GPU
    (N=1; one sensor per GPU at N>1 is the same per-GPU work, scaling weak).
    Per point: B captures per step (B = 16 scaled down so a step's beams stay
    near the default's), GPU-synthesised inputs, 1 warm-up + K timed steps on
    the device path (CUDA events), then one profiled step for the stage
    shares; `frac` = the envelope stage's algorithmic FLOPs
    / its time / the live FP64 (or FP32) FMA peak."""
    import torch
    pts = []
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    for grid in SWEEP_GRIDS:
        for mr in SWEEP_RANGES:
            cfg = sweep_config(sn, grid, mr, args.precision)
            d = cfg.dims()
            n, N = d["n_directions"], d["env_fft_size"]
            B = int(max(1, min(16, round(16 * 3000 * 8192 / (n * N)))))
            t0 = time.perf_counter()
            ws = sn.Workspace(cfg, device=local, max_batch=B)
            setup_s = time.perf_counter() - t0
            scenes = [sn.Scene([sn.Reflector(*r) for r in BENCH_SCENE[:1 if mr < 2 else 2]], 0.01, 7 + k)
                      for k in range(2 * B)]
            pin = torch.empty(2 * B * ws.packed_bytes, dtype=torch.uint8, device=dev)
            sn.synthesize_device(cfg, scenes, pin.data_ptr(), device=local)
            out = torch.empty((B, ws.n_dirs, ws.bins), dtype=torch.float32, device=dev)
            sp = stream.cuda_stream

            def step(k):
                ws.process_device(pin.data_ptr() + (k % 2) * B * ws.packed_bytes, B, out.data_ptr(), sp)

            with torch.cuda.stream(stream):
                step(1)
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for k in range(args.sweep_steps):
                    step(k)
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / args.sweep_steps
                ws.set_profiling(True)
                step(0)
                stream.synchronize()
                st = ws.stage_times()
                ws.set_profiling(False)
            kf = kernel_flops(ws.dims)
            env_tf = kf["envelope"] * B / (st["envelope"] * 1e-3) / 1e12
            pts.append({
                "grid": grid, "n_directions": n, "max_range_m": mr, "frames": d["frames"], "env_fft": N,
                "range_bins": d["range_bins"], "batch": B, "value": B / (ms * 1e-3), "unit": UNIT,
                "ms_per_capture": ms / B, "stage_ms_per_capture": {k: v / B for k, v in st.items()},
                "envelope_frac": env_tf / peak, "setup_s": setup_s,
            })
            del ws, pin, out
            torch.cuda.empty_cache()
    return {"points": pts, "steps": args.sweep_steps,
            "what": "device path (sn_workspace_process_device), GPU-synthesised captures (sn_synthesize_device); "
                    "frac: envelope stage vs the live FMA peak"}


def stream_bench(sn, cfg, ws, pool_h, args, L, C):
    """BASELINE configs[3]: 8 sensors (serials 1..8) x N/8 time-synchronised
    measurements (default 256 x 8) as wire frames through sn_pool (2 workers
    x max_batch 8 on one GPU): sustained throughput unthrottled, then
    per-frame latency (submit -> released) at the 10 Hz-per-sensor rate
    (80 frames/s offered) over a bounded paced sample."""
    n = args.stream_frames
    frames = []
    for k in range(n):
        serial, t = 1 + k % 8, k // 8
        frames.append(sn.measurement_frame(sn.RawMeasurement(serial, 100000 * t, t, 32, ws.frames, cfg.pdm_rate,
                                                             pool_h[k % len(pool_h)])))
    pool = sn.CentralPool(cfg, devices=[0], workers_per_device=2, max_batch=8)
    ptr, nl, st, ser, sq = C.c_void_p(), C.c_uint64(0), C.c_int32(0), C.c_uint32(0), C.c_uint64(0)

    def poll():  # zero-copy view of the released frame (valid until the next poll)
        rc = L.sn_pool_poll_view(pool._h, 60000, C.byref(ptr), C.byref(nl), C.byref(st), C.byref(ser), C.byref(sq))
        if rc != 0 or st.value != 0:
            raise RuntimeError(f"pool poll rc={rc} status={st.value}")

    import threading
    for f in frames[:16]:  # warm-up
        pool.submit(f)
    for _ in range(16):
        poll()
    t0 = time.perf_counter()
    feeder = threading.Thread(target=lambda: [pool.submit(f) for f in frames])
    feeder.start()
    for _ in range(n):
        poll()
    feeder.join()
    sustained = n / (time.perf_counter() - t0)
    # paced: 80 frames/s offered; latency = release time - submit time
    paced_n = args.paced_frames
    sub_t = {}
    done = []

    def paced_feed():
        start = time.perf_counter()
        for k in range(paced_n):
            target = start + k / 80.0
            while time.perf_counter() < target:
                time.sleep(0.0005)
            sub_t[(1 + k % 8, 1000 + k // 8)] = time.perf_counter()
            m = sn.RawMeasurement(1 + k % 8, 0, 1000 + k // 8, 32, ws.frames, cfg.pdm_rate, pool_h[k % len(pool_h)])
            pool.submit(sn.measurement_frame(m))

    feeder = threading.Thread(target=paced_feed)
    feeder.start()
    for _ in range(paced_n):
        poll()
        done.append(((ser.value, sq.value), time.perf_counter()))
    feeder.join()
    lat = [(t - sub_t[key]) * 1e3 for key, t in done]
    pool.close()
    return {"frames": n, "measurements_per_sensor": n // 8, "sensors": 8, "workers": 2, "max_batch": 8,
            "sustained_value": sustained, "unit": UNIT,
            "paced_offered_per_s": 80, "paced_frames": paced_n,
            "latency_ms_p50": float(np.percentile(lat, 50)), "latency_ms_p99": float(np.percentile(lat, 99)),
            "what": "wire frames in (CRC on GPU) -> sn_pool (per-sensor FIFO) -> processed-image frames out "
                    "(zero-copy view of the page-locked result); the paced frame is built on the host inside "
                    "the latency window"}


def run_b200(args):
    import torch
    import paper_2208_10839_b200 as sn
    if args.lib:
        sn.load_library(args.lib)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    if args.only_sweep:
        torch.cuda.set_device(local)
        peak = sn.measure_fp_peak(local, sn.Precision.f64 if args.precision == "f64" else sn.Precision.f32)
        print(json.dumps({"sweep": sweep(sn, args, local, peak)}), flush=True)
        return 0
    cfg = make_config(sn, args.grid, args.precision)
    B = args.batch
    pool_n = max(B, (args.pool // B) * B)
    ws = sn.Workspace(cfg, device=local, max_batch=B, tc_tile_n=args.tc_tile_n)
    d = ws.dims
    serial = rank + 1
    pool_h = synth_pool(sn, cfg, serial, pool_n)
    pool = torch.from_numpy(pool_h).to(dev)
    outs = [torch.empty((B, ws.n_dirs, ws.bins), dtype=torch.float32, device=dev) for _ in range(2)]
    out = outs[0]
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    nchunks = pool_n // B

    # 360-degree view (configs[2]): the C++ NCCL gather (sn_gather_*) of every
    # step's energyscapes to rank 0 on its own stream, double-buffered: step
    # k writes outs[k % 2] while step k - 1's gather reads the other slot
    vg, views = None, None
    if dist is not None and args.gather:
        from paper_2208_10839_b200.distributed import ViewGather
        vg = ViewGather(ws.n_dirs * ws.bins, B, device=local)
        if rank == 0:
            views = [torch.empty((world, B, ws.n_dirs, ws.bins), dtype=torch.float32, device=dev)
                     for _ in range(2)]

    def step(k):
        src = pool[(k % nchunks) * B]
        slot = k % 2
        if vg is not None:
            vg.wait(slot, sptr)  # the slot's previous gather has read outs[slot]
        ws.process_device(src.data_ptr(), B, outs[slot].data_ptr(), sptr)
        if vg is not None:
            ids = [(serial, 100000 * k, k)] * B  # one trigger per step (sync.hpp:16-19)
            vg.start(slot, outs[slot].data_ptr(), ids, views[slot].data_ptr() if rank == 0 else 0, sptr)

    # ---- warm-up ----------------------------------------------------------
    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step(k)
    torch.cuda.synchronize(dev)

    # ---- device-resident timed region ---------------------------------------
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for k in range(args.steps):
                step(k)
            if vg is not None:  # the last steps' gathers belong to the timed region
                for sl in range(2):
                    vg.wait(sl, sptr)
            e1.record(stream)
        torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    gather_res = None
    if vg is not None:
        gather_res = {"ms_last": [vg.elapsed_ms(sl) for sl in range(2)],
                      "bytes_to_root_per_step": (world - 1) * B * ws.n_dirs * ws.bins * 4,
                      "what": "sn_gather (C++ NCCL send/recv to rank 0, own stream, double-buffered view slots)"}
        if rank == 0:
            ids, ok = vg.ids((args.steps - 1) % 2)
            gather_res["triggers_synchronized"] = ok
    launches = ws.last_launches() * args.steps
    if dist is not None:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    value = world * args.steps * B / (elapsed_ms / 1e3)

    # ---- e2e through the public host API (pinned buffers) ---------------------
    # one call = E2E_BLOCKS device batches (sn_workspace_process_batch with
    # E2E_BLOCKS x B captures): the blocks of a call pipeline into each other
    # (upload + front end of block j + 1 under block j's envelope/downloads)
    EB = E2E_BLOCKS * B
    pin_in = torch.from_numpy(pool_h[: EB]).pin_memory()
    pin_out = torch.empty((EB, ws.n_dirs, ws.bins), dtype=torch.float32).pin_memory()
    pin_in_np, pin_out_np = pin_in.numpy(), pin_out.numpy()
    for k in range(max(1, args.warmup // 2)):
        ws.process_packed_host(pin_in_np, pin_out_np)
    if dist is not None:
        dist.barrier()
    e2e_steps = max(8, args.steps // 4)  # >= 1024 captures: stable to ~1% box to box
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        ws.process_packed_host(pin_in_np, pin_out_np)
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * e2e_steps * EB / e2e_s

    # ---- wire path: raw-measurement frames in, processed-image frames out ------
    # (the central node's traffic: CRC-checked on the GPU, AIMG frames encoded
    # and CRC'd on the GPU; sn_workspace_process_frames; pinned host buffers;
    # EB frames per call, whose device batches pipeline into each other like
    # the e2e leg's)
    import ctypes as C
    del pin_in, pin_out, pin_in_np, pin_out_np
    L = sn.lib()
    slot = ws.image_frame_bytes
    WF = EB
    fr = [sn.measurement_frame(sn.RawMeasurement(serial, k, k, 32, ws.frames, cfg.pdm_rate, pool_h[k % pool_n]))
          for k in range(2 * WF)]
    flen = len(fr[0])
    fin = torch.empty((2 * WF, flen), dtype=torch.uint8).pin_memory()
    fin_np = fin.numpy()
    for k in range(2 * WF):
        fin_np[k] = np.frombuffer(fr[k], np.uint8)
    del fr
    fout = torch.empty((WF, slot), dtype=torch.uint8).pin_memory()
    ptrs = [(C.c_void_p * WF)(*[fin_np[h * WF + i].ctypes.data for i in range(WF)]) for h in range(2)]
    lens = (C.c_uint64 * WF)(*([flen] * WF))
    olen, ost = (C.c_uint64 * WF)(), (C.c_int32 * WF)()
    fout_ptr = fout.numpy().ctypes.data

    def wire_step(k):
        rc = L.sn_workspace_process_frames(ws._h, ptrs[k % 2], lens, WF, fout_ptr, slot, olen, ost)
        if rc != 0 or any(ost[i] != 0 for i in range(WF)):
            raise RuntimeError(f"process_frames failed: rc={rc} status={list(ost)}")

    for k in range(max(1, min(args.warmup, 2))):
        wire_step(k)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        wire_step(k)
    wire_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([wire_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wire_s = float(t.item())
    wire_value = world * e2e_steps * WF / wire_s
    del fin, fin_np, fout

    # ---- streaming through the GPU-backed worker pool (BASELINE configs[3]) ---
    stream_res = None
    if args.stream_frames > 0 and rank == 0:
        stream_res = stream_bench(sn, cfg, ws, pool_h, args, L, C)

    # ---- single-capture latency (host API, 1 capture) -------------------------
    # page-locked capture and energyscape buffers (sn_workspace_process_batch
    # with count 1), as a C-ABI caller that cares about latency would hold
    # them; the Python convenience call (ws.process: pageable numpy in, a new
    # 7.9 MB numpy array out, staged through the workspace's pinned buffers)
    # is reported beside it
    lat, lat_pg = [], []
    lat_in = torch.from_numpy(pool_h[:1].copy()).pin_memory()
    lat_out = torch.empty((1, ws.n_dirs, ws.bins), dtype=torch.float32).pin_memory()
    lat_in_np, lat_out_np = lat_in.numpy(), lat_out.numpy()
    for i in range(args.latency_samples + 3):
        t0 = time.perf_counter()
        ws.process_packed_host(lat_in_np, lat_out_np)
        if i >= 3:
            lat.append((time.perf_counter() - t0) * 1e3)
    m = sn.RawMeasurement(serial, 0, 0, 32, ws.frames, cfg.pdm_rate, pool_h[0])
    for i in range(args.latency_samples + 3):
        t0 = time.perf_counter()
        ws.process(m)
        if i >= 3:
            lat_pg.append((time.perf_counter() - t0) * 1e3)
    dev_lat = []
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for i in range(args.latency_samples + 3):
            ev_a.record(stream)
            ws.process_device(pool[i % pool_n].data_ptr(), 1, out.data_ptr(), sptr)
            ev_b.record(stream)
            ev_b.synchronize()
            if i >= 3:
                dev_lat.append(ev_a.elapsed_time(ev_b))

    # ---- per-kernel timing for the roofline (separate pass) --------------------
    ws.set_profiling(True)
    stage_ms = {k: [] for k in sn.STAGES}
    with torch.cuda.stream(stream):
        for k in range(min(20, args.steps)):
            step(k)
            stream.synchronize()
            for kk, v in ws.stage_times().items():
                stage_ms[kk].append(v)
    ws.set_profiling(False)
    stage_avg = {k: float(np.mean(v)) for k, v in stage_ms.items()}
    fe_flops, dir_flops = flops_per_energyscape(d)
    peak = sn.measure_fp_peak(local, sn.Precision.f64 if args.precision == "f64" else sn.Precision.f32)
    kflops = kernel_flops(d)  # per energyscape, SURVEY.md §8(d) rows
    kernels = {}
    for k, ms in stage_avg.items():
        f = kflops[k] * B
        kernels[k] = {"ms": ms, "tflops": f / (ms * 1e-3) / 1e12,
                      "frac": f / (ms * 1e-3) / 1e12 / peak}
    bf = ws.beamformer_info()
    if bf["kind"] == 1:
        # tensor-core delay-and-sum: int8 MACs the MMAs execute per step (dense
        # steering-matrix contraction over (shift, channel), six digit planes)
        macs = bf["sum_R"] * bf["ntiles"] * bf["slices"] * bf["m"] * bf["n"] * bf["k"] * B
        tops = 2 * macs / (stage_avg["beamform"] * 1e-3) / 1e12
        kernels["beamform"].update({
            "path": "tcgen05 kind::i8 (k_digits + k_beamform_tc)", "int8_tops_executed": tops,
            "int8_peak_tops": TC_INT8_PEAK, "tensor_frac": tops / TC_INT8_PEAK,
            "mma": {"m": bf["m"], "n": bf["n"], "k": bf["k"], "clusters": bf["clusters"],
                    "sum_R": bf["sum_R"], "slices": bf["slices"]}})
    dom = max(stage_avg, key=stage_avg.get)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.grid}/{args.precision}/B{B}/{dom}")
        except Exception:
            traffic = None
    total_step_ms = sum(stage_avg.values())
    bytes_per = 32 * d["frames"] // 8 + 4 * d["n_directions"] * d["range_bins"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (product synthesize_measurement, bench scene bench.cpp:113-117, "
                "seeds 7+1000*serial+seq)",
        "config": {**workload_desc(args.grid, d, B, pool_n), "precision": args.precision,
                   "parallelism": f"{world} GPU(s), one sensor per GPU, no data-path collective"
                                  + (", NCCL gather to rank 0" if args.gather else "")},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": EB * 32 * d["frames"] // 8,
                "d2h_bytes_per_step": EB * 4 * d["n_directions"] * d["range_bins"],
                "captures_per_step": EB, "steps": e2e_steps,
                "api": f"Workspace.process_packed_host (sn_workspace_process_batch), pinned buffers, "
                       f"{EB} captures per call ({E2E_BLOCKS} device batches of {B}, pipelined)"},
        "e2e_wire": {"value": wire_value, "unit": UNIT, "h2d_bytes_per_step": WF * flen,
                     "d2h_bytes_per_step": WF * slot, "frames_per_step": WF, "steps": e2e_steps,
                     "api": f"sn_workspace_process_frames: raw-measurement frames in (CRC verified on the GPU), "
                            f"processed-image frames out (AIMG encoded + CRC on the GPU), pinned buffers, "
                            f"{WF} frames per call ({WF // B} device batches of {B}, pipelined)"},
        "latency_ms": {
            "p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
            "device_p50": float(np.percentile(dev_lat, 50)),
            "device_p99": float(np.percentile(dev_lat, 99)),
            "pageable_p50": float(np.percentile(lat_pg, 50)), "pageable_p99": float(np.percentile(lat_pg, 99)),
            "what": "1 capture: host API incl. H2D+D2H, page-locked buffers (p50/p99; "
                    "sn_workspace_process_batch, count 1); the Python ws.process() call with pageable "
                    "buffers and a fresh output array (pageable_*); device-only (device_*)"},
        "roofline": {
            "kernel": dom, "bound": args.precision, "achieved": kernels[dom]["tflops"],
            "peak": peak, "unit": "TFLOP/s", "frac": kernels[dom]["frac"], "traffic": traffic,
            "peak_source": "measured live: FMA-chain microbenchmark (sn_measure_fp_peak) on this "
                           "GPU; MEASURED_PEAKS.json has no CUDA-core FP64/FP32 figure",
            "flops_per_launch": kflops[dom] * B, "kernel_ms": stage_avg[dom],
            "share_of_step": stage_avg[dom] / total_step_ms if total_step_ms else None,
            "kernels": kernels,
            "whole_path_tflops": (fe_flops + dir_flops * d["n_directions"]) * value / world / 1e12,
            "hbm_compulsory_gbs": bytes_per * value / world / 1e9,
        },
        "stream_pool": stream_res,
        "gather": gather_res,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.grid, args.cpu_calls)
        except Exception as e:  # the GPU number stands on its own
            line["cpu_baseline"] = {"error": str(e)}
        if args.cpu_latency_calls > 0:
            try:
                cl = cpu_latency(args.grid, args.cpu_latency_calls)
                line["cpu_baseline"]["latency_ms"] = cl
                line["latency_ms"]["cpu_reference_p50"] = {k: cl[k]["p50"] for k in ("threads_2", "threads_nproc")}
            except Exception as e:
                line["cpu_baseline"]["latency_ms"] = {"error": str(e)}
    if rank == 0 and world == 1 and not args.no_sweep:
        line["sweep"] = sweep(sn, args, local, peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
