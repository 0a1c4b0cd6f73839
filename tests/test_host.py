"""Product host side on CPU (no GPU needed): setup tables, steering tables,
synthesis, validation and the C ABI surface, against the reference oracle
and the golden fixtures."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, TINY, TINY_SCENE, az181, golden, to_oracle

TABLES = range(5)  # demod_rev, demod_lut, premf_rev, chirp_ref, smooth_decimate_rev


def host_ws(sn, cfg):
    return sn.Workspace(cfg, device=-1)


def configs(sn):
    base = sn.default_pipeline_config(sn.GridKind.horizontal90)
    return {
        "h90": base,
        "box1850": sn.default_pipeline_config(sn.GridKind.box1850),
        "hemi3000": sn.default_pipeline_config(sn.GridKind.hemisphere3000),
        "tiny": base.copy(**TINY),
        "small": base.copy(max_range=1.5),
        "az181": base.copy(directions=az181(), grid_kind=3),
        "demod101": base.copy(demod_taps=101),
        "demod_d8": base.copy(demod_decimation=8, demod_cutoff_hz=110e3),
        "smooth63": base.copy(smoothing_taps=63, smoothing_cutoff_hz=8e3),
    }


@pytest.mark.parametrize("name", ["h90", "box1850", "hemi3000", "tiny", "small", "az181",
                                  "demod101", "demod_d8", "smooth63"])
def test_setup_tables_bit_exact_vs_reference(sn, po, ref, name):
    cfg = configs(sn)[name]
    ws = host_ws(sn, cfg)
    rws = ref.workspace(to_oracle(po, cfg))
    for t in TABLES:
        assert np.array_equal(ws.table(t), rws.table(t)), f"table {t}"
    assert np.array_equal(ws.delay_table(), rws.delay_table())
    assert np.array_equal(ws.reference_advances(), rws.reference_advances())
    d = ws.dims
    for k in ("frames", "demod_samples", "mf_samples", "range_bins", "ref_len", "mf_fft_size",
              "env_fft_size", "smoothing_len"):
        assert d[k] == rws.dims[k], k
    assert d["range_bin_size"] == rws.range_bin_size


def test_grids_and_array_match_reference(sn, ref):
    for k in (0, 1, 2):
        assert np.array_equal(sn.direction_grid(k), ref.direction_grid(k))
    for seed in (42, 7, 1234):
        assert np.array_equal(sn.default_array(seed), ref.default_array(seed))


def test_golden_hemi_tables(sn):
    g = golden("hemi.npz")
    ws = host_ws(sn, sn.default_pipeline_config(sn.GridKind.hemisphere3000))
    assert np.array_equal(ws.delay_table(), g["delays"].astype(np.int32))
    assert np.array_equal(ws.reference_advances(), g["advances"].astype(np.int32))
    import hashlib
    assert hashlib.sha256(ws.table(1).tobytes()).hexdigest() == str(g["lut_sha256"])


def test_golden_tiny_tables(sn):
    g = golden("tiny.npz")
    ws = host_ws(sn, sn.default_pipeline_config().copy(**TINY))
    for name, t in (("demod_rev", 0), ("demod_lut", 1), ("premf_rev", 2), ("chirp", 3),
                    ("comp_rev", 4)):
        assert np.array_equal(ws.table(t), g[name]), name
    assert np.array_equal(ws.delay_table(), g["delays"])


@pytest.mark.parametrize("scene", [
    dict(reflectors=[], noise_rms=0.0, seed=0),
    dict(reflectors=[], noise_rms=0.01, seed=3),
    dict(reflectors=[(1.5, 0.2, 0.0, 0.8), (3.0, -0.4, 0.1, 0.5)], noise_rms=0.01, seed=7),
    dict(reflectors=[(0.5, -1.2, 0.3, 2.0)], noise_rms=0.0, seed=0),  # clipping regime
])
def test_synthesis_bit_exact_vs_reference(sn, po, ref, scene):
    cfg = sn.default_pipeline_config()
    m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(*r) for r in scene["reflectors"]],
                                                scene["noise_rms"], scene["seed"]))
    want = ref.synthesize(to_oracle(po, cfg), scene["reflectors"], scene["noise_rms"], scene["seed"])
    assert m.packed.shape == want.shape and np.array_equal(m.packed, want)
    assert m.channels == 32 and m.frames == 144800 and m.packed.size == 579200


def test_synthesis_golden_tiny(sn):
    g = golden("tiny.npz")
    cfg = sn.default_pipeline_config().copy(**TINY)
    m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(*r) for r in TINY_SCENE["reflectors"]],
                                                TINY_SCENE["noise_rms"], TINY_SCENE["seed"]))
    assert np.array_equal(m.packed, g["packed"])


def test_config_derived_rates(sn):
    # test_pipeline.cpp:59-74
    cfg = sn.default_pipeline_config()
    d = cfg.dims()
    assert cfg.demod_rate() == pytest.approx(450000.0)
    assert cfg.mf_rate() == pytest.approx(225000.0)
    assert cfg.final_rate() == pytest.approx(22500.0)
    assert d["frames"] % 8 == 0 and d["frames"] % cfg.demod_decimation == 0
    assert d["demod_samples"] % cfg.pre_mf_decimation == 0
    assert d["mf_samples"] % cfg.post_envelope_decimation == 0
    assert d["frames"] / cfg.pdm_rate >= 2 * cfg.max_range / cfg.speed_of_sound + cfg.chirp_duration
    assert d["range_bins"] >= 1
    assert d["range_bin_size"] == pytest.approx(343.0 / 45000.0)


@pytest.mark.parametrize("change", [
    dict(max_range=-1.0), dict(demod_taps=256), dict(chirp_f_start=200000.0),
    dict(directions=np.zeros((0, 2))), dict(max_range=0.001), dict(smoothing_taps=4),
    dict(speed_of_sound=0.0), dict(pdm_rate=0.0), dict(demod_decimation=0),
    dict(processing_threads=-1), dict(smoothing_cutoff_hz=200e3), dict(demod_cutoff_hz=3e6),
])
def test_config_validation_rejects_nonsense(sn, change):
    # test_pipeline.cpp:76-93 + pipeline.cpp:60-92
    cfg = sn.default_pipeline_config().copy(**change)
    with pytest.raises(sn.ConfigError):
        sn.Workspace(cfg, device=-1)


def test_reference_agrees_on_rejections(sn, po, ref):
    for change in (dict(max_range=-1.0), dict(demod_taps=256), dict(chirp_f_start=200000.0),
                   dict(max_range=0.001)):
        cfg = sn.default_pipeline_config().copy(**change)
        with pytest.raises(po.OracleError) as e:
            ref.workspace(to_oracle(po, cfg))
        assert e.value.status == 1  # ConfigError


def test_geometry_and_direction_argument_errors(sn):
    cfg = sn.default_pipeline_config()
    bad = cfg.mic_xyz.copy()
    bad[3] = bad[4]  # two coincident microphones (geometry.cpp:45-55)
    with pytest.raises(sn.ArgumentError):
        sn.Workspace(cfg.copy(mic_xyz=bad), device=-1)
    far = cfg.mic_xyz.copy()
    far[0, 1] = 0.2  # outside the 5 cm disk
    with pytest.raises(sn.ArgumentError):
        sn.Workspace(cfg.copy(mic_xyz=far), device=-1)
    dirs = cfg.directions.copy()
    dirs[0, 1] = 2.0  # elevation beyond pi/2 (geometry.cpp:151)
    with pytest.raises(sn.ArgumentError):
        sn.Workspace(cfg.copy(directions=dirs), device=-1)


def test_process_validation_all_or_error_on_host(sn):
    # pipeline.cpp:524-540 checks run before any device work (DecodeError),
    # then a host-only workspace refuses to compute (no CPU fallback).
    cfg = sn.default_pipeline_config().copy(**TINY)
    ws = sn.Workspace(cfg, device=-1)
    m = sn.synthesize_measurement(cfg, sn.Scene())
    for bad in (dict(channels=16), dict(frames=m.frames - 8), dict(pdm_rate=1e5),
                dict(packed=m.packed[:-1])):
        mm = sn.RawMeasurement(**{**m.__dict__, **bad})
        with pytest.raises(sn.DecodeError):
            ws.process(mm)
    with pytest.raises(sn.CudaError):
        ws.process(m)
    assert ws.allocation_events() == 0


def test_c_abi_exports_every_declared_symbol(sn):
    header = open(os.path.join(ROOT, "include", "sonarnet_b200.h")).read()
    declared = set(re.findall(r"\b(sn_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 25
    lib = ctypes.CDLL(sn.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", sn.LIB_PATH], capture_output=True, text=True)
    for s in declared:
        assert re.search(rf"\bT {s}\b", out.stdout), s


def test_library_is_sm100a(sn):
    out = subprocess.run(["cuobjdump", "--list-elf", sn.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_status_names_and_abi_version(sn):
    L = sn.lib()
    assert L.sn_abi_version() == 1
    L.sn_status_name.restype = ctypes.c_char_p
    assert [L.sn_status_name(i).decode() for i in range(7)] == [
        "ok", "config", "argument", "decode", "io", "cuda", "internal"]


def test_dims_of_standard_configs(sn):
    d = sn.default_pipeline_config(sn.GridKind.hemisphere3000).dims()
    assert (d["frames"], d["mf_samples"], d["range_bins"], d["n_directions"]) == (144800, 7240, 655, 3000)
    t = sn.default_pipeline_config().copy(**TINY).dims()
    assert (t["frames"], t["range_bins"]) == (13200, 58)
    s = sn.default_pipeline_config().copy(max_range=1.5).dims()
    assert (s["frames"], s["mf_samples"], s["range_bins"], s["env_fft_size"]) == (53000, 2650, 196, 4096)


def test_tensor_core_beamformer_schedule(sn, monkeypatch):
    # host-side cluster schedule of the tcgen05 delay-and-sum (beamform_tc.cu):
    # every direction in one cluster of <= 128 slots with <= 40 shift values
    import math
    for kind in (0, 1, 2):
        cfg = sn.default_pipeline_config(kind)
        ws = sn.Workspace(cfg, device=-1)
        info = ws.beamformer_info()
        n = ws.n_dirs
        assert info["kind"] == 1 and info["m"] == 128 and info["k"] == 32 and info["slices"] == 6
        assert math.ceil(n / 128) <= info["clusters"] <= n
        assert 1 <= info["max_R"] <= 40 and info["sum_R"] <= info["clusters"] * info["max_R"]
        assert info["ntiles"] == math.ceil(ws.dims["mf_samples"] / info["n"])
    assert sn.Workspace(sn.default_pipeline_config(2), device=-1,
                        beamformer=sn.Beamformer.cuda_core).beamformer_info()["kind"] == 0


# ---- round 2: dense grids, workspace options, bench legs (CPU only) --------
def test_fibonacci_hemisphere_matches_the_reference_grid(sn, ref):
    # n = 3000 is the reference's hemisphere3000 (geometry.cpp:206-229), bit for bit
    g = sn.fibonacci_hemisphere(3000)
    assert np.array_equal(g, sn.direction_grid(sn.GridKind.hemisphere3000))
    assert np.array_equal(g, ref.direction_grid(2))


@pytest.mark.parametrize("n", [1, 10, 10000, 30000])
def test_fibonacci_hemisphere_variable_n(sn, n):
    # restated in numpy (same formula and sort); libm vs numpy trig may differ
    # in the last place, so 1e-14 rad
    g = sn.fibonacci_hemisphere(n)
    i = np.arange(n, dtype=np.float64)
    x = (i + 0.5) / n
    r = np.sqrt(1.0 - x * x)
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    az = np.arctan2(r * np.cos(phi), x)
    el = np.arcsin(np.clip(r * np.sin(phi), -1, 1))
    order = np.lexsort((az, el))
    want = np.stack([az[order], el[order]], 1)
    assert g.shape == (n, 2)
    assert np.abs(g - want).max() <= 1e-14
    assert (np.diff(g[:, 1]) >= 0).all() and (np.abs(g[:, 0]) <= np.pi / 2).all()
    with pytest.raises(sn.ConfigError):
        sn.fibonacci_hemisphere(0)


def test_sweep_configs_derived_sizes(sn):
    # frames 53,000 / 144,800 / 276,000; FFT 4096 /
    # 8192 / 16384; bins 196 / 655 / 1,311 at 1.5 / 5 / 10 m
    import bench
    want = {1.5: (53000, 4096, 196), 5.0: (144800, 8192, 655), 10.0: (276000, 16384, 1311)}
    for grid, nd in (("fib30k", 30000), ("fib10k", 10000), ("az181", 181), ("hemisphere3000", 3000)):
        for mr, (fr, nfft, bins) in want.items():
            d = bench.sweep_config(sn, grid, mr, "f64").dims()
            assert (d["n_directions"], d["frames"], d["env_fft_size"], d["range_bins"]) == (nd, fr, nfft, bins)


def test_workspace_options_validated(sn):
    cfg = sn.default_pipeline_config(sn.GridKind.horizontal90)
    with pytest.raises(sn.ArgumentError):
        sn.Workspace(cfg, device=-1, tc_tile_n=100)
    with pytest.raises(sn.ArgumentError):
        sn.Workspace(cfg, device=-1, beamformer=7)
    for n in (64, 96, 128):
        assert sn.Workspace(cfg, device=-1, tc_tile_n=n).beamformer_info()["kind"] == 1


def test_cpu_latency_leg(ref):
    # bench.cpp:63-108 protocol through the reference oracle, both thread legs
    import bench
    r = bench.cpu_latency("horizontal90", 2)
    assert r["threads_2"]["threads"] == 2 and r["threads_2"]["n"] == 2
    assert 0 < r["threads_nproc"]["p50"] and r["threads_2"]["p50"] <= r["threads_2"]["p99"]
    assert "shim" in r["fft"]


def test_trigger_synchronisation_check():
    from paper_2208_10839_b200.distributed import triggers_synchronized
    ids = [(1, 100, 7), (1, 200, 8), (2, 100, 7), (2, 200, 8)]  # world 2, 2 images each
    assert triggers_synchronized(ids, 2)
    assert not triggers_synchronized([(1, 100, 7), (2, 100, 8)], 2)


def test_hot_kernels_register_budget(sn):
    # ptxas resource usage of the production kernels (cuobjdump -res-usage on
    # the in-tree library): the envelope's register allocation is fragile (an
    # extra kernel-parameter field once pushed its stack from 56 to 352 B and
    # cost 23%), so the hot kernels' stack frames are pinned here
    import shutil
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-res-usage", sn.LIB_PATH], capture_output=True, text=True).stdout
    usage, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and cur:
            usage[cur] = (int(m.group(1)), int(m.group(2)))
    limits = {  # mangled name prefix -> max stack bytes
        "_ZN3snb10k_envelopeIdLi2ELi4096ELb1E": 16,   # default FP64 envelope (N = 8192, FFT FIR)
        # FP32 (3 groups at 80 registers): the fused first FIR pass costs a
        # 40 B frame and is still faster (envelope 1.87 -> 1.72 ms)
        "_ZN3snb10k_envelopeIfLi3ELi4096ELb1E": 48,
        "_ZN3snb19k_envelope_pair2048IdE": 0,           # 1.5 m window
        "_ZN3snb20k_envelope_split8192IdE": 32,         # 10 m window
        "_ZN3snb13k_beamform_tcILi96E": 64,             # tensor-core delay-and-sum
        "_ZN3snb7k_demod": 0,
        "_ZN3snb10k_premf_rw": 0,
    }
    for prefix, lim in limits.items():
        hits = [v for k, v in usage.items() if k.startswith(prefix)]
        assert hits, prefix
        assert all(st <= lim for _, st in hits), (prefix, hits)


def test_measurement_dtype_matches_ctypes_layout(sn):
    """process_packed_host fills sn_raw_measurement structs column-wise via a
    numpy dtype built from the ctypes field offsets: same bytes as ctypes."""
    import ctypes as C
    M = sn._Measurement
    dt = sn._measurement_dtype()
    assert dt.itemsize == C.sizeof(M)
    buf = np.zeros(4, dt)
    data = np.zeros((4, 16), np.uint8)
    buf["sensor_serial"] = 7
    buf["timestamp_us"] = 123456789
    buf["seq"] = np.arange(4)
    buf["channels"] = 32
    buf["frames"] = 144800
    buf["pdm_rate"] = 4.5e6
    buf["packed"] = np.uint64(data.ctypes.data) + np.arange(4, dtype=np.uint64) * np.uint64(16)
    buf["packed_len"] = 16
    s = (M * 4).from_buffer(buf)
    for i in range(4):
        ref = M(7, 123456789, i, 32, 144800, 4.5e6, C.cast(data.ctypes.data + 16 * i, C.POINTER(C.c_uint8)), 16)
        assert bytes(s[i]) == bytes(ref)


@pytest.mark.parametrize("c0", [1, 63, 223, 255, 257, 321, 511])
def test_fused_sink_covers_fir_layout_once(c0):
    """k_envelope's fused sink (kernels.cu, FFT FIR): thread m of the last
    inverse pass holds samples t_k = 2m + c0 + 512k (k = 0..15) and runs the
    FIR's radix-3 butterflies over (t, t + 2560, t + 5120) for the five t_k in
    [0, 2560) -- k = 0..4 if t_0 < 512, else k = -1..3 (t_-1 < c0: a zero
    sample). Every slot (sequence a, position u < 768) of the layout must be
    written exactly once, and each butterfly's members must be the slots
    u, u + 256, u + 512 of one sequence."""
    seen = np.zeros((5, 768), np.int32)
    for m in range(256):
        t0 = 2 * m + c0
        hi = t0 >= 512
        for j in range(5):
            ks = (j, j + 5, j + 10) if j < 4 else ((-1, 4, 9) if hi else (4, 9, 14))
            t = t0 - 512 if (j == 4 and hi) else t0 + 512 * j
            assert 0 <= t < 2560 and t % 2 == 1
            for n1, k in enumerate(ks):
                tk = t0 + 512 * k
                assert tk == t + 2560 * n1            # member n1 of the butterfly
                assert k <= 14                        # output k = 15 is never needed
                u, sa = tk // 10, (tk % 10 - 1) // 2
                assert u == t // 10 + 256 * n1 and sa == (t % 10 - 1) // 2
                if k < 0:
                    assert tk < c0                    # the zero sample below the window
                seen[sa, u] += 1
    assert (seen == 1).all()
