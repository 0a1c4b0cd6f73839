"""GPU parity at the configs[4] sweep's sizes and the round-2 test holes:
dense Fibonacci grids (geometry.cpp:206-229 with n free) and long windows
against the unmodified reference, the tensor-core beams themselves against
the reference's beamform_into, a high-dynamic-range scene, the bounded beam
ring (chunked per-direction stage), the GPU load generator against the
reference's synthesize_measurement, allocation counting, and the C++ NCCL
360-degree gather at world size 1.

Tolerances as test_gpu_parity.py: energyscapes within one
float32 ulp (+1e-12 x peak) and relative RMS <= 1e-9 in FP64 mode; beams of
the tensor-core path within 2^-45 x max|filt| of the reference's FP64 sums
(the 46-bit block-floating-point quantisation), the CUDA-core
path's beams bit-identical.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import rel_rms, to_oracle
from test_gpu_parity import capture, cfg_for, check_f64

pytestmark = pytest.mark.gpu

NPROC = os.cpu_count() or 4


@pytest.fixture(scope="module")
def gpu(sn):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return sn


def fib_cfg(sn, n, max_range):
    return sn.default_pipeline_config(sn.GridKind.horizontal90).copy(
        directions=sn.fibonacci_hemisphere(n), grid_kind=3, max_range=max_range)


def ref_energies(po, ref, cfg, packed):
    # processing_threads = nproc: the reference splits the directions over
    # threads (results independent of the count, test_pipeline.cpp:417-432)
    return ref.workspace(to_oracle(po, cfg).copy(processing_threads=NPROC)).process(packed)


@pytest.mark.parametrize("name", ["hemi3000_10m", "fib10k_5m", "fib30k_1.5m"])
def test_sweep_points_vs_reference(gpu, po, ref, name):
    sn = gpu
    if name == "hemi3000_10m":
        cfg = sn.default_pipeline_config(sn.GridKind.hemisphere3000).copy(max_range=10.0)
    elif name == "fib10k_5m":
        cfg = fib_cfg(sn, 10000, 5.0)
    else:
        cfg = fib_cfg(sn, 30000, 1.5)
    refl = [(0.9, 0.25, 0.15, 0.4), (min(cfg.max_range * 0.7, 6.0), -0.3, -0.1, 0.4)]
    m = capture(sn, cfg, refl, 0.01, 61)
    ws = sn.Workspace(cfg, device=0)
    got = ws.process(m).energies
    want = ref_energies(po, ref, cfg, m.packed)
    same = check_f64(got, want)
    assert same >= 0.99, same


def test_fib30k_batch_through_a_small_beam_ring(gpu):
    # 30k directions x 5 m: three captures through a ring that holds one
    # capture (chunk_cap = 1, the memory bound of the large sweep points),
    # identical to one capture at a time
    sn = gpu
    cfg = fib_cfg(sn, 30000, 5.0)
    ms = [capture(sn, cfg, [(1.0 + 0.5 * i, 0.2 * i, 0.1, 0.7)], 0.01, 70 + i, seq=i) for i in range(3)]
    small = sn.Workspace(cfg, device=0, max_batch=3, beam_budget_bytes=1)
    e = np.stack([im.energies for im in small.process_batch(ms)])
    one = sn.Workspace(cfg, device=0, max_batch=1)
    for i in range(3):
        assert np.array_equal(one.process(ms[i]).energies, e[i])


def test_beam_ring_chunking_is_transparent(gpu):
    # every path (host batch, device, CUDA graph, wire frames) with a ring of
    # one capture gives the bytes of the default (whole-batch) ring
    import torch
    sn = gpu
    cfg = cfg_for(sn, "box1850")
    B = 3
    ms = [capture(sn, cfg, [(1.2 + 0.3 * i, 0.1 - 0.1 * i, 0.05, 0.7)], 0.01, 80 + i, seq=i) for i in range(B)]
    big = sn.Workspace(cfg, device=0, max_batch=B)
    small = sn.Workspace(cfg, device=0, max_batch=B, beam_budget_bytes=1)
    want = np.stack([im.energies for im in big.process_batch(ms)])
    assert np.array_equal(np.stack([im.energies for im in small.process_batch(ms)]), want)
    dp = torch.from_numpy(np.stack([m.packed for m in ms])).cuda()
    out = torch.empty((B, small.n_dirs, small.bins), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for graph in (False, True, True):
        out.zero_()
        small.process_device(dp.data_ptr(), B, out.data_ptr(), s.cuda_stream, graph=graph)
        s.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)
    res = small.process_frames([sn.measurement_frame(m) for m in ms])
    res_big = big.process_frames([sn.measurement_frame(m) for m in ms])
    assert [r[0] for r in res] == [0] * B and [r[1] for r in res] == [r[1] for r in res_big]


@pytest.mark.parametrize("name", ["small", "hemi3000"])
def test_tensor_core_beams_vs_reference(gpu, po, ref, name):
    # the hot path's beams (SN_STAGE_BEAMS) against the reference's
    # beamform_into applied to the same matched-filter output
    sn = gpu
    cfg = cfg_for(sn, name)
    m = capture(sn, cfg, [(1.1, 0.3, 0.1, 0.7), (1.3 if name == "small" else 2.5, -0.4, 0.0, 0.4)], 0.01, 17)
    ws = sn.Workspace(cfg, device=0)
    ws.process(m)
    filt = ws.stage(2)
    beams = ws.stage(3)
    want = ref.workspace(to_oracle(po, cfg)).beamform(filt)
    assert beams.shape == want.shape == (ws.n_dirs, ws.dims["mf_samples"])
    bound = 2.0 ** -45 * np.abs(filt).max()
    d = np.abs(beams - want)
    assert d.max() <= bound, (d.max(), bound)
    # relative to the beams' RMS (mostly noise level, far below max|filt|)
    # the same quantisation error is larger: observed ~3e-13 on hemi3000
    assert rel_rms(beams, want) <= 1e-11
    # CUDA-core path: bit-identical beams (channel-order FP64 sums)
    wc = sn.Workspace(cfg, device=0, beamformer=sn.Beamformer.cuda_core)
    wc.process(m)
    assert np.array_equal(wc.stage(3), ref.workspace(to_oracle(po, cfg)).beamform(wc.stage(2)))


def test_high_dynamic_range_scene(gpu, po, ref):
    # strong near echo + weak far echo + tiny noise: the block-floating-point
    # scale follows the strong echo, the weak one must still hold the bar
    sn = gpu
    cfg = cfg_for(sn, "h90")
    # reflectivity = amplitude x range^2 (synth.cpp:11-61): 0.8 at 0.4 m, 1e-3 at 4.2 m
    m = capture(sn, cfg, [(0.4, 0.1, 0.0, 0.8 * 0.16), (4.2, -0.5, 0.0, 1e-3 * 4.2 ** 2)], 1e-5, 5)
    got = sn.Workspace(cfg, device=0).process(m).energies
    want = ref.workspace(to_oracle(po, cfg)).process(m.packed)
    check_f64(got, want)
    # the weak far echo is resolved: far-range region peak at the weak echo's cell
    far = want[:, int(0.7 * want.shape[1]):]
    gfar = got[:, int(0.7 * got.shape[1]):]
    assert np.unravel_index(np.argmax(gfar), gfar.shape) == np.unravel_index(np.argmax(far), far.shape)
    assert rel_rms(gfar, far) <= 1e-9


@pytest.mark.parametrize("name", ["tiny", "h90"])
def test_gpu_synthesis_matches_reference(gpu, po, ref, name):
    # sn_synthesize_device against the unmodified reference's
    # synthesize_measurement (synth.cpp:116-134) directly
    import torch
    sn = gpu
    cfg = cfg_for(sn, name)
    rc = to_oracle(po, cfg)
    scenes = [([(0.6 + 0.1 * i, 0.3 - 0.1 * i, 0.05 * i, 0.8), (1.0 + 0.05 * i, -0.2, 0.0, 0.4)][: 1 + i % 2],
               0.01 * (i % 3), 11 + i) for i in range(4)]
    nbytes = 32 * cfg.frames() // 8
    d = torch.zeros(len(scenes) * nbytes, dtype=torch.uint8, device="cuda")
    sn.synthesize_device(cfg, [sn.Scene([sn.Reflector(*r) for r in rs], nz, sd) for rs, nz, sd in scenes],
                         d.data_ptr(), device=0)
    got = d.cpu().numpy().reshape(len(scenes), nbytes)
    for i, (rs, nz, sd) in enumerate(scenes):
        want = ref.synthesize(rc, rs, nz, sd)
        assert np.array_equal(got[i], want), f"scene {i}: {int((got[i] != want).sum())} bytes differ"


def test_allocation_events_count_runtime_allocations(gpu):
    # test_pipeline.cpp:143-155 on every process path, then the beamform()
    # accessor: its two scratch buffers are allocated on the first call only
    import torch
    sn = gpu
    cfg = cfg_for(sn, "small").copy(max_range=0.8, chirp_duration=1e-3)
    ws = sn.Workspace(cfg, device=0, max_batch=2)
    m = capture(sn, cfg, [(0.5, 0.0, 0.0, 0.2)], 0.0, 0)
    dp = torch.from_numpy(np.stack([m.packed, m.packed])).cuda()
    out = torch.empty((2, ws.n_dirs, ws.bins), dtype=torch.float32, device="cuda")
    fr = sn.measurement_frame(m)
    for i in range(100):
        ws.process(m)
        if i % 10 == 0:
            ws.process_batch([m, m])
            ws.process_device(dp.data_ptr(), 2, out.data_ptr())
            ws.process_device(dp.data_ptr(), 2, out.data_ptr(), graph=True)
            ws.process_frames([fr, fr])
    torch.cuda.synchronize()
    assert ws.allocation_events() == 0
    x = np.random.default_rng(1).uniform(-1, 1, (32, ws.dims["mf_samples"]))
    ws.beamform(x)
    assert ws.allocation_events() == 2
    ws.beamform(x)
    ws.process(m)
    assert ws.allocation_events() == 2


def test_nccl_gather_world1(gpu):
    # the C++ 360-degree gather (sn_gather_*) as a 1-rank communicator: the
    # view is the rank's own images, ids come back with the trigger check
    import torch
    sn = gpu
    L = sn.lib()
    uid = (C.c_uint8 * 128)()
    if L.sn_gather_unique_id(uid) != 0:
        pytest.skip("NCCL unavailable: " + L.sn_last_error().decode())
    h = C.c_void_p()
    assert L.sn_gather_create(0, 1, uid, 0, 1000, 4, C.byref(h)) == 0, L.sn_last_error()
    imgs = torch.arange(3 * 1000, dtype=torch.float32, device="cuda")
    view = [torch.zeros(3 * 1000, dtype=torch.float32, device="cuda") for _ in range(2)]
    ids = (sn.FrameId * 3)(*[sn.FrameId(s, 0, 777, 5) for s in (1, 2, 3)])
    s = torch.cuda.Stream()
    for slot in (0, 1, 0):
        assert L.sn_gather_wait(h, slot, C.c_void_p(s.cuda_stream)) == 0
        assert L.sn_gather_start(h, slot, C.c_void_p(imgs.data_ptr()), ids, 3, C.c_void_p(view[slot].data_ptr()),
                                 C.c_void_p(s.cuda_stream)) == 0, L.sn_last_error()
    assert L.sn_gather_wait(h, 0, None) == 0
    assert torch.equal(view[0], imgs) and torch.equal(view[1], imgs)
    got = (sn.FrameId * 3)()
    ok = C.c_int32(0)
    assert L.sn_gather_ids(h, 0, got, 3, C.byref(ok)) == 0 and ok.value == 1
    assert [(g.sensor_serial, g.timestamp_us, g.seq) for g in got] == [(1, 777, 5), (2, 777, 5), (3, 777, 5)]
    ms = C.c_float(0)
    assert L.sn_gather_elapsed(h, 1, C.byref(ms)) == 0 and ms.value >= 0
    L.sn_gather_destroy(h)


def test_opt_in_log_normalisation_transform(gpu, po, ref):
    # north star stage 4 as an opt-in post-step: the energies keep the
    # reference's max(0, float) values (pipeline.cpp:469-471, one-ulp bar) and
    # the transform of them matches a numpy post-step on the oracle's energies
    import torch
    sn = gpu
    cfg = cfg_for(sn, "h90")
    ms = [capture(sn, cfg, [(1.0 + 0.5 * i, 0.3 - 0.2 * i, 0.0, 0.6)], 0.01, 90 + i, seq=i) for i in range(2)]
    ws = sn.Workspace(cfg, device=0, max_batch=2)
    dp = torch.from_numpy(np.stack([m.packed for m in ms])).cuda()
    e = torch.empty((2, ws.n_dirs, ws.bins), dtype=torch.float32, device="cuda")
    ws.process_device(dp.data_ptr(), 2, e.data_ptr())
    torch.cuda.synchronize()
    raw = e.cpu().numpy()
    r = ref.workspace(to_oracle(po, cfg))
    want = [r.process(m.packed) for m in ms]
    for i in range(2):
        check_f64(raw[i], want[i])
    cells = ws.n_dirs * ws.bins
    out = torch.empty_like(e)
    for mode, floor in ((sn.Transform.normalize, 0.0), (sn.Transform.db, -60.0)):
        sn.energyscape_transform(e.data_ptr(), out.data_ptr(), 2, cells, mode, floor)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        assert np.array_equal(e.cpu().numpy(), raw)  # energies untouched
        for i in range(2):
            w = want[i].astype(np.float64) / want[i].max()
            if mode == sn.Transform.db:
                with np.errstate(divide="ignore"):
                    w = np.maximum(10 * np.log10(w), floor)
                assert np.abs(got[i] - w).max() <= 1e-4  # dB, float32 arithmetic
                assert got[i].max() == 0.0 and got[i].min() >= floor
            else:
                assert np.abs(got[i] - w).max() <= 1e-6
                assert got[i].max() == 1.0
    with pytest.raises(sn.ArgumentError):
        sn.energyscape_transform(e.data_ptr(), e.data_ptr(), 2, cells)


def test_pipelined_host_blocks_match_single_calls(gpu):
    # page-locked buffers: the blocks of one sn_workspace_process_batch call
    # pipeline into each other (events on d_packed / d_energy); results equal
    # one capture per call, and the pageable path (per-block sync) agrees
    import torch
    sn = gpu
    cfg = cfg_for(sn, "box1850")
    ms = [capture(sn, cfg, [(1.0 + 0.25 * i, 0.3 - 0.1 * i, 0.05, 0.7)], 0.01, 120 + i, seq=i) for i in range(7)]
    ws = sn.Workspace(cfg, device=0, max_batch=2)  # 7 captures -> 4 blocks (2, 2, 2, 1)
    pin_in = torch.from_numpy(np.stack([m.packed for m in ms])).pin_memory()
    pin_out = torch.zeros((7, ws.n_dirs, ws.bins), dtype=torch.float32).pin_memory()
    for _ in range(2):
        ws.process_packed_host(pin_in.numpy(), pin_out.numpy())
        one = sn.Workspace(cfg, device=0, max_batch=1)
        for i in (0, 3, 6):
            assert np.array_equal(one.process(ms[i]).energies, pin_out.numpy()[i])
    pageable = np.stack([im.energies for im in ws.process_batch(ms)])
    assert np.array_equal(pageable, pin_out.numpy())
