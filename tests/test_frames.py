"""Wire-format frames around the hot path: CRC-32
(wire.cpp:58-63), the raw-measurement frame a sensor sends (wire.cpp:251-259)
and the central node's frame processing (central_node.cpp:130-160, 238-270)
with the processed-image frame (wire::image_frame(image_to_bytes(img), seq),
wire.cpp:268-276, pipeline.cpp:109-125) encoded and CRC'd on the GPU.

Oracle: the unmodified reference wire/pipeline code (oracle/_ref) and zlib's
CRC-32 (same polynomial, init and xorout)."""
import zlib

import numpy as np
import pytest

from conftest import TINY, rel_rms, to_oracle


def test_crc32_host_matches_zlib_and_reference(sn, ref):
    rng = np.random.default_rng(1)
    for n in [0, 1, 3, 4, 5, 255, 4096, 100003]:
        d = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert sn.crc32(d) == zlib.crc32(d) == ref.crc32(d)
    assert sn.crc32(b"123456789") == 0xCBF43926  # CRC-32 check value


def test_measurement_frame_bytes_match_reference(sn, po, ref):
    cfg = sn.default_pipeline_config(sn.GridKind.horizontal90).copy(**TINY)
    m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.7, 0.1, 0.0, 0.9)], 0.01, 3), 5, 1234, 17)
    ours = sn.measurement_frame(m)
    theirs = ref.measurement_frame(m.packed, m.frames, m.pdm_rate, m.sensor_serial, m.timestamp_us, m.seq)
    assert ours == theirs
    assert zlib.crc32(ours[:-4]) == int.from_bytes(ours[-4:], "little")


# ---------------------------------------------------------------------------
def _frame_parts(frame: bytes, n_dirs: int, bins: int):
    E = 36 + 34 + 8 * n_dirs
    head = frame[:E]
    energies = np.frombuffer(frame[E:E + 4 * n_dirs * bins], np.float32).reshape(n_dirs, bins)
    return head, energies


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny", "h90", "hemi3000"])
def test_process_frames_vs_reference_central_node(sn, po, ref, name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base = sn.default_pipeline_config(sn.GridKind.horizontal90)
    cfg = {"tiny": base.copy(**TINY), "h90": base,
           "hemi3000": sn.default_pipeline_config(sn.GridKind.hemisphere3000)}[name]
    ws = sn.Workspace(cfg, device=0, max_batch=3)
    rws = ref.workspace(to_oracle(po, cfg))
    ms = [sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.6 + 0.2 * i, 0.3 - 0.2 * i, 0.0, 0.8)], 0.01, 40 + i),
                                    serial=2 + i, timestamp_us=1000 * i + 7, seq=11 + i) for i in range(5)]
    frames = [sn.measurement_frame(m) for m in ms]
    got = ws.process_frames(frames)  # 5 frames through a 3-capture workspace: 3 + 2
    nd, nb = ws.n_dirs, ws.bins
    for (st, f), fin in zip(got, frames):
        want = rws.process_frame(fin)
        assert st == 0 and len(f) == len(want) == ws.image_frame_bytes
        assert zlib.crc32(f[:-4]) == int.from_bytes(f[-4:], "little")     # our CRC (GPU) is the frame's CRC
        h_got, e_got = _frame_parts(f, nd, nb)
        h_want, e_want = _frame_parts(want, nd, nb)
        assert h_got == h_want                                              # headers + direction table
        w32 = e_want.astype(np.float32)
        tol = np.spacing(np.abs(w32)).astype(np.float64) + 1e-12 * float(e_want.max())
        assert (np.abs(e_got.astype(np.float64) - e_want) <= tol).all()
        if np.array_equal(e_got, e_want):
            assert f == want                                                # byte-identical frame


@pytest.mark.gpu
def test_process_frames_errors_like_the_central_node(sn, po, ref):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = sn.default_pipeline_config(sn.GridKind.horizontal90).copy(**TINY)
    ws = sn.Workspace(cfg, device=0, max_batch=2)
    rws = ref.workspace(to_oracle(po, cfg))
    m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.7, 0.1, 0.0, 0.9)], 0.01, 3), 5, 1234, 17)
    good = sn.measurement_frame(m)
    # CRC mismatch: discarded (wire.cpp:141-145)
    bad_crc = bytearray(good)
    bad_crc[1000] ^= 0x10
    # wrong pdm rate in a well-formed frame: process() throws -> error frame
    m2 = sn.RawMeasurement(m.sensor_serial, m.timestamp_us, m.seq + 1, 32, m.frames, m.pdm_rate * 1.01, m.packed)
    wrong_rate = sn.measurement_frame(m2)
    # a frame of another configuration (more frames): error frame too
    m3 = sn.RawMeasurement(7, 9, 3, 32, m.frames + 8, m.pdm_rate, np.zeros(4 * (m.frames + 8), np.uint8))
    other_cfg = sn.measurement_frame(m3)
    # garbage / truncated / not a measurement: discarded
    trunc = good[:100]
    got = ws.process_frames([good, bytes(bad_crc), wrong_rate, other_cfg, trunc, b"\0" * 64, good])
    st = [s for s, _ in got]
    assert st == [0, 4, 3, 3, 4, 4, 0]  # ok, discarded, error frame x2, discarded x2, ok
    assert got[0][1] == got[6][1] and got[1][1] == b"" and got[4][1] == b""
    for k, mm in ((2, m2), (3, m3)):
        f = got[k][1]
        assert zlib.crc32(f[:-4]) == int.from_bytes(f[-4:], "little")
        assert int.from_bytes(f[6:8], "little") == 5                      # MsgType::error
        with pytest.raises(po.OracleError) as e:
            rws.process_frame(wrong_rate if k == 2 else other_cfg)
        assert f[36:-4].decode() == e.value.msg                           # the reference's message
    with pytest.raises(po.OracleError):
        rws.process_frame(bytes(bad_crc))
    # a nominal-size frame whose header is corrupted (pdm_rate byte flipped,
    # CRC no longer matching): the reference checks the CRC first and drops
    # it as an integrity error (wire.cpp:136-145) -- discarded, not an error
    # frame carrying the corrupted ids
    bad_rate_crc = bytearray(good)
    bad_rate_crc[66 + 6] ^= 0x01          # a byte of the f64 pdm_rate field
    bad_serial = bytearray(good)
    bad_serial[36] ^= 0x55                # the payload's sensor serial
    got = ws.process_frames([bytes(bad_rate_crc), bytes(bad_serial), good])
    assert [s for s, _ in got] == [4, 4, 0] and got[0][1] == b"" and got[1][1] == b""
    for f in (bad_rate_crc, bad_serial):
        with pytest.raises(po.OracleError):
            rws.process_frame(bytes(f))


# ---------------------------------------------------------------------------
# GPU-backed central-node worker pool: per-sensor FIFO
# release and K-transparency (test_nodes.cpp:396-445: K=1 and K=8 workers give
# identical bytes per sensor)
def _pool_run(sn, cfg, frames, workers, max_batch):
    pool = sn.CentralPool(cfg, devices=[0], workers_per_device=workers, max_batch=max_batch)
    accepted = sum(pool.submit(f) for f in frames)
    out = [pool.poll(timeout_ms=60000) for _ in range(accepted)]
    stats = pool.stats()
    pool.close()
    return accepted, out, stats


@pytest.mark.gpu
def test_central_pool_fifo_and_worker_transparency(sn, po, ref):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = sn.default_pipeline_config(sn.GridKind.horizontal90).copy(**TINY)
    frames, meta = [], []
    for k in range(6):
        for serial in (3, 9, 4):
            m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.5 + 0.05 * k, 0.1 * serial - 0.5, 0.0, 0.8)],
                                                        0.01, 100 * serial + k), serial=serial,
                                          timestamp_us=1000 * k, seq=k)
            frames.append(sn.measurement_frame(m))
            meta.append((serial, k))
    bad = bytearray(frames[4])          # sensor 9, seq 1: CRC mismatch -> discarded in order
    bad[500] ^= 1
    frames[4] = bytes(bad)
    frames.insert(7, b"garbage" * 20)   # dropped at ingest: no ticket
    rws = ref.workspace(to_oracle(po, cfg))
    results = {}
    for workers, mb in ((1, 1), (3, 2)):
        accepted, out, stats = _pool_run(sn, cfg, frames, workers, mb)
        assert accepted == 18 and stats["completed"] == 18 and stats["discarded"] == 1
        per = {}
        for serial, seq, status, f in out:
            per.setdefault(serial, []).append((seq, status, f))
        for serial, lst in per.items():
            assert [s for s, _, _ in lst] == list(range(6))          # per-sensor FIFO
        results[workers] = per
    assert results[1] == results[3]                                    # K-transparent
    # against the reference central node's frames
    fi = 0
    for f in frames:
        if f.startswith(b"garbage"):
            continue
        serial, k = meta[fi]
        fi += 1
        seq, status, got = results[3][serial][k]
        if serial == 9 and k == 1:
            assert status == 4 and got == b""
            continue
        want = rws.process_frame(f)
        assert status == 0 and len(got) == len(want) and got[:36] == want[:36]


@pytest.mark.gpu
def test_process_frames_pipelined_blocks_match_unpipelined(sn):
    """Page-locked frames in and a page-locked output: the blocks of one call
    pipeline into each other (alternating output halves, verdicts read when a
    block's downloads are done). Byte-identical frames and statuses against the
    pageable (block-synchronous) path, with a CRC-corrupted frame (discarded;
    its block's output slots are no longer consecutive, so that block is
    staged) and a mix of page-locked and pageable inputs."""
    import ctypes as C
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = sn.default_pipeline_config(sn.GridKind.horizontal90)
    ws = sn.Workspace(cfg, device=0, max_batch=3)
    n = 13
    frames = []
    for i in range(n):
        m = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.5 + 0.1 * i, 0.2, 0.0, 0.8)], 0.01, 70 + i),
                                      serial=1 + i % 4, timestamp_us=500 * i, seq=i)
        frames.append(bytearray(sn.measurement_frame(m)))
    frames[4][1000] ^= 0x40  # payload corrupted: CRC mismatch, discarded
    frames = [bytes(f) for f in frames]
    want = ws.process_frames(frames)  # pageable: every block finished before the next
    assert [s for s, _ in want].count(0) == n - 1 and want[4][0] != 0

    slot = ws.image_frame_bytes
    flen = len(frames[0])
    L = sn.lib()

    def run(pinned_mask):
        pin = torch.empty((n, flen), dtype=torch.uint8).pin_memory()
        pg = np.empty((n, flen), np.uint8)
        for i, f in enumerate(frames):
            (pin.numpy() if pinned_mask[i] else pg)[i] = np.frombuffer(f, np.uint8)
        ptrs = (C.c_void_p * n)(*[(pin.numpy() if pinned_mask[i] else pg)[i].ctypes.data for i in range(n)])
        lens = (C.c_uint64 * n)(*([flen] * n))
        out = torch.zeros((n, slot), dtype=torch.uint8).pin_memory()
        olen, st = (C.c_uint64 * n)(), (C.c_int32 * n)()
        assert L.sn_workspace_process_frames(ws._h, ptrs, lens, n, out.numpy().ctypes.data, slot, olen, st) == 0
        o = out.numpy()
        return [(int(st[i]), o[i, :olen[i]].tobytes()) for i in range(n)]

    for mask in ([True] * n, [i < 6 for i in range(n)], [i % 5 != 2 for i in range(n)]):
        for _ in range(2):  # twice: the second call starts on the halves the first left
            got = run(mask)
            for i in range(n):
                assert got[i][0] == want[i][0], (mask, i)
                assert got[i][1] == want[i][1], (mask, i)
