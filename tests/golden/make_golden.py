"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists and `make -C oracle ref` has built
oracle/_ref/libsonarnet_ref.so (pinned FP flags). The fixtures travel with the
repo; nothing in the GPU tests reads /root/reference.

    python tests/golden/make_golden.py

Contents (all produced by the reference's own code paths, pipeline.cpp via
oracle/ref_capi.cpp):
  tiny.npz   tiny_config (acceptance.cpp:66-76) + horizontal90, one reflector:
             packed capture, bit rows, demod_buf, mf_buf, filt_buf, energies,
             delay table, advances, setup tables.
  h90.npz    default config (5 m, horizontal90), bench scene (bench.cpp:110-119):
             sha256 of the capture, energies.
  hemi.npz   default hemisphere3000: delay table (int8), advances, sha256 of the
             demod LUT / taps / composite kernel.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

TINY = dict(pdm_rate=1e6, chirp_f_start=20000.0, chirp_f_end=8000.0, chirp_duration=1.5e-3,
            max_range=2.0)
TINY_SCENE = dict(reflectors=[(1.0, 0.3, 0.0, 0.5)], noise_rms=0.01, seed=5)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = po.Ref()
    # ---- tiny -----------------------------------------------------------
    cfg = ref.default_config(po.GRID_H90).copy(**TINY)
    ws = ref.workspace(cfg)
    pk = ref.synthesize(cfg, TINY_SCENE["reflectors"], TINY_SCENE["noise_rms"], TINY_SCENE["seed"],
                        serial=1, ts=1000)
    e = ws.process(pk, serial=1, ts=1000)
    np.savez_compressed(
        os.path.join(HERE, "tiny.npz"),
        packed=pk, bit_rows=ws.bit_rows(), demod=ws.stage(0), mf=ws.stage(1), filt=ws.stage(2),
        energies=e, delays=ws.delay_table(), advances=ws.reference_advances(),
        demod_rev=ws.table(0), demod_lut=ws.table(1), premf_rev=ws.table(2), chirp=ws.table(3),
        comp_rev=ws.table(4), dims=np.array([ws.dims[k] for k in po.RefWorkspace.DIM_NAMES]),
        range_bin_size=np.array(ws.range_bin_size))
    # ---- default h90, bench scene ---------------------------------------
    cfg = ref.default_config(po.GRID_H90)
    ws = ref.workspace(cfg)
    pk = ref.synthesize(cfg, po.BENCH_SCENE, po.BENCH_NOISE, po.BENCH_SEED)
    e = ws.process(pk)
    np.savez_compressed(os.path.join(HERE, "h90.npz"), packed_sha256=np.array(sha(pk)),
                        energies=e, demod_sha256=np.array(sha(ws.stage(0))),
                        mf_sha256=np.array(sha(ws.stage(1))))
    # ---- hemisphere3000 setup tables --------------------------------------
    cfg = ref.default_config(po.GRID_HEMI3000)
    ws = ref.workspace(cfg)
    dl = ws.delay_table()
    assert dl.min() >= -128 and dl.max() < 128
    np.savez_compressed(
        os.path.join(HERE, "hemi.npz"), delays=dl.astype(np.int8),
        advances=ws.reference_advances().astype(np.int16), directions=cfg.directions,
        mic_xyz=cfg.mic_xyz, lut_sha256=np.array(sha(ws.table(1))),
        demod_rev_sha256=np.array(sha(ws.table(0))), premf_rev_sha256=np.array(sha(ws.table(2))),
        chirp_sha256=np.array(sha(ws.table(3))), comp_rev_sha256=np.array(sha(ws.table(4))))
    for f in ("tiny.npz", "h90.npz", "hemi.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
