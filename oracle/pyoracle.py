"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the parity oracles.

* ``Ref``  : oracle/_ref/libsonarnet_ref.so — the UNMODIFIED reference C++
  core (/root/reference/proj/core/src) built by oracle/Makefile with a
  test-only FFTW shim and pinned FP flags. ``Ref(fast=True)`` loads the
  timing build (reference default Release flags) used as the CPU baseline.
* ``Port`` : oracle/_build/libsonarnet_port.so — the plain-C restatement
  (oracle/sonarnet_port.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module. The product (paper_2208_10839_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsonarnet_ref.so")
REF_FAST_SO = os.path.join(HERE, "_ref", "libsonarnet_ref_fast.so")
PORT_SO = os.path.join(HERE, "_build", "libsonarnet_port.so")

GRID_H90, GRID_BOX1850, GRID_HEMI3000, GRID_CUSTOM = 0, 1, 2, 3
GRID_SIZES = {GRID_H90: 90, GRID_BOX1850: 1850, GRID_HEMI3000: 3000}


class OrcConfig(C.Structure):
    _fields_ = [
        ("mic_xyz", C.c_double * 96),
        ("directions", C.POINTER(C.c_double)),
        ("n_directions", C.c_uint64),
        ("grid_kind", C.c_int32),
        ("processing_threads", C.c_int32),
        ("pdm_rate", C.c_double),
        ("chirp_f_start", C.c_double),
        ("chirp_f_end", C.c_double),
        ("chirp_duration", C.c_double),
        ("demod_cutoff_hz", C.c_double),
        ("demod_taps", C.c_int32),
        ("demod_decimation", C.c_int32),
        ("pre_mf_decimation", C.c_int32),
        ("post_envelope_decimation", C.c_int32),
        ("smoothing_cutoff_hz", C.c_double),
        ("smoothing_taps", C.c_int32),
        ("precision", C.c_int32),
        ("speed_of_sound", C.c_double),
        ("max_range", C.c_double),
    ]


class OrcMeasurement(C.Structure):
    _fields_ = [
        ("sensor_serial", C.c_uint32),
        ("timestamp_us", C.c_uint64),
        ("seq", C.c_uint64),
        ("channels", C.c_uint16),
        ("frames", C.c_uint64),
        ("pdm_rate", C.c_double),
        ("packed", C.POINTER(C.c_uint8)),
        ("packed_len", C.c_uint64),
    ]


class OrcReflector(C.Structure):
    _fields_ = [("range", C.c_double), ("azimuth", C.c_double),
                ("elevation", C.c_double), ("reflectivity", C.c_double)]


class OrcScene(C.Structure):
    _fields_ = [("reflectors", C.POINTER(OrcReflector)), ("n_reflectors", C.c_uint64),
                ("noise_rms", C.c_double), ("seed", C.c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


@dataclass
class Config:
    """Python-side PipelineConfig (pipeline.hpp:22-55) that renders to the flat struct."""
    mic_xyz: np.ndarray
    directions: np.ndarray  # (n, 2) az, el
    grid_kind: int = GRID_H90
    processing_threads: int = 0
    pdm_rate: float = 4.5e6
    chirp_f_start: float = 90e3
    chirp_f_end: float = 25e3
    chirp_duration: float = 3e-3
    demod_cutoff_hz: float = 126e3
    demod_taps: int = 255
    demod_decimation: int = 10
    pre_mf_decimation: int = 2
    post_envelope_decimation: int = 10
    smoothing_cutoff_hz: float = 10e3
    smoothing_taps: int = 127
    precision: int = 0
    speed_of_sound: float = 343.0
    max_range: float = 5.0

    def to_struct(self):
        c = OrcConfig()
        xyz = np.ascontiguousarray(self.mic_xyz, dtype=np.float64).reshape(96)
        for i in range(96):
            c.mic_xyz[i] = float(xyz[i])
        dirs = np.ascontiguousarray(self.directions, dtype=np.float64).reshape(-1, 2)
        c.directions = dirs.ctypes.data_as(C.POINTER(C.c_double))
        c.n_directions = dirs.shape[0]
        for name, _ in OrcConfig._fields_:
            if name in ("mic_xyz", "directions", "n_directions"):
                continue
            setattr(c, name, getattr(self, name))
        return c, dirs  # keep dirs alive alongside the struct

    def copy(self, **kw):
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


def _lib_load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


class Ref:
    """The unmodified reference, via oracle/ref_capi.cpp."""

    def __init__(self, fast: bool = False):
        self.lib = _lib_load(REF_FAST_SO if fast else REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_ws_create.restype = C.c_void_p
        L.ref_ws_create.argtypes = [C.POINTER(OrcConfig), C.POINTER(C.c_int)]
        L.ref_ws_destroy.argtypes = [C.c_void_p]
        L.ref_ws_dims.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_ws_process.argtypes = [C.c_void_p, C.POINTER(OrcMeasurement), C.c_void_p]
        L.ref_ws_stage.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
        L.ref_ws_table.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64,
                                   C.POINTER(C.c_uint64)]
        L.ref_ws_delays.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.ref_ws_advances.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.ref_ws_alloc_events.restype = C.c_uint64
        L.ref_ws_alloc_events.argtypes = [C.c_void_p]
        L.ref_ws_beamform.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.ref_synthesize.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcScene), C.c_uint32,
                                     C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_latency.argtypes = [C.c_void_p, C.POINTER(OrcMeasurement), C.c_int, C.c_void_p]
        L.ref_throughput.argtypes = [C.POINTER(OrcConfig), C.c_void_p, C.c_uint64, C.c_int,
                                     C.c_uint64, C.c_void_p]
        L.ref_default_array.argtypes = [C.c_uint64, C.c_void_p]
        L.ref_direction_grid.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_default_config.argtypes = [C.c_int, C.POINTER(OrcConfig), C.c_void_p, C.c_uint64]
        L.ref_crc32.restype = C.c_uint32
        L.ref_crc32.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_measurement_frame.argtypes = [C.POINTER(OrcMeasurement), C.c_void_p, C.c_uint64,
                                            C.POINTER(C.c_uint64)]
        L.ref_ws_process_frame.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                           C.POINTER(C.c_uint64)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    # --- setup helpers -------------------------------------------------
    def default_array(self, seed=42):
        out = np.zeros(96, np.float64)
        self._check(self.lib.ref_default_array(seed, out.ctypes.data))
        return out.reshape(32, 3)

    def direction_grid(self, kind):
        n = C.c_uint64(0)
        self._check(self.lib.ref_direction_grid(kind, None, 0, C.byref(n)))
        out = np.zeros((n.value, 2), np.float64)
        self._check(self.lib.ref_direction_grid(kind, out.ctypes.data, n.value, C.byref(n)))
        return out

    def default_config(self, kind=GRID_H90) -> Config:
        c = OrcConfig()
        buf = np.zeros((3000, 2), np.float64)
        self._check(self.lib.ref_default_config(kind, C.byref(c), buf.ctypes.data, 3000))
        cfg = Config(mic_xyz=np.array(c.mic_xyz[:]).reshape(32, 3),
                     directions=buf[: c.n_directions].copy())
        for name, _ in OrcConfig._fields_:
            if name in ("mic_xyz", "directions", "n_directions"):
                continue
            setattr(cfg, name, getattr(c, name))
        return cfg

    def synthesize(self, cfg: Config, reflectors, noise_rms=0.0, seed=0, serial=1, ts=0, seq=0):
        st, _keep = cfg.to_struct()
        refl = (OrcReflector * max(1, len(reflectors)))()
        for i, r in enumerate(reflectors):
            refl[i] = OrcReflector(*r)
        scene = OrcScene(refl, len(reflectors), noise_rms, seed)
        frames = self.frames_for(cfg)
        out = np.zeros(32 * frames // 8, np.uint8)
        self._check(self.lib.ref_synthesize(C.byref(st), C.byref(scene), serial, ts, seq,
                                            out.ctypes.data, out.size))
        return out

    def frames_for(self, cfg: Config) -> int:
        ws = self.workspace(cfg)
        return ws.dims["frames"]

    def workspace(self, cfg: Config) -> "RefWorkspace":
        return RefWorkspace(self, cfg)

    # --- wire format (wire.cpp) ----------------------------------------
    def crc32(self, data) -> int:
        b = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else data,
                                 dtype=np.uint8)
        return int(self.lib.ref_crc32(b.ctypes.data, b.size))

    def measurement_frame(self, packed, frames, pdm_rate, serial=1, ts=0, seq=0, channels=32) -> bytes:
        m, _k = measurement_struct(packed, frames, pdm_rate, serial, ts, seq, channels)
        n = C.c_uint64(0)
        self._check(self.lib.ref_measurement_frame(C.byref(m), None, 0, C.byref(n)))
        out = np.zeros(n.value, np.uint8)
        self._check(self.lib.ref_measurement_frame(C.byref(m), out.ctypes.data, out.size, C.byref(n)))
        return out.tobytes()

    def throughput(self, cfg: Config, pool: np.ndarray, threads: int, calls_per_worker: int):
        st, _keep = cfg.to_struct()
        pool = np.ascontiguousarray(pool, dtype=np.uint8)
        stats = np.zeros(2, np.float64)
        self._check(self.lib.ref_throughput(C.byref(st), pool.ctypes.data, pool.shape[0],
                                            threads, calls_per_worker, stats.ctypes.data))
        return float(stats[0]), int(stats[1])


def measurement_struct(packed: np.ndarray, frames: int, pdm_rate: float, serial=1, ts=0, seq=0,
                       channels=32):
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    m = OrcMeasurement(serial, ts, seq, channels, frames, pdm_rate,
                       packed.ctypes.data_as(C.POINTER(C.c_uint8)), packed.size)
    return m, packed


class RefWorkspace:
    DIM_NAMES = ["frames", "demod_samples", "mf_samples", "range_bins", "n_dirs", "ref_len",
                 "mf_fft_size", "env_fft_size", "smoothing_len", "lut_octets"]

    def __init__(self, ref: Ref, cfg: Config):
        self.ref, self.cfg = ref, cfg
        st, self._keep = cfg.to_struct()
        status = C.c_int(0)
        self.h = ref.lib.ref_ws_create(C.byref(st), C.byref(status))
        if status.value != 0:
            raise OracleError(status.value, ref.lib.ref_last_error().decode())
        d = (C.c_uint64 * 10)()
        rbs = C.c_double(0)
        ref._check(ref.lib.ref_ws_dims(self.h, d, C.byref(rbs)))
        self.dims = {k: int(d[i]) for i, k in enumerate(self.DIM_NAMES)}
        self.range_bin_size = rbs.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_ws_destroy(self.h)
            self.h = None

    def process(self, packed, serial=1, ts=0, seq=0, frames=None, pdm_rate=None, channels=32):
        frames = self.dims["frames"] if frames is None else frames
        pdm_rate = self.cfg.pdm_rate if pdm_rate is None else pdm_rate
        m, _k = measurement_struct(packed, frames, pdm_rate, serial, ts, seq, channels)
        out = np.zeros((self.dims["n_dirs"], self.dims["range_bins"]), np.float32)
        self.ref._check(self.ref.lib.ref_ws_process(self.h, C.byref(m), out.ctypes.data))
        return out

    def process_frame(self, frame: bytes) -> bytes:
        """Central-node path for one received frame: decode_packet (CRC) ->
        decode_raw_measurement -> process -> wire::image_frame(image, seq)."""
        f = np.frombuffer(frame, np.uint8)
        cap = 64 + 8 * self.dims["n_dirs"] + 4 * self.dims["n_dirs"] * self.dims["range_bins"] + 64
        out = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        self.ref._check(self.ref.lib.ref_ws_process_frame(self.h, f.ctypes.data, f.size, out.ctypes.data,
                                                          out.size, C.byref(n)))
        return out[: n.value].tobytes()

    def stage(self, which: int):
        d = self.dims
        if which == 0:
            out = np.zeros((32, d["demod_samples"]), np.float64)
        elif which in (1, 2):
            out = np.zeros((32, d["mf_samples"]), np.float64)
        else:
            raise ValueError(which)
        self.ref._check(self.ref.lib.ref_ws_stage(self.h, which, out.ctypes.data, out.size))
        return out

    def bit_rows(self):
        stride = self.dims["frames"] // 8 + self.dims["lut_octets"]
        out = np.zeros(32 * stride, np.uint8)
        self.ref._check(self.ref.lib.ref_ws_stage(self.h, 3, out.ctypes.data, out.size))
        return out.reshape(32, stride)

    def table(self, which: int):
        n = C.c_uint64(0)
        self.ref._check(self.ref.lib.ref_ws_table(self.h, which, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.float64)
        self.ref._check(self.ref.lib.ref_ws_table(self.h, which, out.ctypes.data, n.value,
                                                  C.byref(n)))
        return out

    def delay_table(self):
        out = np.zeros((self.dims["n_dirs"], 32), np.int32)
        self.ref._check(self.ref.lib.ref_ws_delays(self.h, out.ctypes.data, out.size))
        return out

    def reference_advances(self):
        out = np.zeros(self.dims["n_dirs"], np.int32)
        self.ref._check(self.ref.lib.ref_ws_advances(self.h, out.ctypes.data, out.size))
        return out

    def allocation_events(self):
        return int(self.ref.lib.ref_ws_alloc_events(self.h))

    def beamform(self, filt: np.ndarray):
        filt = np.ascontiguousarray(filt, dtype=np.float64)
        out = np.zeros((self.dims["n_dirs"], filt.shape[1]), np.float64)
        self.ref._check(self.ref.lib.ref_ws_beamform(self.h, filt.ctypes.data, filt.shape[0],
                                                     filt.shape[1], out.ctypes.data))
        return out

    def latency(self, packed, n: int):
        m, _k = measurement_struct(packed, self.dims["frames"], self.cfg.pdm_rate)
        out = np.zeros(n, np.float64)
        self.ref._check(self.ref.lib.ref_latency(self.h, C.byref(m), n, out.ctypes.data))
        return out


# Fixed configurations used across tests / bench.
BENCH_SCENE = [(1.5, 0.2, 0.0, 0.8), (3.0, -0.4, 0.1, 0.5)]  # bench.cpp:113-117
BENCH_NOISE, BENCH_SEED = 0.01, 7


def az181_directions():
    """Custom 181-azimuth grid, -90..+90 deg step 1 deg, el 0."""
    az = np.deg2rad(np.arange(-90, 91, dtype=np.float64))
    return np.stack([az, np.zeros_like(az)], axis=1)


class Port:
    """The plain-C restatement (oracle/sonarnet_port.c)."""

    def __init__(self):
        self.lib = _lib_load(PORT_SO)
        L = self.lib
        L.port_last_error.restype = C.c_char_p
        L.port_dims.argtypes = [C.POINTER(OrcConfig), C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.port_process.argtypes = [C.POINTER(OrcConfig), C.c_void_p, C.c_uint64, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
        L.port_table.argtypes = [C.POINTER(OrcConfig), C.c_int, C.c_void_p, C.c_uint64,
                                 C.POINTER(C.c_uint64)]
        L.port_steering.argtypes = [C.POINTER(OrcConfig), C.c_void_p, C.c_void_p]
        L.port_synthesize.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcScene), C.c_void_p,
                                      C.c_uint64]
        L.port_default_array.argtypes = [C.c_uint64, C.c_void_p]
        L.port_direction_grid.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.port_last_error().decode())

    def default_array(self, seed=42):
        out = np.zeros(96, np.float64)
        self._check(self.lib.port_default_array(seed, out.ctypes.data))
        return out.reshape(32, 3)

    def direction_grid(self, kind):
        n = C.c_uint64(0)
        self._check(self.lib.port_direction_grid(kind, None, 0, C.byref(n)))
        out = np.zeros((n.value, 2), np.float64)
        self._check(self.lib.port_direction_grid(kind, out.ctypes.data, n.value, C.byref(n)))
        return out

    def dims(self, cfg: Config):
        st, _k = cfg.to_struct()
        d = (C.c_uint64 * 10)()
        rbs = C.c_double(0)
        self._check(self.lib.port_dims(C.byref(st), d, C.byref(rbs)))
        return {k: int(d[i]) for i, k in enumerate(RefWorkspace.DIM_NAMES)}

    def table(self, cfg: Config, which: int):
        st, _k = cfg.to_struct()
        n = C.c_uint64(0)
        self._check(self.lib.port_table(C.byref(st), which, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.float64)
        self._check(self.lib.port_table(C.byref(st), which, out.ctypes.data, n.value, C.byref(n)))
        return out

    def steering(self, cfg: Config):
        st, _k = cfg.to_struct()
        n = st.n_directions
        delays = np.zeros((n, 32), np.int32)
        adv = np.zeros(n, np.int32)
        self._check(self.lib.port_steering(C.byref(st), delays.ctypes.data, adv.ctypes.data))
        return delays, adv

    def synthesize(self, cfg: Config, reflectors, noise_rms=0.0, seed=0):
        st, _k = cfg.to_struct()
        refl = (OrcReflector * max(1, len(reflectors)))()
        for i, r in enumerate(reflectors):
            refl[i] = OrcReflector(*r)
        scene = OrcScene(refl, len(reflectors), noise_rms, seed)
        frames = self.dims(cfg)["frames"]
        out = np.zeros(32 * frames // 8, np.uint8)
        self._check(self.lib.port_synthesize(C.byref(st), C.byref(scene), out.ctypes.data,
                                             out.size))
        return out

    def process(self, cfg: Config, packed, stages=False):
        st, _k = cfg.to_struct()
        d = self.dims(cfg)
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.zeros((d["n_dirs"], d["range_bins"]), np.float32)
        if stages:
            dm = np.zeros((32, d["demod_samples"]), np.float64)
            mf = np.zeros((32, d["mf_samples"]), np.float64)
            fl = np.zeros((32, d["mf_samples"]), np.float64)
            self._check(self.lib.port_process(C.byref(st), packed.ctypes.data, packed.size,
                                              out.ctypes.data, dm.ctypes.data, mf.ctypes.data,
                                              fl.ctypes.data))
            return out, dm, mf, fl
        self._check(self.lib.port_process(C.byref(st), packed.ctypes.data, packed.size,
                                          out.ctypes.data, None, None, None))
        return out
