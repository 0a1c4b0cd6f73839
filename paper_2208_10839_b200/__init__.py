"""paper_2208_10839_b200 — B200-native eRTIS image-formation path.

Python mirror of the reference's processing API (sonarnet, pipeline.hpp:22-130)
over the C ABI in include/sonarnet_b200.h (libsonarnet_b200.so, built in-tree
by ``paper_2208_10839_b200.build``). Names, argument meaning and error
behaviour follow the reference:

    cfg = default_pipeline_config(GridKind.hemisphere3000)
    ws  = Workspace(cfg)                      # ConfigError on a bad config
    m   = synthesize_measurement(cfg, scene, serial=1, timestamp_us=0)
    img = ws.process(m)                       # DecodeError on a mismatched capture
    img.argmax(), img.energies                # (directions x range_bins) float32

There is no CPU fallback: importing works without a GPU (setup helpers and
host-only workspaces are usable for parity checks of the setup tables), but
``process`` requires the CUDA library and a device and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libsonarnet_b200.so")

__all__ = [
    "GridKind", "Precision", "PipelineConfig", "RawMeasurement", "AcousticImage", "Reflector",
    "Scene", "Workspace", "default_pipeline_config", "direction_grid", "default_array",
    "synthesize_measurement", "SonarError", "ConfigError", "ArgumentError", "DecodeError",
    "IoError", "CudaError", "lib", "crc32", "measurement_frame", "CentralPool", "synthesize_device",
    "fibonacci_hemisphere", "Beamformer", "load_library", "Transform", "energyscape_transform",
]


# ---------------------------------------------------------------------------
# errors (errors.hpp:11-29)
class SonarError(RuntimeError):
    status = 6


class ConfigError(SonarError):
    status = 1


class ArgumentError(SonarError, ValueError):
    status = 2


class DecodeError(SonarError):
    status = 3


class IoError(SonarError):
    status = 4


class CudaError(SonarError):
    status = 5


_ERRORS = {1: ConfigError, 2: ArgumentError, 3: DecodeError, 4: IoError, 5: CudaError}


class GridKind(enum.IntEnum):  # geometry.hpp:65
    horizontal90 = 0
    box1850 = 1
    hemisphere3000 = 2
    custom = 3


class Precision(enum.IntEnum):
    f64 = 0
    f32 = 1


class Beamformer(enum.IntEnum):  # sn_beamformer_kind
    tensor_core = 0
    cuda_core = 1


class _Options(C.Structure):  # sn_workspace_options
    _fields_ = [("beamformer", C.c_int32), ("tc_tile_n", C.c_int32), ("beam_budget_bytes", C.c_uint64)]


# ---------------------------------------------------------------------------
# ctypes mirror of the C ABI structs
class _Config(C.Structure):
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


class _Measurement(C.Structure):
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


_MEAS_DTYPE = None


def _measurement_dtype():
    """numpy dtype with _Measurement's field offsets (pointers as uint64)."""
    global _MEAS_DTYPE
    if _MEAS_DTYPE is None:
        conv = {C.c_uint32: np.uint32, C.c_uint64: np.uint64, C.c_uint16: np.uint16, C.c_double: np.float64}
        names = [n for n, _ in _Measurement._fields_]
        _MEAS_DTYPE = np.dtype({"names": names,
                                "formats": [conv.get(t, np.uint64) for _, t in _Measurement._fields_],
                                "offsets": [getattr(_Measurement, n).offset for n in names],
                                "itemsize": C.sizeof(_Measurement)})
    return _MEAS_DTYPE


class _Dims(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "frames", "demod_samples", "mf_samples", "range_bins", "n_directions", "ref_len",
        "mf_fft_size", "env_fft_size", "smoothing_len")] + [
        ("range_bin_size", C.c_double), ("demod_rate", C.c_double), ("mf_rate", C.c_double),
        ("final_rate", C.c_double), ("max_batch", C.c_uint64)]


class _Reflector(C.Structure):
    _fields_ = [("range", C.c_double), ("azimuth", C.c_double), ("elevation", C.c_double),
                ("reflectivity", C.c_double)]


class _Scene(C.Structure):
    _fields_ = [("reflectors", C.POINTER(_Reflector)), ("n_reflectors", C.c_uint64),
                ("noise_rms", C.c_double), ("seed", C.c_uint64)]


class FrameId(C.Structure):  # sn_frame_id: one image's trigger identity (sync.hpp:16-19)
    _fields_ = [("sensor_serial", C.c_uint32), ("reserved", C.c_uint32), ("timestamp_us", C.c_uint64),
                ("seq", C.c_uint64)]


_lib: Optional[C.CDLL] = None

STAGES = ("demod", "premf", "matched_filter", "beamform", "envelope")


class _BfInfo(C.Structure):  # sn_beamformer_info
    _fields_ = [("kind", C.c_int32), ("clusters", C.c_int32), ("sum_R", C.c_int64), ("max_R", C.c_int32),
                ("ntiles", C.c_int32), ("slices", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
                ("k", C.c_int32)]


def load_library(path: str) -> C.CDLL:
    """Bind another build of the same sources (developer A/B builds) instead
    of the in-tree library; call before anything else touches lib()."""
    global _lib, LIB_PATH
    if _lib is not None:
        raise RuntimeError("the library is already loaded")
    LIB_PATH = path
    return lib()


def lib() -> C.CDLL:
    """Load libsonarnet_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2208_10839_b200.build`")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
    L.sn_last_error.restype = C.c_char_p
    L.sn_abi_version.restype = C.c_int
    L.sn_default_config.argtypes = [i32, C.POINTER(_Config), vp, u64]
    L.sn_default_array.argtypes = [u64, vp]
    L.sn_direction_grid.argtypes = [i32, vp, u64, C.POINTER(u64)]
    L.sn_config_dims.argtypes = [C.POINTER(_Config), C.POINTER(_Dims)]
    L.sn_synthesize_packed.argtypes = [C.POINTER(_Config), C.POINTER(_Scene), vp, u64]
    L.sn_workspace_create.argtypes = [C.POINTER(_Config), C.c_int, u64, C.POINTER(vp)]
    L.sn_workspace_create_ex.argtypes = [C.POINTER(_Config), C.c_int, u64, C.POINTER(_Options), C.POINTER(vp)]
    L.sn_fibonacci_hemisphere.argtypes = [u64, vp, u64]
    L.sn_workspace_destroy.argtypes = [vp]
    L.sn_workspace_dims.argtypes = [vp, C.POINTER(_Dims)]
    L.sn_workspace_process.argtypes = [vp, C.POINTER(_Measurement), vp]
    L.sn_workspace_process_batch.argtypes = [vp, C.POINTER(_Measurement), u64, vp]
    L.sn_workspace_process_device.argtypes = [vp, vp, u64, vp, vp]
    L.sn_workspace_process_device_graph.argtypes = [vp, vp, u64, vp, vp]
    L.sn_workspace_beamform.argtypes = [vp, vp, u64, u64, vp]
    L.sn_workspace_delay_table.argtypes = [vp, vp, u64]
    L.sn_workspace_reference_advances.argtypes = [vp, vp, u64]
    L.sn_workspace_allocation_events.argtypes = [vp]
    L.sn_workspace_allocation_events.restype = u64
    L.sn_workspace_last_launches.argtypes = [vp]
    L.sn_workspace_last_launches.restype = u64
    L.sn_workspace_table.argtypes = [vp, i32, vp, u64, C.POINTER(u64)]
    L.sn_workspace_stage.argtypes = [vp, i32, u64, vp, u64]
    L.sn_workspace_set_profiling.argtypes = [vp, C.c_int]
    L.sn_workspace_stage_times.argtypes = [vp, vp]
    L.sn_measure_fp_peak.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    L.sn_workspace_beamformer_info.argtypes = [vp, C.POINTER(_BfInfo)]
    L.sn_pool_create.argtypes = [C.POINTER(_Config), C.POINTER(C.c_int), C.c_int, C.c_int, u64, C.POINTER(vp)]
    L.sn_pool_destroy.argtypes = [vp]
    L.sn_pool_submit.argtypes = [vp, vp, u64]
    L.sn_pool_poll.argtypes = [vp, C.c_int, vp, u64, C.POINTER(u64), C.POINTER(C.c_int32),
                               C.POINTER(C.c_uint32), C.POINTER(u64)]
    L.sn_pool_stats.argtypes = [vp, C.POINTER(u64)]
    L.sn_pool_poll_view.argtypes = [vp, C.c_int, C.POINTER(C.c_void_p), C.POINTER(u64), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_uint32), C.POINTER(u64)]
    L.sn_pool_frame_bytes.restype = u64
    L.sn_pool_frame_bytes.argtypes = [vp]
    L.sn_synthesize_device.argtypes = [C.POINTER(_Config), C.POINTER(_Scene), u64, C.c_int, vp, vp]
    L.sn_crc32.restype = C.c_uint32
    L.sn_crc32.argtypes = [vp, u64]
    L.sn_measurement_frame.argtypes = [C.POINTER(_Measurement), vp, u64, C.POINTER(u64)]
    L.sn_workspace_image_frame_bytes.restype = u64
    L.sn_workspace_image_frame_bytes.argtypes = [vp]
    L.sn_workspace_process_frames.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(u64), u64, vp, u64,
                                              C.POINTER(u64), C.POINTER(C.c_int32)]
    # (bound when present: load_library() may A/B an older build of the
    # sources; the in-tree library exports every symbol of the header, which
    # tests/test_host.py checks)
    optional = {
        "sn_energyscape_transform": [vp, vp, u64, u64, i32, C.c_float, vp],
        "sn_gather_unique_id": [vp],
        "sn_gather_create": [C.c_int, C.c_int, vp, C.c_int, u64, u64, C.POINTER(vp)],
        "sn_gather_destroy": [vp],
        "sn_gather_start": [vp, C.c_int, vp, C.POINTER(FrameId), u64, vp, vp],
        "sn_gather_wait": [vp, C.c_int, vp],
        "sn_gather_ids": [vp, C.c_int, C.POINTER(FrameId), u64, C.POINTER(C.c_int32)],
        "sn_gather_elapsed": [vp, C.c_int, C.POINTER(C.c_float)],
    }
    for name, args in optional.items():
        if hasattr(L, name):
            getattr(L, name).argtypes = args
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().sn_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SonarError)(msg)


def measure_fp_peak(device: int = 0, precision: Precision = Precision.f64) -> float:
    """FMA throughput of the CUDA cores in TFLOP/s (FMA = 2 flops)."""
    v = C.c_double(0)
    _check(lib().sn_measure_fp_peak(device, int(precision), C.byref(v)))
    return v.value


# ---------------------------------------------------------------------------
class CentralPool:
    """GPU-backed central-node worker pool (sn_pool_*; central_node.cpp:48-53,
    130-160, 224-336): K workers with one Workspace each, per-sensor FIFO release.

        pool = CentralPool(cfg, devices=[0], workers_per_device=2, max_batch=8)
        pool.submit(frame)                  # raw-measurement frame (wire bytes)
        serial, seq, status, frame = pool.poll(timeout_ms=1000)
    """

    def __init__(self, cfg: PipelineConfig, devices=(0,), workers_per_device: int = 1, max_batch: int = 1):
        st, self._keep = cfg._struct()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(lib().sn_pool_create(C.byref(st), devs, len(devices), workers_per_device, max_batch, C.byref(h)))
        self._h = h
        self.frame_bytes = int(lib().sn_pool_frame_bytes(self._h))
        self._buf = np.empty(self.frame_bytes, np.uint8)

    def submit(self, frame: bytes) -> bool:
        """False when the ingest would drop the frame (bad magic/length/type)."""
        b = np.frombuffer(frame, np.uint8)
        rc = lib().sn_pool_submit(self._h, b.ctypes.data, b.size)
        if rc == IoError.status:
            return False
        _check(rc)
        return True

    def poll(self, timeout_ms: int = -1):
        """Next released result (serial, seq, status, frame_bytes), or None on timeout."""
        n, st, ser, seq = C.c_uint64(0), C.c_int32(0), C.c_uint32(0), C.c_uint64(0)
        rc = lib().sn_pool_poll(self._h, timeout_ms, self._buf.ctypes.data, self._buf.size, C.byref(n),
                                C.byref(st), C.byref(ser), C.byref(seq))
        if rc == 7:  # SN_ERR_NOT_READY
            return None
        _check(rc)
        return int(ser.value), int(seq.value), int(st.value), self._buf[:n.value].tobytes()

    def stats(self) -> dict:
        s = (C.c_uint64 * 4)()
        _check(lib().sn_pool_stats(self._h, s))
        return {"submitted": s[0], "completed": s[1], "discarded": s[2], "workers": s[3]}

    def close(self):
        if getattr(self, "_h", None):
            lib().sn_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Transform(enum.IntEnum):  # sn_transform
    normalize = 1
    db = 2


def energyscape_transform(d_energies_ptr: int, d_out_ptr: int, count: int, cells: int,
                          mode: Transform = Transform.db, floor_db: float = -60.0, stream: int = 0) -> None:
    """Opt-in display transform (north star stage 4) of `count` finished
    energyscapes in device memory into a separate device buffer; the
    reference-parity energies (max(0, float), pipeline.cpp:469-471) are left
    untouched. normalize: e / max(e); db: max(10 log10(e / max(e)), floor_db)."""
    _check(lib().sn_energyscape_transform(C.c_void_p(d_energies_ptr), C.c_void_p(d_out_ptr), int(count), int(cells),
                                          int(mode), float(floor_db), C.c_void_p(stream or 1)))


def crc32(data) -> int:
    """wire::crc32 (wire.cpp:58-63), host implementation of the C ABI."""
    b = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8))
    return int(lib().sn_crc32(b.ctypes.data if b.size else None, b.size))


def measurement_frame(m: "RawMeasurement") -> bytes:
    """wire::measurement_frame (wire.cpp:251-259): the frame a sensor sends."""
    st, _keep = m._struct()
    n = C.c_uint64(0)
    _check(lib().sn_measurement_frame(C.byref(st), None, 0, C.byref(n)))
    out = np.empty(n.value, np.uint8)
    _check(lib().sn_measurement_frame(C.byref(st), out.ctypes.data, out.size, C.byref(n)))
    return out.tobytes()


def default_array(seed: int = 42) -> np.ndarray:
    """geometry.cpp:69-96 — 32 x 3 microphone positions (m)."""
    out = np.zeros(96, np.float64)
    _check(lib().sn_default_array(seed, out.ctypes.data))
    return out.reshape(32, 3)


def direction_grid(kind: GridKind) -> np.ndarray:
    """geometry.cpp:181-235 — n x (azimuth, elevation) radians."""
    n = C.c_uint64(0)
    _check(lib().sn_direction_grid(int(kind), None, 0, C.byref(n)))
    out = np.zeros((n.value, 2), np.float64)
    _check(lib().sn_direction_grid(int(kind), out.ctypes.data, n.value, C.byref(n)))
    return out


def fibonacci_hemisphere(n: int) -> np.ndarray:
    """geometry.cpp:206-229 with n points (n = 3000: hemisphere3000) — n x (az, el)."""
    out = np.zeros((int(n), 2), np.float64)
    _check(lib().sn_fibonacci_hemisphere(int(n), out.ctypes.data, int(n)))
    return out


@dataclass
class PipelineConfig:
    """sonarnet::PipelineConfig (pipeline.hpp:22-55), flattened."""
    mic_xyz: np.ndarray = field(default_factory=lambda: default_array(42))
    directions: np.ndarray = field(default_factory=lambda: direction_grid(GridKind.horizontal90))
    grid_kind: int = GridKind.horizontal90
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
    precision: int = Precision.f64
    speed_of_sound: float = 343.0
    max_range: float = 5.0

    def _struct(self):
        c = _Config()
        xyz = np.ascontiguousarray(self.mic_xyz, dtype=np.float64).reshape(96)
        C.memmove(c.mic_xyz, xyz.ctypes.data, 96 * 8)
        dirs = np.ascontiguousarray(self.directions, dtype=np.float64).reshape(-1, 2)
        c.directions = dirs.ctypes.data_as(C.POINTER(C.c_double))
        c.n_directions = dirs.shape[0]
        for name, _ in _Config._fields_[3:]:
            setattr(c, name, type(getattr(c, name))(getattr(self, name)))
        return c, dirs

    # derived quantities (pipeline.hpp:38-50)
    def dims(self) -> dict:
        st, _k = self._struct()
        d = _Dims()
        _check(lib().sn_config_dims(C.byref(st), C.byref(d)))
        return {n: getattr(d, n) for n, _ in _Dims._fields_}

    def frames(self) -> int:
        return int(self.dims()["frames"])

    def range_bins(self) -> int:
        return int(self.dims()["range_bins"])

    def demod_rate(self) -> float:
        return self.pdm_rate / self.demod_decimation

    def mf_rate(self) -> float:
        return self.demod_rate() / self.pre_mf_decimation

    def final_rate(self) -> float:
        return self.mf_rate() / self.post_envelope_decimation

    def range_bin_size(self) -> float:
        return self.speed_of_sound / (2.0 * self.final_rate())

    def validate(self):
        self.dims()

    def copy(self, **kw) -> "PipelineConfig":
        d = dict(self.__dict__)
        d.update(kw)
        return PipelineConfig(**d)


def default_pipeline_config(kind: GridKind = GridKind.horizontal90) -> PipelineConfig:
    """pipeline.cpp:94-99."""
    return PipelineConfig(mic_xyz=default_array(42), directions=direction_grid(kind),
                          grid_kind=int(kind))


@dataclass
class RawMeasurement:
    """wire::RawMeasurement (wire.hpp:97-107)."""
    sensor_serial: int = 0
    timestamp_us: int = 0
    seq: int = 0
    channels: int = 0
    frames: int = 0
    pdm_rate: float = 0.0
    packed: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    def _struct(self):
        pk = np.ascontiguousarray(self.packed, dtype=np.uint8)
        return _Measurement(self.sensor_serial, self.timestamp_us, self.seq, self.channels,
                            self.frames, self.pdm_rate, pk.ctypes.data_as(C.POINTER(C.c_uint8)),
                            pk.size), pk


@dataclass
class Reflector:  # synth.hpp:13-18
    range: float = 1.0
    azimuth: float = 0.0
    elevation: float = 0.0
    reflectivity: float = 1.0


@dataclass
class Scene:  # synth.hpp:20-24
    reflectors: List[Reflector] = field(default_factory=list)
    noise_rms: float = 0.0
    seed: int = 0


def synthesize_measurement(cfg: PipelineConfig, scene: Scene, serial: int = 1,
                           timestamp_us: int = 0, seq: int = 0) -> RawMeasurement:
    """synth.cpp:116-134 (host-side load generator, bit-exact with the reference)."""
    st, _k = cfg._struct()
    n = len(scene.reflectors)
    arr = (_Reflector * max(1, n))()
    for i, r in enumerate(scene.reflectors):
        arr[i] = _Reflector(r.range, r.azimuth, r.elevation, r.reflectivity)
    sc = _Scene(arr, n, scene.noise_rms, scene.seed)
    frames = cfg.frames()
    out = np.zeros(32 * frames // 8, np.uint8)
    _check(lib().sn_synthesize_packed(C.byref(st), C.byref(sc), out.ctypes.data, out.size))
    return RawMeasurement(serial, timestamp_us, seq, 32, frames, cfg.pdm_rate, out)


def synthesize_device(cfg: PipelineConfig, scenes: Sequence[Scene], d_packed_ptr: int, device: int = 0,
                      stream: int = 0) -> None:
    """GPU load generator (sn_synthesize_device): len(scenes) packed captures
    (32 * frames / 8 bytes each, synth.cpp:116-134) written to device memory at
    d_packed_ptr, one capture per GPU thread."""
    st, _k = cfg._struct()
    n = len(scenes)
    keep = []
    arr = (_Scene * max(1, n))()
    for i, sc in enumerate(scenes):
        refl = (_Reflector * max(1, len(sc.reflectors)))()
        for k, r in enumerate(sc.reflectors):
            refl[k] = _Reflector(r.range, r.azimuth, r.elevation, r.reflectivity)
        keep.append(refl)
        arr[i] = _Scene(refl, len(sc.reflectors), sc.noise_rms, sc.seed)
    _check(lib().sn_synthesize_device(C.byref(st), arr, n, device, d_packed_ptr, stream))


@dataclass
class AcousticImage:
    """pipeline.hpp:66-81."""
    sensor_serial: int
    timestamp_us: int
    directions: np.ndarray
    range_bin_size: float
    range_bins: int
    energies: np.ndarray  # (n_dirs, range_bins) float32

    def at(self, direction: int, bin: int) -> float:
        return float(self.energies[direction, bin])

    def range_for_bin(self, bin: int) -> float:
        return bin * self.range_bin_size

    def argmax(self):
        i = int(np.argmax(self.energies.reshape(-1)))  # first maximum, like pipeline.cpp:101-107
        return i // self.range_bins, i % self.range_bins


class Workspace:
    """sonarnet::Workspace (pipeline.hpp:95-130) on one B200.

    device=None picks the current torch device if torch is initialised, else 0;
    device=-1 builds the host tables only (no GPU needed; process raises).
    beamformer / tc_tile_n / beam_budget_bytes: sn_workspace_options.
    """

    def __init__(self, cfg: PipelineConfig, device: Optional[int] = 0, max_batch: int = 1,
                 beamformer: Beamformer = Beamformer.tensor_core, tc_tile_n: int = 0,
                 beam_budget_bytes: int = 0):
        self._cfg = cfg
        st, _k = cfg._struct()
        h = C.c_void_p()
        dev = 0 if device is None else int(device)
        opt = _Options(int(beamformer), int(tc_tile_n), int(beam_budget_bytes))
        _check(lib().sn_workspace_create_ex(C.byref(st), dev, max(1, int(max_batch)), C.byref(opt), C.byref(h)))
        self._h = h
        d = _Dims()
        _check(lib().sn_workspace_dims(h, C.byref(d)))
        self.dims = {n: getattr(d, n) for n, _ in _Dims._fields_}
        self.n_dirs = int(d.n_directions)
        self.bins = int(d.range_bins)
        self.frames = int(d.frames)
        self.max_batch = int(d.max_batch)
        self.packed_bytes = 32 * self.frames // 8

    def close(self):
        if getattr(self, "_h", None):
            lib().sn_workspace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def config(self) -> PipelineConfig:
        return self._cfg

    def process(self, m: RawMeasurement) -> AcousticImage:
        st, _pk = m._struct()
        out = np.empty((self.n_dirs, self.bins), np.float32)
        _check(lib().sn_workspace_process(self._h, C.byref(st), out.ctypes.data))
        return AcousticImage(m.sensor_serial, m.timestamp_us, np.array(self._cfg.directions),
                             self.dims["range_bin_size"], self.bins, out)

    def process_batch(self, ms: Sequence[RawMeasurement]) -> List[AcousticImage]:
        structs = (_Measurement * max(1, len(ms)))()
        keep = []
        for i, m in enumerate(ms):
            s, pk = m._struct()
            structs[i] = s
            keep.append(pk)
        out = np.empty((len(ms), self.n_dirs, self.bins), np.float32)
        _check(lib().sn_workspace_process_batch(self._h, structs, len(ms), out.ctypes.data))
        return [AcousticImage(m.sensor_serial, m.timestamp_us, np.array(self._cfg.directions),
                              self.dims["range_bin_size"], self.bins, out[i])
                for i, m in enumerate(ms)]

    @property
    def image_frame_bytes(self) -> int:
        """Size of one processed-image frame (wire::image_frame) of this config."""
        return int(lib().sn_workspace_image_frame_bytes(self._h))

    def process_frames(self, frames: Sequence[bytes], out: Optional[np.ndarray] = None):
        """The central node's path for received frames (sn_workspace_process_frames):
        returns [(status, frame_bytes)] — status 0 with the processed-image
        frame, DecodeError.status with the reference's error frame, IoError.status
        (discarded: malformed / CRC mismatch / not a measurement) with b""."""
        n = len(frames)
        slot = self.image_frame_bytes
        keep = [np.frombuffer(f, np.uint8) for f in frames]
        ptrs = (C.c_void_p * max(1, n))(*[k.ctypes.data for k in keep])
        lens = (C.c_uint64 * max(1, n))(*[k.size for k in keep])
        if out is None or out.size < n * slot:
            out = np.empty(max(1, n) * slot, np.uint8)
        olen = (C.c_uint64 * max(1, n))()
        st = (C.c_int32 * max(1, n))()
        _check(lib().sn_workspace_process_frames(self._h, ptrs, lens, n, out.ctypes.data, slot, olen, st))
        return [(int(st[i]), out[i * slot:i * slot + olen[i]].tobytes()) for i in range(n)]

    def process_packed_host(self, packed: np.ndarray, out: np.ndarray):
        """Fast host path for B equal-sized captures already packed as
        (B, packed_bytes) uint8 (e.g. pinned); out (B, n_dirs, bins) f32."""
        B = packed.shape[0]
        # the sn_raw_measurement array built column-wise in numpy (a Python
        # loop over ctypes structs cost 0.3 ms per 128 captures)
        a = np.zeros(B, _measurement_dtype())
        a["sensor_serial"] = 1
        a["seq"] = np.arange(B, dtype=np.uint64)
        a["channels"] = 32
        a["frames"] = self.frames
        a["pdm_rate"] = self._cfg.pdm_rate
        a["packed"] = np.uint64(packed.ctypes.data) + np.arange(B, dtype=np.uint64) * np.uint64(packed.strides[0])
        a["packed_len"] = self.packed_bytes
        structs = (_Measurement * B).from_buffer(a)
        _check(lib().sn_workspace_process_batch(self._h, structs, B, out.ctypes.data))
        return out

    def process_device(self, d_packed_ptr: int, count: int, d_energy_ptr: int, stream: int = 0,
                       graph: bool = False):
        """Device-resident path (raw device pointers, e.g. torch tensor data_ptr())."""
        # stream 0 is torch's legacy default stream: pass cudaStreamLegacy (0x1),
        # since NULL at the C ABI selects the workspace's own stream.
        fn = lib().sn_workspace_process_device_graph if graph else lib().sn_workspace_process_device
        _check(fn(self._h, C.c_void_p(d_packed_ptr), count, C.c_void_p(d_energy_ptr),
                  C.c_void_p(stream if stream else 1)))

    def beamform(self, filtered: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(filtered, dtype=np.float64)
        if f.ndim != 2:
            raise ArgumentError("beamform: expected a (channels, samples) matrix")
        out = np.empty((self.n_dirs, f.shape[1]), np.float64)
        _check(lib().sn_workspace_beamform(self._h, f.ctypes.data, f.shape[0], f.shape[1],
                                           out.ctypes.data))
        return out

    def delay_table(self) -> np.ndarray:
        out = np.empty((self.n_dirs, 32), np.int32)
        _check(lib().sn_workspace_delay_table(self._h, out.ctypes.data, out.size))
        return out

    def reference_advances(self) -> np.ndarray:
        out = np.empty(self.n_dirs, np.int32)
        _check(lib().sn_workspace_reference_advances(self._h, out.ctypes.data, out.size))
        return out

    def allocation_events(self) -> int:
        return int(lib().sn_workspace_allocation_events(self._h))

    def last_launches(self) -> int:
        return int(lib().sn_workspace_last_launches(self._h))

    def table(self, which: int) -> np.ndarray:
        n = C.c_uint64(0)
        _check(lib().sn_workspace_table(self._h, which, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        _check(lib().sn_workspace_table(self._h, which, out.ctypes.data, n.value, C.byref(n)))
        return out

    def beamformer_info(self) -> dict:
        """Delay-and-sum schedule (sn_workspace_beamformer_info): kind 1 =
        tensor-core path with its cluster / tile / MMA-shape figures."""
        info = _BfInfo()
        _check(lib().sn_workspace_beamformer_info(self._h, C.byref(info)))
        return {f: getattr(info, f) for f, _ in _BfInfo._fields_}

    def set_profiling(self, enable: bool = True):
        _check(lib().sn_workspace_set_profiling(self._h, int(enable)))

    def stage_times(self) -> dict:
        """Device ms of {demod, premf, matched_filter, beamform, envelope} of the last call."""
        out = np.zeros(5, np.float32)
        _check(lib().sn_workspace_stage_times(self._h, out.ctypes.data))
        return dict(zip(STAGES, map(float, out)))

    def stage(self, which: int, item: int = 0) -> np.ndarray:
        """Stage buffers of capture `item` of the last call: 0 demod, 1 pre-MF,
        2 matched filter (32 x samples), 3 beams (n_dirs x mf_samples)."""
        L = self.dims["demod_samples"] if which == 0 else self.dims["mf_samples"]
        out = np.empty((self.n_dirs if which == 3 else 32, L), np.float64)
        _check(lib().sn_workspace_stage(self._h, which, item, out.ctypes.data, out.size))
        return out
