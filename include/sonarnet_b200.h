/*
 * sonarnet_b200 — C ABI of the B200-native eRTIS image-formation path.
 *
 * Drop-in boundary for the reference's only caller contract, the pimpl class
 * `sonarnet::Workspace` (/root/reference/proj/core/include/sonarnet/pipeline.hpp:95-130,
 * implementation pipeline.cpp:191-591). Plain pointers and sizes only; no
 * exceptions and no torch types cross this boundary. Every entry point returns
 * an sn_status that mirrors the reference error taxonomy
 * (errors.hpp:11-29; CLI exit-code mapping tools/main.cpp:332-350):
 *
 *   SN_ERR_CONFIG   <- sonarnet::ConfigError   (Workspace ctor / validate)
 *   SN_ERR_ARGUMENT <- sonarnet::ArgumentError (beamform shape, geometry)
 *   SN_ERR_DECODE   <- sonarnet::DecodeError   (process input mismatch)
 *   SN_ERR_IO       <- sonarnet::IoError
 *   SN_ERR_CUDA     device / driver failure (no reference analogue)
 *
 * The message of the last failure on the calling thread is available from
 * sn_last_error().
 *
 * Threading (pipeline.hpp:95-97): one in-flight call per
 * workspace; many workspaces may share a device. Each workspace owns one CUDA
 * stream and all of its device buffers, allocated at creation; process calls
 * never allocate (allocation_events stays 0, test_pipeline.cpp:143-155).
 */
#ifndef SONARNET_B200_H
#define SONARNET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SN_CHANNELS 32 /* geometry.hpp:11 kChannelCount */
#define SN_ABI_VERSION 1

typedef enum sn_status {
    SN_OK = 0,
    SN_ERR_CONFIG = 1,
    SN_ERR_ARGUMENT = 2,
    SN_ERR_DECODE = 3,
    SN_ERR_IO = 4,
    SN_ERR_CUDA = 5,
    SN_ERR_INTERNAL = 6,
    SN_ERR_NOT_READY = 7   /* sn_pool_poll: nothing released within the timeout */
} sn_status;

/* geometry.hpp:65 GridKind */
typedef enum sn_grid_kind {
    SN_GRID_HORIZONTAL90 = 0,
    SN_GRID_BOX1850 = 1,
    SN_GRID_HEMISPHERE3000 = 2,
    SN_GRID_CUSTOM = 3
} sn_grid_kind;

/* Arithmetic of the per-direction stage (beamform, Hilbert envelope,
 * smoothing). The front end (demodulation, pre-MF decimation) is always the
 * reference's FP64 arithmetic, bit-exact; the matched filter is FP64. */
typedef enum sn_precision {
    SN_PRECISION_F64 = 0, /* FP64 throughout (default) */
    SN_PRECISION_F32 = 1  /* FP32 per-direction stage, FP64 front end */
} sn_precision;

/* Flat restatement of sonarnet::PipelineConfig (pipeline.hpp:22-55).
 * `directions` is borrowed for the duration of sn_workspace_create only. */
typedef struct sn_pipeline_config {
    double mic_xyz[SN_CHANNELS * 3]; /* ArrayGeometry positions (x,y,z) m      */
    const double* directions;        /* n_directions x (azimuth, elevation) rad */
    uint64_t n_directions;
    int32_t grid_kind;               /* sn_grid_kind, informational            */
    int32_t processing_threads;      /* accepted for API parity; unused on GPU */
    double pdm_rate;                 /* Hz, default 4.5e6                       */
    double chirp_f_start;            /* Hz, default 90e3                        */
    double chirp_f_end;              /* Hz, default 25e3                        */
    double chirp_duration;           /* s,  default 3e-3                        */
    double demod_cutoff_hz;          /* default 126e3                           */
    int32_t demod_taps;              /* default 255                             */
    int32_t demod_decimation;        /* default 10                              */
    int32_t pre_mf_decimation;       /* default 2                               */
    int32_t post_envelope_decimation;/* default 10                              */
    double smoothing_cutoff_hz;      /* default 10e3                            */
    int32_t smoothing_taps;          /* default 127                             */
    int32_t precision;               /* sn_precision                            */
    double speed_of_sound;           /* m/s, default 343                        */
    double max_range;                /* m, default 5                            */
} sn_pipeline_config;

/* wire::RawMeasurement (wire.hpp:97-107). `packed` is frame-major, bit index
 * = frame*channels + channel, MSB first, 1 -> +1 (dsp.hpp:67-69). */
typedef struct sn_raw_measurement {
    uint32_t sensor_serial;
    uint64_t timestamp_us;
    uint64_t seq;
    uint16_t channels;
    uint64_t frames;
    double pdm_rate;
    const uint8_t* packed;
    uint64_t packed_len;
} sn_raw_measurement;

/* Derived sizes (pipeline.hpp:44-50, pipeline.cpp:40-52, 250-259). */
typedef struct sn_dims {
    uint64_t frames;
    uint64_t demod_samples;
    uint64_t mf_samples;
    uint64_t range_bins;
    uint64_t n_directions;
    uint64_t ref_len;        /* reference chirp length at the MF rate */
    uint64_t mf_fft_size;    /* next_pow2(mf_samples + ref_len - 1)   */
    uint64_t env_fft_size;   /* next_pow2(mf_samples)                  */
    uint64_t smoothing_len;  /* composite smoothing+anti-alias taps    */
    double range_bin_size;   /* m */
    double demod_rate, mf_rate, final_rate;
    uint64_t max_batch;      /* measurements per device launch          */
} sn_dims;

/* synth.hpp:13-25 Reflector / Scene. `reflectors` borrowed for the call. */
typedef struct sn_reflector {
    double range;
    double azimuth;
    double elevation;
    double reflectivity;
} sn_reflector;

typedef struct sn_scene {
    const sn_reflector* reflectors;
    uint64_t n_reflectors;
    double noise_rms;
    uint64_t seed;
} sn_scene;

typedef struct sn_workspace sn_workspace;

/* Intermediate stage buffers (test / parity access; Workspace::Impl members
 * pipeline.cpp:211-220). */
typedef enum sn_stage {
    SN_STAGE_DEMOD = 0, /* 32 x demod_samples f64 (demod_buf)   */
    SN_STAGE_PREMF = 1, /* 32 x mf_samples f64    (mf_buf)      */
    SN_STAGE_FILT = 2,  /* 32 x mf_samples f64    (filt_buf)    */
    SN_STAGE_BEAMS = 3  /* n_directions x mf_samples: the hot path's delay-and-sum
                           of that measurement (beamform_into, pipeline.cpp:432-446),
                           direction order, f64 (f32 beams widened in F32 mode);
                           recomputed on demand by the same kernels (deterministic) */
} sn_stage;

/* ---- library ---------------------------------------------------------- */
int sn_abi_version(void);
const char* sn_last_error(void);
const char* sn_status_name(sn_status s);

/* ---- setup helpers (host only; no GPU needed) ------------------------- */
/* PipelineConfig defaults + default_array(42) + grid (pipeline.cpp:94-99).
 * For a built-in grid the direction table is written into `dir_buf`
 * (capacity in directions) and cfg->directions points at it. */
sn_status sn_default_config(int32_t grid_kind, sn_pipeline_config* cfg, double* dir_buf,
                            uint64_t dir_capacity);
/* geometry.cpp:69-96 default_array(seed) -> 96 doubles */
sn_status sn_default_array(uint64_t seed, double* mic_xyz_out);
/* geometry.cpp:181-235 direction_grid(kind) -> n x (az, el) */
sn_status sn_direction_grid(int32_t grid_kind, double* out, uint64_t capacity,
                            uint64_t* n_out);
/* The Fibonacci lattice of hemisphere3000 (geometry.cpp:206-229) with n
 * points instead of 3000 (n = 3000 reproduces the built-in grid exactly):
 * n x (az, el) into `out`; the configs[4] sweep's dense custom grids. */
sn_status sn_fibonacci_hemisphere(uint64_t n, double* out, uint64_t capacity);
/* pipeline.cpp:60-92 PipelineConfig::validate + derived sizes. */
sn_status sn_config_dims(const sn_pipeline_config* cfg, sn_dims* dims);
/* synth.cpp:116-134 synthesize_measurement: packed bytes of one capture.
 * `packed_out` must hold 32*frames/8 bytes. */
sn_status sn_synthesize_packed(const sn_pipeline_config* cfg, const sn_scene* scene,
                               uint8_t* packed_out, uint64_t capacity);

/* Synthetic captures on the GPU (load generation): `count` scenes (each with
 * its own seed, <= 8 reflectors) -> count x (32 * frames / 8) packed bytes in
 * DEVICE memory on `device`, identical to sn_synthesize_packed (synth.cpp:
 * 116-134) up to last-place differences of the device log() (a sigma-delta
 * decision changes only where |integrator + x| < ~1e-16). One capture per
 * GPU thread (the noise stream is sequential); a batch runs in parallel. */
sn_status sn_synthesize_device(const sn_pipeline_config* cfg, const sn_scene* scenes, uint64_t count, int device,
                               uint8_t* d_packed, void* stream);

/* ---- workspace (Workspace, pipeline.hpp:98-130) ------------------------ */
/* device >= 0: allocate every device buffer on that CUDA device (no
 * allocation ever happens later). device < 0: host tables only (setup
 * parity checks on machines without a GPU); process calls then fail with
 * SN_ERR_CUDA. max_batch: largest batch a single process call may carry. */
sn_status sn_workspace_create(const sn_pipeline_config* cfg, int device, uint64_t max_batch,
                              sn_workspace** out);
/* Device-side choices of a workspace (no effect on results beyond the
 * per-stage tolerances of DESIGN.md §5); zero-initialised = defaults. */
typedef enum sn_beamformer_kind {
    SN_BEAMFORMER_TENSOR_CORE = 0, /* tcgen05 int8 delay-and-sum (default)        */
    SN_BEAMFORMER_CUDA_CORE = 1    /* FP64 CUDA-core tiles, bit-identical beams   */
} sn_beamformer_kind;
typedef struct sn_workspace_options {
    int32_t beamformer;          /* sn_beamformer_kind                                 */
    int32_t tc_tile_n;           /* tensor-core tile width: 0 = 96; 64, 96 or 128      */
    uint64_t beam_budget_bytes;  /* 0 = 4 GiB: device bytes of the beam ring (beams +
                                    digit planes of the captures one chunk of a batch
                                    holds); larger grids/windows run more chunks      */
} sn_workspace_options;
/* sn_workspace_create with options (NULL = defaults). */
sn_status sn_workspace_create_ex(const sn_pipeline_config* cfg, int device, uint64_t max_batch,
                                 const sn_workspace_options* options, sn_workspace** out);
void sn_workspace_destroy(sn_workspace* ws);
sn_status sn_workspace_dims(const sn_workspace* ws, sn_dims* dims);

/* Workspace::process (pipeline.cpp:522-574): host bytes in, host energies
 * out (n_directions x range_bins f32, row-major). All-or-error. */
sn_status sn_workspace_process(sn_workspace* ws, const sn_raw_measurement* m,
                               float* energies_out);
/* B measurements, identical per-measurement semantics; results do not
 * depend on B. Validates every measurement before any device work. */
sn_status sn_workspace_process_batch(sn_workspace* ws, const sn_raw_measurement* ms,
                                     uint64_t count, float* energies_out);
/* Device-resident variant: d_packed = count x (32*frames/8) bytes already in
 * device memory, d_energies = count x n_dirs x bins f32 device buffer.
 * Enqueued on `stream` (cudaStream_t, NULL = the workspace stream); does not
 * synchronise. Inputs are trusted (no host-side validation possible). */
sn_status sn_workspace_process_device(sn_workspace* ws, const uint8_t* d_packed,
                                      uint64_t count, float* d_energies, void* stream);

/* Workspace::beamform (pipeline.cpp:576-591): filtered = 32 x mf_samples
 * f64 host, out = n_dirs x mf_samples f64 host. ArgumentError on shape. */
sn_status sn_workspace_beamform(sn_workspace* ws, const double* filtered, uint64_t channels,
                                uint64_t samples, double* out);

/* Accessors (pipeline.hpp:108-125). */
sn_status sn_workspace_delay_table(const sn_workspace* ws, int32_t* out, uint64_t capacity);
sn_status sn_workspace_reference_advances(const sn_workspace* ws, int32_t* out,
                                          uint64_t capacity);
uint64_t sn_workspace_allocation_events(const sn_workspace* ws);

/* Setup tables (host copies), for parity tests of the setup stage. */
typedef enum sn_table {
    SN_TABLE_DEMOD_TAPS_REV = 0,   /* demod_rev, demod_taps f64              */
    SN_TABLE_DEMOD_LUT = 1,        /* 8 x octets x 256 f64                   */
    SN_TABLE_PREMF_TAPS_REV = 2,   /* premf_rev f64                          */
    SN_TABLE_CHIRP_REF = 3,        /* reference chirp @ mf rate, ref_len f64 */
    SN_TABLE_SMOOTH_REV = 4        /* smooth_decimate_rev f64                */
} sn_table;
sn_status sn_workspace_table(const sn_workspace* ws, int32_t table, double* out,
                             uint64_t capacity, uint64_t* n_out);

/* Stage dump of the measurement most recently processed (index `item`
 * of that batch): sn_stage buffers as f64 host arrays. */
sn_status sn_workspace_stage(sn_workspace* ws, int32_t stage, uint64_t item, double* out,
                             uint64_t capacity);

/* Number of kernel launches issued by the last process call (for the bench
 * `gpu_launches` claim). */
uint64_t sn_workspace_last_launches(const sn_workspace* ws);

/* CUDA-graph replay of the device path for a fixed (count, d_packed,
 * d_energies) triple: captured on first use, replayed afterwards. */
sn_status sn_workspace_process_device_graph(sn_workspace* ws, const uint8_t* d_packed,
                                            uint64_t count, float* d_energies, void* stream);

/* Per-stage device timing of the next process calls (CUDA events on the
 * launching stream). stage_times: ms for {demod, premf, matched filter,
 * beamform, envelope} of the most recent call. Diagnostics for the roofline
 * report. */
sn_status sn_workspace_set_profiling(sn_workspace* ws, int enable);
sn_status sn_workspace_stage_times(sn_workspace* ws, float* ms5);

/* Delay-and-sum schedule of a device workspace. kind 1: tensor-core path
 * (tcgen05 int8 MMAs over direction clusters, beamform_tc.cu); kind 0: the
 * CUDA-core tiled kernel (SNB_BEAMFORMER=tiles). For kind 1, the MMA work of
 * one capture is sum_R * ntiles * slices MMAs of m x n x k int8 MACs. */
typedef struct sn_beamformer_info {
    int32_t kind;
    int32_t clusters;     /* direction clusters (<= m directions each)        */
    int64_t sum_R;        /* sum over clusters of the shift values R_c        */
    int32_t max_R;
    int32_t ntiles;       /* time tiles of n samples per capture              */
    int32_t slices;       /* int8 digit planes of the 46-bit samples          */
    int32_t m, n, k;      /* MMA shape                                        */
} sn_beamformer_info;
sn_status sn_workspace_beamformer_info(const sn_workspace* ws, sn_beamformer_info* info);

/* ---- wire format (protocol.md) ------------------------------------------
 * The central node's traffic around Workspace::process: raw-measurement frames
 * in (wire::measurement_frame, wire.cpp:251-259), processed-image frames out
 * (wire::image_frame(image_to_bytes(img), seq), wire.cpp:268-276,
 * pipeline.cpp:109-125). CRC-32 as wire::crc32 (wire.cpp:58-63). */
uint32_t sn_crc32(const uint8_t* bytes, uint64_t n);
sn_status sn_measurement_frame(const sn_raw_measurement* m, uint8_t* out, uint64_t capacity, uint64_t* n_out);
/* Size of one processed-image frame of this workspace's configuration. */
uint64_t sn_workspace_image_frame_bytes(const sn_workspace* ws);
/* Process `count` received frames (central_node.cpp:130-160, 238-270):
 * per frame i, out + i * slot_bytes receives out_lens[i] bytes and status[i] is
 *   SN_OK          the processed-image frame (AIMG payload, CRC) — encoded and
 *                  CRC'd on the GPU, input CRC verified on the GPU
 *   SN_ERR_DECODE  process() rejected the measurement: wire::error_frame
 *   SN_ERR_IO      malformed, CRC mismatch or not a measurement: discarded (0 bytes)
 * slot_bytes >= sn_workspace_image_frame_bytes(ws). */
sn_status sn_workspace_process_frames(sn_workspace* ws, const uint8_t* const* frames, const uint64_t* lens,
                                      uint64_t count, uint8_t* out, uint64_t slot_bytes, uint64_t* out_lens,
                                      int32_t* status);

/* ---- GPU-backed central-node worker pool (central_node.cpp:48-53, 130-160,
 * 224-336) ----------------------------------------------------------------
 * K = n_devices x workers_per_device workers, each owning a Workspace; frames
 * are ticketed per sensor at submission, processed in device batches of up to
 * max_batch (sn_workspace_process_frames), and released strictly in per-sensor
 * submission order. submit blocks while the input queue is full (backpressure)
 * and returns SN_ERR_IO for a frame the ingest would drop (bad magic, length,
 * version or type). poll returns the next released result: status SN_OK with
 * the processed-image frame, SN_ERR_DECODE with the reference's error frame,
 * SN_ERR_IO (CRC mismatch, discarded) with no bytes; out == NULL peeks at the
 * length without consuming. */
typedef struct sn_pool sn_pool;
sn_status sn_pool_create(const sn_pipeline_config* cfg, const int* devices, int n_devices,
                         int workers_per_device, uint64_t max_batch, sn_pool** out);
void sn_pool_destroy(sn_pool* pool);
sn_status sn_pool_submit(sn_pool* pool, const uint8_t* frame, uint64_t len);
sn_status sn_pool_poll(sn_pool* pool, int timeout_ms, uint8_t* out, uint64_t capacity, uint64_t* len,
                       int32_t* status, uint32_t* serial, uint64_t* seq);
/* Zero-copy variant: *data points at the released frame inside the pool's
 * page-locked result block, valid until the next sn_pool_poll_view call. */
sn_status sn_pool_poll_view(sn_pool* pool, int timeout_ms, const uint8_t** data, uint64_t* len, int32_t* status,
                            uint32_t* serial, uint64_t* seq);
/* stats: submitted, completed, discarded (CRC), workers */
sn_status sn_pool_stats(sn_pool* pool, uint64_t* stats4);
uint64_t sn_pool_frame_bytes(const sn_pool* pool);

/* ---- multi-sensor 360-degree view (BASELINE configs[2]) ---
 * One sensor per GPU, one process per GPU; the energyscapes of a trigger are
 * gathered to rank 0 over NCCL (bound at run time from libnccl.so.2) on the
 * gather's own stream, into one of two view slots (double buffering: step k's
 * gather overlaps step k + 1). The ids travel with the images; a trigger is
 * the same (timestamp_us, seq) on every sensor (nodes/sync.hpp:16-19).
 * Replaces the reference's per-sensor fan-out of images to subscribers
 * (central_node.cpp:272-336) for the co-located 8-GPU network. */
#define SN_GATHER_ID_BYTES 128 /* NCCL_UNIQUE_ID_BYTES */
typedef struct sn_frame_id {
    uint32_t sensor_serial;
    uint32_t reserved;
    uint64_t timestamp_us;
    uint64_t seq;
} sn_frame_id;
typedef struct sn_gather sn_gather;
/* rank 0 creates the id and shares it out of band (e.g. a TCP store). */
sn_status sn_gather_unique_id(uint8_t* id_out /* SN_GATHER_ID_BYTES */);
/* collective over the `world` ranks; image_floats = n_dirs * range_bins;
 * max_count = images per rank per gather. */
sn_status sn_gather_create(int rank, int world, const uint8_t* id, int device, uint64_t image_floats,
                           uint64_t max_count, sn_gather** out);
void sn_gather_destroy(sn_gather* g);
/* After the work already enqueued on `stream` (the producer of d_images),
 * gather `count` images (count x image_floats f32, device) and their ids
 * (host) from every rank into slot `slot` (0/1) of rank 0's d_view (device,
 * world x count x image_floats, rank-major; ignored elsewhere). Returns once
 * enqueued (after waiting on the host for the slot's previous gather, whose
 * id staging it reuses); collective: every rank calls it with the same slot
 * and count. */
sn_status sn_gather_start(sn_gather* g, int slot, const float* d_images, const sn_frame_id* ids, uint64_t count,
                          float* d_view, void* stream);
/* Make `stream` wait for slot's last gather (NULL: block the host) — call
 * before overwriting the images or reading the view of that slot. */
sn_status sn_gather_wait(sn_gather* g, int slot, void* stream);
/* rank 0: the gathered ids of slot (world x count, rank-major, blocks until
 * done) and whether every rank's image i belongs to the same trigger. */
sn_status sn_gather_ids(sn_gather* g, int slot, sn_frame_id* out, uint64_t capacity, int32_t* synchronized);
/* device ms of slot's last gather (its own stream, CUDA events). */
sn_status sn_gather_elapsed(sn_gather* g, int slot, float* ms);

/* ---- opt-in display transform (north star stage 4: log/normalisation) ----
 * Not part of Workspace::process: the reference writes max(0, float) energies
 * (pipeline.cpp:469-471) and so does every process entry point. This maps
 * `count` finished energyscapes of `cells` floats each (device memory) into a
 * SEPARATE device buffer, per image: NORMALIZE e / max(e); DB
 * max(10 log10(e / max(e)), floor_db) (floor_db where e == 0). Enqueued on
 * `stream`; in == out is rejected (the energies stay untouched). */
typedef enum sn_transform {
    SN_TRANSFORM_NORMALIZE = 1,
    SN_TRANSFORM_DB = 2
} sn_transform;
sn_status sn_energyscape_transform(const float* d_energies, float* d_out, uint64_t count, uint64_t cells,
                                   int32_t mode, float floor_db, void* stream);

/* FMA-throughput microbenchmark on `device` (TFLOP/s, FMA = 2 flops); the
 * roofline denominator for CUDA-core kernels (no tensor cores involved). */
sn_status sn_measure_fp_peak(int device, int precision, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* SONARNET_B200_H */
