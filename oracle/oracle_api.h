/* TEST INFRASTRUCTURE ONLY — the oracle's C interface.
 *
 * Two implementations export this interface:
 *   oracle/_ref/libsonarnet_ref.so   the UNMODIFIED reference C++ sources
 *                                    (/root/reference/proj/core/src/*.cpp)
 *                                    compiled by oracle/Makefile, wrapped by
 *                                    oracle/ref_capi.cpp   (prefix ref_)
 *   oracle/_build/libsonarnet_port.so a plain-C restatement of the same path,
 *                                    oracle/sonarnet_port.c (prefix port_)
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load either library; the product never does.
 *
 * The config/measurement/scene structs are layout-identical to the product's
 * sn_pipeline_config / sn_raw_measurement / sn_scene (include/sonarnet_b200.h)
 * so one ctypes description serves both.
 */
#ifndef SONARNET_ORACLE_API_H
#define SONARNET_ORACLE_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_config {
    double mic_xyz[96];
    const double* directions;
    uint64_t n_directions;
    int32_t grid_kind;
    int32_t processing_threads;
    double pdm_rate;
    double chirp_f_start;
    double chirp_f_end;
    double chirp_duration;
    double demod_cutoff_hz;
    int32_t demod_taps;
    int32_t demod_decimation;
    int32_t pre_mf_decimation;
    int32_t post_envelope_decimation;
    double smoothing_cutoff_hz;
    int32_t smoothing_taps;
    int32_t precision;
    double speed_of_sound;
    double max_range;
} orc_config;

typedef struct orc_measurement {
    uint32_t sensor_serial;
    uint64_t timestamp_us;
    uint64_t seq;
    uint16_t channels;
    uint64_t frames;
    double pdm_rate;
    const uint8_t* packed;
    uint64_t packed_len;
} orc_measurement;

typedef struct orc_reflector {
    double range, azimuth, elevation, reflectivity;
} orc_reflector;

typedef struct orc_scene {
    const orc_reflector* reflectors;
    uint64_t n_reflectors;
    double noise_rms;
    uint64_t seed;
} orc_scene;

/* dims[]: frames, demod_samples, mf_samples, range_bins, n_dirs, ref_len,
 *         mf_fft_size, env_fft_size, smoothing_len, lut_octets */
#define ORC_NDIMS 10

/* status: 0 ok, 1 config, 2 argument, 3 decode, 4 io, 6 other */

/* wire format (protocol.md, wire.cpp) */
uint32_t ref_crc32(const uint8_t* bytes, uint64_t n);
int ref_measurement_frame(const orc_measurement* m, uint8_t* out, uint64_t cap, uint64_t* n_out);
int ref_ws_process_frame(void* ws, const uint8_t* frame, uint64_t len, uint8_t* out, uint64_t cap,
                         uint64_t* n_out);

#ifdef __cplusplus
}
#endif

#endif
