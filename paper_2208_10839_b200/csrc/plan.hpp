// Host-side plan: every table the device path needs, derived once from a
// PipelineConfig (reference: Workspace::Impl::Impl, pipeline.cpp:250-319).
//
// Compiled with -ffp-contract=off: the FP64 demodulation lookup table and the
// pre-MF taps must be the exact doubles the reference builds, because the
// device reproduces the reference's summation order bit for bit.
#pragma once

#include "sonarnet_b200.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace snb {

// Error taxonomy (reference errors.hpp:11-29) carried through the C ABI as
// sn_status codes.
struct Error : std::runtime_error {
    sn_status status;
    Error(sn_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};
// message returned by sn_last_error() on this thread (sn_api.cu)
void set_last_error(const std::string& m);

[[noreturn]] inline void config_error(const std::string& m) { throw Error(SN_ERR_CONFIG, m); }
[[noreturn]] inline void argument_error(const std::string& m) { throw Error(SN_ERR_ARGUMENT, m); }
[[noreturn]] inline void decode_error(const std::string& m) { throw Error(SN_ERR_DECODE, m); }

constexpr int kCh = SN_CHANNELS;

// Derived sizes of one configuration (pipeline.hpp:38-50, pipeline.cpp:40-52).
struct Sizes {
    uint64_t frames = 0, row_bytes = 0, demod_len = 0, mf_len = 0, bins = 0;
    uint64_t ref_len = 0, n_dirs = 0, mf_fft = 0, env_fft = 0, lut_octets = 0;
    uint64_t comp_len = 0, premf_taps = 0;
    double demod_rate = 0, mf_rate = 0, final_rate = 0, range_bin_size = 0;
    // demodulation output window (pipeline.cpp:395-399)
    int64_t m_lo = 0, m_hi = 0;
};

struct Plan {
    sn_pipeline_config cfg{};         // copy (directions pointer cleared)
    std::vector<double> directions;   // n_dirs x 2
    Sizes sz;
    std::vector<double> demod_rev;    // reversed demod taps
    std::vector<double> demod_lut;    // 8 x octets x 256
    std::vector<double> premf_rev;    // reversed pre-MF taps
    std::vector<double> chirp_ref;    // reference chirp at the MF rate (ref_len)
    std::vector<double> comp_rev;     // reversed composite smoothing+anti-alias kernel
    std::vector<int32_t> delays;      // n_dirs x 32 at the MF rate
    std::vector<int32_t> advances;    // n_dirs
    // Device scheduling of the direction loop (no effect on results: every
    // direction is independent, pipeline.cpp:225-226):
    std::vector<int32_t> order;       // slot -> direction, Morton order of (u_y, u_z)
    std::vector<int32_t> shifts;      // slot-major [n_dirs][32]: delay - advance
    std::vector<int32_t> tc_leaves;   // first slot of every <= kTcLeafDirs k-d subtree (+ n_dirs)
    int32_t halo = 0;                 // max |shift| over all directions/channels
};

constexpr int kClusterDirs = 8;  // k-d leaf size of the direction schedule
constexpr int kTcLeafDirs = 128; // upper k-d level: tensor-core beamformer clusters

// Validates (pipeline.cpp:60-92; geometry.cpp:27-57 invariants; Direction
// ranges geometry.cpp:146-155) and derives every table. Throws Error.
Plan make_plan(const sn_pipeline_config& cfg);
// tensor-core cluster planning (cluster.cpp): replaces the k-d leaves and the
// cluster bounds by balanced k-means clusters when that lowers the sum of R_c
void rebalance_tc_clusters(Plan& p, uint64_t n, std::vector<int32_t>& leaves, std::vector<int32_t>& tc_leaves);
Sizes derive_sizes(const sn_pipeline_config& cfg); // validate + sizes only

// Setup helpers restated from the reference.
std::vector<double> design_lowpass(double cutoff_hz, double sample_rate, int taps);
int decimation_filter_taps(int factor);
void default_array(uint64_t seed, double* xyz96);
std::vector<double> direction_grid(int kind); // n x (az, el)
std::vector<double> fibonacci_hemisphere(uint64_t n); // n x (az, el), geometry.cpp:206-229
void default_config(int kind, sn_pipeline_config* cfg);

// synth.cpp:116-134: packed bytes of one capture (frame-major, MSB first).
// Echo geometry of one synthetic scene (synth.cpp:11-61): the pulse at the
// PDM rate, per reflector its amplitude and per channel its onset sample.
struct SceneEchoes {
    uint64_t frames = 0;
    std::vector<double> pulse;
    std::vector<double> amplitude;   // [reflector]
    std::vector<int64_t> onset;      // [reflector][32]
};
SceneEchoes scene_echoes(const sn_pipeline_config& c, const sn_scene& scene);
void synthesize_packed(const sn_pipeline_config& cfg, const sn_scene& scene, uint8_t* out);

} // namespace snb
