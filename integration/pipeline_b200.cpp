// Reference-side binding: sonarnet::Workspace
// re-implemented on the C ABI of libsonarnet_b200.so. Built by
// integration/Makefile together with the reference's own sources (its
// pipeline.cpp compiled with the class renamed, so everything else in that
// file — config derivation, validation, AIMG/CSV — stays the reference's) and
// linked into the reference's UNMODIFIED acceptance runner.
#include "sonarnet/pipeline.hpp"
#include "sonarnet/errors.hpp"
#include <sonarnet_b200.h>

namespace sonarnet {

namespace {
[[noreturn]] void rethrow(sn_status s) {          // errors.hpp:11-29
    const std::string m = sn_last_error();
    switch (s) {
        case SN_ERR_CONFIG:   throw ConfigError(m);
        case SN_ERR_ARGUMENT: throw ArgumentError(m);
        case SN_ERR_DECODE:   throw DecodeError(m);
        case SN_ERR_IO:       throw IoError(m);
        default:              throw std::runtime_error(m);
    }
}
void check(sn_status s) { if (s != SN_OK) rethrow(s); }

sn_pipeline_config flatten(const PipelineConfig& c, std::vector<double>& dirs) {
    sn_pipeline_config f{};
    for (int i = 0; i < kChannelCount; ++i) {
        const Vec3& p = c.geometry.position(i);
        f.mic_xyz[3 * i] = p.x; f.mic_xyz[3 * i + 1] = p.y; f.mic_xyz[3 * i + 2] = p.z;
    }
    for (const Direction& d : c.directions.directions) { dirs.push_back(d.azimuth); dirs.push_back(d.elevation); }
    f.directions = dirs.data();
    f.n_directions = c.directions.size();
    f.grid_kind = static_cast<int32_t>(c.directions.kind);
    f.processing_threads = c.processing_threads;
    f.pdm_rate = c.pdm_rate;
    f.chirp_f_start = c.chirp.f_start; f.chirp_f_end = c.chirp.f_end; f.chirp_duration = c.chirp.duration;
    f.demod_cutoff_hz = c.demod.cutoff_hz; f.demod_taps = c.demod.taps; f.demod_decimation = c.demod.decimation;
    f.pre_mf_decimation = c.pre_mf_decimation; f.post_envelope_decimation = c.post_envelope_decimation;
    f.smoothing_cutoff_hz = c.envelope_smoothing.cutoff_hz; f.smoothing_taps = c.envelope_smoothing.taps;
    f.precision = SN_PRECISION_F64;                // bit-identical mode
    f.speed_of_sound = c.speed_of_sound; f.max_range = c.max_range;
    return f;
}
} // namespace

struct Workspace::Impl {
    PipelineConfig cfg;
    sn_workspace* ws = nullptr;
    sn_dims dims{};
    std::vector<int32_t> delays, advances;
    ~Impl() { sn_workspace_destroy(ws); }
};

Workspace::Workspace(PipelineConfig cfg) : impl_(std::make_unique<Impl>()) {
    std::vector<double> dirs;
    const sn_pipeline_config f = flatten(cfg, dirs);
    check(sn_workspace_create(&f, /*device=*/0, /*max_batch=*/1, &impl_->ws));
    check(sn_workspace_dims(impl_->ws, &impl_->dims));
    impl_->delays.resize(impl_->dims.n_directions * kChannelCount);
    impl_->advances.resize(impl_->dims.n_directions);
    check(sn_workspace_delay_table(impl_->ws, impl_->delays.data(), impl_->delays.size()));
    check(sn_workspace_reference_advances(impl_->ws, impl_->advances.data(), impl_->advances.size()));
    impl_->cfg = std::move(cfg);
}

Workspace::~Workspace() = default;
Workspace::Workspace(Workspace&&) noexcept = default;
Workspace& Workspace::operator=(Workspace&&) noexcept = default;

AcousticImage Workspace::process(const wire::RawMeasurement& m) {
    const sn_raw_measurement r{m.sensor_serial, m.timestamp_us, m.seq, m.channels, m.frames,
                               m.pdm_rate, m.packed.data(), m.packed.size()};
    AcousticImage image;
    image.sensor_serial = m.sensor_serial;
    image.timestamp_us = m.timestamp_us;
    image.directions = impl_->cfg.directions;
    image.range_bin_size = impl_->dims.range_bin_size;
    image.range_bins = impl_->dims.range_bins;
    image.energies.resize(impl_->dims.n_directions * impl_->dims.range_bins);
    check(sn_workspace_process(impl_->ws, &r, image.energies.data()));   // DecodeError all-or-error
    return image;
}

SignalMatrix Workspace::beamform(const SignalMatrix& x) const {
    SignalMatrix out(impl_->dims.n_directions, x.samples, x.sample_rate);
    check(sn_workspace_beamform(impl_->ws, x.data.data(), x.channels, x.samples, out.data.data()));
    return out;
}

const PipelineConfig& Workspace::config() const { return impl_->cfg; }
const std::vector<int32_t>& Workspace::delay_table() const { return impl_->delays; }
const std::vector<int32_t>& Workspace::reference_advances() const { return impl_->advances; }
size_t Workspace::allocation_events() const { return sn_workspace_allocation_events(impl_->ws); }

} // namespace sonarnet
