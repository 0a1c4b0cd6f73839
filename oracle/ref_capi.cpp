// TEST INFRASTRUCTURE ONLY — C wrapper around the UNMODIFIED reference.
//
// Compiled by oracle/Makefile into oracle/_ref/libsonarnet_ref*.so together
// with the reference's own core sources straight from /root/reference (no
// source is copied into this repository). Used by tests/ as the parity
// oracle and by bench.py --impl reference / cpu_baseline as the CPU arm.
//
// Stage buffers (demod_buf, mf_buf, filt_buf, demod_lut, ...) live in the
// private pimpl `Workspace::Impl` (pipeline.cpp:191-506). SURVEY.md Appendix
// B step 4: this TU includes pipeline.cpp itself with `private` widened to
// `public` for the class declaration, so the members are readable after
// process(); pipeline.o is therefore NOT linked separately.

// Every standard header pipeline.cpp and its includes use, first, so the
// access-specifier trick below never touches the standard library.
#include <algorithm>
#include <array>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <iosfwd>
#include <memory>
#include <numbers>
#include <numeric>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "sonarnet/detail/bytes.hpp"
#include "sonarnet/detail/filters.hpp"
#include "sonarnet/dsp.hpp"
#include "sonarnet/errors.hpp"
#include "sonarnet/fft.hpp"
#include "sonarnet/geometry.hpp"
#include "sonarnet/rng.hpp"
#include "sonarnet/wire.hpp"

#define private public
#include "sonarnet/pipeline.hpp"
#undef private

#include "sonarnet/synth.hpp"

#include "pipeline.cpp" // /root/reference/proj/core/src/pipeline.cpp via -I

#include "oracle_api.h"

using namespace sonarnet;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_error = e.what();
        return 1;
    } catch (const ArgumentError& e) {
        g_error = e.what();
        return 2;
    } catch (const DecodeError& e) {
        g_error = e.what();
        return 3;
    } catch (const ProtocolError& e) { // CLI maps protocol errors to 3 as well (errors.hpp:9)
        g_error = e.what();
        return 3;
    } catch (const IoError& e) {
        g_error = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 6;
    }
}

PipelineConfig to_config(const orc_config& c) {
    std::array<Vec3, kChannelCount> pos{};
    for (int i = 0; i < kChannelCount; ++i) {
        pos[static_cast<size_t>(i)] = Vec3{c.mic_xyz[3 * i], c.mic_xyz[3 * i + 1],
                                           c.mic_xyz[3 * i + 2]};
    }
    PipelineConfig cfg = default_pipeline_config(GridKind::horizontal90);
    cfg.geometry = ArrayGeometry::from_positions(pos);
    DirectionSet set;
    set.kind = static_cast<GridKind>(c.grid_kind);
    set.directions.reserve(c.n_directions);
    for (uint64_t d = 0; d < c.n_directions; ++d) {
        set.directions.emplace_back(c.directions[2 * d], c.directions[2 * d + 1]);
    }
    cfg.directions = std::move(set);
    cfg.pdm_rate = c.pdm_rate;
    cfg.chirp.f_start = c.chirp_f_start;
    cfg.chirp.f_end = c.chirp_f_end;
    cfg.chirp.duration = c.chirp_duration;
    cfg.chirp.sample_rate = c.pdm_rate;
    cfg.demod.cutoff_hz = c.demod_cutoff_hz;
    cfg.demod.taps = c.demod_taps;
    cfg.demod.decimation = c.demod_decimation;
    cfg.pre_mf_decimation = c.pre_mf_decimation;
    cfg.post_envelope_decimation = c.post_envelope_decimation;
    cfg.envelope_smoothing.cutoff_hz = c.smoothing_cutoff_hz;
    cfg.envelope_smoothing.taps = c.smoothing_taps;
    cfg.speed_of_sound = c.speed_of_sound;
    cfg.max_range = c.max_range;
    cfg.processing_threads = c.processing_threads;
    return cfg;
}

wire::RawMeasurement to_measurement(const orc_measurement& m) {
    wire::RawMeasurement r;
    r.sensor_serial = m.sensor_serial;
    r.timestamp_us = m.timestamp_us;
    r.seq = m.seq;
    r.channels = m.channels;
    r.frames = m.frames;
    r.pdm_rate = m.pdm_rate;
    r.packed.assign(m.packed, m.packed + m.packed_len);
    return r;
}

template <typename T>
int copy_out(const std::vector<T>& v, T* out, uint64_t cap, uint64_t* n_out) {
    if (n_out) *n_out = v.size();
    if (out == nullptr) return 0;
    if (cap < v.size()) {
        g_error = "output capacity too small";
        return 2;
    }
    std::copy(v.begin(), v.end(), out);
    return 0;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_default_array(uint64_t seed, double* out) {
    return guarded([&] {
        const auto g = default_array(seed);
        for (int i = 0; i < kChannelCount; ++i) {
            out[3 * i] = g.position(i).x;
            out[3 * i + 1] = g.position(i).y;
            out[3 * i + 2] = g.position(i).z;
        }
    });
}

int ref_direction_grid(int kind, double* out, uint64_t cap, uint64_t* n_out) {
    return guarded([&] {
        const auto set = direction_grid(static_cast<GridKind>(kind));
        *n_out = set.size();
        if (out == nullptr) return;
        if (cap < set.size()) throw ArgumentError("capacity too small");
        for (size_t d = 0; d < set.size(); ++d) {
            out[2 * d] = set[d].azimuth;
            out[2 * d + 1] = set[d].elevation;
        }
    });
}

int ref_default_config(int kind, orc_config* c, double* dir_buf, uint64_t cap) {
    return guarded([&] {
        const PipelineConfig cfg = default_pipeline_config(static_cast<GridKind>(kind));
        for (int i = 0; i < kChannelCount; ++i) {
            c->mic_xyz[3 * i] = cfg.geometry.position(i).x;
            c->mic_xyz[3 * i + 1] = cfg.geometry.position(i).y;
            c->mic_xyz[3 * i + 2] = cfg.geometry.position(i).z;
        }
        if (cap < cfg.directions.size()) throw ArgumentError("capacity too small");
        for (size_t d = 0; d < cfg.directions.size(); ++d) {
            dir_buf[2 * d] = cfg.directions[d].azimuth;
            dir_buf[2 * d + 1] = cfg.directions[d].elevation;
        }
        c->directions = dir_buf;
        c->n_directions = cfg.directions.size();
        c->grid_kind = static_cast<int32_t>(cfg.directions.kind);
        c->processing_threads = cfg.processing_threads;
        c->pdm_rate = cfg.pdm_rate;
        c->chirp_f_start = cfg.chirp.f_start;
        c->chirp_f_end = cfg.chirp.f_end;
        c->chirp_duration = cfg.chirp.duration;
        c->demod_cutoff_hz = cfg.demod.cutoff_hz;
        c->demod_taps = cfg.demod.taps;
        c->demod_decimation = cfg.demod.decimation;
        c->pre_mf_decimation = cfg.pre_mf_decimation;
        c->post_envelope_decimation = cfg.post_envelope_decimation;
        c->smoothing_cutoff_hz = cfg.envelope_smoothing.cutoff_hz;
        c->smoothing_taps = cfg.envelope_smoothing.taps;
        c->precision = 0;
        c->speed_of_sound = cfg.speed_of_sound;
        c->max_range = cfg.max_range;
    });
}

void* ref_ws_create(const orc_config* c, int* status) {
    Workspace* ws = nullptr;
    *status = guarded([&] { ws = new Workspace(to_config(*c)); });
    return ws;
}

void ref_ws_destroy(void* ws) { delete static_cast<Workspace*>(ws); }

int ref_ws_dims(void* p, uint64_t* dims, double* range_bin_size) {
    return guarded([&] {
        auto& w = *static_cast<Workspace*>(p)->impl_;
        dims[0] = w.frames;
        dims[1] = w.demod_len;
        dims[2] = w.mf_len;
        dims[3] = w.bins;
        dims[4] = w.n_dirs;
        dims[5] = w.ref_len;
        dims[6] = w.mf_fft.size();
        dims[7] = w.scratch.empty() ? 0 : w.scratch[0]->env_fft.size();
        dims[8] = w.smooth_decimate_rev.size();
        dims[9] = w.lut_octets;
        *range_bin_size = w.cfg.range_bin_size();
    });
}

int ref_ws_process(void* p, const orc_measurement* m, float* out) {
    return guarded([&] {
        auto* ws = static_cast<Workspace*>(p);
        const auto img = ws->process(to_measurement(*m));
        std::copy(img.energies.begin(), img.energies.end(), out);
    });
}

// stage: 0 demod_buf, 1 mf_buf, 2 filt_buf, 3 bit_rows (as bytes into out)
int ref_ws_stage(void* p, int stage, double* out, uint64_t cap) {
    return guarded([&] {
        auto& w = *static_cast<Workspace*>(p)->impl_;
        switch (stage) {
            case 0: copy_out(w.demod_buf, out, cap, nullptr); break;
            case 1: copy_out(w.mf_buf, out, cap, nullptr); break;
            case 2: copy_out(w.filt_buf, out, cap, nullptr); break;
            case 3: {
                if (cap < w.bit_rows.size()) throw ArgumentError("capacity too small");
                std::memcpy(out, w.bit_rows.data(), w.bit_rows.size());
                break;
            }
            default: throw ArgumentError("bad stage");
        }
    });
}

// table: 0 demod_rev, 1 demod_lut, 2 premf_rev, 3 chirp ref (mf rate),
//        4 smooth_decimate_rev, 5 ref_spec (complex interleaved)
int ref_ws_table(void* p, int table, double* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        auto& w = *static_cast<Workspace*>(p)->impl_;
        int rc = 0;
        switch (table) {
            case 0: rc = copy_out(w.demod_rev, out, cap, n); break;
            case 1: rc = copy_out(w.demod_lut, out, cap, n); break;
            case 2: rc = copy_out(w.premf_rev, out, cap, n); break;
            case 3: {
                const SignalMatrix ref = generate_chirp(w.cfg.chirp_at(w.cfg.mf_rate()));
                rc = copy_out(ref.data, out, cap, n);
                break;
            }
            case 4: rc = copy_out(w.smooth_decimate_rev, out, cap, n); break;
            case 5: {
                std::vector<double> flat;
                for (const auto& z : w.ref_spec) {
                    flat.push_back(z.real());
                    flat.push_back(z.imag());
                }
                rc = copy_out(flat, out, cap, n);
                break;
            }
            default: throw ArgumentError("bad table");
        }
        if (rc != 0) throw ArgumentError(g_error);
    });
}

int ref_ws_delays(void* p, int32_t* out, uint64_t cap) {
    return guarded([&] {
        const auto& v = static_cast<Workspace*>(p)->delay_table();
        if (cap < v.size()) throw ArgumentError("capacity too small");
        std::copy(v.begin(), v.end(), out);
    });
}

int ref_ws_advances(void* p, int32_t* out, uint64_t cap) {
    return guarded([&] {
        const auto& v = static_cast<Workspace*>(p)->reference_advances();
        if (cap < v.size()) throw ArgumentError("capacity too small");
        std::copy(v.begin(), v.end(), out);
    });
}

uint64_t ref_ws_alloc_events(void* p) { return static_cast<Workspace*>(p)->allocation_events(); }

int ref_ws_beamform(void* p, const double* filt, uint64_t channels, uint64_t samples,
                    double* out) {
    return guarded([&] {
        auto* ws = static_cast<Workspace*>(p);
        SignalMatrix x(channels, samples, ws->config().mf_rate());
        std::copy(filt, filt + channels * samples, x.data.begin());
        const auto y = ws->beamform(x);
        std::copy(y.data.begin(), y.data.end(), out);
    });
}

int ref_synthesize(const orc_config* c, const orc_scene* s, uint32_t serial, uint64_t ts,
                   uint64_t seq, uint8_t* out, uint64_t cap) {
    return guarded([&] {
        const PipelineConfig cfg = to_config(*c);
        Scene scene;
        scene.noise_rms = s->noise_rms;
        scene.seed = s->seed;
        for (uint64_t i = 0; i < s->n_reflectors; ++i) {
            const auto& r = s->reflectors[i];
            scene.reflectors.push_back({r.range, r.azimuth, r.elevation, r.reflectivity});
        }
        const auto m = synthesize_measurement(cfg, scene, serial, ts, seq);
        if (cap < m.packed.size()) throw ArgumentError("capacity too small");
        std::copy(m.packed.begin(), m.packed.end(), out);
    });
}

// Latency protocol of bench::run_benchmark (bench.cpp:63-108): one warm-up
// process() call, then n timed calls on steady_clock.
int ref_latency(void* p, const orc_measurement* m, int n, double* durations_ms) {
    return guarded([&] {
        auto* ws = static_cast<Workspace*>(p);
        const auto meas = to_measurement(*m);
        (void)ws->process(meas);
        for (int i = 0; i < n; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            (void)ws->process(meas);
            const auto t1 = std::chrono::steady_clock::now();
            durations_ms[i] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
    });
}

// Throughput protocol (central-node model, central_node.cpp:48-53,238-270):
// `threads` workers, each owning one Workspace (processing_threads = 1 unless
// the config says otherwise), each processing `calls_per_worker`
// measurements drawn round-robin from the pool. Workspace construction and
// one warm-up call per worker are excluded. stats = {elapsed_s, total_calls}.
int ref_throughput(const orc_config* c, const uint8_t* pool, uint64_t pool_n, int threads,
                   uint64_t calls_per_worker, double* stats) {
    return guarded([&] {
        const PipelineConfig cfg = to_config(*c);
        const size_t bytes = size_t{kChannelCount} * cfg.frames() / 8;
        std::vector<wire::RawMeasurement> ms(pool_n);
        for (uint64_t i = 0; i < pool_n; ++i) {
            auto& r = ms[i];
            r.sensor_serial = 1;
            r.seq = i;
            r.channels = kChannelCount;
            r.frames = cfg.frames();
            r.pdm_rate = cfg.pdm_rate;
            r.packed.assign(pool + i * bytes, pool + (i + 1) * bytes);
        }
        std::vector<std::unique_ptr<Workspace>> wss;
        for (int t = 0; t < threads; ++t) wss.push_back(std::make_unique<Workspace>(cfg));
        std::atomic<int> ready{0};
        std::atomic<bool> go{false};
        std::vector<std::thread> pool_threads;
        std::vector<std::exception_ptr> errors(static_cast<size_t>(threads));
        std::chrono::steady_clock::time_point t0;
        for (int t = 0; t < threads; ++t) {
            pool_threads.emplace_back([&, t] {
                try {
                    auto& ws = *wss[static_cast<size_t>(t)];
                    (void)ws.process(ms[static_cast<size_t>(t) % pool_n]);
                    ready.fetch_add(1);
                    while (!go.load()) std::this_thread::yield();
                    for (uint64_t k = 0; k < calls_per_worker; ++k) {
                        (void)ws.process(ms[(static_cast<size_t>(t) + k * threads) % pool_n]);
                    }
                } catch (...) {
                    errors[static_cast<size_t>(t)] = std::current_exception();
                    ready.fetch_add(1);
                }
            });
        }
        while (ready.load() < threads) std::this_thread::yield();
        t0 = std::chrono::steady_clock::now();
        go.store(true);
        for (auto& th : pool_threads) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errors) {
            if (e) std::rethrow_exception(e);
        }
        stats[0] = std::chrono::duration<double>(t1 - t0).count();
        stats[1] = static_cast<double>(calls_per_worker) * threads;
    });
}

// ---- wire format (protocol.md; wire.cpp) -----------------------------------
uint32_t ref_crc32(const uint8_t* bytes, uint64_t n) { return wire::crc32({bytes, static_cast<size_t>(n)}); }

// wire::measurement_frame (wire.cpp:251-259): the frame a sensor node sends.
int ref_measurement_frame(const orc_measurement* m, uint8_t* out, uint64_t cap, uint64_t* n_out) {
    return guarded([&] {
        const auto f = wire::measurement_frame(to_measurement(*m));
        copy_out(f, out, cap, n_out);
    });
}

// The central node's processing of one received frame (central_node.cpp:
// decode_packet -> decode_raw_measurement -> Workspace::process ->
// wire::image_frame(image, seq)). Returns the reference's error classes
// (3: decode/protocol); a CRC mismatch throws ProtocolError from decode_packet.
int ref_ws_process_frame(void* p, const uint8_t* frame, uint64_t len, uint8_t* out, uint64_t cap,
                         uint64_t* n_out) {
    return guarded([&] {
        auto* ws = static_cast<Workspace*>(p);
        size_t consumed = 0;
        const auto pkt = wire::decode_packet({frame, static_cast<size_t>(len)}, &consumed);
        if (pkt.msg_type != wire::MsgType::raw_measurement) throw DecodeError("not a raw measurement frame");
        const auto m = wire::decode_raw_measurement(pkt.payload);
        const auto img = ws->process(m);
        const auto f = wire::image_frame(img, m.seq);
        copy_out(f, out, cap, n_out);
    });
}

} // extern "C"
