// Multi-sensor 360-degree view (BASELINE configs[2]): the
// energyscapes of one trigger, processed one sensor per GPU, gathered to a
// root rank over NCCL (NVLink 5 / NVSwitch) — the only collective of the
// sensor network; the data path itself has none (central_node.cpp:48-53).
//
// Trigger semantics follow the reference's shared-clock fan-out
// (nodes/sync.hpp:16-19, sync.cpp:45-82): every sensor of one trigger carries
// the same (timestamp_us, seq). Each rank sends its images together with
// their (serial, timestamp_us, seq) ids; the root checks that all ranks'
// images of a slot belong to the same trigger (sn_gather_ids).
//
// The gather runs on its own stream after an event on the producer's stream,
// into one of two view slots, so step k's gather overlaps step k + 1's
// processing (double buffering): before the producer overwrites the images of
// slot s it waits for that slot's previous gather (sn_gather_wait).
//
// NCCL is bound at run time (dlopen "libnccl.so.2": the copy torch already
// loaded when running under torch.distributed, else the system library), so
// the library has no link-time NCCL dependency and single-GPU users never
// load it.
#include "sonarnet_b200.h"
#include "plan.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) {
            n.error = std::string("NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [&](const char* s) {
            void* p = dlsym(n.h, s);
            if (!p && n.error.empty()) n.error = std::string("NCCL symbol missing: ") + s;
            return p;
        };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
        n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    return n;
}

struct GatherError : std::runtime_error {
    sn_status status;
    GatherError(sn_status s, const std::string& w) : std::runtime_error(w), status(s) {}
};

void ckc(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw GatherError(SN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ckn(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw GatherError(SN_ERR_IO, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

template <typename F>
sn_status guarded(F&& f) {
    try {
        f();
        return SN_OK;
    } catch (const GatherError& e) {
        snb::set_last_error(e.what());
        return e.status;
    } catch (const std::exception& e) {
        snb::set_last_error(e.what());
        return SN_ERR_INTERNAL;
    }
}

struct Dev {
    int prev = -1;
    explicit Dev(int d) {
        cudaGetDevice(&prev);
        if (prev != d) ckc(cudaSetDevice(d), "cudaSetDevice");
    }
    ~Dev() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

} // namespace

struct sn_gather {
    int rank = 0, world = 1, device = 0;
    uint64_t image_floats = 0, max_count = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ready[2] = {}, done[2] = {}, t0[2] = {}, t1[2] = {};
    sn_frame_id* d_ids[2] = {};   // [world][max_count] on the root, [max_count] elsewhere
    sn_frame_id* h_ids[2] = {};   // page-locked staging of the ids
    uint64_t last_count[2] = {};
    bool started[2] = {};

    ~sn_gather() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
        for (int s = 0; s < 2; ++s) {
            for (cudaEvent_t e : {ready[s], done[s], t0[s], t1[s]})
                if (e) cudaEventDestroy(e);
            if (d_ids[s]) cudaFree(d_ids[s]);
            if (h_ids[s]) cudaFreeHost(h_ids[s]);
        }
        if (stream) cudaStreamDestroy(stream);
        if (prev >= 0) cudaSetDevice(prev);
    }
};

extern "C" {

sn_status sn_gather_unique_id(uint8_t* id_out) {
    return guarded([&] {
        if (!id_out) throw GatherError(SN_ERR_ARGUMENT, "null argument");
        const Nccl& n = nccl();
        if (!n.error.empty()) throw GatherError(SN_ERR_CUDA, n.error);
        ncclUniqueId id;
        ckn(n.GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, id.internal, SN_GATHER_ID_BYTES);
    });
}

sn_status sn_gather_create(int rank, int world, const uint8_t* id, int device, uint64_t image_floats,
                           uint64_t max_count, sn_gather** out) {
    return guarded([&] {
        if (!id || !out || world < 1 || rank < 0 || rank >= world || device < 0 || image_floats == 0 ||
            max_count == 0)
            throw GatherError(SN_ERR_ARGUMENT, "sn_gather_create: bad argument");
        *out = nullptr;
        const Nccl& n = nccl();
        if (!n.error.empty()) throw GatherError(SN_ERR_CUDA, n.error);
        Dev g(device);
        auto gt = new sn_gather;
        std::unique_ptr<sn_gather> own(gt);
        gt->rank = rank;
        gt->world = world;
        gt->device = device;
        gt->image_floats = image_floats;
        gt->max_count = max_count;
        ckc(cudaStreamCreateWithFlags(&gt->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        for (int s = 0; s < 2; ++s) {
            ckc(cudaEventCreateWithFlags(&gt->ready[s], cudaEventDisableTiming), "cudaEventCreate");
            ckc(cudaEventCreateWithFlags(&gt->done[s], cudaEventDisableTiming), "cudaEventCreate");
            ckc(cudaEventCreate(&gt->t0[s]), "cudaEventCreate");
            ckc(cudaEventCreate(&gt->t1[s]), "cudaEventCreate");
            const uint64_t nid = (rank == 0 ? (uint64_t)world : 1) * max_count;
            ckc(cudaMalloc(&gt->d_ids[s], nid * sizeof(sn_frame_id)), "cudaMalloc");
            ckc(cudaMallocHost(&gt->h_ids[s], nid * sizeof(sn_frame_id)), "cudaMallocHost");
        }
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, SN_GATHER_ID_BYTES);
        ckn(n.CommInitRank(&gt->comm, world, uid, rank), "ncclCommInitRank");
        *out = own.release();
    });
}

void sn_gather_destroy(sn_gather* g) { delete g; }

sn_status sn_gather_start(sn_gather* g, int slot, const float* d_images, const sn_frame_id* ids, uint64_t count,
                          float* d_view, void* stream) {
    return guarded([&] {
        if (!g || slot < 0 || slot > 1 || !d_images || !ids || count == 0 || count > g->max_count ||
            (g->rank == 0 && !d_view))
            throw GatherError(SN_ERR_ARGUMENT, "sn_gather_start: bad argument");
        const Nccl& n = nccl();
        Dev dv(g->device);
        const size_t per = count * g->image_floats;
        // the slot's staging is reused: its previous gather must be done
        if (g->started[slot]) ckc(cudaEventSynchronize(g->done[slot]), "gather slot sync");
        std::memcpy(g->h_ids[slot], ids, count * sizeof(sn_frame_id));
        ckc(cudaEventRecord(g->ready[slot], static_cast<cudaStream_t>(stream)), "event");
        ckc(cudaStreamWaitEvent(g->stream, g->ready[slot], 0), "wait");
        ckc(cudaEventRecord(g->t0[slot], g->stream), "event");
        sn_frame_id* dids = g->d_ids[slot];
        ckc(cudaMemcpyAsync(dids, g->h_ids[slot], count * sizeof(sn_frame_id), cudaMemcpyHostToDevice, g->stream),
            "H2D ids");
        const size_t id_bytes = count * sizeof(sn_frame_id);
        if (g->rank == 0) {
            ckc(cudaMemcpyAsync(d_view, d_images, per * sizeof(float), cudaMemcpyDeviceToDevice, g->stream), "D2D");
            ckn(n.GroupStart(), "ncclGroupStart");
            for (int r = 1; r < g->world; ++r) {
                ckn(n.Recv(d_view + (size_t)r * per, per, ncclFloat32, r, g->comm, g->stream), "ncclRecv");
                ckn(n.Recv(reinterpret_cast<uint8_t*>(dids) + (size_t)r * id_bytes, id_bytes, ncclUint8, r, g->comm,
                           g->stream), "ncclRecv ids");
            }
            ckn(n.GroupEnd(), "ncclGroupEnd");
            ckc(cudaMemcpyAsync(g->h_ids[slot], dids, g->world * id_bytes, cudaMemcpyDeviceToHost, g->stream),
                "D2H ids");
        } else {
            ckn(n.GroupStart(), "ncclGroupStart");
            ckn(n.Send(d_images, per, ncclFloat32, 0, g->comm, g->stream), "ncclSend");
            ckn(n.Send(dids, id_bytes, ncclUint8, 0, g->comm, g->stream), "ncclSend ids");
            ckn(n.GroupEnd(), "ncclGroupEnd");
        }
        ckc(cudaEventRecord(g->t1[slot], g->stream), "event");
        ckc(cudaEventRecord(g->done[slot], g->stream), "event");
        g->last_count[slot] = count;
        g->started[slot] = true;
    });
}

sn_status sn_gather_wait(sn_gather* g, int slot, void* stream) {
    return guarded([&] {
        if (!g || slot < 0 || slot > 1) throw GatherError(SN_ERR_ARGUMENT, "sn_gather_wait: bad argument");
        if (!g->started[slot]) return;
        Dev dv(g->device);
        if (stream) ckc(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), g->done[slot], 0), "wait");
        else ckc(cudaEventSynchronize(g->done[slot]), "gather sync");
    });
}

sn_status sn_gather_ids(sn_gather* g, int slot, sn_frame_id* out, uint64_t capacity, int32_t* synchronized) {
    return guarded([&] {
        if (!g || slot < 0 || slot > 1 || !out) throw GatherError(SN_ERR_ARGUMENT, "sn_gather_ids: bad argument");
        if (g->rank != 0) throw GatherError(SN_ERR_ARGUMENT, "sn_gather_ids: root rank only");
        const uint64_t c = g->last_count[slot], n = (uint64_t)g->world * c;
        if (capacity < n) throw GatherError(SN_ERR_ARGUMENT, "buffer too small");
        Dev dv(g->device);
        ckc(cudaEventSynchronize(g->done[slot]), "gather sync");
        std::memcpy(out, g->h_ids[slot], n * sizeof(sn_frame_id));
        // sync.hpp:16-19: one trigger = one (timestamp_us, seq) for every sensor
        int32_t ok = 1;
        for (uint64_t r = 1; r < (uint64_t)g->world; ++r)
            for (uint64_t i = 0; i < c; ++i)
                if (out[r * c + i].timestamp_us != out[i].timestamp_us || out[r * c + i].seq != out[i].seq) ok = 0;
        if (synchronized) *synchronized = ok;
    });
}

sn_status sn_gather_elapsed(sn_gather* g, int slot, float* ms) {
    return guarded([&] {
        if (!g || slot < 0 || slot > 1 || !ms) throw GatherError(SN_ERR_ARGUMENT, "sn_gather_elapsed: bad argument");
        Dev dv(g->device);
        ckc(cudaEventSynchronize(g->t1[slot]), "gather sync");
        ckc(cudaEventElapsedTime(ms, g->t0[slot], g->t1[slot]), "elapsed");
    });
}

} // extern "C"
