// GPU-backed central-node worker pool.
//
// Mirrors CentralNode's processing core (central_node.cpp:48-53, 130-160,
// 224-336): received raw-measurement frames get a per-sensor ticket at
// submission (ingest thread), K workers each owning a Workspace pull work from a
// bounded input queue (blocking push = backpressure, central_node.cpp:153-156),
// results enter a bounded reorder window, and a release step hands them out
// strictly in per-sensor ticket order (dispatch_loop). Differences from the
// reference, by design: a worker takes up to `max_batch` queued frames at once
// and runs them as one device batch (sn_workspace_process_frames: CRC, decode,
// the pipeline and the AIMG frame encode all on the GPU); workers may live on
// several devices; results are polled (sn_pool_poll) instead of being written
// to subscriber sockets. Frames whose CRC fails on the GPU are released as
// "discarded" (status SN_ERR_IO, no bytes) so later tickets of that sensor
// are not held back.
#include "sonarnet_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace {

struct Item {
    uint32_t serial = 0;
    uint64_t ticket = 0;
    std::vector<uint8_t> frame;
};

// Page-locked result block of one worker batch (max_batch slots): the GPU
// writes the image frames straight into it; outcomes reference their slot and
// the block returns to its worker's free list when the last one is polled.
struct Block {
    uint8_t* data = nullptr;
    std::mutex* m = nullptr;
    std::vector<uint8_t*>* free_list = nullptr;
};
struct BlockRelease {
    void operator()(Block* b) const {
        {
            std::lock_guard<std::mutex> lk(*b->m);
            b->free_list->push_back(b->data);
        }
        delete b;
    }
};

struct Outcome {
    uint32_t serial = 0;
    uint64_t seq = 0;
    int32_t status = SN_OK;
    std::shared_ptr<Block> block; // frame bytes at block->data + offset
    uint64_t offset = 0, len = 0;
};

} // namespace

struct sn_pool {
    std::vector<sn_workspace*> workspaces;
    std::vector<std::thread> workers;
    uint64_t max_batch = 1;
    size_t input_capacity = 1, window_capacity = 1;
    std::mutex m;
    std::condition_variable cv_in, cv_space, cv_out;
    std::deque<Item> input;
    std::map<uint32_t, uint64_t> next_ticket, next_release;
    std::map<std::pair<uint32_t, uint64_t>, Outcome> pending;
    std::deque<Outcome> released;
    Outcome view; // result handed out by sn_pool_poll_view, valid until the next call
    bool closing = false;
    uint64_t submitted = 0, completed = 0, discarded = 0;
    std::string worker_error;
    std::mutex blocks_m;
    std::vector<uint8_t*> free_blocks, all_blocks;
    uint64_t block_bytes = 0;

    uint8_t* take_block() {
        {
            std::lock_guard<std::mutex> lk(blocks_m);
            if (!free_blocks.empty()) {
                uint8_t* b = free_blocks.back();
                free_blocks.pop_back();
                return b;
            }
        }
        uint8_t* b = nullptr;
        if (cudaMallocHost(&b, block_bytes) != cudaSuccess) return nullptr;
        std::lock_guard<std::mutex> lk(blocks_m);
        all_blocks.push_back(b);
        return b;
    }

    ~sn_pool() {
        {
            std::lock_guard<std::mutex> lk(m);
            closing = true;
        }
        cv_in.notify_all();
        cv_space.notify_all();
        for (auto& t : workers) {
            if (t.joinable()) t.join();
        }
        pending.clear();
        released.clear();
        view = Outcome{};
        for (auto* w : workspaces) sn_workspace_destroy(w);
        for (uint8_t* b : all_blocks) cudaFreeHost(b);
    }

    // move every outcome whose ticket is next for its sensor to `released`
    void release_locked() {
        bool moved = true;
        while (moved) {
            moved = false;
            for (auto it = pending.begin(); it != pending.end();) {
                auto& nr = next_release[it->first.first];
                if (nr == it->first.second) {
                    const uint32_t serial = it->first.first;
                    ++nr;
                    released.push_back(std::move(it->second));
                    it = pending.erase(it);
                    moved = true;
                    // a sensor with nothing queued, in flight or pending drops
                    // its counters (the ticket is assigned before the CRC is
                    // verified, so a corrupted serial would otherwise leave a
                    // map entry behind for good); its next frame restarts at 0
                    auto nt = next_ticket.find(serial);
                    if (nt != next_ticket.end() && nt->second == nr) {
                        next_ticket.erase(nt);
                        next_release.erase(serial);
                    }
                } else {
                    ++it;
                }
            }
        }
    }

    void worker_loop(size_t index) {
        sn_workspace* ws = workspaces[index];
        const uint64_t slot = sn_workspace_image_frame_bytes(ws);
        std::vector<uint64_t> out_lens(max_batch);
        std::vector<int32_t> status(max_batch);
        std::vector<const uint8_t*> ptrs(max_batch);
        std::vector<uint64_t> lens(max_batch);
        while (true) {
            std::vector<Item> batch;
            {
                std::unique_lock<std::mutex> lk(m);
                cv_in.wait(lk, [&] { return closing || !input.empty(); });
                if (input.empty()) return; // closing and drained
                while (!input.empty() && batch.size() < max_batch) {
                    batch.push_back(std::move(input.front()));
                    input.pop_front();
                }
            }
            cv_space.notify_all();
            for (size_t i = 0; i < batch.size(); ++i) {
                ptrs[i] = batch[i].frame.data();
                lens[i] = batch[i].frame.size();
            }
            uint8_t* raw = take_block();
            sn_status rc = SN_ERR_CUDA;
            std::shared_ptr<Block> block;
            if (raw) {
                block.reset(new Block{raw, &blocks_m, &free_blocks}, BlockRelease{});
                rc = sn_workspace_process_frames(ws, ptrs.data(), lens.data(), batch.size(), raw, slot,
                                                 out_lens.data(), status.data());
            }
            std::vector<Outcome> outs(batch.size());
            for (size_t i = 0; i < batch.size(); ++i) {
                Outcome& o = outs[i];
                o.serial = batch[i].serial;
                std::memcpy(&o.seq, batch[i].frame.data() + 48, 8); // payload seq (checked at submit)
                if (rc != SN_OK) {
                    o.status = rc;
                } else {
                    o.status = status[i];
                    o.block = block;
                    o.offset = i * slot;
                    o.len = out_lens[i];
                }
            }
            {
                std::unique_lock<std::mutex> lk(m);
                if (rc != SN_OK && worker_error.empty()) worker_error = sn_last_error();
                // bounded reorder window (central_node.cpp:224-236): wait while it
                // is full unless one of ours is the next to be released
                cv_space.wait(lk, [&] {
                    if (closing || pending.size() + released.size() + outs.size() <= window_capacity) return true;
                    for (size_t i = 0; i < batch.size(); ++i)
                        if (next_release[batch[i].serial] == batch[i].ticket) return true;
                    return false;
                });
                for (size_t i = 0; i < batch.size(); ++i) {
                    if (outs[i].status == SN_ERR_IO) ++discarded;
                    ++completed;
                    pending[{batch[i].serial, batch[i].ticket}] = std::move(outs[i]);
                }
                release_locked();
            }
            cv_out.notify_all();
            cv_space.notify_all();
        }
    }
};

extern "C" {

sn_status sn_pool_create(const sn_pipeline_config* cfg, const int* devices, int n_devices, int workers_per_device,
                         uint64_t max_batch, sn_pool** out) {
    if (!cfg || !devices || n_devices <= 0 || workers_per_device <= 0 || !out) return SN_ERR_ARGUMENT;
    *out = nullptr;
    auto pool = std::make_unique<sn_pool>();
    pool->max_batch = std::max<uint64_t>(1, max_batch);
    for (int d = 0; d < n_devices; ++d) {
        if (devices[d] < 0) return SN_ERR_ARGUMENT;
        for (int k = 0; k < workers_per_device; ++k) {
            sn_workspace* ws = nullptr;
            const sn_status rc = sn_workspace_create(cfg, devices[d], pool->max_batch, &ws);
            if (rc != SN_OK) return rc;
            pool->workspaces.push_back(ws);
        }
    }
    const size_t k = pool->workspaces.size();
    pool->block_bytes = pool->max_batch * sn_workspace_image_frame_bytes(pool->workspaces[0]);
    pool->input_capacity = 4 * k * pool->max_batch;
    pool->window_capacity = 2 * k * pool->max_batch;
    // result blocks for the steady state: one in flight per worker, the
    // bounded window's worth, one being viewed (allocated up front: page-locked
    // allocations are slow)
    const size_t nblocks = 2 * k + pool->window_capacity / pool->max_batch + 1;
    for (size_t i = 0; i < nblocks; ++i) {
        uint8_t* b = nullptr;
        if (cudaMallocHost(&b, pool->block_bytes) != cudaSuccess) return SN_ERR_CUDA;
        pool->all_blocks.push_back(b);
        pool->free_blocks.push_back(b);
    }
    for (size_t i = 0; i < k; ++i) {
        sn_pool* p = pool.get();
        pool->workers.emplace_back([p, i] { p->worker_loop(i); });
    }
    *out = pool.release();
    return SN_OK;
}

void sn_pool_destroy(sn_pool* pool) { delete pool; }

sn_status sn_pool_submit(sn_pool* pool, const uint8_t* frame, uint64_t len) {
    if (!pool || (!frame && len)) return SN_ERR_ARGUMENT;
    // ingest-side packet/payload check (central_node.cpp:133-151): only
    // well-formed raw-measurement frames get a ticket; the CRC is verified by
    // the worker on the GPU
    if (len < 40 + 38) return SN_ERR_IO;
    uint32_t magic;
    uint16_t version, type;
    uint64_t plen;
    std::memcpy(&magic, frame, 4);
    std::memcpy(&version, frame + 4, 2);
    std::memcpy(&type, frame + 6, 2);
    std::memcpy(&plen, frame + 28, 8);
    if (magic != 0x45525449u || len != 40 + plen || version != 1 || type != 1) return SN_ERR_IO;
    Item item;
    std::memcpy(&item.serial, frame + 36, 4);
    item.frame.assign(frame, frame + len);
    {
        std::unique_lock<std::mutex> lk(pool->m);
        pool->cv_space.wait(lk, [&] { return pool->closing || pool->input.size() < pool->input_capacity; });
        if (pool->closing) return SN_ERR_ARGUMENT;
        item.ticket = pool->next_ticket[item.serial]++;
        pool->input.push_back(std::move(item));
        ++pool->submitted;
    }
    pool->cv_in.notify_one();
    return SN_OK;
}

sn_status sn_pool_poll(sn_pool* pool, int timeout_ms, uint8_t* out, uint64_t capacity, uint64_t* len,
                       int32_t* status, uint32_t* serial, uint64_t* seq) {
    if (!pool || !len || !status) return SN_ERR_ARGUMENT;
    std::unique_lock<std::mutex> lk(pool->m);
    auto ready = [&] { return !pool->released.empty(); };
    if (timeout_ms < 0) pool->cv_out.wait(lk, ready);
    else if (!pool->cv_out.wait_for(lk, std::chrono::milliseconds(timeout_ms), ready)) {
        *len = 0;
        return SN_ERR_NOT_READY;
    }
    Outcome& o = pool->released.front();
    *len = o.len;
    *status = o.status;
    if (serial) *serial = o.serial;
    if (seq) *seq = o.seq;
    if (!out) return SN_OK; // peek
    if (capacity < o.len) return SN_ERR_ARGUMENT;
    Outcome taken = std::move(o);
    pool->released.pop_front();
    lk.unlock(); // copy outside the lock; the block stays alive through `taken`
    pool->cv_space.notify_all();
    if (taken.len) std::memcpy(out, taken.block->data + taken.offset, taken.len);
    return SN_OK;
}

sn_status sn_pool_poll_view(sn_pool* pool, int timeout_ms, const uint8_t** data, uint64_t* len, int32_t* status,
                            uint32_t* serial, uint64_t* seq) {
    if (!pool || !data || !len || !status) return SN_ERR_ARGUMENT;
    Outcome old;
    {
        std::unique_lock<std::mutex> lk(pool->m);
        auto ready = [&] { return !pool->released.empty(); };
        if (timeout_ms < 0) pool->cv_out.wait(lk, ready);
        else if (!pool->cv_out.wait_for(lk, std::chrono::milliseconds(timeout_ms), ready)) {
            *len = 0;
            *data = nullptr;
            return SN_ERR_NOT_READY;
        }
        old = std::move(pool->view);
        pool->view = std::move(pool->released.front());
        pool->released.pop_front();
        const Outcome& o = pool->view;
        *data = o.len ? o.block->data + o.offset : nullptr;
        *len = o.len;
        *status = o.status;
        if (serial) *serial = o.serial;
        if (seq) *seq = o.seq;
    }
    pool->cv_space.notify_all();
    return SN_OK; // `old` (the previous view) is released here, outside the lock
}

sn_status sn_pool_stats(sn_pool* pool, uint64_t* stats4) {
    if (!pool || !stats4) return SN_ERR_ARGUMENT;
    std::lock_guard<std::mutex> lk(pool->m);
    stats4[0] = pool->submitted;
    stats4[1] = pool->completed;
    stats4[2] = pool->discarded;
    stats4[3] = pool->workspaces.size();
    return SN_OK;
}

uint64_t sn_pool_frame_bytes(const sn_pool* pool) {
    return pool && !pool->workspaces.empty() ? sn_workspace_image_frame_bytes(pool->workspaces[0]) : 0;
}

} // extern "C"
