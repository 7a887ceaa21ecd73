// Device memory and host<->device copies of the B200 GaBP engine: the process-wide cache of large
// device blocks behind Engine::dalloc / dfree, and the pinned stager for pageable caller buffers.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <omp.h>
#include <string>
#include <vector>

#include "engine.h"

namespace bgabp {

// Engine allocations go through a process-wide cache of large device blocks (exact rounded size,
// per device): a handle created after another was destroyed -- the multigrid hierarchies of one
// solve after another, the shards of a re-partitioned system -- reuses its blocks instead of
// paying cudaFree / cudaMalloc and the driver's re-zeroing of freed pages (~0.15 s for a config-5
// hierarchy).  Blocks stay whole cudaMalloc allocations (CUDA IPC of shard buffers works).
// BGABP_NO_BLOCK_CACHE=1 frees immediately; at most BGABP_BLOCK_CACHE_GB (default 32) GB are held
// (all devices).
namespace {
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> free_blocks;
    std::map<void*, std::pair<int, size_t>> sizes;  // every block handed out, with its rounded size
    size_t held = 0;
    bool off = getenv("BGABP_NO_BLOCK_CACHE") != nullptr;
    static constexpr size_t kMin = size_t(1) << 20, kGran = size_t(2) << 20;
    // idle blocks kept: 32 GB of the B200's 180 GB by default (a config-5 hierarchy holds ~12 GB, and
    // a fresh cudaMalloc / cudaFree of its blocks costs 0.1-0.3 s); BGABP_BLOCK_CACHE_GB overrides
    size_t kCap = [] {
        const char* e = getenv("BGABP_BLOCK_CACHE_GB");
        const long gb = e ? std::atol(e) : 32;
        return size_t(gb < 0 ? 0 : gb) << 30;
    }();
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache();
    return *c;
}
size_t round_block(size_t b) {
    return b < BlockCache::kMin ? b : (b + BlockCache::kGran - 1) / BlockCache::kGran * BlockCache::kGran;
}
// free every idle block of device `dev` (-1: all devices); caller holds C.mu
void trim_locked(BlockCache& C, int dev) {
    for (auto it = C.free_blocks.begin(); it != C.free_blocks.end();) {
        if (dev >= 0 && it->first.first != dev) {
            ++it;
            continue;
        }
        cudaFree(it->second);
        C.held -= it->first.second;
        it = C.free_blocks.erase(it);
    }
}
}  // namespace

// idle cached blocks back to the driver (e.g. before another library allocates)
void trim_block_cache() {
    BlockCache& C = block_cache();
    std::lock_guard<std::mutex> lock(C.mu);
    trim_locked(C, -1);
}

void* Engine::dalloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    const size_t rb = round_block(bytes);
    BlockCache& C = block_cache();
    if (rb >= BlockCache::kMin && !C.off) {
        int dev = 0;
        ck(cudaGetDevice(&dev), "device");
        std::lock_guard<std::mutex> lock(C.mu);
        auto it = C.free_blocks.find({dev, rb});
        if (it != C.free_blocks.end()) {
            p = it->second;
            C.free_blocks.erase(it);
            C.held -= rb;
        } else if (cudaMalloc(&p, rb) != cudaSuccess) {
            // out of memory with idle cached blocks of other sizes: give them back, retry once
            cudaGetLastError();
            trim_locked(C, dev);
            ck(cudaMalloc(&p, rb), "cudaMalloc");
        }
        C.sizes[p] = {dev, rb};
    } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        int dev = 0;
        ck(cudaGetDevice(&dev), "device");
        {
            std::lock_guard<std::mutex> lock(C.mu);
            trim_locked(C, dev);
        }
        ck(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    allocs.push_back(p);
    device_bytes += (long long)bytes;
    return p;
}

// return a block to the cache (large) or the driver (small, or cache full / off)
void release_block(void* p) {
    BlockCache& C = block_cache();
    {
        std::lock_guard<std::mutex> lock(C.mu);
        auto it = C.sizes.find(p);
        if (it != C.sizes.end()) {
            const auto key = it->second;
            C.sizes.erase(it);
            if (C.held + key.second <= C.kCap) {
                C.free_blocks.emplace(key, p);
                C.held += key.second;
                return;
            }
        }
    }
    cudaFree(p);
}

void Engine::dfree(void* p) {
    auto it = std::find(allocs.begin(), allocs.end(), p);
    if (it == allocs.end()) return;
    allocs.erase(it);
    DeviceGuard g(device);
    ck(cudaDeviceSynchronize(), "sync");  // the block may be handed out again at once (as cudaFree)
    release_block(p);
}


// upload from pageable caller memory through two pinned staging buffers (parallel host copies
// overlapped with the DMA of the previous chunk).  The staging pair is process-wide (allocated
// once: pinning 64 MB per engine cost ~30 ms) and serialised by a mutex.
namespace {
struct Stager {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    static constexpr size_t kMaxChunk = size_t(64) << 20;
    size_t chunk = size_t(32) << 20;
    int threads = 16;
    void init() {
        if (buf[0]) return;
        if (const char* e = getenv("BGABP_STAGE_MB")) chunk = std::min(kMaxChunk, size_t(std::max(1, atoi(e))) << 20);
        if (const char* e = getenv("BGABP_STAGE_THREADS")) threads = std::max(1, atoi(e));
        for (int k = 0; k < 2; ++k) {
            ck(cudaMallocHost(&buf[k], chunk), "cudaMallocHost");
            ck(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming), "event");
        }
    }
};
void par_copy(char* dst, const char* src, size_t len, int threads) {
    const int T = std::max(1, std::min(omp_get_max_threads(), threads));
    const size_t piece = (len + T - 1) / T;
#pragma omp parallel for num_threads(T) schedule(static)
    for (int t = 0; t < T; ++t) {
        const size_t a = std::min(len, (size_t)t * piece), b = std::min(len, a + piece);
        if (b > a) std::memcpy(dst + a, src + a, b - a);
    }
}
Stager& stager() {
    static Stager* s = new Stager();  // leaked on purpose: no teardown-order issues at exit
    return *s;
}
}  // namespace

// memory the DMA engines can read or write directly: pinned host, device or managed memory
static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host -> device on `st`.  Pinned sources and small copies go straight to the DMA engine (an
// asynchronous copy: the source must stay valid until `st` is synchronised -- every caller does
// so before returning); large pageable ones through the stager: parallel host copies into one
// pinned chunk overlapped with the DMA of the other, after which the source may be reused.
void host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes <= (size_t(1) << 20) || is_pinned(src)) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st), "H2D");
        return;
    }
    Stager& S = stager();
    std::lock_guard<std::mutex> lock(S.mu);
    S.init();
    const size_t kChunk = S.chunk;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    int k = 0;
    bool used[2] = {false, false};
    for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
        const size_t len = std::min(kChunk, bytes - off);
        if (used[k]) ck(cudaEventSynchronize(S.ev[k]), "stage wait");
        par_copy(static_cast<char*>(S.buf[k]), s + off, len, S.threads);
        ck(cudaMemcpyAsync(d + off, S.buf[k], len, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaEventRecord(S.ev[k], st), "event");
        used[k] = true;
    }
    for (int q = 0; q < 2; ++q)  // the buffers are reused by the next caller (any stream)
        if (used[q]) ck(cudaEventSynchronize(S.ev[q]), "stage wait");
}

// Device -> host on `st`, ordered after the work already on `st`.  Pinned destinations (and small
// copies) are enqueued and complete with the caller's next synchronisation; large pageable ones
// go through the stager and have landed in `dst` on return.
void device_to_host(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes <= (size_t(1) << 20) || is_pinned(dst)) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st), "D2H");
        return;
    }
    Stager& S = stager();
    std::lock_guard<std::mutex> lock(S.mu);
    S.init();
    const size_t kChunk = S.chunk;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    // chunk i lands in buffer i & 1; the host copy-out of chunk i overlaps the DMA of chunk i+1
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto enqueue = [&](size_t i) {
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        ck(cudaMemcpyAsync(S.buf[i & 1], s + off, len, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaEventRecord(S.ev[i & 1], st), "event");
    };
    enqueue(0);
    for (size_t i = 0; i < nch; ++i) {
        if (i + 1 < nch) enqueue(i + 1);
        ck(cudaEventSynchronize(S.ev[i & 1]), "stage wait");
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        par_copy(d + off, static_cast<const char*>(S.buf[i & 1]), len, S.threads);
    }
}

void Engine::upload_host(void* dst, const void* src, size_t bytes) { host_to_device(dst, src, bytes, st); }


}  // namespace bgabp
