// scratch.cuh -- library-owned device memory: a per-device memory pool and
// persistent, stream-ordered scratch arenas (host code, included by hexval.cu).
//
// Every call needs scratch for its control block, its work queues and the
// subdivision kernel's per-warp node stacks (sized for the warps that can be
// resident, ~1.1 MB per warp: the depth-sorted stack's worst case, DESIGN.md
// section 5).  Instead of allocating that per call, a call borrows an arena:
//   * an arena last used on the same stream is taken first (no wait at all);
//   * else an arena whose last use has completed (its event has fired);
//   * else a new arena is created -- so the number of arenas is the number of
//     streams with calls in flight at the same time, not the number of calls.
// Before using an arena last touched by another stream the call makes its
// stream wait for that use (cudaStreamWaitEvent), so reuse is stream-ordered
// and needs no host synchronisation.  An arena grows (stream-ordered free +
// allocation) only when a call needs more than it holds; in steady state a
// call allocates nothing.  Memory comes from a pool the library owns
// (cudaMemPoolCreate, release threshold on that pool only): the process's
// default pool is left alone.  hexval_scratch_release() frees every arena.
//
// Calls made while their stream is being captured into a CUDA graph allocate
// per call from the same pool instead (graph memory nodes), since an arena
// shared with eager work cannot be referenced from a replayable graph.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <vector>

namespace hexval_scratch {

struct Arena {
    char* base = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;           // recorded after the last call that used the arena
    unsigned long long stream_id = 0;   // stream of that call (0: never used)
    bool busy = false;                  // a host thread is enqueueing work that uses it
};

struct DevicePool {
    bool init = false;
    cudaMemPool_t pool = nullptr;
    std::vector<Arena*> arenas;
};

inline std::mutex& mu() {
    static std::mutex m;
    return m;
}
inline DevicePool* pools() {
    static DevicePool p[64];
    return p;
}

inline cudaMemPool_t device_pool(int dev) {
    DevicePool& d = pools()[dev & 63];
    if (!d.init) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&d.pool, &props) != cudaSuccess) {
            cudaGetLastError();
            d.pool = nullptr;
        } else {
            uint64_t thr = UINT64_MAX;                       // keep freed blocks: calls re-borrow them
            cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        d.init = true;
    }
    return d.pool;
}

// stream-ordered allocation from the library's pool (default pool if it could not be created)
inline cudaError_t alloc_async(void** p, size_t bytes, cudaStream_t stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu());
        pool = device_pool(dev);
    }
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, stream) : cudaMallocAsync(p, bytes, stream);
}

// A borrowed block of scratch: base pointer valid for the work the caller enqueues on
// `stream` between acquire() and release().
struct Lease {
    char* base = nullptr;
    Arena* arena = nullptr;             // null: per-call allocation (graph capture)
    int dev = 0;
};

inline bool capturing(cudaStream_t stream) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st != cudaStreamCaptureStatusNone;
}

inline cudaError_t acquire(Lease& L, size_t bytes, cudaStream_t stream) {
    cudaGetDevice(&L.dev);
    if (capturing(stream)) {
        L.arena = nullptr;
        return alloc_async((void**)&L.base, bytes, stream);
    }
    unsigned long long sid = 0;
    if (cudaStreamGetId(stream, &sid) != cudaSuccess) return cudaGetLastError();
    Arena* a = nullptr;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu());
        pool = device_pool(L.dev);
        auto& list = pools()[L.dev & 63].arenas;
        for (Arena* x : list)                               // same stream: already ordered
            if (!x->busy && x->stream_id == sid) { a = x; break; }
        if (!a)
            for (Arena* x : list)                           // idle: its last use has completed
                if (!x->busy && (x->stream_id == 0 || cudaEventQuery(x->ev) == cudaSuccess)) { a = x; break; }
        if (!a) {
            a = new Arena();
            list.push_back(a);
        }
        a->busy = true;
    }
    cudaGetLastError();                                     // cudaEventQuery's cudaErrorNotReady
    if (!a->ev && cudaEventCreateWithFlags(&a->ev, cudaEventDisableTiming) != cudaSuccess) {
        a->busy = false;
        return cudaErrorMemoryAllocation;
    }
    if (a->stream_id != 0 && a->stream_id != sid) cudaStreamWaitEvent(stream, a->ev, 0);
    if (a->cap < bytes) {
        if (a->base) cudaFreeAsync(a->base, stream);
        a->base = nullptr;
        a->cap = 0;
        const size_t want = bytes + bytes / 4;              // headroom: grow rarely
        const cudaError_t e = pool ? cudaMallocFromPoolAsync((void**)&a->base, want, pool, stream)
                                   : cudaMallocAsync((void**)&a->base, want, stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            a->base = nullptr;
            std::lock_guard<std::mutex> lk(mu());
            a->busy = false;
            return e;
        }
        a->cap = want;
    }
    L.arena = a;
    L.base = a->base;
    return cudaSuccess;
}

inline void release(Lease& L, cudaStream_t stream) {
    if (!L.arena) {
        if (L.base) cudaFreeAsync(L.base, stream);
        L.base = nullptr;
        return;
    }
    unsigned long long sid = 0;
    cudaStreamGetId(stream, &sid);
    cudaEventRecord(L.arena->ev, stream);
    std::lock_guard<std::mutex> lk(mu());
    L.arena->stream_id = sid;
    L.arena->busy = false;
    L.arena = nullptr;
}

// bytes reserved by the arenas of `dev` and their number
inline void info(int dev, size_t* bytes, int* count) {
    std::lock_guard<std::mutex> lk(mu());
    size_t b = 0;
    for (Arena* x : pools()[dev & 63].arenas) b += x->cap;
    if (bytes) *bytes = b;
    if (count) *count = (int)pools()[dev & 63].arenas.size();
}

// free every idle arena of `dev` (waits for their last uses); returns the number freed
inline int release_all(int dev) {
    std::lock_guard<std::mutex> lk(mu());
    auto& list = pools()[dev & 63].arenas;
    int freed = 0;
    std::vector<Arena*> keep;
    for (Arena* x : list) {
        if (x->busy) { keep.push_back(x); continue; }
        if (x->ev) cudaEventSynchronize(x->ev);
        if (x->base) cudaFree(x->base);
        if (x->ev) cudaEventDestroy(x->ev);
        delete x;
        ++freed;
    }
    list.swap(keep);
    if (pools()[dev & 63].pool) cudaMemPoolTrimTo(pools()[dev & 63].pool, 0);
    return freed;
}

}  // namespace hexval_scratch
