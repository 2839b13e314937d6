// util.cuh -- error plumbing and small device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <unordered_map>
#include <string>
#include <vector>

namespace ipcg {

// error kinds mirror the reference's exception types (ipcomp_b200.h)
enum ErrKind : int { OK = 0, EINVAL_ = 1, ERUNTIME = 2, EDOMAIN = 3, EINFEASIBLE = 4, ECUDA = 5 };

struct Error : std::runtime_error {
    int kind;
    Error(int k, const std::string &m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char *what, const char *file, int line) {
    throw Error(ECUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                           std::to_string(line));
}
#define CK(x)                                                          \
    do {                                                               \
        cudaError_t _e = (x);                                          \
        if (_e != cudaSuccess) ::ipcg::throw_cuda(_e, #x, __FILE__, __LINE__); \
    } while (0)
// every kernel launch goes through CKL(): checks the launch and counts it on the counter of
// the context whose API call runs on this thread (ipcg_kernel_launches); a process-wide one
// outside any call
inline unsigned long long *&current_launches() {
    thread_local unsigned long long *p = nullptr;
    return p;
}
inline unsigned long long &launch_counter() {
    static unsigned long long global = 0;
    unsigned long long *c = current_launches();
    return c ? *c : global;
}
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
// true the first time it is called for the current device (per-device one-time setup such as
// cudaFuncSetAttribute, which applies to the device current when it is called)
template <int Slot>
inline bool first_on_device() {
    static unsigned long long mask = 0;  // devices 0..63
    const unsigned long long bit = 1ull << (current_device() & 63);
    const bool first = !(__atomic_fetch_or(&mask, bit, __ATOMIC_RELAXED) & bit);
    return first;
}
#define CKL()                              \
    do {                                   \
        ++::ipcg::launch_counter();        \
        CK(cudaGetLastError());            \
    } while (0)

// Small device->host result reads on the hot path (sizes, CRCs, status words) go through
// mapped page-locked memory: a kernel stores them over PCIe, then the stream is synchronized.
// A cudaMemcpy D2H would queue on the copy engine behind any bulk transfer in flight (a
// host-async copy-out of 512 MiB holds it ~10 ms).  Synchronizes `st`; defined in ipcg.cu.
void readback(void *dst, const void *src_dev, size_t bytes, cudaStream_t st);

// Optional per-kernel-family timing: CUDA events recorded on the launching stream
// around each family (enabled by ipcg_profile_enable); read back by ipcg_profile_read.
struct Profiler {
    bool enabled = false;
    struct Rec {
        const char *name;
        cudaEvent_t a, b;
        uint64_t bytes;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t ev() {
        if (pool.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
};
// the profiler of the context whose API call runs on this thread (a process-wide one otherwise)
inline Profiler *&current_profiler() {
    thread_local Profiler *p = nullptr;
    return p;
}
inline Profiler &profiler() {
    static Profiler global;
    Profiler *p = current_profiler();
    return p ? *p : global;
}
struct ProfScope {
    int idx = -1;
    cudaStream_t st;
    ProfScope(const char *name, cudaStream_t s, uint64_t bytes = 0) : st(s) {
        Profiler &p = profiler();
        if (!p.enabled) return;
        Profiler::Rec r{name, p.ev(), p.ev(), bytes};
        cudaEventRecord(r.a, s);
        p.recs.push_back(r);
        idx = (int)p.recs.size() - 1;
    }
    ~ProfScope() {
        if (idx >= 0) cudaEventRecord(profiler().recs[idx].b, st);
    }
};

// Grow-only device scratch owned by a context.  Blocks are handed out best-fit (within
// 25% + 1 MiB of the request) and go back to the pool, not to CUDA: every user enqueues on
// the context's stream, so a block returned by one call is reused, stream-ordered, by the
// next.  (cudaMallocAsync of multi-GB buffers per call was measured blocking the host for
// up to 200 ms whenever the CUDA pool had to map memory again, leaving the GPU idle.)
//
// Graph capture (ipcg.cu, compress graphs): while `arena` is set every request is carved from
// that caller-owned slab by a bump pointer and never returned, so the captured kernels keep
// valid addresses for every replay; `tally` sums a call's (rounded) requests -- the slab size
// the next call of the same shape needs.
struct ScratchPool {
    std::multimap<size_t, void *> free_;
    std::unordered_map<void *, size_t> size_;
    uint8_t *arena = nullptr;
    size_t arena_cap = 0, arena_off = 0;
    bool arena_over = false;
    size_t tally = 0;
    void *get(size_t bytes, cudaStream_t st) {
        bytes = (bytes + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        tally += bytes;
        if (arena) {
            if (arena_off + bytes > arena_cap) {  // the capture is discarded (never launched)
                arena_over = true;
                return arena;
            }
            void *p = arena + arena_off;
            arena_off += bytes;
            return p;
        }
        auto it = free_.lower_bound(bytes);
        if (it != free_.end() && it->first <= bytes + bytes / 4 + (size_t(1) << 20)) {
            void *p = it->second;
            free_.erase(it);
            return p;
        }
        void *p = nullptr;
        CK(cudaMallocAsync(&p, bytes, st));
        size_[p] = bytes;
        return p;
    }
    void put(void *p) {
        if (arena) return;
        if (p) free_.emplace(size_.at(p), p);
    }
    void release_all(cudaStream_t st) {  // caller has synchronized
        for (auto &kv : size_) cudaFreeAsync(kv.first, st);
        free_.clear();
        size_.clear();
    }
};
// the pool of the context whose API call is running on this thread (set by the C-ABI entry)
inline ScratchPool *&current_scratch() {
    thread_local ScratchPool *p = nullptr;
    return p;
}
inline void *scratch_get(size_t bytes, cudaStream_t st) {
    if (ScratchPool *sp = current_scratch()) return sp->get(bytes, st);
    void *p = nullptr;
    CK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
    return p;
}
inline void scratch_put(void *p, cudaStream_t st) {
    if (!p) return;
    if (ScratchPool *sp = current_scratch()) sp->put(p);
    else cudaFreeAsync(p, st);
}

// stream-ordered temporaries released together
struct DevAlloc {
    std::vector<void *> ptrs;
    cudaStream_t st = nullptr;
    void *get(size_t bytes, cudaStream_t s) {
        void *p = scratch_get(bytes, s);
        ptrs.push_back(p);
        st = s;
        return p;
    }
    ~DevAlloc() {
        for (void *p : ptrs) scratch_put(p, st);
    }
};

// dev timeline marks from inside the stages (IPCG_DEBUG_TIMELINE): named events, printed and
// released by ipcg.cu's Timeline after the call's final sync
inline std::vector<std::pair<std::string, cudaEvent_t>> &debug_marks() {
    static std::vector<std::pair<std::string, cudaEvent_t>> v;
    return v;
}
inline void debug_mark(const char *name, int level, cudaStream_t s) {
    static const bool on = getenv("IPCG_DEBUG_TIMELINE") != nullptr;
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    debug_marks().push_back({std::string(name) + std::to_string(level), e});
}

// SM count of the current device (cached per device)
inline int num_sms() {
    static int cache[64] = {0};
    const int dev = current_device() & 63;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device());
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
    uint64_t g = (n + block - 1) / block;
    if (g == 0) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

#if defined(__CUDACC__)
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
#endif

}  // namespace ipcg
