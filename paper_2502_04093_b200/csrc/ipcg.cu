// ipcg.cu -- orchestration of the B200 hot path behind the C-ABI (include/ipcomp_b200.h).
//
//   compress_field   (pipeline.hpp:140-223): range scan -> per level L..1: one
//                    predict+quantize launch per (level, axis) pass -> loss-table replay
//                    -> transpose bitplanes + XOR -> DeflateBatch (32 planes) -> one sync ->
//                    host index (archive.cpp:31-65) -> device payload gather.
//   reconstruct_field (pipeline.hpp:227-287) / refine_field (:294-352): host plans the
//                    block reads (partial-bitplane fetch, byte accounting), device gathers
//                    the blocks, CRC-32 + inflate, XOR-decode+merge, per-pass reconstruction
//                    with in-traversal outlier overwrite.
// All device work of a call is ordered on the context's stream; temporaries, archive
// payloads and session codewords come from the context's grow-only ScratchPool
// (util.cuh), so steady-state calls allocate nothing.
#include <functional>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../include/ipcomp_b200.h"
#include "assemble.cuh"
#include "deflate.cuh"
#include "grid.h"
#include "host.h"
#include "inflate.cuh"
#include "numerics.cuh"

using namespace ipcg;

namespace ipcg {
namespace rb {
__global__ void k_readback(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
struct MappedBuf {  // grow-only mapped page-locked staging, one per host thread
    void *h = nullptr;
    size_t cap = 0;
    ~MappedBuf() {
        if (h) cudaFreeHost(h);
    }
};
}  // namespace rb

void compute_metrics_device(int scalar, const void *a, const void *b, uint64_t n, double out[3], cudaStream_t st);

// several device ranges read back behind one stream synchronization
struct RbPart {
    void *dst;
    const void *src;
    size_t bytes;
};
void readback_parts(const RbPart *parts, int np, cudaStream_t st) {
    size_t total = 0;
    for (int i = 0; i < np; ++i) total += (parts[i].bytes + 15) & ~size_t(15);
    if (!total) return;
    thread_local rb::MappedBuf mb;
    if (total > mb.cap) {
        CK(cudaStreamSynchronize(st));
        if (mb.h) CK(cudaFreeHost(mb.h));
        mb.h = nullptr;
        const size_t cap = std::max<size_t>(total, 64 << 10);
        CK(cudaHostAlloc(&mb.h, cap, cudaHostAllocMapped));
        mb.cap = cap;
    }
    void *d = nullptr;
    CK(cudaHostGetDevicePointer(&d, mb.h, 0));
    size_t off = 0;
    for (int i = 0; i < np; ++i) {
        const size_t b = parts[i].bytes;
        if (b) {
            rb::k_readback<<<(unsigned)std::min<size_t>((b + 255) / 256, 64), 256, 0, st>>>(
                static_cast<const uint8_t *>(parts[i].src), static_cast<uint8_t *>(d) + off, b);
            CKL();
        }
        off += (b + 15) & ~size_t(15);
    }
    CK(cudaStreamSynchronize(st));
    off = 0;
    for (int i = 0; i < np; ++i) {
        std::memcpy(parts[i].dst, static_cast<uint8_t *>(mb.h) + off, parts[i].bytes);
        off += (parts[i].bytes + 15) & ~size_t(15);
    }
}
void readback(void *dst, const void *src_dev, size_t bytes, cudaStream_t st) {
    const RbPart p{dst, src_dev, bytes};
    readback_parts(&p, 1, st);
}
}  // namespace ipcg

struct ipcg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;  // all work is ordered on this stream (forks join back)
    cudaStream_t own_stream = nullptr;
    std::vector<cudaStream_t> side;  // fork targets (per-level chains)
    std::vector<cudaStream_t> loss;  // per-level loss-table streams (highest priority)
    std::vector<cudaStream_t> odside;  // per-level streams of the deflate on-demand parse
    cudaStream_t quant = nullptr;      // compress's prediction/quantization chain (highest priority)
    cudaStream_t h2d = nullptr;        // compress's upload of a host field
    // a host field uploaded ahead of its compress (ipcg_stage_field): context-owned device copy
    struct Staged {
        cudaStream_t stream = nullptr;
        cudaEvent_t ready = nullptr;
        void *dev = nullptr;
        size_t cap = 0;
        const void *host = nullptr;  // the staged field (nullptr: none pending)
        size_t bytes = 0, issued = 0;  // bytes whose copy is enqueued so far (stage_pump)
    } staged;
    std::vector<cudaEvent_t> events;
    size_t events_used = 0;
    ScratchPool scratch;  // per-call device scratch, reused across calls (also archive/session memory)
    Profiler prof;        // per-family timing (ipcg_profile_enable)
    unsigned long long launches = 0;  // kernels this context launched (ipcg_kernel_launches)
    std::string err;
    void *pinned = nullptr;
    size_t pinned_cap = 0;
    void *src_pinned = nullptr;  // staging of block reads from a seekable archive source
    size_t src_pinned_cap = 0;
    // host-async mode (ipcg_set_host_async): a retrieval's device->host copy of its values
    // runs on `copy` from a ring of device output buffers, so the next call's kernels (and
    // its host->device uploads: PCIe is full duplex) overlap it
    bool host_async = false;
    cudaStream_t copy = nullptr;
    struct OutSlot {
        void *p = nullptr;
        size_t cap = 0;
        cudaEvent_t ready = nullptr, done = nullptr;  // values final (on stream) / copied out
    };
    std::vector<OutSlot> ring;
    size_t ring_next = 0;
    cudaEvent_t copy_tail = nullptr;  // the last copy enqueued
    bool copy_pending = false;
    // compress graphs (compress_entry): a device-resident field of a shape seen before replays
    // the whole captured kernel sequence of its compress with one launch
    struct CGraph {
        int scalar, nd, interp, lp;
        uint64_t dims[4], cap, eb_bits;
        int state = 0;        // 0 seen once (its scratch tallied), 1 captured, 2 not capturable
        size_t need = 0;      // scratch bytes one compress of this shape requests
        uint8_t *slab = nullptr;  // input slot + every scratch block the captured calls use
        cudaGraphExec_t exec = nullptr;
        void *aout = nullptr;     // AsmOut in the slab
        uint8_t *arch = nullptr;  // assembled archive in the slab
        unsigned long long nlaunch = 0;
        uint64_t used = 0;
    };
    std::vector<CGraph> graphs;
    uint64_t graph_clock = 0;
    cudaStream_t capture = nullptr;  // graphs are captured on this stream
};

struct ipcg_archive {
    ipcg_index ix{};
    const uint8_t *bytes = nullptr;
    uint64_t size = 0;
    bool on_device = false;
    uint8_t *owned = nullptr;  // device buffer when produced by ipcg_compress
    cudaStream_t owner = nullptr;  // stream `owned` was allocated on (reused there, stream-ordered)
    ScratchPool *pool = nullptr;   // the creating context's pool `owned` returns to
    uint64_t payload_read = 0;
    int device = 0;
    ipcg_read_fn read = nullptr;  // seekable source (ipcg_archive_open_source): bytes == nullptr
    void *user = nullptr;
    // device archives: the 21-byte header of every plane block, [level-1][plane], read back once
    // on the first retrieval (the archive is immutable) instead of per call
    std::vector<uint8_t> hdr_all;
};

struct ipcg_session {
    uint32_t archive_crc = 0;
    int levels = 0, lp = 0;
    int k[IPCG_MAX_LEVELS] = {0};
    uint64_t count[IPCG_MAX_LEVELS] = {0};
    uint32_t *merged[IPCG_MAX_LEVELS] = {nullptr};  // device, progressive levels only
    cudaStream_t owner = nullptr;                     // stream the merged arrays are released on
    ScratchPool *pool = nullptr;                      // and the pool they return to
    int device = 0;
};

namespace {

// ------------------------------------------------------------------ helpers
struct DBuf {  // stream-ordered device allocation
    void *p = nullptr;
    cudaStream_t st = nullptr;
    DBuf() = default;
    DBuf(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes) p = scratch_get(bytes, s);
    }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
    DBuf &operator=(DBuf &&o) noexcept {
        release();
        p = o.p;
        st = o.st;
        o.p = nullptr;
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        scratch_put(p, st);
        p = nullptr;
    }
    template <class T>
    T *as() const {
        return static_cast<T *>(p);
    }
};

// side stream i: 0 carries work off the critical path (lowest priority), the others the
// critical chains (highest priority), so the scheduler fills the gaps of the latter with it
// Stream priorities for compress: level 1's lossless chain (side stream 1) is the critical
// path but throughput-bound -- it runs at the lowest priority and fills whatever the
// others leave; the coarser levels' latency-bound chains and the loss tables run at the
// highest, so their few CTAs are dispatched as soon as an SM frees up instead of queueing
// behind level 1's kernels.  Measured on cfg2: 46.4 ms per compress and run-to-run stable,
// vs 57 ms (loss tables on one shared stream) and a bimodal 48-58 ms (level 1 highest).
static int prio_for(bool low) {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    return low ? least : greatest;
}
// dev: IPCG_PRIO_MODE=1 inverts the lossless streams (level 1 highest, coarser levels lowest),
// 2 puts every lossless stream at the default priority
static int lossless_prio(bool level1) {
    static const int mode = getenv("IPCG_PRIO_MODE") ? atoi(getenv("IPCG_PRIO_MODE")) : 0;
    if (mode == 2) return 0;
    return prio_for(mode == 1 ? !level1 : level1);
}

cudaStream_t side_stream(ipcg_ctx *c, size_t i) {
    while (c->side.size() <= i) {
        cudaStream_t s;
        CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, lossless_prio(c->side.size() == 1)));
        c->side.push_back(s);
    }
    return c->side[i];
}

cudaStream_t loss_stream(ipcg_ctx *c, size_t i) {
    while (c->loss.size() <= i) {
        cudaStream_t s;
        CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio_for(false)));
        c->loss.push_back(s);
    }
    return c->loss[i];
}

// the stream compress runs its level-by-level quantization chain on: highest priority, because
// level 1's quantization starts the critical path (its lossless stage) and otherwise queued
// behind the coarser levels' lossless kernels (measured: level-1 quant done at 4.4 ms instead of ~1)
cudaStream_t quant_stream(ipcg_ctx *c) {
    if (!c->quant) CK(cudaStreamCreateWithPriority(&c->quant, cudaStreamNonBlocking, prio_for(false)));
    return c->quant;
}

// level li's on-demand-parse stream (level 1, throughput-bound, at the lowest priority like its
// main deflate chain; the latency-bound coarser levels at the highest)
cudaStream_t od_stream(ipcg_ctx *c, size_t li) {
    while (c->odside.size() <= li) {
        cudaStream_t s;
        // the on-demand parse streams at the highest priority: level 1's latency-bound parse then
        // ends (IPCG_DEBUG_TIMELINE "O14") at ~20 ms instead of last at ~27 ms, behind the dense
        // search it shares the GPU with; compress 29.9 -> 29.1 ms (IPCG_OD_PRIO=0: the old order)
        static const int od_hi = getenv("IPCG_OD_PRIO") ? atoi(getenv("IPCG_OD_PRIO")) : 1;
        CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, od_hi ? prio_for(false) : lossless_prio(c->odside.size() == 0)));
        c->odside.push_back(s);
    }
    return c->odside[li];
}

// an event from the context's pool (reused across calls: a wait captures the event's
// state at enqueue time)
cudaEvent_t pool_event(ipcg_ctx *c) {
    if (c->events_used == c->events.size()) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->events.push_back(e);
    }
    return c->events[c->events_used++];
}

// `to` waits for everything enqueued on `from` so far
void stream_dep(ipcg_ctx *c, cudaStream_t from, cudaStream_t to) {
    cudaEvent_t e = pool_event(c);
    CK(cudaEventRecord(e, from));
    CK(cudaStreamWaitEvent(to, e, 0));
}

void *pinned(ipcg_ctx *c, size_t bytes) {
    if (bytes > c->pinned_cap) {
        if (c->pinned) CK(cudaFreeHost(c->pinned));
        size_t cap = std::max<size_t>(bytes, 1 << 20);
        CK(cudaMallocHost(&c->pinned, cap));
        c->pinned_cap = cap;
    }
    return c->pinned;
}

// next output buffer of the host-async ring (grown to `bytes` once its last copy is done)
constexpr size_t RING_SLOTS = 4;
ipcg_ctx::OutSlot &out_slot(ipcg_ctx *c, size_t bytes) {
    if (c->ring.empty()) {
        c->ring.resize(RING_SLOTS);
        for (auto &sl : c->ring) {
            CK(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
        }
    }
    ipcg_ctx::OutSlot &sl = c->ring[c->ring_next];
    c->ring_next = (c->ring_next + 1) % c->ring.size();
    if (sl.cap < bytes) {
        CK(cudaEventSynchronize(sl.done));
        if (sl.p) CK(cudaFree(sl.p));
        sl.p = nullptr;
        CK(cudaMalloc(&sl.p, bytes));
        sl.cap = bytes;
    }
    return sl;
}

// host-async copies issued so far have landed in host memory
void drain_copies(ipcg_ctx *c) {
    if (c->copy && c->copy_pending) {
        CK(cudaStreamSynchronize(c->copy));
        c->copy_pending = false;
    }
}

thread_local std::string g_host_err;  // errors of context-free (host-only) calls

template <class F>
int guarded(ipcg_ctx *c, F &&f) {
    std::string &err = c ? c->err : g_host_err;
    struct Bind {  // this call's scratch pool, profiler and launch counter
        ScratchPool *prev;
        Profiler *prev_prof;
        unsigned long long *prev_launches;
        explicit Bind(ipcg_ctx *c)
            : prev(current_scratch()), prev_prof(current_profiler()), prev_launches(current_launches()) {
            current_scratch() = c ? &c->scratch : nullptr;
            current_profiler() = c ? &c->prof : nullptr;
            current_launches() = c ? &c->launches : nullptr;
        }
        ~Bind() {
            current_scratch() = prev;
            current_profiler() = prev_prof;
            current_launches() = prev_launches;
        }
    } bind(c);
    try {
        if (c) CK(cudaSetDevice(c->device));
        f();
        return IPCG_OK;
    } catch (const Error &e) {
        err = e.what();
        return e.kind;
    } catch (const std::bad_alloc &) {
        err = "out of host memory";
        return IPCG_ERUNTIME;
    } catch (const std::exception &e) {
        err = e.what();
        return IPCG_ERUNTIME;
    }
}

void validate_dims(const uint64_t *dims, int nd) {  // common.hpp:35-42
    if (nd < 1 || nd > 4) throw Error(EINVAL_, "grid must have between 1 and 4 dimensions");
    for (int i = 0; i < nd; ++i)
        if (dims[i] < 1) throw Error(EINVAL_, "grid extents must be positive");
}

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// ------------------------------------------------------------- byte gather
struct CopyDesc {
    const uint8_t *src;
    uint64_t dst_off;
    uint64_t len;
};

__global__ void __launch_bounds__(512) k_gather(const CopyDesc *d, int nd, uint8_t *dst) {
    const int i = blockIdx.x;
    if (i >= nd) return;
    const CopyDesc c = d[i];
    uint8_t *o = dst + c.dst_off;
    const uint8_t *s = c.src;
    uint64_t len = c.len;
    // bytes until the destination is 16-byte aligned (plane rows are), then 16-byte stores whose
    // source words are funnel-shifted from aligned 4-byte loads (archive payloads start at
    // arbitrary bytes), then the tail bytes
    const uint64_t head = min(len, (uint64_t)((16 - ((uintptr_t)o & 15)) & 15));
    if (threadIdx.x < head) o[threadIdx.x] = s[threadIdx.x];
    o += head, s += head, len -= head;
    const uint64_t nv = len / 16;
    const unsigned sh = (unsigned)((uintptr_t)s & 3) * 8;
    const uint32_t *sw = reinterpret_cast<const uint32_t *>((uintptr_t)s & ~uintptr_t(3));
    uint4 *ov = reinterpret_cast<uint4 *>(o);
    for (uint64_t k = threadIdx.x; k < nv; k += blockDim.x) {
        const uint32_t *q = sw + 4 * k;
        const uint32_t w0 = __ldg(q), w1 = __ldg(q + 1), w2 = __ldg(q + 2), w3 = __ldg(q + 3);
        const uint32_t w4 = sh ? __ldg(q + 4) : 0u;  // only read when the source is unaligned
        ov[k] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                           __funnelshift_r(w3, w4, sh));
    }
    for (uint64_t k = nv * 16 + threadIdx.x; k < len; k += blockDim.x) o[k] = s[k];
}

// dst == nullptr: dst_off are absolute device addresses
void gather(ipcg_ctx *c, std::vector<CopyDesc> descs, uint8_t *dst) {
    // split long copies so every SM participates
    std::vector<CopyDesc> pieces;
    pieces.reserve(descs.size());
    const uint64_t piece = 64 << 10;
    for (const CopyDesc &d : descs)
        for (uint64_t o = 0; o < d.len; o += piece)
            pieces.push_back(CopyDesc{d.src + o, d.dst_off + o, std::min(piece, d.len - o)});
    if (pieces.empty()) return;
    DBuf dd(pieces.size() * sizeof(CopyDesc), c->stream);
    // from pageable memory: the driver stages it before returning, so no stream sync is needed
    // to reuse `pieces` (a pinned staging buffer cost a sync per call)
    CK(cudaMemcpyAsync(dd.p, pieces.data(), pieces.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice, c->stream));
    k_gather<<<(unsigned)pieces.size(), 512, 0, c->stream>>>(dd.as<CopyDesc>(), (int)pieces.size(), dst);
    CKL();
}

// ---------------------------------------------------------------- compress
// dev timeline (IPCG_DEBUG_TIMELINE=1): when each stream reaches the marked points of a compress
struct Timeline {
    bool on = getenv("IPCG_DEBUG_TIMELINE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    cudaEvent_t mark(const std::string &name, cudaStream_t s) {
        if (!on) return nullptr;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, s));
        ev.push_back({name, e});
        return e;
    }
    void print() {
        if (!on || ev.empty()) return;
        CK(cudaDeviceSynchronize());
        for (auto &x : debug_marks()) ev.push_back(x);
        debug_marks().clear();
        std::vector<std::pair<float, std::string>> t;
        for (auto &x : ev) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ev[0].second, x.second));
            t.push_back({ms, x.first});
        }
        std::sort(t.begin(), t.end());
        fprintf(stderr, "[timeline]");
        for (auto &x : t) fprintf(stderr, " %s@%.1f", x.second.c_str(), x.first);
        fprintf(stderr, "\n");
        for (auto &x : ev) cudaEventDestroy(x.second);
        ev.clear();
    }
};

// host-side phase timer (IPCG_DEBUG_TIMING=1): where a call's wall time goes
struct PhaseTimer {
    bool on = getenv("IPCG_DEBUG_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    std::string line;
    void mark(const char *what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        snprintf(buf, sizeof(buf), " %s %.2f", what, std::chrono::duration<double, std::milli>(now - last).count());
        line += buf;
        last = now;
    }
    ~PhaseTimer() {
        if (on) fprintf(stderr, "[ipcg timing]%s total %.2f ms\n", line.c_str(),
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

// what a captured compress leaves for its replays (compress graphs, below)
struct CaptureOut {
    AsmOut *aout = nullptr;
    uint8_t *arch = nullptr;
    uint64_t capacity = 0;
};

// index bytes of an archive (host.cpp serialize_index: 12-byte preamble, dims, 20 bytes of
// header fields, 808 bytes per level)
inline uint64_t index_bytes_for(int nd, int levels) { return 12 + 8 * (uint64_t)nd + 20 + 808 * (uint64_t)levels; }

ipcg_archive *compress_impl(ipcg_ctx *c, int scalar, const void *values, int on_dev, const uint64_t *dims, int nd,
                            double eb, int interp, int lp_opt, uint64_t cap, CaptureOut *capture = nullptr) {
    PhaseTimer tm;
    validate_dims(dims, nd);
    if (scalar != 0 && scalar != 1) throw Error(EINVAL_, "field scalars must be f32 or f64");
    if (!(eb > 0.0) || !std::isfinite(eb)) throw Error(EINVAL_, "error bound must be positive and finite");
    const Geometry G = make_geometry(dims, nd, max_levels_for_cap(cap));
    const int L = G.levels;
    const int lp = lp_opt == 0 ? L : lp_opt;
    if (lp < 1 || lp > L) throw Error(EINVAL_, "first progressive level out of range");
    if (L > IPCG_MAX_LEVELS) throw Error(EINVAL_, "too many levels for this build");
    const bool cubic = interp == 1;
    const int w = scalar == 0 ? 4 : 8;
    const uint64_t n = G.n;
    cudaStream_t st = c->stream;

    DBuf vals_buf;
    const void *vals = values;
    if (!on_dev) {
        vals_buf = DBuf(n * w, st);
        vals = vals_buf.p;
    }
    DBuf state(n * w, st), dev(n * 8, st);
    CK(cudaMemsetAsync(state.p, 0, n * w, st));
    CK(cudaMemsetAsync(dev.p, 0, n * 8, st));
    // small per-call device state (assemble.cuh)
    using Small = AsmSmall;
    DBuf small(sizeof(Small), st);
    tm.mark("setup");
    Timeline tline;
    tline.mark("start", st);
    Small *sd = small.as<Small>();
    CK(cudaMemsetAsync(small.p, 0, sizeof(Small), st));
    // outliers: a bitmap over each level's ordinals and the exact values by ordinal
    uint64_t flag_words = 0;
    std::vector<uint64_t> fbase(L);
    for (int li = 0; li < L; ++li) fbase[li] = flag_words, flag_words += (G.level[li].count + 31) / 32;
    DBuf bits(n * 8, st), oflags(std::max<uint64_t>(flag_words, 1) * 4, st);
    CK(cudaMemsetAsync(oflags.p, 0, std::max<uint64_t>(flag_words, 1) * 4, st));
    const bool serial0 = profiler().enabled;
    c->events_used = 0;
    const cudaStream_t qs = serial0 ? st : quant_stream(c);
    if (qs != st) stream_dep(c, st, qs);
    // A host field is uploaded in two parts: first the rows whose leading coordinates are all even
    // -- every point the levels coarser than 1 read or write lies in them (their strides are >= 2
    // on every axis) -- then the rest, so the coarse levels' quantization and lossless stages run
    // while ~3/4 of the field is still crossing PCIe; level 1 and the range wait for all of it.
    cudaEvent_t all_ready = nullptr;
    if (!on_dev) {
        if (serial0) {
            CK(cudaMemcpyAsync(vals_buf.p, values, n * w, cudaMemcpyHostToDevice, st));
        } else {
            if (!c->h2d) CK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
            const cudaStream_t hs = c->h2d;
            stream_dep(c, st, hs);  // the buffer's stream-ordered allocation
            const bool split = L >= 2 && (nd == 2 || nd == 3) && dims[0] >= 2;
            uint8_t *dst = vals_buf.as<uint8_t>();
            const uint8_t *src = static_cast<const uint8_t *>(values);
            if (split) {
                const size_t rowb = (size_t)dims[nd - 1] * w;
                const size_t Y = nd == 3 ? (size_t)dims[1] : (size_t)dims[0], Z = nd == 3 ? (size_t)dims[0] : 1;
                auto rows3d = [&](size_t off, size_t height) {  // rows y = off, off+2, ... of every even z
                    if (!height) return;
                    cudaMemcpy3DParms m{};
                    m.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t *>(src) + off * rowb, 2 * rowb, rowb, Y);
                    m.dstPtr = make_cudaPitchedPtr(dst + off * rowb, 2 * rowb, rowb, Y);
                    m.extent = make_cudaExtent(rowb, height, nd == 3 ? (Z + 1) / 2 : 1);
                    m.kind = cudaMemcpyHostToDevice;
                    CK(cudaMemcpy3DAsync(&m, hs));
                };
                rows3d(0, (Y + 1) / 2);  // coarse rows: even y (and even z)
                cudaEvent_t coarse = pool_event(c);
                CK(cudaEventRecord(coarse, hs));
                CK(cudaStreamWaitEvent(qs, coarse, 0));
                rows3d(1, Y / 2);  // odd y of even z
                if (nd == 3 && Z >= 2) {  // odd z slabs
                    const size_t slab = Y * rowb;
                    CK(cudaMemcpy2DAsync(dst + slab, 2 * slab, src + slab, 2 * slab, slab, Z / 2, cudaMemcpyHostToDevice, hs));
                }
            } else {
                CK(cudaMemcpyAsync(dst, src, n * w, cudaMemcpyHostToDevice, hs));
            }
            all_ready = pool_event(c);
            CK(cudaEventRecord(all_ready, hs));
            if (!split) CK(cudaStreamWaitEvent(qs, all_ready, 0));
            if (qs != st) CK(cudaStreamWaitEvent(st, all_ready, 0));  // (st joins qs later anyway)
        }
    }
    auto range_once = [&] {
        ProfScope ps("range", qs, n * w);
        launch_range(vals, scalar, n, sd->range_part, sd->rng, qs);
    };
    if (!all_ready) range_once();

    // (Forking each level's lossless stage and the loss tables onto side streams was
    // measured: no gain -- level 1's kernels saturate the GPU, so overlap only hides the
    // small levels' latency tails, and those are a few ms.)
    // Only quantization is sequential across levels (level l predicts from the state the
    // coarser levels left).  Each level's lossless stage (bitplanes + deflate) forks onto its
    // own side stream and its loss table onto its own highest-priority stream: the small
    // levels' latency-bound chains (zlib's serial Huffman builds, single-CTA scans) then run
    // under level 1's throughput-bound kernels.  Everything joins back into `st` before the
    // results are read.
    // With the per-family profiler on (bench.py's roofline step, never the timed loop) all
    // of it stays on `st`, so each family's CUDA-event span covers only its own kernels.
    const bool serial = serial0;
    auto fork = [&](size_t i) { return serial ? st : side_stream(c, i); };
    cudaEvent_t fb_done = nullptr;  // last per-pass loss fallback (they share `dev`)
    std::vector<DBuf> nbs(L), wss(L), planes(L), outs(L);
    std::vector<uint64_t> pb(L), plane_stride(L), out_stride(L), sink_base(L);
    uint64_t base = 0;
    for (int level = L; level >= 1; --level) {
        const LevelGeom &lg = G.level[level - 1];
        const int li = level - 1;
        if (level == 1 && all_ready) {  // the whole field is on the device
            CK(cudaStreamWaitEvent(qs, all_ready, 0));
            range_once();
        }
        sink_base[li] = base;
        base += lg.count;
        pb[li] = (lg.count + 7) / 8;
        const uint64_t words = (lg.count + 31) / 32;
        plane_stride[li] = round_up(std::max<uint64_t>(words, 1), 4);  // words, 16-byte rows
        out_stride[li] = round_up(pb[li] + 16, 16);
        nbs[li] = DBuf(std::max<uint64_t>(lg.count, 1) * 4, st);
        wss[li] = DBuf(DeflateBatch::workspace_bytes(32, pb[li]), st);
        planes[li] = DBuf(32 * plane_stride[li] * 4, st);
        outs[li] = DBuf(32 * out_stride[li], st);
        tm.mark("alloc_l");
        uint32_t *nb = nbs[li].as<uint32_t>();
        const OutlierSink sink{&sd->ocount[li], oflags.as<uint32_t>() + fbase[li], bits.as<uint64_t>() + sink_base[li]};
        {
            ProfScope ps("quant_pass", qs, lg.count * (uint64_t)(2 * w + 4) + lg.count * (uint64_t)w);
            for (const PassDesc &pd : lg.passes)
                launch_quant_pass(vals, state.p, scalar, cubic, pd, eb, nb, &sd->lowor[li], sink, G.dims[G.nd - 1], qs);
        }
        tm.mark("quant");
        tline.mark("q" + std::to_string(level), qs);
        // lossless stage.  (No memset: k_bitplanes writes every word below the row length, zero
        // past `count`; the deflate stage never reads a row past its n = ceil(count/8) bytes.)
        cudaStream_t ds = fork(1 + (size_t)li);
        if (ds != st) stream_dep(c, qs, ds);
        {
            ProfScope ps("bitplanes", ds, lg.count * 8);
            launch_bitplanes(nb, lg.count, planes[li].as<uint32_t>(), plane_stride[li], ds);
        }
        cudaEvent_t after_match = tline.on ? nullptr : pool_event(c);
        if (tline.on) {
            CK(cudaEventCreate(&after_match));
            tline.ev.push_back({"m" + std::to_string(level), after_match});
        }
        const BackendResults res{sd->backend[li], sd->length[li], sd->crc[li], sd->payload[li]};
        cudaStream_t os = serial ? nullptr : od_stream(c, (size_t)li);
        DeflateBatch::run(planes[li].as<uint8_t>(), plane_stride[li] * 4, 32, pb[li], outs[li].as<uint8_t>(),
                          out_stride[li], wss[li].p, res, ds, after_match, os, os ? pool_event(c) : nullptr,
                          os ? pool_event(c) : nullptr);
        tline.mark("d" + std::to_string(level), ds);
        // loss table (measure_loss_table): replay per dropped-digit count d, on the level's own
        // highest-priority stream, started once this level's match search is done so it
        // overlaps the latency-bound parse/Huffman phases instead of competing with the
        // throughput-bound ones.  (One loss stream shared by all levels put level 1's table
        // behind level 2's, whose match search finishes late under level 1's kernels:
        // measured 57 ms per compress vs 39 ms without loss tables.)
        cudaStream_t ls = serial ? st : loss_stream(c, (size_t)li);
        static const int loss_early = getenv("IPCG_LOSS_EARLY") ? atoi(getenv("IPCG_LOSS_EARLY")) : 0;  // dev
        if (ls != st) {
            stream_dep(c, qs, ls);
            if (!loss_early) CK(cudaStreamWaitEvent(ls, after_match, 0));
        }
        {
            ProfScope psl("loss_table", ls, lg.count * 4);
            if (!launch_loss_fused(nb, G, level, cubic, 2.0 * eb, &sd->lowor[li], sd->raw[li], ls)) {
                // the per-pass fallback shares `dev` across levels: chain those in order
                if (fb_done) CK(cudaStreamWaitEvent(ls, fb_done, 0));
                for (int d = 1; d <= 32; ++d)
                    for (const PassDesc &pd : lg.passes)
                        launch_loss_pass(nb, dev.as<double>(), pd, cubic, 2.0 * eb, d, &sd->lowor[li], sd->raw[li], ls);
                for (const PassDesc &pd : lg.passes) launch_zero_pass(dev.as<double>(), pd, ls);
                if (ls != st) {
                    fb_done = pool_event(c);
                    CK(cudaEventRecord(fb_done, ls));
                }
            }
            launch_loss_finalize(sd->raw[li], &sd->lowor[li], sd->delta[li], ls);
        }
        tline.mark("L" + std::to_string(level), ls);
        tm.mark("deflate");
    }
    if (!serial) {
        stream_dep(c, qs, st);
        for (int li = 0; li < L; ++li) {
            stream_dep(c, loss_stream(c, (size_t)li), st);
            stream_dep(c, side_stream(c, 1 + (size_t)li), st);
        }
    }
    tm.mark("enqueue");
    // the archive, assembled on the device (assemble.cu): offsets by a device prefix sum, index,
    // block headers, payload gather, outlier blocks compacted in ordinal order.  One readback at
    // the end (the finished index); the host parses it like the reference's reader.
    AsmParams P{};
    P.scalar = scalar, P.interp = interp, P.nd = nd, P.levels = L, P.lp = lp, P.cap = (int)(uint8_t)cap;
    for (int i = 0; i < nd; ++i) P.dims[i] = dims[i];
    P.eb = eb;
    for (int li = 0; li < L; ++li) P.count[li] = G.level[li].count;
    std::vector<const uint32_t *> ofl(L);
    std::vector<const uint64_t *> obt(L);
    uint64_t max_tiles = 1;
    for (int li = 0; li < L; ++li) {
        ofl[li] = oflags.as<uint32_t>() + fbase[li];
        obt[li] = bits.as<uint64_t>() + sink_base[li];
        max_tiles = std::max<uint64_t>(max_tiles, ((G.level[li].count + 31) / 32 + 8191) / 8192);
    }
    DBuf descs((size_t)L * 32 * sizeof(AsmDesc), st), aout(sizeof(AsmOut), st), tiles(max_tiles * 4, st);
    ipcg_archive *a = new ipcg_archive;
    a->device = c->device;
    a->owner = st;
    a->pool = &c->scratch;
    a->on_device = true;
    uint64_t capacity = asm_capacity(P);
    AsmOut ho{};
    // the index's size is fixed by the shape: it comes back with the assembly result, behind
    // the call's one synchronization
    std::vector<uint8_t> index(index_bytes_for(nd, L));
    for (int attempt = 0; attempt < 2; ++attempt) {
        // stream-ordered pool memory: a cudaMalloc/cudaFree pair per call would synchronize the device
        a->owned = static_cast<uint8_t *>(c->scratch.get(std::max<uint64_t>(capacity, 1), st));
        launch_assemble(P, sd, a->owned, capacity, descs.as<AsmDesc>(), aout.as<AsmOut>(), ofl.data(), obt.data(),
                        tiles.as<uint32_t>(), st);
        if (capture) {  // enqueue only: the replays read the results back
            capture->aout = aout.as<AsmOut>();
            capture->arch = a->owned;
            capture->capacity = capacity;
            delete a;
            return nullptr;
        }
        const RbPart parts[2] = {{&ho, aout.p, sizeof(AsmOut)}, {index.data(), a->owned, index.size()}};
        readback_parts(parts, 2, st);
        tline.print();
        if (ho.fits) break;
        c->scratch.put(a->owned);  // more outliers than the 1/64 allowance: assemble again at the exact size
        a->owned = nullptr;
        capacity = ho.total;
    }
    if (!ho.fits || ho.index_bytes != index.size()) {
        delete a;
        throw Error(ERUNTIME, "archive assembly overflow");
    }
    tm.mark("assemble");
    try {
        parse_index(index.data(), index.size(), a->ix);  // also the identity (crc32 of the index)
    } catch (...) {
        c->scratch.put(a->owned);
        delete a;
        throw;
    }
    a->bytes = a->owned;
    a->size = ho.total;
    tm.mark("index");
    return a;
}

// ------------------------------------------------------------ compress graphs
// A small field's compress is bound by the host: ~230 launches, events and stream forks take
// ~0.9 ms to enqueue on cfg1 (64^3), while level 1's chain waits for them.  A device-resident
// field whose shape, error bound and options were compressed before replays that call's
// kernel sequence as one CUDA graph: the first call runs normally and tallies its scratch
// requests, the second is captured (multi-stream: the side, loss-table and parse streams join
// the capture through their events; per-node priorities kept) with every scratch block carved
// from a slab the graph owns, and every later call copies the field into the slab's input slot,
// launches the graph and reads back the assembly result and index behind one synchronization.
// The archive is then copied out of the slab into a block of its own.
constexpr uint64_t kGraphMaxBytes = 128ull << 20;  // fields up to 128 MiB (their slab: ~120 B/point)
constexpr size_t kGraphsKept = 4;

void free_graph(ipcg_ctx::CGraph &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.slab) cudaFree(g.slab);
    g.exec = nullptr, g.slab = nullptr;
}

ipcg_archive *compress_entry(ipcg_ctx *c, int scalar, const void *values, int on_dev, const uint64_t *dims, int nd,
                             double eb, int interp, int lp, uint64_t cap) {
    static const bool off = getenv("IPCG_NO_GRAPH") != nullptr;  // dev A/B knob
    const int w = scalar == 0 ? 4 : 8;
    uint64_t n = 1;
    bool shape_ok = nd >= 1 && nd <= 4 && (scalar == 0 || scalar == 1);
    for (int i = 0; shape_ok && i < nd; ++i) shape_ok = dims[i] >= 1 && dims[i] <= kGraphMaxBytes, n *= dims[i];
    const bool eligible = !off && on_dev && shape_ok && n * w <= kGraphMaxBytes && !profiler().enabled &&
                          !getenv("IPCG_DEBUG_TIMELINE") && std::isfinite(eb) && eb > 0.0;
    if (!eligible) return compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
    uint64_t eb_bits;
    std::memcpy(&eb_bits, &eb, 8);
    ipcg_ctx::CGraph *g = nullptr;
    for (auto &x : c->graphs) {
        bool same = x.scalar == scalar && x.nd == nd && x.interp == interp && x.lp == lp && x.cap == cap &&
                    x.eb_bits == eb_bits;
        for (int i = 0; same && i < nd; ++i) same = x.dims[i] == dims[i];
        if (same) g = &x;
    }
    if (!g) {  // first sight: a normal call, tallying its scratch requests
        const size_t t0 = c->scratch.tally;
        ipcg_archive *a = compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
        if (c->graphs.size() >= kGraphsKept) {  // evict the least recently used
            auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                        [](const auto &a1, const auto &b1) { return a1.used < b1.used; });
            if (lru->slab) CK(cudaStreamSynchronize(c->stream));
            free_graph(*lru);
            c->graphs.erase(lru);
        }
        ipcg_ctx::CGraph ng{};
        ng.scalar = scalar, ng.nd = nd, ng.interp = interp, ng.lp = lp, ng.cap = cap, ng.eb_bits = eb_bits;
        for (int i = 0; i < nd; ++i) ng.dims[i] = dims[i];
        ng.need = c->scratch.tally - t0;
        ng.used = ++c->graph_clock;
        c->graphs.push_back(ng);
        return a;
    }
    g->used = ++c->graph_clock;
    if (g->state == 2) return compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
    const uint64_t in_bytes = (n * w + 255) & ~uint64_t(255);
    if (g->state == 0) {  // second sight: capture
        g->state = 2;  // unless the capture below succeeds
        const size_t arena = g->need + (g->need >> 4) + (1u << 20);
        void *slab = nullptr;
        if (cudaMalloc(&slab, in_bytes + arena) != cudaSuccess) {
            cudaGetLastError();
            return compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
        }
        g->slab = static_cast<uint8_t *>(slab);
        if (!c->capture) CK(cudaStreamCreateWithFlags(&c->capture, cudaStreamNonBlocking));
        const cudaStream_t real = c->stream;
        const unsigned long long l0 = c->launches;
        c->stream = c->capture;
        c->scratch.arena = g->slab + in_bytes, c->scratch.arena_cap = arena, c->scratch.arena_off = 0;
        c->scratch.arena_over = false;
        CaptureOut co;
        bool ok = cudaStreamBeginCapture(c->capture, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        cudaGraph_t graph = nullptr;
        if (ok) {
            try {
                compress_impl(c, scalar, g->slab, 1, dims, nd, eb, interp, lp, cap, &co);
            } catch (...) {
                ok = false;
            }
            ok = cudaStreamEndCapture(c->capture, &graph) == cudaSuccess && ok;
        }
        ok = ok && !c->scratch.arena_over && co.aout && graph;
        c->stream = real;
        c->scratch.arena = nullptr;
        g->nlaunch = c->launches - l0;
        c->launches = l0;
        if (ok) ok = cudaGraphInstantiateWithFlags(&g->exec, graph, cudaGraphInstantiateFlagUseNodePriority) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();  // a failed capture leaves its error here; the call falls back
        if (!ok) {
            free_graph(*g);
            return compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
        }
        g->aout = co.aout, g->arch = co.arch;
        g->state = 1;
    }
    // replay
    const cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(g->slab, values, n * w, cudaMemcpyDeviceToDevice, st));
    CK(cudaGraphLaunch(g->exec, st));
    c->launches += g->nlaunch;
    const Geometry G = make_geometry(dims, nd, max_levels_for_cap(cap));
    AsmOut ho{};
    std::vector<uint8_t> index(index_bytes_for(nd, G.levels));
    const RbPart parts[2] = {{&ho, g->aout, sizeof(AsmOut)}, {index.data(), g->arch, index.size()}};
    readback_parts(parts, 2, st);
    if (!ho.fits || ho.index_bytes != index.size())  // more outliers than the slab's assembly allows
        return compress_impl(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
    ipcg_archive *a = new ipcg_archive;
    a->device = c->device;
    a->owner = st;
    a->pool = &c->scratch;
    a->on_device = true;
    try {
        parse_index(index.data(), index.size(), a->ix);
        a->owned = static_cast<uint8_t *>(c->scratch.get(std::max<uint64_t>(ho.total, 1), st));
        CK(cudaMemcpyAsync(a->owned, g->arch, ho.total, cudaMemcpyDeviceToDevice, st));
    } catch (...) {
        if (a->owned) c->scratch.put(a->owned);
        delete a;
        throw;
    }
    a->bytes = a->owned;
    a->size = ho.total;
    return a;
}

// ---------------------------------------------------------------- retrieval
struct PlaneRef {
    int level, plane;
    uint64_t block_off;  // offset of the block (header) in the staged/device source
    uint8_t backend;
    uint64_t plen;
    uint32_t crc;
};

// diff[i] = 1 when the two ranges of pair i differ (src vs dst_off-as-address)
__global__ void k_compare(const CopyDesc *pairs, int n, int *diff) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const CopyDesc c = pairs[i];
    const uint8_t *b = reinterpret_cast<const uint8_t *>(c.dst_off);
    for (uint64_t k = threadIdx.x; k < c.len; k += blockDim.x)
        if (c.src[k] != b[k]) {
            diff[i] = 1;
            break;
        }
}

// offs[2i] = block offset, offs[2i+1] = block length (a block shorter than its 21-byte header
// copies only its own bytes; the host length checks then reject it)
__global__ void k_copy_headers(const uint8_t *src, const uint64_t *offs, int n, uint8_t *dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t len = offs[2 * i + 1] < 21 ? offs[2 * i + 1] : 21;
    for (uint64_t k = 0; k < len; ++k) dst[i * 21 + k] = src[offs[2 * i] + k];
}

// read `len` bytes at absolute archive offset `off` through a seekable source
void source_read(const ipcg_archive *a, uint64_t off, void *dst, uint64_t len, const char *short_msg) {
    uint64_t done = 0;
    while (done < len) {
        const int64_t got = a->read(a->user, off + done, static_cast<uint8_t *>(dst) + done, len - done);
        if (got <= 0) throw Error(ERUNTIME, short_msg);
        done += std::min<uint64_t>((uint64_t)got, len - done);
    }
}

void *src_pinned(ipcg_ctx *c, size_t bytes) {
    if (bytes > c->src_pinned_cap) {
        if (c->src_pinned) {
            CK(cudaStreamSynchronize(c->stream));  // earlier uploads from it have landed
            CK(cudaFreeHost(c->src_pinned));
        }
        c->src_pinned = nullptr;
        const size_t cap = std::max<size_t>(bytes, 1 << 20);
        CK(cudaMallocHost(&c->src_pinned, cap));
        c->src_pinned_cap = cap;
    }
    return c->src_pinned;
}

// Enqueue up to `budget` more bytes of a pending ipcg_stage_field upload.  The copy engine serves
// host->device copies in issue order, so the whole field enqueued at once sits in front of every
// upload -- block spans, descriptor tables -- of the retrievals that follow (measured on cfg2: the
// fresh retrieval 6.8 -> 13.5 ms; with a share enqueued right after each retrieval's block uploads,
// that call's later table uploads waited instead: 3.3 -> 9 ms).  So each retrieval enqueues a share
// once all its own work is enqueued -- the pieces cross PCIe under its merge and reconstruction
// kernels -- and the compress that takes the field enqueues whatever is left.  (A zero-copy
// kernel reading the pinned field instead of the copy engine was measured too: it slowed the
// concurrent archive write and the fresh retrieval by as much as it saved.)
void stage_pump(ipcg_ctx *c, size_t budget) {
    ipcg_ctx::Staged &sg = c->staged;
    if (!sg.host || sg.issued >= sg.bytes) return;
    const size_t piece = size_t(32) << 20;
    while (sg.issued < sg.bytes && budget > 0) {
        const size_t len = std::min<size_t>({piece, sg.bytes - sg.issued, budget});
        CK(cudaMemcpyAsync(static_cast<uint8_t *>(sg.dev) + sg.issued, static_cast<const uint8_t *>(sg.host) + sg.issued,
                           len, cudaMemcpyHostToDevice, sg.stream));
        sg.issued += len, budget -= len;
    }
    if (sg.issued == sg.bytes) CK(cudaEventRecord(sg.ready, sg.stream));
}

void retrieve_impl(ipcg_ctx *c, ipcg_archive *a, int scalar, const int *k, void *out, int out_on_dev,
                   uint64_t out_count, const ipcg_session *prev_sess, const void *previous, int prev_on_dev,
                   uint64_t prev_count, ipcg_session **sess_out, ipcg_retrieve_stats *stats) {
    PhaseTimer tm;
    if (!a) throw Error(EINVAL_, "archive is null");
    if (!k) throw Error(EINVAL_, "plan is null");
    const ipcg_index &ix = a->ix;
    if (ix.scalar != scalar) throw Error(EINVAL_, "scalar kind does not match archive");
    validate_plan(ix, k);
    const bool refine = prev_sess != nullptr;
    if (refine) {
        if (prev_sess->archive_crc != ix.identity) throw Error(ERUNTIME, "session does not belong to this archive");
        if (prev_sess->levels != ix.levels) throw Error(ERUNTIME, "session level count does not match archive");
    }
    const Geometry G = make_geometry(ix.dims, ix.ndims, max_levels_for_cap(ix.anchor_cap));
    if (!refine && G.levels != ix.levels) throw Error(ERUNTIME, "archive level count does not match its dimensions");
    const int L = ix.levels;
    const int w = scalar == 0 ? 4 : 8;
    const uint64_t n = G.n;
    if (refine && (prev_count != n || !previous)) throw Error(EINVAL_, "previous reconstruction has wrong size");
    if (out_count != n || !out) throw Error(EINVAL_, "output buffer has wrong size");
    if (refine) {
        for (int level = 1; level <= L; ++level)
            if (k[level - 1] < prev_sess->k[level - 1])
                throw Error(EINVAL_, "refinement plan must not drop planes the session already loaded");
    }
    cudaStream_t st = c->stream;
    c->events_used = 0;  // this call's events (the previous call has drained)
    // ---- plan the block reads (read_range accounting, archive.cpp:172-200)
    struct LevelPlan {
        int p0, p1;
        bool active;
        uint64_t ob_off;  // outlier block source offset (staged or archive payload)
    };
    std::vector<LevelPlan> lv(L);
    std::vector<PlaneRef> refs;
    uint64_t read = 0;
    // overflow-safe forms of read_range's checks (archive.cpp:173,178); a source's size is only
    // known when a read comes up short
    auto range_ok = [&](uint64_t off, uint64_t len) {
        if (len > ix.payload_bytes || off > ix.payload_bytes - len) throw Error(ERUNTIME, "block offset outside payload");
        if (a->read) return;
        if (a->size < ix.index_bytes || len > a->size - ix.index_bytes || off > a->size - ix.index_bytes - len)
            throw Error(ERUNTIME, "truncated archive payload");
    };
    std::vector<std::pair<uint64_t, uint64_t>> spans;  // payload-relative (off, len) in read order
    for (int level = L; level >= 1; --level) {
        const int li = level - 1;
        const ipcg_level_record &r = ix.records[li];
        LevelPlan &p = lv[li];
        p.active = !refine || level <= ix.progressive_levels;
        p.p0 = refine ? prev_sess->k[li] : 0;
        p.p1 = k[li];
        if (!p.active) continue;
        if (refine) {
            if (prev_sess->count[li] != r.count || (p.p0 > 0 && !prev_sess->merged[li]))
                throw Error(ERUNTIME, "session codeword array has wrong length");
        } else if (r.count != G.level[li].count) {
            throw Error(ERUNTIME, "level point count does not match its dimensions");
        }
        for (int q = p.p0; q < p.p1; ++q) {
            range_ok(r.plane_offset[q], r.plane_length[q]);
            spans.push_back({r.plane_offset[q], r.plane_length[q]});
            refs.push_back(PlaneRef{level, q, 0, 0, 0, 0});
            read += r.plane_length[q];
        }
        const uint64_t e = 8 + (uint64_t)w;
        if (r.outlier_length % e != 0 || r.outlier_length / e != r.outlier_count)
            throw Error(ERUNTIME, "outlier block length does not match its count");
        range_ok(r.outlier_offset, r.outlier_length);
        spans.push_back({r.outlier_offset, r.outlier_length});
        read += r.outlier_length;
    }
    // ---- bring the blocks to the device
    cudaEvent_t stage_def = nullptr, stage_all = nullptr;  // two-phase host staging (below)
    uint64_t staged = 0;
    for (auto &s : spans) staged += s.second;
    DBuf stage;
    const uint8_t *src_dev;  // device base the block offsets below refer to
    std::vector<uint64_t> src_off(spans.size());
    std::vector<uint8_t> headers(refs.size() * 21);
    if (a->on_device) {
        src_dev = a->bytes + ix.index_bytes;
        for (size_t i = 0; i < spans.size(); ++i) src_off[i] = spans[i].first;
        if (!refs.empty()) {
            if (a->hdr_all.empty()) {  // every plane block's header, once per archive
                std::vector<uint64_t> hoffs;  // (offset, length) per plane block, [level-1][plane]
                for (int li = 0; li < L; ++li)
                    for (int q = 0; q < 32; ++q) {
                        const uint64_t off = ix.records[li].plane_offset[q], len = ix.records[li].plane_length[q];
                        const bool ok = len <= ix.payload_bytes && off <= ix.payload_bytes - len;
                        hoffs.push_back(ok ? off : 0), hoffs.push_back(ok ? len : 0);
                    }
                const size_t nh = hoffs.size() / 2;
                DBuf ho(hoffs.size() * 8, st), hd(nh * 21, st);
                CK(cudaMemcpyAsync(ho.p, hoffs.data(), hoffs.size() * 8, cudaMemcpyHostToDevice, st));
                CK(cudaMemsetAsync(hd.p, 0, nh * 21, st));
                k_copy_headers<<<(unsigned)((nh + 127) / 128), 128, 0, st>>>(src_dev, ho.as<uint64_t>(), (int)nh,
                                                                            hd.as<uint8_t>());
                CKL();
                std::vector<uint8_t> all(nh * 21);
                readback(all.data(), hd.p, all.size(), st);
                a->hdr_all.swap(all);
            }
            size_t ri = 0;
            for (int level = L; level >= 1; --level) {
                const LevelPlan &p = lv[level - 1];
                if (!p.active) continue;
                for (int q = p.p0; q < p.p1; ++q, ++ri)
                    std::memcpy(&headers[ri * 21], &a->hdr_all[((size_t)(level - 1) * 32 + q) * 21], 21);
            }
        }
    } else {
        // straight from the caller's buffer (no host-side staging copy): spans that are
        // adjacent in the archive (a level's planes and its outlier block) go as one copy,
        // which is a DMA from page-locked memory and a driver-pipelined copy otherwise.  The
        // call returns only after the stream drains, so the buffer is not read after return.
        // A seekable source is read span by span (the reference's read_range order) into
        // page-locked staging, each span's upload overlapping the next span's read.
        stage = DBuf(std::max<uint64_t>(staged, 1), st);
        uint8_t *sp = a->read ? static_cast<uint8_t *>(src_pinned(c, std::max<uint64_t>(staged, 1))) : nullptr;
        const uint8_t *hb = a->read ? sp : a->bytes + ix.index_bytes;
        // From a caller's buffer the spans upload on the context's h2d stream in two rounds: the
        // deflate-coded plane blocks first (the inflate starts on them), then the identity planes
        // and outlier blocks, whose upload runs under the inflate.
        const bool two_phase = !a->read && !profiler().enabled;
        std::vector<uint8_t> is_plane(spans.size(), 0);
        {
            size_t si = 0;
            for (int level = L; level >= 1; --level) {
                if (!lv[level - 1].active) continue;
                for (int q = lv[level - 1].p0; q < lv[level - 1].p1; ++q) is_plane[si++] = 1;
                ++si;  // outlier block
            }
        }
        auto deflate_span = [&](size_t i) { return is_plane[i] && spans[i].second >= 1 && hb[spans[i].first] == 1; };
        cudaStream_t hs = st;
        if (two_phase) {
            if (!c->h2d) CK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
            hs = c->h2d;
            stream_dep(c, st, hs);  // the stage buffer's stream-ordered allocation
        }
        uint64_t o = 0;
        for (size_t i = 0; i < spans.size(); ++i) src_off[i] = o, o += spans[i].second;
        for (int phase = two_phase ? 0 : 1; phase < 2; ++phase) {
            // phase 0: deflate plane blocks; phase 1: the rest (everything when not two-phase)
            for (size_t i = 0; i < spans.size();) {
                const bool mine = !two_phase || (phase == 0) == deflate_span(i);
                if (!mine) {
                    ++i;
                    continue;
                }
                size_t e = i + 1;
                while (e < spans.size() && spans[e].first == spans[e - 1].first + spans[e - 1].second &&
                       (!two_phase || (phase == 0) == deflate_span(e)))
                    ++e;
                const uint64_t len = spans[e - 1].first + spans[e - 1].second - spans[i].first;
                const uint8_t *from = hb + spans[i].first;
                if (a->read) {
                    source_read(a, ix.index_bytes + spans[i].first, sp + src_off[i], len, "truncated archive payload");
                    from = sp + src_off[i];
                }
                if (len) CK(cudaMemcpyAsync(stage.as<uint8_t>() + src_off[i], from, len, cudaMemcpyHostToDevice, hs));
                i = e;
            }
            if (two_phase) {
                cudaEvent_t ev = pool_event(c);
                CK(cudaEventRecord(ev, hs));
                (phase == 0 ? stage_def : stage_all) = ev;
            }
        }
        size_t si = 0, ri = 0;
        for (int level = L; level >= 1; --level) {
            const LevelPlan &p = lv[level - 1];
            if (!p.active) continue;
            for (int q = p.p0; q < p.p1; ++q, ++ri, ++si)  // (a short block fails the length checks below)
                std::memcpy(&headers[ri * 21], a->read ? sp + src_off[si] : hb + spans[si].first,
                            std::min<uint64_t>(21, spans[si].second));
            ++si;
        }
        src_dev = stage.as<uint8_t>();
    }
    a->payload_read += read;
    tm.mark("stage");
    // ---- block headers (read_block + load_plane checks, backend.cpp:75-86, archive.cpp:183-191)
    {
        size_t si = 0, ri = 0;
        for (int level = L; level >= 1; --level) {
            LevelPlan &p = lv[level - 1];
            if (!p.active) continue;
            const ipcg_level_record &r = ix.records[level - 1];
            for (int q = p.p0; q < p.p1; ++q, ++ri, ++si) {
                const uint64_t blen = r.plane_length[q];
                const uint8_t *h = &headers[ri * 21];
                if (blen < 1) throw Error(ERUNTIME, "truncated input while parsing");
                if (h[0] > 1) throw Error(ERUNTIME, "unknown backend id");
                if (blen < 21) throw Error(ERUNTIME, "truncated input while parsing");
                uint64_t raw_bits = 0, plen = 0;
                uint32_t crc = 0;
                for (int i = 0; i < 8; ++i) raw_bits |= (uint64_t)h[1 + i] << (8 * i);
                for (int i = 0; i < 8; ++i) plen |= (uint64_t)h[9 + i] << (8 * i);
                for (int i = 0; i < 4; ++i) crc |= (uint32_t)h[17 + i] << (8 * i);
                if (blen - 21 < plen) throw Error(ERUNTIME, "truncated input while parsing");
                if (blen - 21 != plen) throw Error(ERUNTIME, "plane block has trailing bytes");
                if (raw_bits != r.count) throw Error(ERUNTIME, "plane bit count does not match level");
                refs[ri].block_off = src_off[si];
                refs[ri].backend = h[0];
                refs[ri].plen = plen;
                refs[ri].crc = crc;
            }
            p.ob_off = src_off[si++];
        }
    }
    // ---- CRC-32 of every payload, then identity copies / inflate into plane rows
    const size_t R = refs.size();
    uint64_t maxp = 1;
    for (const PlaneRef &r : refs) maxp = std::max(maxp, r.plen);
    std::vector<DBuf> planes(L);
    std::vector<uint64_t> stride(L, 0);
    for (int level = 1; level <= L; ++level) {
        const LevelPlan &p = lv[level - 1];
        if (!p.active) continue;
        const uint64_t count = ix.records[level - 1].count;
        stride[level - 1] = round_up(std::max<uint64_t>((count + 31) / 32, 1), 4);
        planes[level - 1] = DBuf(32 * stride[level - 1] * 4, st);
    }
    // plane rows the merge reads (duplicates may alias one decoded row)
    std::vector<std::vector<const uint32_t *>> rows(L, std::vector<const uint32_t *>(32, nullptr));
    for (int l = 0; l < L; ++l)
        if (planes[l].p)
            for (int q = 0; q < 32; ++q) rows[l][q] = planes[l].as<uint32_t>() + (uint64_t)q * stride[l];
    // checks made once the merge and reconstruction are enqueued (finish_checks): the payload
    // CRCs and the inflate's Adler-32/status run on side streams under them
    DBuf crcws, crcs, pd, ld;
    cudaStream_t cs = st;
    DevAlloc inflate_tmp;
    DBuf inflate_status;
    size_t inflate_jobs = 0;
    cudaStream_t inflate_check = nullptr;
    cudaEvent_t inflate_done = nullptr;
    struct JoinCheck {  // an exception before finish_checks still orders inflate_tmp's release
        cudaStream_t &check, &st;
        cudaEvent_t &done;
        ~JoinCheck() {
            if (check) cudaStreamWaitEvent(st, done, 0);
        }
    } join_check{inflate_check, st, inflate_done};
    std::function<void()> finish_checks = [] {};
    if (R) {
        std::vector<const uint8_t *> ptrs(R);
        std::vector<uint64_t> lens(R);
        std::vector<InflateJob> jobs;
        std::vector<int> job_level, job_plane;
        std::vector<uint32_t> job_crc;
        std::vector<CopyDesc> copies;
        for (size_t i = 0; i < R; ++i) {
            const PlaneRef &r = refs[i];
            ptrs[i] = src_dev + r.block_off + 21;
            lens[i] = r.plen;
            const int li = r.level - 1;
            const uint64_t pbytes = (ix.records[li].count + 7) / 8;
            uint8_t *row = planes[li].as<uint8_t>() + (uint64_t)r.plane * stride[li] * 4;
            if (r.backend == 0) {  // identity: the length check follows the CRC check, as in backend_decode
                copies.push_back(CopyDesc{ptrs[i], (uint64_t)reinterpret_cast<uintptr_t>(row), std::min(r.plen, pbytes)});
            } else {
                jobs.push_back(InflateJob{ptrs[i], r.plen, row, pbytes});
                job_level.push_back(li);
                job_plane.push_back(r.plane);
                job_crc.push_back(r.crc);
            }
        }
        const size_t cw = crc32_batch_workspace((int)R, maxp);
        crcws = DBuf(cw, st), crcs = DBuf(R * 4, st), pd = DBuf(R * 8, st), ld = DBuf(R * 8, st);
        // (pageable sources: staged by the driver on return, no stream sync)
        CK(cudaMemcpyAsync(pd.p, ptrs.data(), R * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ld.p, lens.data(), R * 8, cudaMemcpyHostToDevice, st));
        // CRC-32 of every payload on a side stream, concurrent with the copies and the inflate
        // (which validate everything they read and never fault on corrupt input); the checks
        // run after the inflate in backend_decode's order -- every checksum, then identity
        // lengths, then the inflate status -- so the reported error is unchanged
        cs = profiler().enabled ? st : side_stream(c, 0);
        if (cs != st) stream_dep(c, st, cs);
        if (stage_all) CK(cudaStreamWaitEvent(cs, stage_all, 0));
        {
            uint64_t cb = 0;
            for (uint64_t x : lens) cb += x;
            ProfScope ps("crc_check", cs, cb);
            crc32_batch(pd.as<const uint8_t *>(), ld.as<uint64_t>(), (int)R, maxp, crcs.as<uint32_t>(), crcws.p, cw, cs);
        }
        struct JoinOnExit {  // an exception before check_crcs still orders the CRC's buffers' release
            ipcg_ctx *c;
            cudaStream_t from, to;
            ~JoinOnExit() {
                if (from != to) {
                    cudaEvent_t e = pool_event(c);
                    cudaEventRecord(e, from);
                    cudaStreamWaitEvent(to, e, 0);
                }
            }
        } join_crc{c, cs, st};
        auto check_crcs = [&] {
            if (cs != st) stream_dep(c, cs, st);
            std::vector<uint32_t> hcrc(R);
            readback(hcrc.data(), crcs.p, R * 4, st);
            for (size_t i = 0; i < R; ++i)
                if (hcrc[i] != refs[i].crc) throw Error(ERUNTIME, "block checksum mismatch");
            for (size_t i = 0; i < R; ++i) {
                const uint64_t pbytes = (ix.records[refs[i].level - 1].count + 7) / 8;
                if (refs[i].backend == 0 && refs[i].plen != pbytes) throw Error(ERUNTIME, "identity block has wrong length");
            }
        };
    tm.mark("crc");
    tm.mark("copies");
        if (stage_def) CK(cudaStreamWaitEvent(st, stage_def, 0));
        // identical deflate payloads (typically the all-zero high planes) decode once:
        // same (length, crc, plane size) and byte-equal on the device -> alias the row
        std::vector<int> rep_of(jobs.size(), -1);
        {
            std::vector<std::pair<int, int>> pairs;  // (dup job, rep job)
            for (size_t a = 0; a < jobs.size(); ++a) {
                for (size_t b = 0; b < a; ++b) {
                    if (rep_of[b] >= 0) continue;
                    if (jobs[a].src_len == jobs[b].src_len && jobs[a].dst_len == jobs[b].dst_len &&
                        job_crc[a] == job_crc[b]) {
                        pairs.push_back({(int)a, (int)b});
                        break;
                    }
                }
            }
            if (!pairs.empty()) {
                std::vector<CopyDesc> cmp;
                for (auto &pr : pairs)
                    cmp.push_back(CopyDesc{jobs[pr.first].src, (uint64_t)reinterpret_cast<uintptr_t>(jobs[pr.second].src),
                                           jobs[pr.first].src_len});
                DBuf cd(cmp.size() * sizeof(CopyDesc), st), diff(cmp.size() * 4, st);
                CK(cudaMemcpyAsync(cd.p, cmp.data(), cmp.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice, st));
                CK(cudaMemsetAsync(diff.p, 0, cmp.size() * 4, st));
                k_compare<<<(unsigned)cmp.size(), 256, 0, st>>>(cd.as<CopyDesc>(), (int)cmp.size(), diff.as<int>());
                CKL();
                std::vector<int> hd(cmp.size());
                readback(hd.data(), diff.p, cmp.size() * 4, st);
                for (size_t q = 0; q < pairs.size(); ++q)
                    if (!hd[q]) rep_of[pairs[q].first] = pairs[q].second;
            }
        }
        std::vector<InflateJob> todo;
    tm.mark("dedupe");
        for (size_t a = 0; a < jobs.size(); ++a)
            if (rep_of[a] < 0) todo.push_back(jobs[a]);
            else rows[job_level[a]][job_plane[a]] = rows[job_level[rep_of[a]]][job_plane[rep_of[a]]];
        if (!todo.empty()) {
            inflate_status = DBuf(todo.size() * 4, st);
            inflate_jobs = todo.size();
            uint64_t ib = 0;
            for (const InflateJob &j : todo) ib += j.src_len + j.dst_len;
            ProfScope ps("inflate", st, ib);
            // the inflate's Adler-32 and status run on a side stream under the merge and
            // reconstruction below; every check is made before returning (finish_checks)
            if (!profiler().enabled) {
                inflate_check = quant_stream(c);  // (compress's stream: idle here; side stream 0 carries the CRC)
                inflate_done = pool_event(c);
                inflate_batch_host(todo, inflate_status.as<int>(), inflate_tmp, st, inflate_check, pool_event(c),
                                   inflate_done);
            } else {
                inflate_batch_host(todo, inflate_status.as<int>(), inflate_tmp, st);
            }
        }
        // identity planes: their upload (second staging round) ran under the inflate
        if (stage_all) CK(cudaStreamWaitEvent(st, stage_all, 0));
        if (!copies.empty()) gather(c, copies, nullptr);
        finish_checks = [&, check_crcs] {
            if (inflate_check) CK(cudaStreamWaitEvent(st, inflate_done, 0));
            check_crcs();
            if (inflate_jobs) {
                std::vector<int> status(inflate_jobs);
                readback(status.data(), inflate_status.p, inflate_jobs * 4, st);
                for (int s : status)
                    if (s) throw Error(ERUNTIME, "deflate backend failed to decompress block");
            }
        };
    tm.mark("inflate");
    }
    if (stage_all) CK(cudaStreamWaitEvent(st, stage_all, 0));  // outlier blocks (and no planes at all)
    DBuf rows_d((size_t)L * 32 * sizeof(void *), st);
    {
        std::vector<const uint32_t *> flat((size_t)L * 32, nullptr);
        for (int l = 0; l < L; ++l)
            for (int q = 0; q < 32; ++q) flat[(size_t)l * 32 + q] = rows[l][q];
        CK(cudaMemcpyAsync(rows_d.p, flat.data(), flat.size() * sizeof(void *), cudaMemcpyHostToDevice, st));
    }
    tm.mark("rows");
    // ---- merge + reconstruct, coarsest first
    DBuf out_buf;
    void *state = out;
    ipcg_ctx::OutSlot *slot = nullptr;
    if (!out_on_dev) {
        if (c->host_async) {
            slot = &out_slot(c, n * w);
            CK(cudaStreamWaitEvent(st, slot->done, 0));  // its previous copy-out has finished
            state = slot->p;
        } else {
            out_buf = DBuf(n * w, st);
            state = out_buf.p;
        }
    }
    // refine_field starts from `previous` and replays the progressive levels (pipeline.hpp:
    // 310-349); the replay rewrites every point of those levels, so `previous` only
    // contributes the points of non-progressive levels: copy it only if there are any.
    bool keeps_previous = false;
    for (int l = 0; l < L; ++l) keeps_previous |= !lv[l].active;
    if (refine && keeps_previous) {
        // `previous` may be the host destination of a copy-out still in flight
        if (!prev_on_dev && c->copy_pending) CK(cudaStreamWaitEvent(st, c->copy_tail, 0));
        CK(cudaMemcpyAsync(state, previous, n * w, prev_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    }
    ipcg_session *ns = new ipcg_session;
    ns->archive_crc = ix.identity;
    ns->levels = L;
    ns->lp = ix.progressive_levels;
    ns->owner = st;
    ns->pool = &c->scratch;
    ns->device = c->device;
    DBuf napplied(8 * IPCG_MAX_LEVELS, st);
    try {
        for (int level = L; level >= 1; --level) {
            const int li = level - 1;
            const LevelPlan &p = lv[li];
            ns->k[li] = k[li];
            ns->count[li] = ix.records[li].count;
            if (!p.active) {
                if (refine) ns->k[li] = prev_sess->k[li];
                continue;
            }
            const uint64_t count = ix.records[li].count;
            uint32_t *merged = nullptr;
            merged = static_cast<uint32_t *>(scratch_get(std::max<uint64_t>(count, 1) * 4 + 16, st));
            const uint32_t *min = refine ? prev_sess->merged[li] : nullptr;
            {
                ProfScope ps("merge", st, count * 4 + (uint64_t)(p.p1 - p.p0) * ((count + 7) / 8));
                launch_merge(rows_d.as<const uint32_t *>() + (size_t)li * 32, min, merged, count, p.p0, p.p1, st);
            }
            const uint8_t *ob = src_dev + p.ob_off;
            const uint64_t no = ix.records[li].outlier_count;
            if (no) launch_outlier_prefix(ob, no, scalar, count, napplied.as<uint64_t>() + li, st);
            {
                ProfScope psr("recon_pass", st, count * (uint64_t)(4 + 2 * w));
                for (const PassDesc &pd : G.level[li].passes) {
                    launch_recon_pass(state, scalar, ix.interp == 1, pd, ix.eb, merged, G.dims[G.nd - 1], st);
                    if (no) launch_outlier_apply(state, scalar, pd, ob, napplied.as<uint64_t>() + li, no, st);
                }
            }
            if (level <= ix.progressive_levels) ns->merged[li] = merged;
            else scratch_put(merged, st);
        }
        {
            // a field staged for the next compress (ipcg_stage_field): a share of its upload now,
            // behind everything this call uploads and under the kernels it still has to run
            static const size_t pump_mib = getenv("IPCG_STAGE_PUMP") ? strtoull(getenv("IPCG_STAGE_PUMP"), nullptr, 10) : 64;  // dev knob (MiB per retrieval; measured on cfg2's e2e step, 56.3 ms without staging: 64 -> 54.7, 96 -> 54.4-55.8, 128 -> 55.0, 192 -> 55.2 -- larger shares delay the third retrieval's uploads by more than they save the compress)
            stage_pump(c, pump_mib << 20);
        }
        finish_checks();  // every checksum, then identity lengths, then the inflate status
        if (slot) {
            CK(cudaEventRecord(slot->ready, st));
            CK(cudaStreamWaitEvent(c->copy, slot->ready, 0));
            CK(cudaMemcpyAsync(out, state, n * w, cudaMemcpyDeviceToHost, c->copy));
            CK(cudaEventRecord(slot->done, c->copy));
            CK(cudaEventRecord(c->copy_tail, c->copy));
            c->copy_pending = true;
        } else if (!out_on_dev) {
            CK(cudaMemcpyAsync(out, state, n * w, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
    tm.mark("recon");
    } catch (...) {
        for (int l = 0; l < IPCG_MAX_LEVELS; ++l)
            if (ns->merged[l]) scratch_put(ns->merged[l], st);
        delete ns;
        throw;
    }
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->payload_bytes_loaded = read;
        for (int l = 0; l < L; ++l) stats->level_visits[l] = lv[l].active ? 1 : 0;  // pipeline.hpp:275,346
    }
    if (sess_out) *sess_out = ns;
    else {
        for (int l = 0; l < IPCG_MAX_LEVELS; ++l)
            if (ns->merged[l]) scratch_put(ns->merged[l], st);
        delete ns;
    }
}

}  // namespace

// ================================================================== C-ABI
extern "C" {

int ipcg_ctx_create(int device, ipcg_ctx **out) {
    ipcg_ctx *c = new ipcg_ctx;
    c->device = device;
    const int rc = guarded(c, [&] {
        int cnt = 0;
        CK(cudaGetDeviceCount(&cnt));
        if (device < 0 || device >= cnt) throw Error(ECUDA, "no such CUDA device");
        CK(cudaSetDevice(device));
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
    });
    if (rc != IPCG_OK) {
        *out = nullptr;
        delete c;
        return rc;
    }
    *out = c;
    return IPCG_OK;
}

void ipcg_ctx_destroy(ipcg_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->copy) cudaStreamSynchronize(c->copy);
    for (auto &sl : c->ring) {
        if (sl.p) cudaFree(sl.p);
        cudaEventDestroy(sl.ready);
        cudaEventDestroy(sl.done);
    }
    if (c->copy_tail) cudaEventDestroy(c->copy_tail);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaStream_t s : c->side) cudaStreamSynchronize(s);
    for (cudaStream_t s : c->loss) cudaStreamSynchronize(s);
    for (cudaStream_t s : c->odside) cudaStreamSynchronize(s);
    if (c->quant) cudaStreamSynchronize(c->quant);
    if (c->h2d) cudaStreamSynchronize(c->h2d);
    if (c->staged.stream) {
        cudaStreamSynchronize(c->staged.stream);
        cudaStreamDestroy(c->staged.stream);
        cudaEventDestroy(c->staged.ready);
        if (c->staged.dev) cudaFree(c->staged.dev);
    }
    if (c->capture) cudaStreamSynchronize(c->capture);
    for (auto &g : c->graphs) free_graph(g);
    if (c->capture) cudaStreamDestroy(c->capture);
    c->scratch.release_all(c->own_stream);
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->src_pinned) cudaFreeHost(c->src_pinned);
    for (cudaStream_t s : c->side) cudaStreamDestroy(s);
    for (cudaStream_t s : c->loss) cudaStreamDestroy(s);
    for (cudaStream_t s : c->odside) cudaStreamDestroy(s);
    if (c->quant) cudaStreamDestroy(c->quant);
    if (c->h2d) cudaStreamDestroy(c->h2d);
    for (cudaEvent_t e : c->events) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

const char *ipcg_last_error(const ipcg_ctx *c) { return c ? c->err.c_str() : g_host_err.c_str(); }

int ipcg_set_stream(ipcg_ctx *c, void *s) {
    return guarded(c, [&] {
        drain_copies(c);
        CK(cudaStreamSynchronize(c->stream));
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    });
}

int ipcg_synchronize(ipcg_ctx *c) {
    return guarded(c, [&] {
        drain_copies(c);
        CK(cudaStreamSynchronize(c->stream));
        if (c->staged.stream) CK(cudaStreamSynchronize(c->staged.stream));  // enqueued pieces of a staged field
    });
}

int ipcg_set_host_async(ipcg_ctx *c, int enable) {
    return guarded(c, [&] {
        drain_copies(c);
        if (enable && !c->copy) {
            CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->copy_tail, cudaEventDisableTiming));
        }
        c->host_async = enable != 0;
    });
}

int ipcg_stage_field(ipcg_ctx *c, const void *host_values, uint64_t bytes) {
    return guarded(c, [&] {
        ipcg_ctx::Staged &sg = c->staged;
        if (!host_values || !bytes) throw Error(EINVAL_, "stage_field: null field");
        if (!sg.stream) {
            CK(cudaStreamCreateWithFlags(&sg.stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&sg.ready, cudaEventDisableTiming));
        }
        // the last compress that read the staging buffer has returned (compress synchronizes), and
        // a pending upload that was never consumed is simply overwritten behind it in stream order
        if (bytes > sg.cap) {
            CK(cudaStreamSynchronize(sg.stream));
            if (sg.dev) CK(cudaFree(sg.dev));
            sg.dev = nullptr, sg.cap = 0;
            CK(cudaMalloc(&sg.dev, bytes));
            sg.cap = bytes;
        }
        sg.host = host_values, sg.bytes = bytes, sg.issued = 0;
        // (the copies are enqueued by stage_pump: in shares by the retrievals that follow, the rest
        // by the compress that takes the field)
    });
}

int ipcg_compress(ipcg_ctx *c, int scalar, const void *values, int on_dev, const uint64_t *dims, int nd, double eb,
                  int interp, int lp, uint64_t cap, ipcg_archive **out) {
    return guarded(c, [&] {
        // a host field staged ahead (ipcg_stage_field) is compressed from its device copy
        ipcg_ctx::Staged &sg = c->staged;
        if (!on_dev && values && sg.host == values) {
            uint64_t n = 1;
            bool ok = nd >= 1 && nd <= 4 && dims;
            for (int i = 0; ok && i < nd; ++i) ok = dims[i] >= 1 && n <= sg.bytes / dims[i], n *= ok ? dims[i] : 1;
            if (ok && n * (scalar == 0 ? 4u : 8u) == sg.bytes) {
                stage_pump(c, sg.bytes);
                CK(cudaStreamWaitEvent(c->stream, sg.ready, 0));
                values = sg.dev, on_dev = 1;
            }
            sg.host = nullptr;
        }
        *out = compress_entry(c, scalar, values, on_dev, dims, nd, eb, interp, lp, cap);
    });
}

int ipcg_archive_open(ipcg_ctx *c, const void *bytes, uint64_t size, int on_device, ipcg_archive **out) {
    if (!c && on_device) return IPCG_EINVAL;
    return guarded(c, [&] {
        std::vector<uint8_t> head(std::min<uint64_t>(size, kMaxIndexBytes));
        if (on_device) {
            if (!head.empty()) CK(cudaMemcpy(head.data(), bytes, head.size(), cudaMemcpyDeviceToHost));
        } else if (!head.empty()) {
            std::memcpy(head.data(), bytes, head.size());
        }
        ipcg_archive *a = new ipcg_archive;
        try {
            parse_index(head.data(), head.size(), a->ix);
        } catch (...) {
            delete a;
            throw;
        }
        a->bytes = static_cast<const uint8_t *>(bytes);
        a->size = size;
        a->on_device = on_device != 0;
        a->device = c ? c->device : 0;
        *out = a;
    });
}

int ipcg_archive_open_source(ipcg_ctx *c, ipcg_read_fn read, void *user, ipcg_archive **out) {
    if (out) *out = nullptr;
    return guarded(c, [&] {
        if (!read || !out) throw Error(EINVAL_, "archive source needs a read function");
        ipcg_archive *a = new ipcg_archive;
        try {
            parse_index(IndexSource{read, user}, a->ix);
        } catch (...) {
            delete a;
            throw;
        }
        a->read = read;
        a->user = user;
        a->size = a->ix.index_bytes + a->ix.payload_bytes;  // as the index describes it
        a->device = c ? c->device : 0;
        *out = a;
    });
}

int ipcg_archive_read_range(ipcg_ctx *c, ipcg_archive *a, uint64_t off, uint64_t len, void *dst) {
    return guarded(c, [&] {
        const ipcg_index &ix = a->ix;
        if (len > ix.payload_bytes || off > ix.payload_bytes - len) throw Error(ERUNTIME, "block offset outside payload");
        if (len && !dst) throw Error(EINVAL_, "read_range: null destination");
        if (a->read) {
            source_read(a, ix.index_bytes + off, dst, len, "truncated archive payload");
        } else {
            if (a->size < ix.index_bytes || len > a->size - ix.index_bytes || off > a->size - ix.index_bytes - len)
                throw Error(ERUNTIME, "truncated archive payload");
            if (!len) {
            } else if (a->on_device) {
                CK(cudaMemcpyAsync(dst, a->bytes + ix.index_bytes + off, len, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            } else {
                std::memcpy(dst, a->bytes + ix.index_bytes + off, len);
            }
        }
        a->payload_read += len;
    });
}

int ipcg_archive_copy(ipcg_ctx *c, const ipcg_archive *a, uint64_t off, uint64_t len, void *dst, int dst_on_device) {
    return guarded(c, [&] {
        if (!len) return;
        if (!dst) throw Error(EINVAL_, "archive copy: null destination");
        if (a->read) {
            if (dst_on_device) {
                void *h = pinned(c, len);
                source_read(a, off, h, len, "truncated archive");
                CK(cudaMemcpyAsync(dst, h, len, cudaMemcpyHostToDevice, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            } else {
                source_read(a, off, dst, len, "truncated archive");
            }
            return;
        }
        if (len > a->size || off > a->size - len) throw Error(EINVAL_, "archive copy outside the archive");
        if (!a->on_device && !dst_on_device) {
            std::memcpy(dst, a->bytes + off, len);
            return;
        }
        const cudaMemcpyKind kind = a->on_device ? (dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost)
                                                 : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(dst, a->bytes + off, len, kind, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ipcg_archive_index(const ipcg_archive *a, ipcg_index *out) {
    if (!a || !out) return IPCG_EINVAL;
    *out = a->ix;
    return IPCG_OK;
}

int ipcg_index_serialize(const ipcg_index *ix, uint8_t *dst, uint64_t capacity, uint64_t *size_out) {
    return guarded(nullptr, [&] {
        if (!ix) throw Error(EINVAL_, "index is null");
        if (ix->levels > IPCG_MAX_LEVELS) throw Error(EINVAL_, "archive has more levels than supported");
        const std::vector<uint8_t> b = serialize_index(*ix);
        if (size_out) *size_out = b.size();
        if (!dst || capacity < b.size()) throw Error(EINVAL_, "index buffer too small");
        std::memcpy(dst, b.data(), b.size());
    });
}

int ipcg_index_parse(const uint8_t *bytes, uint64_t size, ipcg_index *out) {
    return guarded(nullptr, [&] {
        if (!out || (size && !bytes)) throw Error(EINVAL_, "index_parse: null argument");
        parse_index(bytes, size, *out);
    });
}

uint32_t ipcg_crc32(const void *bytes, uint64_t len) {
    return len ? crc32_host(static_cast<const uint8_t *>(bytes), len) : 0u;
}

uint64_t ipcg_archive_size(const ipcg_archive *a) { return a ? a->size : 0; }

int ipcg_archive_write(ipcg_ctx *c, const ipcg_archive *a, void *dst, int dst_on_device, uint64_t capacity) {
    return guarded(c, [&] {
        if (a->read) throw Error(EINVAL_, "archive opened from a source: copy it with ipcg_archive_copy");
        if (capacity < a->size) throw Error(EINVAL_, "destination too small for the archive");
        const cudaMemcpyKind kind = a->on_device ? (dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost)
                                                 : (dst_on_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost);
        CK(cudaMemcpyAsync(dst, a->bytes, a->size, kind, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

uint64_t ipcg_archive_payload_bytes_read(const ipcg_archive *a) { return a ? a->payload_read : 0; }

void ipcg_archive_free(ipcg_archive *a) {
    if (!a) return;
    if (a->owned) {
        cudaSetDevice(a->device);
        if (a->pool) a->pool->put(a->owned);  // reused stream-ordered by the context's next calls
        else cudaFreeAsync(a->owned, a->owner);
    }
    delete a;
}

int ipcg_reconstruct(ipcg_ctx *c, ipcg_archive *a, int scalar, const int *k, void *out, int out_on_device,
                     uint64_t out_count, ipcg_session **session_out, ipcg_retrieve_stats *stats) {
    if (session_out) *session_out = nullptr;
    return guarded(c, [&] {
        retrieve_impl(c, a, scalar, k, out, out_on_device, out_count, nullptr, nullptr, 0, 0, session_out, stats);
    });
}

int ipcg_refine(ipcg_ctx *c, ipcg_archive *a, int scalar, const ipcg_session *s, const void *previous, int prev_on_dev,
                uint64_t previous_count, const int *k, void *out, int out_on_device, uint64_t out_count,
                ipcg_session **session_out, ipcg_retrieve_stats *stats) {
    if (session_out) *session_out = nullptr;
    return guarded(c, [&] {
        if (!s) throw Error(EINVAL_, "refinement needs a session");
        retrieve_impl(c, a, scalar, k, out, out_on_device, out_count, s, previous, prev_on_dev, previous_count,
                      session_out, stats);
    });
}

// RetrievalSession from host data (session.hpp:19-34), validated the way a refinement would use
// it: plane counts in 0..32, 32 above the progressive bound, codewords for every progressive
// level that has planes loaded
int ipcg_session_create(ipcg_ctx *c, const ipcg_archive *a, const int *planes_loaded, const uint32_t *const *merged,
                        ipcg_session **out) {
    if (out) *out = nullptr;
    return guarded(c, [&] {
        if (!a || !planes_loaded || !out) throw Error(EINVAL_, "session_create: null argument");
        const int L = a->ix.levels, lp = a->ix.progressive_levels;
        for (int l = 0; l < L; ++l) {
            const int kk = planes_loaded[l];
            if (kk < 0 || kk > 32) throw Error(EINVAL_, "plane index out of range");
            if (l + 1 > lp && kk != 32) throw Error(EINVAL_, "non-progressive levels must load all planes");
            if (l + 1 <= lp && kk > 0 && !(merged && merged[l]))
                throw Error(ERUNTIME, "session codeword array has wrong length");
        }
        ipcg_session *s = new ipcg_session;
        s->archive_crc = a->ix.identity;
        s->levels = L;
        s->lp = lp;
        s->owner = c->stream;
        s->pool = &c->scratch;
        s->device = c->device;
        try {
            for (int l = 0; l < L; ++l) {
                s->k[l] = planes_loaded[l];
                s->count[l] = a->ix.records[l].count;
                if (l + 1 <= lp && merged && merged[l]) {
                    const uint64_t cnt = s->count[l];
                    s->merged[l] = static_cast<uint32_t *>(c->scratch.get(std::max<uint64_t>(cnt, 1) * 4 + 16, c->stream));
                    CK(cudaMemcpyAsync(s->merged[l], merged[l], cnt * 4, cudaMemcpyHostToDevice, c->stream));
                }
            }
            CK(cudaStreamSynchronize(c->stream));
        } catch (...) {
            ipcg_session_free(s);
            throw;
        }
        *out = s;
    });
}

int ipcg_session_levels(const ipcg_session *s) { return s ? s->levels : 0; }
uint32_t ipcg_session_archive_crc(const ipcg_session *s) { return s ? s->archive_crc : 0; }
int ipcg_session_planes_loaded(const ipcg_session *s, int *k_out) {
    if (!s) return IPCG_EINVAL;
    for (int l = 0; l < s->levels; ++l) k_out[l] = s->k[l];
    return IPCG_OK;
}
uint64_t ipcg_session_count(const ipcg_session *s, int level) {
    if (!s || level < 1 || level > s->levels || !s->merged[level - 1]) return 0;
    return s->count[level - 1];
}
int ipcg_session_merged(ipcg_ctx *c, const ipcg_session *s, int level, uint32_t *dst, int dst_on_device) {
    return guarded(c, [&] {
        if (level < 1 || level > s->levels) throw Error(EINVAL_, "level index out of range");
        const uint32_t *m = s->merged[level - 1];
        if (!m) return;
        CK(cudaMemcpyAsync(dst, m, s->count[level - 1] * 4, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}
void ipcg_session_free(ipcg_session *s) {
    if (!s) return;
    cudaSetDevice(s->device);
    for (int l = 0; l < IPCG_MAX_LEVELS; ++l)
        if (s->merged[l]) {
            if (s->pool) s->pool->put(s->merged[l]);
            else cudaFreeAsync(s->merged[l], s->owner);
        }
    delete s;
}

// ------------------------------------------------------------------ session file
// write_session / read_session (src/session.cpp:8-61): "IPS1", u32 archive identity, then per
// level (coarsest first) u8 planes_loaded + one backend block (backend.cpp:67-86) holding the
// level's merged codewords as u32 little-endian -- the device layout of the session's arrays,
// so they are deflated (DeflateBatch, zlib-1.3-exact) and inflated in place on the GPU.
uint64_t ipcg_session_write_bound(const ipcg_session *s) {
    if (!s) return 0;
    uint64_t b = 8;
    for (int l = 0; l < s->levels; ++l) b += 1 + 21 + (s->merged[l] ? s->count[l] * 4 : 0);
    return b;
}

int ipcg_session_write(ipcg_ctx *c, const ipcg_session *s, void *dst, int dst_on_device, uint64_t capacity,
                       uint64_t *size_out) {
    return guarded(c, [&] {
        if (!s) throw Error(EINVAL_, "session is null");
        cudaStream_t st = c->stream;
        const int L = s->levels;
        struct Enc {
            uint8_t be = 0;
            uint64_t raw = 0, len = 0;
            uint32_t crc = 0;
            const uint8_t *payload = nullptr;  // device
        };
        std::vector<Enc> enc(L);
        std::vector<DBuf> keep;  // deflate outputs, alive until the copy-out below
        for (int l = L; l >= 1; --l) {
            const uint32_t *m = s->merged[l - 1];
            if (!m) continue;
            Enc &e = enc[l - 1];
            const uint64_t n = s->count[l - 1] * 4;
            e.raw = n;
            if (n == 0) continue;  // empty identity block, crc32("") = 0
            const uint64_t out_stride = round_up(n + 16, 16);
            keep.emplace_back(out_stride, st);
            DBuf ws(DeflateBatch::workspace_bytes(1, n), st), be(16, st), ln(16, st), cr(16, st), pl(16, st);
            const BackendResults res{be.as<uint8_t>(), ln.as<uint64_t>(), cr.as<uint32_t>(), pl.as<const uint8_t *>()};
            // merged arrays carry >= 16 bytes of padding (session allocations), as DeflateBatch reads padded rows
            DeflateBatch::run(reinterpret_cast<const uint8_t *>(m), round_up(n, 16), 1, n, keep.back().as<uint8_t>(),
                              out_stride, ws.p, res, st);
            readback(&e.be, be.p, 1, st);
            readback(&e.len, ln.p, 8, st);
            readback(&e.crc, cr.p, 4, st);
            readback(&e.payload, pl.p, 8, st);
        }
        uint64_t size = 8;
        for (int l = 0; l < L; ++l) size += 1 + 21 + enc[l].len;
        if (size_out) *size_out = size;
        if (!dst || capacity < size) throw Error(EINVAL_, "session buffer too small");
        std::vector<uint8_t> head(8 + 22 * (size_t)L);
        auto put = [](uint8_t *p, uint64_t v, int nb) {
            for (int i = 0; i < nb; ++i) p[i] = (uint8_t)(v >> (8 * i));
        };
        std::memcpy(head.data(), "IPS1", 4);
        put(head.data() + 4, s->archive_crc, 4);
        struct Piece {
            const void *src;
            bool dev;
            uint64_t len, off;
        };
        std::vector<Piece> pieces{{head.data(), false, 8, 0}};
        uint64_t o = 8;
        for (int l = L, hi = 0; l >= 1; --l, ++hi) {
            const Enc &e = enc[l - 1];
            uint8_t *h = head.data() + 8 + 22 * (size_t)hi;
            h[0] = (uint8_t)s->k[l - 1];
            h[1] = e.be;
            put(h + 2, e.raw * 8, 8);
            put(h + 10, e.len, 8);
            put(h + 18, e.crc, 4);
            pieces.push_back({h, false, 22, o});
            o += 22;
            if (e.len) pieces.push_back({e.payload, true, e.len, o});
            o += e.len;
        }
        uint8_t *d = static_cast<uint8_t *>(dst);
        for (const Piece &pc : pieces) {
            if (!dst_on_device && !pc.dev) std::memcpy(d + pc.off, pc.src, pc.len);
            else
                CK(cudaMemcpyAsync(d + pc.off, pc.src, pc.len,
                                   pc.dev ? (dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost)
                                          : cudaMemcpyHostToDevice,
                                   st));
        }
        CK(cudaStreamSynchronize(st));
    });
}

int ipcg_session_read(ipcg_ctx *c, const ipcg_archive *a, const void *bytes, uint64_t size, int on_device,
                      ipcg_session **out) {
    if (out) *out = nullptr;
    return guarded(c, [&] {
        cudaStream_t st = c->stream;
        const ipcg_index &ix = a->ix;
        const int L = ix.levels, lp = ix.progressive_levels;
        const uint8_t *src = static_cast<const uint8_t *>(bytes);
        // small host reads of the (possibly device-resident) file: the headers only
        auto fetch = [&](uint64_t off, uint64_t len, uint8_t *h) {
            if (!on_device) std::memcpy(h, src + off, len);
            else if (len) CK(cudaMemcpy(h, src + off, len, cudaMemcpyDeviceToHost));
        };
        auto rd = [](const uint8_t *p, int nb) {
            uint64_t v = 0;
            for (int i = 0; i < nb; ++i) v |= (uint64_t)p[i] << (8 * i);
            return v;
        };
        const char *const trunc = "truncated input while parsing";  // ByteReader (common.hpp:98)
        uint8_t h[22];
        if (size < 4) throw Error(ERUNTIME, trunc);
        fetch(0, 4, h);
        if (std::memcmp(h, "IPS1", 4) != 0) throw Error(ERUNTIME, "not a session file: bad magic");
        if (size < 8) throw Error(ERUNTIME, trunc);
        fetch(4, 4, h);
        const uint32_t crc = (uint32_t)rd(h, 4);
        if (crc != ix.identity) throw Error(ERUNTIME, "session does not belong to this archive");
        // parse every level's header in file order; the first parse error is raised only after
        // the blocks of the levels before it decoded cleanly (the reference works level by level)
        struct Blk {
            int level, k;
            uint8_t be;
            uint64_t raw_bits, plen, off;
            uint32_t crc;
        };
        std::vector<Blk> blks;
        std::string parse_err;
        uint64_t pos = 8;
        for (int level = L; level >= 1; --level) {
            Blk b{level, 0, 0, 0, 0, 0, 0};
            if (size - pos < 1) { parse_err = trunc; break; }
            fetch(pos, 1, h);
            b.k = h[0];
            pos += 1;
            if (b.k > 32) { parse_err = "session plane count out of range"; break; }
            if (level > lp && b.k != 32) { parse_err = "session has partial non-progressive level"; break; }
            if (size - pos < 1) { parse_err = trunc; break; }
            fetch(pos, 1, h);
            if (h[0] > 1) { parse_err = "unknown backend id"; break; }
            if (size - pos < 21) { parse_err = trunc; break; }
            fetch(pos, 21, h);
            b.be = h[0];
            b.raw_bits = rd(h + 1, 8);
            b.plen = rd(h + 9, 8);
            b.crc = (uint32_t)rd(h + 17, 4);
            pos += 21;
            if (size - pos < b.plen) { parse_err = trunc; break; }
            b.off = pos;
            pos += b.plen;
            blks.push_back(b);
        }
        if (parse_err.empty() && pos != size) parse_err = "session file has trailing bytes";
        // payload bytes on the device
        DBuf staged;
        const uint8_t *dsrc = src;
        if (!on_device) {
            staged = DBuf(std::max<uint64_t>(pos, 1), st);
            CK(cudaMemcpyAsync(staged.p, src, pos, cudaMemcpyHostToDevice, st));
            dsrc = staged.as<uint8_t>();
        }
        const size_t B = blks.size();
        std::vector<uint32_t> hcrc(B, 0);
        if (B) {
            uint64_t maxp = 1;
            for (const Blk &b : blks) maxp = std::max(maxp, b.plen);
            std::vector<const uint8_t *> ptrs(B);
            std::vector<uint64_t> lens(B);
            for (size_t i = 0; i < B; ++i) ptrs[i] = dsrc + blks[i].off, lens[i] = blks[i].plen;
            const size_t cw = crc32_batch_workspace((int)B, maxp);
            DBuf crcws(cw, st), crcs(B * 4, st), pd(B * 8, st), ld(B * 8, st);
            CK(cudaMemcpyAsync(pd.p, ptrs.data(), B * 8, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(ld.p, lens.data(), B * 8, cudaMemcpyHostToDevice, st));
            crc32_batch(pd.as<const uint8_t *>(), ld.as<uint64_t>(), (int)B, maxp, crcs.as<uint32_t>(), crcws.p, cw, st);
            readback(hcrc.data(), crcs.p, B * 4, st);
        }
        ipcg_session *ns = new ipcg_session;
        ns->archive_crc = ix.identity;
        ns->levels = L;
        ns->lp = lp;
        ns->owner = st;
        ns->pool = &c->scratch;
        ns->device = c->device;
        std::vector<DBuf> scratch_out;  // decode targets of blocks whose size is then rejected
        try {
            // decode every block (identity: copy, deflate: inflate) into its target
            std::vector<InflateJob> jobs;
            std::vector<size_t> job_blk;
            std::vector<CopyDesc> copies;
            std::vector<std::string> blk_err(B);
            for (size_t i = 0; i < B; ++i) {
                const Blk &b = blks[i];
                const int li = b.level - 1;
                ns->k[li] = b.k;
                ns->count[li] = ix.records[li].count;
                if (hcrc[i] != b.crc) { blk_err[i] = "block checksum mismatch"; continue; }
                const uint64_t rb = (b.raw_bits + 7) / 8;
                if (b.be == 0 && b.plen != rb) { blk_err[i] = "identity block has wrong length"; continue; }
                const bool fits = b.level <= lp ? rb == ix.records[li].count * 4 : rb == 0;
                uint8_t *dst = nullptr;
                if (fits && b.level <= lp) {
                    const uint64_t cnt = ix.records[li].count;
                    ns->merged[li] = static_cast<uint32_t *>(scratch_get(std::max<uint64_t>(cnt, 1) * 4 + 16, st));
                    dst = reinterpret_cast<uint8_t *>(ns->merged[li]);
                } else if (rb) {
                    if (rb > (uint64_t(1) << 36)) { blk_err[i] = "std::bad_alloc"; continue; }
                    scratch_out.emplace_back(rb, st);
                    dst = scratch_out.back().as<uint8_t>();
                }
                if (!fits) blk_err[i] = b.level <= lp ? "session codeword array has wrong length"
                                                      : "session stores codewords for a non-progressive level";
                if (!rb) continue;
                if (b.be == 0) copies.push_back(CopyDesc{dsrc + b.off, (uint64_t)reinterpret_cast<uintptr_t>(dst), rb});
                else jobs.push_back(InflateJob{dsrc + b.off, b.plen, dst, rb}), job_blk.push_back(i);
            }
            if (!copies.empty()) gather(c, copies, nullptr);
            if (!jobs.empty()) {
                DevAlloc tmp;
                DBuf sd(jobs.size() * 4, st);
                inflate_batch_host(jobs, sd.as<int>(), tmp, st);
                std::vector<int> js(jobs.size());
                readback(js.data(), sd.p, jobs.size() * 4, st);
                for (size_t k = 0; k < jobs.size(); ++k)
                    if (js[k]) blk_err[job_blk[k]] = "deflate backend failed to decompress block";
            }
            CK(cudaStreamSynchronize(st));
            for (size_t i = 0; i < B; ++i)
                if (!blk_err[i].empty()) throw Error(ERUNTIME, blk_err[i]);
            if (!parse_err.empty()) throw Error(ERUNTIME, parse_err);
        } catch (...) {
            for (int l = 0; l < IPCG_MAX_LEVELS; ++l)
                if (ns->merged[l]) scratch_put(ns->merged[l], st);
            delete ns;
            throw;
        }
        *out = ns;
    });
}

// compute_metrics<T> (pipeline.hpp:354-372) on the device (metrics.cu)
int ipcg_compute_metrics(ipcg_ctx *c, int scalar, const void *original, int original_on_device, uint64_t n_original,
                         const void *decoded, int decoded_on_device, uint64_t n_decoded, double *max_error,
                         double *mse, double *psnr) {
    return guarded(c, [&] {
        if (scalar != 0 && scalar != 1) throw Error(EINVAL_, "field scalars must be f32 or f64");
        if (n_original != n_decoded) throw Error(EINVAL_, "metrics inputs differ in size");
        cudaStream_t st = c->stream;
        const uint64_t bytes = n_original * (scalar == 0 ? 4 : 8);
        DBuf ua, ub;
        const void *a = original, *b = decoded;
        if (!original_on_device && bytes) {
            ua = DBuf(bytes, st);
            CK(cudaMemcpyAsync(ua.p, original, bytes, cudaMemcpyHostToDevice, st));
            a = ua.p;
        }
        if (!decoded_on_device && bytes) {
            ub = DBuf(bytes, st);
            CK(cudaMemcpyAsync(ub.p, decoded, bytes, cudaMemcpyHostToDevice, st));
            b = ub.p;
        }
        double r[3];
        compute_metrics_device(scalar, a, b, n_original, r, st);
        if (max_error) *max_error = r[0];
        if (mse) *mse = r[1];
        if (psnr) *psnr = r[2];
    });
}

int ipcg_plan_for_error(ipcg_ctx *c, const ipcg_archive *a, double max_error, int *k_out) {
    return guarded(c, [&] { plan_for_error(a->ix, max_error, k_out); });
}
int ipcg_plan_for_size(ipcg_ctx *c, const ipcg_archive *a, uint64_t budget, int *k_out) {
    return guarded(c, [&] { plan_for_size(a->ix, budget, k_out); });
}
double ipcg_bound_for_plan(const ipcg_archive *a, const int *k) { return bound_for_plan(a->ix, k); }
uint64_t ipcg_plan_payload_bytes(const ipcg_archive *a, const int *k) { return plan_payload_bytes(a->ix, k); }

int ipcg_build_error_model(const ipcg_index *ix, ipcg_error_model *out) {
    return guarded(nullptr, [&] {
        if (!ix || !out) throw Error(EINVAL_, "build_error_model: null argument");
        if (ix->levels > IPCG_MAX_LEVELS) throw Error(EINVAL_, "archive has more levels than supported");
        build_error_model(*ix, *out);
    });
}
int ipcg_model_plan_for_error(const ipcg_error_model *m, double max_error, int *k_out) {
    return guarded(nullptr, [&] {
        check_model(*m);
        plan_for_error(*m, max_error, k_out);
    });
}
int ipcg_model_plan_device(ipcg_ctx *c, const ipcg_error_model *m, int by_size, double max_error, uint64_t byte_budget,
                           int *k_out) {
    return guarded(c, [&] {
        if (!c || !m || !k_out) throw Error(EINVAL_, "plan_device: null argument");
        plan_on_device(*m, by_size ? 1 : 0, max_error, byte_budget, k_out, c->stream);
        ++c->launches;
    });
}
int ipcg_model_plan_for_size(const ipcg_error_model *m, uint64_t budget, int *k_out) {
    return guarded(nullptr, [&] {
        check_model(*m);
        plan_for_size(*m, budget, k_out);
    });
}
double ipcg_model_bound_for_plan(const ipcg_error_model *m, const int *k) { return bound_for_plan(*m, k); }
uint64_t ipcg_model_plan_payload_bytes(const ipcg_error_model *m, const int *k) { return plan_payload_bytes(*m, k); }
uint64_t ipcg_model_mandatory_payload_bytes(const ipcg_error_model *m) { return mandatory_payload_bytes(*m); }
uint64_t ipcg_model_total_payload_bytes(const ipcg_error_model *m) { return total_payload_bytes(*m); }

int ipcg_backend_encode(ipcg_ctx *c, const uint8_t *raw, int raw_on_device, uint64_t plane_bytes, uint64_t raw_stride,
                        int count, uint8_t *backend, uint64_t *length, uint32_t *crc, uint8_t *out_payload,
                        uint64_t out_capacity) {
    return guarded(c, [&] {
        if (count <= 0) return;
        cudaStream_t st = c->stream;
        const uint64_t in_stride = round_up(std::max<uint64_t>(plane_bytes, 1), 16);
        DBuf in((uint64_t)count * in_stride, st);
        for (int i = 0; i < count; ++i)
            CK(cudaMemcpyAsync(in.as<uint8_t>() + i * in_stride, raw + i * raw_stride, plane_bytes,
                               raw_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        const uint64_t out_stride = round_up(plane_bytes + 16, 16);
        DBuf outb((uint64_t)count * out_stride, st), ws(DeflateBatch::workspace_bytes(count, plane_bytes), st);
        DBuf be(count, st), ln(count * 8, st), cr(count * 4, st), pl(count * 8, st);
        const BackendResults res{be.as<uint8_t>(), ln.as<uint64_t>(), cr.as<uint32_t>(), pl.as<const uint8_t *>()};
        DeflateBatch::run(in.as<uint8_t>(), in_stride, count, plane_bytes, outb.as<uint8_t>(), out_stride, ws.p, res, st);
        std::vector<const uint8_t *> ptrs(count);
        CK(cudaMemcpyAsync(backend, be.p, count, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(length, ln.p, count * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(crc, cr.p, count * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ptrs.data(), pl.p, count * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        uint64_t o = 0;
        for (int i = 0; i < count; ++i) {
            if (o + length[i] > out_capacity) throw Error(EINVAL_, "output capacity too small");
            CK(cudaMemcpyAsync(out_payload + o, ptrs[i], length[i], cudaMemcpyDeviceToHost, st));
            o += length[i];
        }
        CK(cudaStreamSynchronize(st));
    });
}

int ipcg_backend_decode(ipcg_ctx *c, const uint8_t *payloads, const uint64_t *payload_len, const uint8_t *backend,
                        const uint32_t *crc, const uint64_t *raw_bytes, int count, uint8_t *out, int *status) {
    return guarded(c, [&] {
        if (count <= 0) return;
        cudaStream_t st = c->stream;
        uint64_t tin = 0, tout = 0, maxp = 1;
        std::vector<uint64_t> in_off(count), out_off(count);
        for (int i = 0; i < count; ++i) {
            in_off[i] = tin;
            out_off[i] = tout;
            tin += payload_len[i];
            tout += raw_bytes[i];
            maxp = std::max(maxp, payload_len[i]);
        }
        DBuf din(tin + 16, st), dout(tout + 16, st);
        CK(cudaMemcpyAsync(din.p, payloads, tin, cudaMemcpyHostToDevice, st));
        std::vector<const uint8_t *> ptrs(count);
        for (int i = 0; i < count; ++i) ptrs[i] = din.as<uint8_t>() + in_off[i];
        const size_t cw = crc32_batch_workspace(count, maxp);
        DBuf crcws(cw, st), crcs(count * 4, st), pd(count * 8, st), ld(count * 8, st);
        CK(cudaMemcpyAsync(pd.p, ptrs.data(), count * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ld.p, payload_len, count * 8, cudaMemcpyHostToDevice, st));
        crc32_batch(pd.as<const uint8_t *>(), ld.as<uint64_t>(), count, maxp, crcs.as<uint32_t>(), crcws.p, cw, st);
        std::vector<uint32_t> hcrc(count);
        CK(cudaMemcpyAsync(hcrc.data(), crcs.p, count * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<InflateJob> jobs;
        std::vector<int> job_of;
        std::vector<CopyDesc> copies;
        for (int i = 0; i < count; ++i) {
            status[i] = 0;
            if (hcrc[i] != crc[i]) {
                status[i] = 1;
                continue;
            }
            uint8_t *dst = dout.as<uint8_t>() + out_off[i];
            if (backend[i] == 0) {
                if (payload_len[i] != raw_bytes[i]) status[i] = 3;
                else copies.push_back(CopyDesc{ptrs[i], (uint64_t)reinterpret_cast<uintptr_t>(dst), raw_bytes[i]});
            } else {
                jobs.push_back(InflateJob{ptrs[i], payload_len[i], dst, raw_bytes[i]});
                job_of.push_back(i);
            }
        }
        if (!copies.empty()) gather(c, copies, nullptr);
        if (!jobs.empty()) {
            DevAlloc tmp;
            DBuf sd(jobs.size() * 4, st);
            inflate_batch_host(jobs, sd.as<int>(), tmp, st);
            std::vector<int> js(jobs.size());
            CK(cudaMemcpyAsync(js.data(), sd.p, jobs.size() * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            for (size_t k = 0; k < jobs.size(); ++k)
                if (js[k]) status[job_of[k]] = 2;
        }
        CK(cudaMemcpyAsync(out, dout.p, tout, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

// ---------------------------------------------------------- bitplane API
// split / xor_encode / xor_decode / merge (bitplane.cpp:7-59) on host plane arrays: staged
// through 32 device word rows (16-byte aligned, zero-padded past the plane's bytes)
namespace {
struct PlaneRows {
    DBuf buf;
    uint64_t stride = 0, nbytes = 0;
    PlaneRows(uint64_t count, cudaStream_t st) {
        nbytes = (count + 7) / 8;
        stride = round_up(std::max<uint64_t>((count + 31) / 32, 1), 4);
        buf = DBuf(32 * stride * 4, st);
        CK(cudaMemsetAsync(buf.p, 0, 32 * stride * 4, st));
    }
    uint32_t *row(int p) const { return buf.as<uint32_t>() + (uint64_t)p * stride; }
    void upload(const uint8_t *const *planes, int np, cudaStream_t st) {
        for (int p = 0; p < np; ++p)
            if (nbytes) CK(cudaMemcpyAsync(row(p), planes[p], nbytes, cudaMemcpyHostToDevice, st));
    }
    void download(uint8_t *const *planes, int np, cudaStream_t st) {
        for (int p = 0; p < np; ++p)
            if (nbytes) CK(cudaMemcpyAsync(planes[p], row(p), nbytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
};
}  // namespace

int ipcg_split(ipcg_ctx *c, const uint32_t *codewords, uint64_t count, int xor_encode, uint8_t *const *planes) {
    return guarded(c, [&] {
        if (!planes || (count && !codewords)) throw Error(EINVAL_, "split: null argument");
        cudaStream_t st = c->stream;
        PlaneRows r(count, st);
        DBuf codes(std::max<uint64_t>(count, 1) * 4, st);
        if (count) CK(cudaMemcpyAsync(codes.p, codewords, count * 4, cudaMemcpyHostToDevice, st));
        launch_split(codes.as<uint32_t>(), count, r.row(0), r.stride, xor_encode != 0, st);
        r.download(planes, 32, st);
    });
}

int ipcg_plane_xor(ipcg_ctx *c, uint8_t *const *planes, uint64_t count, int np, int decode) {
    return guarded(c, [&] {
        if (np < 0 || np > 32) throw Error(EINVAL_, "plane count out of range");
        if (!planes) throw Error(EINVAL_, "plane_xor: null argument");
        cudaStream_t st = c->stream;
        PlaneRows r(count, st);
        r.upload(planes, np, st);
        launch_plane_xor(r.row(0), r.stride, count, np, decode != 0, st);
        r.download(planes, np, st);
    });
}

int ipcg_merge(ipcg_ctx *c, const uint8_t *const *planes, uint64_t count, int k, uint32_t *codewords) {
    return guarded(c, [&] {
        if (k < 0 || k > 32) throw Error(EINVAL_, "plane count out of range");
        if ((k && !planes) || (count && !codewords)) throw Error(EINVAL_, "merge: null argument");
        cudaStream_t st = c->stream;
        PlaneRows r(count, st);
        r.upload(planes, k, st);
        DBuf out(std::max<uint64_t>(count, 1) * 4, st);
        launch_merge_raw(r.row(0), r.stride, count, k, out.as<uint32_t>(), st);
        if (count) CK(cudaMemcpyAsync(codewords, out.p, count * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

uint64_t ipcg_kernel_launches(const ipcg_ctx *c) { return c ? c->launches : launch_counter(); }

int ipcg_profile_enable(ipcg_ctx *c, int enable) {
    return guarded(c, [&] {
        CK(cudaStreamSynchronize(c->stream));
        Profiler &p = c->prof;
        for (auto &r : p.recs) p.pool.push_back(r.a), p.pool.push_back(r.b);
        p.recs.clear();
        p.enabled = enable != 0;
    });
}

// JSON object {family: [total_ms, scopes, algorithmic_bytes], ...}; clears the records
int ipcg_profile_read(ipcg_ctx *c, char *json, uint64_t capacity) {
    return guarded(c, [&] {
        CK(cudaStreamSynchronize(c->stream));
        Profiler &p = c->prof;
        std::vector<std::string> names;
        std::vector<double> ms;
        std::vector<uint64_t> cnt, bytes;
        for (auto &r : p.recs) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, r.a, r.b));
            size_t i = 0;
            while (i < names.size() && names[i] != r.name) ++i;
            if (i == names.size()) names.push_back(r.name), ms.push_back(0), cnt.push_back(0), bytes.push_back(0);
            ms[i] += t;
            cnt[i] += 1;
            bytes[i] += r.bytes;
            p.pool.push_back(r.a);
            p.pool.push_back(r.b);
        }
        p.recs.clear();
        std::string out = "{";
        for (size_t i = 0; i < names.size(); ++i) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "%s\"%s\": [%.6f, %llu, %llu]", i ? ", " : "", names[i].c_str(), ms[i],
                          (unsigned long long)cnt[i], (unsigned long long)bytes[i]);
            out += buf;
        }
        out += "}";
        if (out.size() + 1 > capacity) throw Error(EINVAL_, "profile buffer too small");
        std::memcpy(json, out.c_str(), out.size() + 1);
    });
}

}  // extern "C"
