// deflate.cu -- sm_100a implementation of DeflateBatch: the zlib-1.3 compress2(level 6)
// byte stream for many equal-length bitplanes at once.  Stage semantics live in
// deflate_core.cuh (shared with the CPU model in tests/native/zmodel.cpp, which is
// diffed against libz); this file only maps the stages onto the GPU:
//   scan (zero test, Adler-32) -> prevlinks (warp-serial hash heads in smem) ->
//   match search (thread/position) -> anchors (block max-scan) -> chunk bounds ->
//   chunk transfer maps (thread per chunk x tag) -> resolve (warp scan of 4->4 maps) ->
//   symbol emission -> per-block Huffman plans -> bit layout -> bit emission ->
//   CRC-32 (chunked + GF(2) combine).
// All-zero planes (most high planes) are compressed once per batch and shared.
#include <cstdlib>
#include "deflate.cuh"
#include "deflate_core.cuh"

namespace ipcg {

using namespace ipz;

namespace {

constexpr int CH = DeflateBatch::CH;
constexpr int PL_WARPS = 3;  // prevlink warps per CTA (64 KiB head table each)
constexpr int CRC_CHUNK = 1024;  // bytes per thread (4 KiB left the 30 MB of a refine's identity planes at ~7K threads)

struct StreamMeta {
    unsigned long long nonzero, adA, adB, zeros;
    uint32_t adler;
    int active, rep, final_tag;
    int od;  // parsed by the on-demand walkers (sparse streams) instead of the all-position search
    unsigned long long S_loop, nsyms, nblocks, total_bits, comp_len;
};

struct Bump {
    uint8_t *p;
    size_t off = 0;
    template <class T>
    T *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T *r = reinterpret_cast<T *>(p + off);
        off += count * sizeof(T) + 16;
        return r;
    }
};

struct RunTask {  // a long periodic stretch of match(258) symbols, written in parallel
    uint64_t a0, g0, m;
    int j;
};

struct Work {
    StreamMeta *meta;
    RunTask *runs;
    unsigned long long *nruns;
    uint16_t *prevd;
    uint64_t *rec;
    uint64_t *first_anchor, *bnd;
    uint32_t *nbreak;  // first chunk >= k that is not entirely 258-byte matches
    uint8_t *exit4;
    uint32_t *cnt4;
    uint8_t *entry;
    uint64_t *symoff;
    uint8_t *seg_exit4, *seg_entry;  // the same per SEG-chunk segment (two-level resolve;
                                     // seg_symoff/seg_cnt4 first serve the bounds scan)
    uint32_t *seg_cnt4;
    uint64_t *seg_symoff;
    uint32_t *syms;
    uint64_t *blk_top, *blk_start, *blk_bitpos;
    BlockTrees *trees;
    uint32_t *crc_part;
    uint32_t *crc_tab;
    uint64_t nchunks, nseg, maxb, ncrc;
    // on-demand parse (streams < 2^31 bytes): per-position visit words, the chunk walks'
    // symbols and loop-top offsets (all three alias `rec`, which only the wide path uses)
    uint16_t *od_vis, *od_spos;
    uint32_t *od_ssym;
    struct OdChunk *od_chunks;
    uint64_t od_nch;
    uint32_t od_C;
    // next byte-change position at or after each 64-byte group (suffix minimum): run lengths in
    // O(1) for the continuation walks' run jumps
    uint32_t *od_chg;
    uint64_t od_ng;
    uint64_t *od_cbuf;  // OD_CB continuation symbols (sym | loop top << 32) per chunk
    uint4 *od_link;     // per chunk (nxt, nidx, nsym, ncont), packed for the path resolution
    struct OdSc *od_sc; // per chunk as a superchunk entry (k_od_sc_jump)
    uint4 *od_entry;    // per superchunk: the path's entry (chunk, join index, output offset)
    uint64_t od_nsc;
};

constexpr uint64_t SEG = 32;  // chunks per resolve segment
constexpr int OD_CB = 4;      // continuation symbols buffered per chunk by k_od_sync
constexpr int OD_SC = 1024;   // chunks per superchunk of the path resolution

// one chunk of the on-demand parse (deflate_core.cuh Walker): its walk from (start, A), the
// continuation from the walk's exit, and its place on the true parse
struct OdChunk {
    uint32_t nsym;                        // symbols of the chunk's own walk
    uint32_t ex_p, ex_tag, ex_pl, ex_pd;  // the walk's exit state (first loop top past the chunk)
    uint32_t nxt;                         // chunk whose walk the continuation joins (od_nch: stream end)
    uint32_t nidx;                        // ... at that walk's symbol index; the final tag at the end
    uint32_t ncont;                       // symbols the continuation emits before it joins
    uint32_t adopted, aidx;               // on the true parse; its first own symbol on it
    uint32_t cbuf_ok;                     // the continuation's symbols are in od_cbuf (no re-walk)
    uint64_t aoff, coff;                  // output offsets of the adopted own symbols / the continuation
};

static uint32_t od_chunk_size() {
    static const uint32_t c = getenv("IPCG_OD_CHUNK") ? (uint32_t)atoi(getenv("IPCG_OD_CHUNK")) : 64u;
    return c < 16 ? 16u : c > 8192 ? 8192u : c;
}

Work carve(void *ws, int S, uint64_t n, size_t *size_out = nullptr) {
    Bump b{static_cast<uint8_t *>(ws)};
    Work w;
    w.nchunks = (n + CH - 1) / CH;
    w.nseg = (w.nchunks + SEG - 1) / SEG;
    w.maxb = n / BLOCK_SYMS + 2;
    w.ncrc = (n + 64 + CRC_CHUNK - 1) / CRC_CHUNK + 1;
    w.meta = b.take<StreamMeta>(S);
    w.runs = b.take<RunTask>((size_t)S * (w.nchunks + 2));
    w.nruns = b.take<unsigned long long>(1);
    w.prevd = b.take<uint16_t>((size_t)S * n);
    w.rec = b.take<uint64_t>((size_t)S * n);
    w.od_C = od_chunk_size();
    w.od_nch = (n + w.od_C - 1) / w.od_C;
    w.od_vis = b.take<uint16_t>((size_t)S * n);
    w.od_spos = b.take<uint16_t>((size_t)S * n);
    w.od_ssym = b.take<uint32_t>((size_t)S * n);
    w.od_chunks = b.take<OdChunk>((size_t)S * w.od_nch);
    w.od_cbuf = b.take<uint64_t>((size_t)S * w.od_nch * OD_CB);
    w.od_link = b.take<uint4>((size_t)S * w.od_nch);
    w.od_nsc = (w.od_nch + OD_SC - 1) / OD_SC;
    w.od_sc = b.take<OdSc>((size_t)S * w.od_nsc * OD_SC);
    w.od_entry = b.take<uint4>((size_t)S * w.od_nsc);
    w.od_ng = (n + 63) / 64;
    w.od_chg = b.take<uint32_t>((size_t)S * (w.od_ng + 1));
    w.first_anchor = b.take<uint64_t>((size_t)S * w.nchunks);
    w.nbreak = b.take<uint32_t>((size_t)S * (w.nchunks + 1));
    w.bnd = b.take<uint64_t>((size_t)S * (w.nchunks + 1));
    w.exit4 = b.take<uint8_t>((size_t)S * w.nchunks * 4);
    w.cnt4 = b.take<uint32_t>((size_t)S * w.nchunks * 4);
    w.entry = b.take<uint8_t>((size_t)S * (w.nchunks + 1));
    w.symoff = b.take<uint64_t>((size_t)S * w.nchunks);
    w.seg_exit4 = b.take<uint8_t>((size_t)S * w.nseg * 4);
    w.seg_cnt4 = b.take<uint32_t>((size_t)S * w.nseg * 4);
    w.seg_entry = b.take<uint8_t>((size_t)S * (w.nseg + 1));
    w.seg_symoff = b.take<uint64_t>((size_t)S * w.nseg);
    w.syms = b.take<uint32_t>((size_t)S * (n + 1));
    w.blk_top = b.take<uint64_t>((size_t)S * w.maxb);
    w.blk_start = b.take<uint64_t>((size_t)S * w.maxb);
    w.blk_bitpos = b.take<uint64_t>((size_t)S * w.maxb);
    w.trees = b.take<BlockTrees>((size_t)S * w.maxb);
    w.crc_part = b.take<uint32_t>((size_t)S * w.ncrc);
    w.crc_tab = b.take<uint32_t>(8 * 256);
    if (size_out) *size_out = b.off + 256;
    return w;
}

size_t carve_size(int S, uint64_t n) {
    size_t sz = 0;
    carve(nullptr, S, n, &sz);
    return sz;
}

struct InBytes {
    const uint8_t *p;  // 8-byte aligned stream base; rows are padded to 16 bytes
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return __ldg(p + i); }
    __device__ __forceinline__ uint64_t load8(int64_t i) const {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p + i);
        const uint64_t *w = reinterpret_cast<const uint64_t *>(a & ~uintptr_t(7));
        const unsigned sh = (unsigned)(a & 7) * 8;
        const uint64_t lo = __ldg(w);
        return sh ? (lo >> sh) | (__ldg(w + 1) << (64 - sh)) : lo;
    }
    // common prefix length of the strings at a and b, capped at maxlen (8 bytes per step)
    __device__ __forceinline__ int64_t match_len(int64_t a, int64_t b, int64_t maxlen) const {
        int64_t len = 0;
        for (; len + 8 <= maxlen; len += 8) {
            const uint64_t x = load8(a + len) ^ load8(b + len);
            if (x) return len + (__ffsll((long long)x) - 1) / 8;
        }
        while (len < maxlen && p[a + len] == p[b + len]) ++len;
        return len;
    }
};
// InBytes for a thread that walks a stream forward (k_emit_syms: the lanes of a warp walk chunks
// 256 bytes apart, so every byte load is 32 separate L1 accesses): the aligned 8 bytes holding
// the last byte asked for stay in a register.  (Rows are 8-byte aligned and padded to 16 bytes.)
struct InBytesCached {
    const uint8_t *p;
    mutable int64_t base = -8;
    mutable uint64_t w = 0;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const {
        const int64_t b = i & ~int64_t(7);
        if (b != base) {
            base = b;
            w = __ldg(reinterpret_cast<const uint64_t *>(p + b));
        }
        return (uint32_t)(w >> (8 * (unsigned)(i - b))) & 0xffu;
    }
};
struct PrevD {
    const uint16_t *p;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return __ldg(p + i); }
};
struct PrevD32 {
    const uint16_t *p;
    __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return __ldg(p + i); }
};
// 4-byte words of a stream whose base is 16-byte aligned and whose row is padded to 16
// bytes, so a word whose first byte is < n is always inside the allocation.
struct InWords {
    const uint8_t *p;  // stream base
    __device__ __forceinline__ uint32_t word(uint32_t k) const { return __ldg(reinterpret_cast<const uint32_t *>(p) + k); }
    __device__ __forceinline__ uint32_t byte(uint32_t i) const { return __ldg(p + i); }
    __device__ __forceinline__ const uint8_t *at(uint32_t off) const { return p + off; }
};

// ------------------------------------------------------------------ 1. scan
// Adler-32 B = sum_i (n - i) b_i = n A - sum_i i b_i (mod 65521): each thread takes 16 bytes per
// step (rows are 16-byte aligned and padded), sums and byte-index-weighted sums by dp4a in exact
// 64-bit integers, reduced mod 65521 once per thread (a per-byte 64-bit modulo made this pass
// ALU-bound at ~0.5 TB/s).
__global__ void k_scan(const uint8_t *in, uint64_t in_stride, uint64_t n, StreamMeta *meta) {
    const int j = blockIdx.y;
    const uint8_t *p = in + (uint64_t)j * in_stride;
    unsigned long long nz = 0, A = 0, W = 0, zc = 0;  // zc: zero bytes x 8 (vcmpeq4 sets 8 bits per byte)
    const uint64_t nv = n / 16;
    const uint4 *pv = reinterpret_cast<const uint4 *>(p);
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 q = __ldg(pv + v);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t s = 0, ws = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t sk = __dp4a(w[k], 0x01010101u, 0u);
            s += sk;
            ws += __dp4a(w[k], 0x03020100u, 0u) + 4u * k * sk;
        }
        nz |= q.x | q.y | q.z | q.w;
        zc += __popc(__vcmpeq4(q.x, 0u)) + __popc(__vcmpeq4(q.y, 0u)) + __popc(__vcmpeq4(q.z, 0u)) +
              __popc(__vcmpeq4(q.w, 0u));
        A += s;
        W += (unsigned long long)(16 * v) * s + ws;
    }
    for (uint64_t i = nv * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = p[i];
        nz |= b;
        zc += b == 0 ? 8u : 0u;
        A += b;
        W += (unsigned long long)i * b;
    }
    const unsigned long long M = 65521;
    unsigned long long B = ((n % M) * (A % M) + M - W % M) % M;
    nz = __reduce_or_sync(0xffffffffu, (unsigned)(nz != 0));
    for (int o = 16; o > 0; o >>= 1) {
        A += __shfl_down_sync(0xffffffffu, A, o);
        B += __shfl_down_sync(0xffffffffu, B, o);
        zc += __shfl_down_sync(0xffffffffu, zc, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&meta[j].zeros, zc / 8);
        if (nz) atomicOr(&meta[j].nonzero, 1ull);
        atomicAdd(&meta[j].adA, A);
        atomicAdd(&meta[j].adB, B % 65521u);
    }
}

__global__ void k_select(StreamMeta *meta, int S, uint64_t n, int od_mode, int od_zeros_pct) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int rep = -1;
    for (int j = 0; j < S; ++j)
        if (!meta[j].nonzero) {
            rep = j;
            break;
        }
    for (int j = 0; j < S; ++j) {
        StreamMeta &m = meta[j];
        m.rep = rep;
        m.active = (m.nonzero || j == rep) && n > 0;
        // on-demand parse for sparse streams: mostly zero bytes means long matches, and the lazy
        // parse then visits few of the positions the all-position search would cover (measured
        // on cfg2 level-1 planes: 92% zeros -> 14% of the search work)
        m.od = od_mode == 1 || (od_mode == 0 && m.zeros * 100 >= (unsigned long long)n * od_zeros_pct);
        const uint32_t a = (uint32_t)((1 + m.adA) % 65521u);
        const uint32_t b = (uint32_t)((m.adB + n) % 65521u);
        m.adler = (b << 16) | a;
    }
}

// ------------------------------------------------------------- 2. prevlinks
// zlib's head/prev insertion order is sequential; one warp walks 32 positions per step
// through a 64 KiB shared-memory head table (match_any resolves same-step collisions).
// Each warp owns `span` 32 KiB windows (chosen per launch from a wave model: longer spans
// amortise the warm-up, shorter ones fill the SMs) and warms up on the window before them.  Table
// entries hold positions (relative to the warm-up start) modulo 65536: at the start of
// window W every entry older than WSIZE-1 relative to the window start becomes the sentinel
// S_W = ((W-1)*WSIZE) mod 65536 -- valid entries during W lie in [W*WSIZE - 32767,
// (W+1)*WSIZE), which covers every residue but that one -- so a lookup's distance is
// (p - entry) mod 65536.  Only the head-table read/write chain is serial: a batch of AHEAD
// steps has its bytes loaded one batch ahead (one byte per lane + two spill bytes, the rest
// by shuffles) and all its match_any masks computed before the chain runs; head reads are
// consumed only after the batch (ncu: using them inside the chain, packing the two loaded
// bytes at fetch time, or inlining the sweep each cost 1.5-2.5x).
// Window-boundary sweep of a prevlinks head table (out of line: it runs once per 32 KiB
// window and would otherwise cost the chain loop registers).
__device__ __noinline__ uint32_t prevlinks_sweep(uint16_t *head, unsigned lane, uint32_t rel0, uint32_t sent) {
    const uint32_t nsent = (rel0 - WSIZE) & 0xFFFF;
    uint4 *h4 = reinterpret_cast<uint4 *>(head);
    for (int i = lane; i < 32768 / 8; i += 32) {
        uint4 v = h4[i];
        uint32_t *w = reinterpret_cast<uint32_t *>(&v);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t sh = (k & 1) * 16, e = (w[k >> 1] >> sh) & 0xFFFF, age = (rel0 - e) & 0xFFFF;
            if (e == sent || age == 0 || age >= (uint32_t)WSIZE) w[k >> 1] = (w[k >> 1] & ~(0xFFFFu << sh)) | (nsent << sh);
        }
        h4[i] = v;
    }
    __syncwarp();
    return nsent;
}

__global__ void __launch_bounds__(PL_WARPS * 32) k_prevlinks(const uint8_t *in, uint64_t in_stride, uint64_t n,
                                                           const StreamMeta *meta, uint16_t *prevd_all, int span) {
    extern __shared__ uint16_t heads[];
    const int j = blockIdx.y;
    if (!meta[j].active) return;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t out0 = ((uint64_t)blockIdx.x * PL_WARPS + warp) * (uint64_t)span * WSIZE;
    if (out0 >= n) return;
    uint16_t *head = heads + (size_t)warp * 32768;
    for (int i = lane; i < 32768; i += 32) head[i] = 0x8000;  // S_0
    __syncwarp();
    const uint8_t *p = in + (uint64_t)j * in_stride;
    uint16_t *prevd = prevd_all + (uint64_t)j * n;
    const uint64_t base = out0 == 0 ? 0 : out0 - WSIZE;
    const uint64_t end = min(n, out0 + (uint64_t)span * WSIZE);
    constexpr int AHEAD = 16;
    uint32_t b0[AHEAD], bx[AHEAD];  // byte at q; lanes 0,1: byte at q + 32
    auto fetch = [&](uint64_t pos0) {
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            b0[k] = q < n ? __ldg(p + q) : 0u;
            bx[k] = (lane < 2 && q + 32 < n) ? __ldg(p + q + 32) : 0u;
        }
    };
    fetch(base);
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t sent = 0x8000;
    for (uint64_t pos0 = base; pos0 < end; pos0 += 32 * AHEAD) {
        const uint32_t rel0 = (uint32_t)(pos0 - base);
        if (rel0 != 0 && (rel0 & (WSIZE - 1)) == 0) {  // window boundary (32*AHEAD divides WSIZE)
            sent = prevlinks_sweep(head, lane, rel0, sent);
        }
        uint32_t hs[AHEAD], mk[AHEAD];
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            const uint32_t v1 = __shfl_sync(0xffffffffu, b0[k], (lane + 1) & 31);
            const uint32_t e1 = __shfl_sync(0xffffffffu, bx[k], (lane + 1) & 31);
            const uint32_t v2 = __shfl_sync(0xffffffffu, b0[k], (lane + 2) & 31);
            const uint32_t e2 = __shfl_sync(0xffffffffu, bx[k], (lane + 2) & 31);
            const uint32_t c1 = lane == 31 ? e1 : v1, c2 = lane >= 30 ? e2 : v2;
            const bool valid = q + MIN_MATCH <= n && q < end;
            hs[k] = valid ? hash3(b0[k], c1, c2) : (0x10000u + lane);
        }
        if (pos0 + 32 * AHEAD < end) fetch(pos0 + 32 * AHEAD);
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) mk[k] = __match_any_sync(0xffffffffu, hs[k]);
        uint32_t prel[AHEAD];
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint32_t h = hs[k];
            const bool valid = h < 0x10000u;
            const uint32_t rel = (uint32_t)(pos0 + 32 * k + lane - base);
            const unsigned lower = mk[k] & lt_mask;
            prel[k] = sent;
            if (lower) prel[k] = rel - (lane - (31u - __clz(lower)));
            else if (valid) prel[k] = head[h];
            __syncwarp();
            if (valid && lane == 31u - __clz(mk[k])) head[h] = (uint16_t)rel;
            __syncwarp();
        }
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            if (q >= out0 && q < end) {
                const uint32_t e = prel[k] & 0xFFFF, d = ((uint32_t)(q - base) - e) & 0xFFFF;
                prevd[q] = (uint16_t)(hs[k] < 0x10000u && e != sent && d < (uint32_t)WSIZE ? d : 0u);
            }
        }
    }
}

// Two warps per head table.  With one warp per table (three per SM) the kernel runs at one warp's
// dependent-issue latency: ~100 instructions per 32 positions of which only the head-table
// read/write chain is serial.  Here warps A and B of a pair take alternate batches of a span: each
// prepares its batch (bytes, hashes, match_any) and stores its links on its own, and only the
// chain (and the window sweep) is a critical section handed back and forth with two named
// barriers (bar.arrive by the warp that leaves it, bar.sync by the one that enters).
__device__ __forceinline__ void pl_bar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void pl_bar_arrive(int id) {
    __threadfence_block();
    asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

template <int NW>  // warps per head table
__global__ void __launch_bounds__(PL_WARPS * NW * 32) k_prevlinks_pair(const uint8_t *in, uint64_t in_stride, uint64_t n,
                                                                     const StreamMeta *meta, uint16_t *prevd_all, int span) {
    extern __shared__ uint16_t heads[];
    const int j = blockIdx.y;
    if (!meta[j].active) return;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned pair = warp / NW, par = warp % NW;  // table of the group; warp `par` takes batches par, par + NW, ...
    const uint64_t out0 = ((uint64_t)blockIdx.x * PL_WARPS + pair) * (uint64_t)span * WSIZE;
    if (out0 >= n) return;  // (both warps of the pair)
    uint16_t *head = heads + (size_t)pair * 32768;
    // barrier "warp g of the group left the chain": 1 + NW * group + g
    const int bar_mine = 1 + NW * (int)pair + (int)par, bar_prev = 1 + NW * (int)pair + (int)((par + NW - 1) % NW);
    if (par == 0) {
        for (int i = lane; i < 32768; i += 32) head[i] = 0x8000;  // S_0
        __syncwarp();
    }
    const uint8_t *p = in + (uint64_t)j * in_stride;
    uint16_t *prevd = prevd_all + (uint64_t)j * n;
    const uint64_t base = out0 == 0 ? 0 : out0 - WSIZE;
    const uint64_t end = min(n, out0 + (uint64_t)span * WSIZE);
    constexpr int AHEAD = 16;
    constexpr uint64_t BATCH = 32 * AHEAD;
    uint32_t b0[AHEAD], bx[AHEAD];  // byte at q; lanes 0,1: byte at q + 32
    auto fetch = [&](uint64_t pos0) {
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            b0[k] = q < n ? __ldg(p + q) : 0u;
            bx[k] = (lane < 2 && q + 32 < n) ? __ldg(p + q + 32) : 0u;
        }
    };
    const uint64_t first = base + par * BATCH;
    if (first < end) fetch(first);
    const unsigned lt_mask = (1u << lane) - 1u;
    for (uint64_t pos0 = first; pos0 < end; pos0 += NW * BATCH) {
        const uint32_t rel0 = (uint32_t)(pos0 - base);
        uint32_t hs[AHEAD], mk[AHEAD];
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            const uint32_t v1 = __shfl_sync(0xffffffffu, b0[k], (lane + 1) & 31);
            const uint32_t e1 = __shfl_sync(0xffffffffu, bx[k], (lane + 1) & 31);
            const uint32_t v2 = __shfl_sync(0xffffffffu, b0[k], (lane + 2) & 31);
            const uint32_t e2 = __shfl_sync(0xffffffffu, bx[k], (lane + 2) & 31);
            const uint32_t c1 = lane == 31 ? e1 : v1, c2 = lane >= 30 ? e2 : v2;
            const bool valid = q + MIN_MATCH <= n && q < end;
            hs[k] = valid ? hash3(b0[k], c1, c2) : (0x10000u + lane);
        }
        if (pos0 + NW * BATCH < end) fetch(pos0 + NW * BATCH);
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) mk[k] = __match_any_sync(0xffffffffu, hs[k]);
        // ---- the critical section: every batch but the first waits for the previous one's
        if (pos0 != base) pl_bar_sync(bar_prev);
        // the sentinel of this batch's window W = rel0 / WSIZE is ((W - 1) * WSIZE) mod 65536; the
        // batch that opens a window sweeps the table (from the previous window's sentinel)
        const uint32_t W = rel0 / (uint32_t)WSIZE;
        uint32_t sent = ((W - 1u) * (uint32_t)WSIZE) & 0xFFFFu;
        if (rel0 != 0 && (rel0 & (WSIZE - 1)) == 0) sent = prevlinks_sweep(head, lane, rel0, ((W - 2u) * (uint32_t)WSIZE) & 0xFFFFu);
        uint32_t prel[AHEAD];
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint32_t h = hs[k];
            const bool valid = h < 0x10000u;
            const uint32_t rel = (uint32_t)(pos0 + 32 * k + lane - base);
            const unsigned lower = mk[k] & lt_mask;
            prel[k] = sent;
            if (lower) prel[k] = rel - (lane - (31u - __clz(lower)));
            else if (valid) prel[k] = head[h];
            __syncwarp();
            if (valid && lane == 31u - __clz(mk[k])) head[h] = (uint16_t)rel;
            __syncwarp();
        }
        pl_bar_arrive(bar_mine);
        // ---- links of the batch
#pragma unroll
        for (int k = 0; k < AHEAD; ++k) {
            const uint64_t q = pos0 + 32 * k + lane;
            if (q >= out0 && q < end) {
                const uint32_t e = prel[k] & 0xFFFF, d = ((uint32_t)(q - base) - e) & 0xFFFF;
                prevd[q] = (uint16_t)(hs[k] < 0x10000u && e != sent && d < (uint32_t)WSIZE ? d : 0u);
            }
        }
    }
}

// ------------------------------------------------------------ 3. match search
// One thread per position runs zlib's longest_match for chain limits 128 and 32 (one
// walk, the 32-limit result snapshotted on the way).  Measured alternatives that lost:
// staging the tile in shared memory (the walk is latency-, not bandwidth-bound: 70 ms vs
// 43 ms) and a per-lane state machine that refills idle lanes (87 ms: neighbouring
// positions have similar chain lengths, so the extra state costs more than divergence).
// A CTA takes a contiguous chunk of `chunk` positions (tile after tile of blockDim positions), so
// its lookups stay inside one slowly sliding window -- 32 KiB of bytes + 64 KiB of links -- that
// lives in L1; a grid-stride loop moved every CTA to a new window each iteration (ncu: 59% L1 hits,
// two thirds of the stall samples on the L2 round trips of the scattered link / byte loads).
template <bool WIDE, int BLOCK>  // WIDE: streams of 2^31 bytes or more (64-bit positions)
__global__ void __launch_bounds__(BLOCK) k_match(const uint8_t *in, uint64_t in_stride, uint64_t n,
                                                const StreamMeta *meta, const uint16_t *prevd_all, uint64_t *rec_all,
                                                uint32_t chunk) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    uint64_t *rec = rec_all + (uint64_t)j * n;
    if constexpr (!WIDE) {
        // the stream bases go through an empty asm so the compiler keeps them in registers
        // (it otherwise recomputed prevd_all + j*n from the constant bank on every chain step)
        const uint8_t *inj = in + (uint64_t)j * in_stride;
        const uint16_t *pvj = prevd_all + (uint64_t)j * n;
        asm volatile("" : "+l"(inj), "+l"(pvj));
        const InWords words{inj};
        const PrevD32 prev{pvj};
        const uint32_t p0 = blockIdx.x * chunk, p1 = (uint32_t)min((uint64_t)p0 + chunk, n);
        for (uint32_t p = p0 + threadIdx.x; p < p1; p += BLOCK) rec[p] = match_search32(p, (uint32_t)n, words, prev);
    } else {
        const InBytes bytes{in + (uint64_t)j * in_stride};
        const PrevD prev{prevd_all + (uint64_t)j * n};
        const uint64_t p0 = (uint64_t)blockIdx.x * chunk, p1 = min(p0 + chunk, n);
        for (uint64_t p = p0 + threadIdx.x; p < p1; p += BLOCK) rec[p] = match_search((int64_t)p, (int64_t)n, bytes, prev);
    }
}

// ---------------------------------------------------------------- 4. anchors
// p is an anchor iff no match found at q < p reaches past p: max_{q<p}(q+max(L128,1)) <= p.
// One CTA scans a 2048-position tile (plus the 258-position reach-in) and reports the
// first anchor of each of its CH-sized chunks.
constexpr int TILE = 2048;
__global__ void __launch_bounds__(256) k_anchor(uint64_t n, const StreamMeta *meta, const uint64_t *rec_all,
                                               uint64_t nchunks, uint64_t *first_anchor) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t c0 = (uint64_t)blockIdx.x * TILE;
    if (c0 >= n) return;
    const uint64_t *rec = rec_all + (uint64_t)j * n;
    const uint64_t c1 = min(n, c0 + TILE);
    const uint64_t r0 = c0 >= MAX_MATCH ? c0 - MAX_MATCH : 0;
    const uint64_t len = c1 - r0;
    const uint64_t per = (len + blockDim.x - 1) / blockDim.x;
    const uint64_t s0 = r0 + threadIdx.x * per, s1 = min(c1, s0 + per);
    __shared__ uint64_t scan[256];
    __shared__ unsigned long long best[TILE / CH];
    __shared__ unsigned full[TILE / CH];
    if (threadIdx.x < TILE / CH) {
        best[threadIdx.x] = ~0ull;
        full[threadIdx.x] = 1u;
    }
    __syncthreads();
    uint64_t mx = 0;
    for (uint64_t q = s0; q < s1; ++q) {
        const uint32_t l = mrec_l128(rec[q]);
        const uint64_t r = q + (l ? l : 1);
        mx = r > mx ? r : mx;
        if (q >= c0 && l != MAX_MATCH) full[(q - c0) / CH] = 0u;
    }
    scan[threadIdx.x] = mx;
    __syncthreads();
    for (unsigned o = 1; o < blockDim.x; o <<= 1) {  // inclusive max-scan
        const uint64_t v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        if (v > scan[threadIdx.x]) scan[threadIdx.x] = v;
        __syncthreads();
    }
    uint64_t run = threadIdx.x ? scan[threadIdx.x - 1] : 0;
    int last = -1;
    for (uint64_t q = s0; q < s1; ++q) {
        if (q >= c0 && run <= q) {
            const int ch = (int)((q - c0) / CH);
            if (ch != last) {
                atomicMin(&best[ch], (unsigned long long)q);
                last = ch;
            }
        }
        const uint32_t l = mrec_l128(rec[q]);
        const uint64_t r = q + (l ? l : 1);
        run = r > run ? r : run;
    }
    __syncthreads();
    const uint64_t k = c0 / CH + threadIdx.x;
    if (threadIdx.x < TILE / CH && k < nchunks)
        first_anchor[(uint64_t)j * nchunks + k] =
            (best[threadIdx.x] == ~0ull ? (~0ull >> 2) : best[threadIdx.x]) |  // "none" stays huge, bit 63 clear
            ((uint64_t)(full[threadIdx.x] && k * CH + CH <= n) << 63);
}

// chunk boundaries: bnd[k] = first anchor >= k*CH (suffix-min over chunks)
// bnd[k] = first anchor >= k*CH (suffix min of the per-chunk first anchors), and
// nbreak[k] = first chunk >= k that is not entirely 258-byte matches (bit 63 of the
// record).  Three phases like the resolve: per-segment minima, one warp per stream
// scanning the segments, per-segment expansion.
__device__ __forceinline__ void bound_item(uint64_t raw, uint64_t k, uint64_t &v, uint32_t &nb) {
    v = raw & ~(1ull << 63);
    nb = !(raw >> 63) ? (uint32_t)k : 0xffffffffu;
}

__global__ void __launch_bounds__(256) k_bounds_seg(const StreamMeta *meta, uint64_t nchunks, uint64_t nseg,
                                                   const uint64_t *first_anchor, uint64_t *segv_all,
                                                   uint32_t *segnb_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nseg) return;
    const uint64_t *fa = first_anchor + (uint64_t)j * nchunks;
    uint64_t v = ~0ull;
    uint32_t nb = 0xffffffffu;
    for (uint64_t k = g * SEG; k < min(nchunks, (g + 1) * SEG); ++k) {
        uint64_t x;
        uint32_t y;
        bound_item(fa[k], k, x, y);
        v = x < v ? x : v;
        nb = y < nb ? y : nb;
    }
    segv_all[(uint64_t)j * nseg + g] = v;
    segnb_all[(uint64_t)j * nseg + g] = nb;
}

// in place: segv[g] <- min(segv[g..], n), segnb[g] <- min(segnb[g..], nchunks)
__global__ void k_bounds_scan(uint64_t n, const StreamMeta *meta, uint64_t nchunks, uint64_t nseg, uint64_t *segv_all,
                              uint32_t *segnb_all) {
    const int j = blockIdx.x;
    if (!meta[j].active || meta[j].od) return;
    const unsigned lane = threadIdx.x;
    uint64_t *segv = segv_all + (uint64_t)j * nseg;
    uint32_t *segnb = segnb_all + (uint64_t)j * nseg;
    uint64_t carry = n;
    uint32_t carry_nb = (uint32_t)nchunks;
    for (int64_t g = (int64_t)((nseg + 31) / 32) - 1; g >= 0; --g) {
        const uint64_t k = (uint64_t)g * 32 + lane;
        uint64_t v = k < nseg ? segv[k] : ~0ull;
        uint32_t nb = k < nseg ? segnb[k] : 0xffffffffu;
        for (int o = 1; o < 32; o <<= 1) {  // suffix min
            const uint64_t w = __shfl_down_sync(0xffffffffu, v, o);
            const uint32_t x = __shfl_down_sync(0xffffffffu, nb, o);
            if (lane + o < 32 && w < v) v = w;
            if (lane + o < 32 && x < nb) nb = x;
        }
        v = v < carry ? v : carry;
        nb = nb < carry_nb ? nb : carry_nb;
        if (k < nseg) segv[k] = v, segnb[k] = nb;
        carry = __shfl_sync(0xffffffffu, v, 0);
        carry_nb = __shfl_sync(0xffffffffu, nb, 0);
    }
}

__global__ void __launch_bounds__(256) k_bounds_expand(uint64_t n, const StreamMeta *meta, uint64_t nchunks,
                                                      uint64_t nseg, const uint64_t *first_anchor,
                                                      const uint64_t *segv_all, const uint32_t *segnb_all,
                                                      uint64_t *bnd_all, uint32_t *nbreak_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g > nseg) return;
    uint64_t *bnd = bnd_all + (uint64_t)j * (nchunks + 1);
    uint32_t *nbreak = nbreak_all + (uint64_t)j * (nchunks + 1);
    if (g == nseg) {
        bnd[nchunks] = n;
        nbreak[nchunks] = (uint32_t)nchunks;
        return;
    }
    const uint64_t *fa = first_anchor + (uint64_t)j * nchunks;
    uint64_t carry = g + 1 < nseg ? segv_all[(uint64_t)j * nseg + g + 1] : n;
    uint32_t carry_nb = g + 1 < nseg ? segnb_all[(uint64_t)j * nseg + g + 1] : (uint32_t)nchunks;
    for (int64_t k = (int64_t)min(nchunks, (g + 1) * SEG) - 1; k >= (int64_t)(g * SEG); --k) {
        uint64_t v;
        uint32_t nb;
        bound_item(fa[k], (uint64_t)k, v, nb);
        carry = v < carry ? v : carry;
        carry_nb = nb < carry_nb ? nb : carry_nb;
        bnd[k] = k == 0 ? 0 : carry;
        nbreak[k] = carry_nb;
    }
}

// Inside a run of chunks whose every position has a 258-byte chain-128 match, the lazy
// parse is periodic: (a, A) holds the match found at a, (a+1, C128) emits match(258) and
// lands on (a+258, A).  Returns how many A-positions a = p + 258*i stay inside the run
// (kept clear of the last 520 bytes, where lookahead caps and tail slides apply).
__device__ __forceinline__ int64_t periodic_run(int64_t p, int tag, uint64_t n, const uint32_t *nbreak) {
    if (tag != TAG_A) return 0;
    const uint64_t kk = (uint64_t)p / CH;
    const uint32_t nb = nbreak[kk];
    if (nb <= kk) return 0;
    int64_t limit = (int64_t)nb * CH;
    if (limit > (int64_t)n - 520) limit = (int64_t)n - 520;
    if (limit <= p) return 0;
    return (limit - p + MAX_MATCH - 1) / MAX_MATCH;
}

// ------------------------------------------------------ 5. chunk transfer maps
// Every chunk is walked from each of the 4 entry tags.  (Staging the records of a few
// chunks in shared memory was measured slower than reading them through L1: the smem
// footprint capped occupancy and left 3/4 of the lanes of the emit walk idle.)
struct NoBytes {
    __device__ __forceinline__ uint32_t operator()(int64_t) const { return 0; }
};

struct RecG {
    const uint64_t *rec;
    __device__ __forceinline__ uint64_t operator()(int64_t q) const { return __ldg(rec + q); }
};

// Thread per chunk: the walks from the 4 entry tags run together, the one at the lowest
// position stepping next.  Two walks that reach the same (position, tag) state evolve
// identically from then on, so the higher-numbered one stops and keeps only its symbol
// count offset (the lowest-position-first order guarantees a shared state is seen while
// both walks sit on it; a merge missed across a periodic jump only costs time).  The
// four walks usually converge within a few steps, so a chunk costs about one walk.
__global__ void __launch_bounds__(256) k_sim(uint64_t n, const StreamMeta *meta, const uint64_t *rec_all,
                                            uint64_t nchunks, const uint64_t *bnd_all,
                                            const uint32_t *nbreak_all, uint8_t *exit4, uint32_t *cnt4) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nchunks) return;
    const RecG R{rec_all + (uint64_t)j * n};
    const uint64_t *bnd = bnd_all + (uint64_t)j * (nchunks + 1);
    const int64_t b0 = (int64_t)bnd[k], b1 = (int64_t)bnd[k + 1];
    const NoBytes bytes;
    const uint32_t *nbreak = nbreak_all + (uint64_t)j * (nchunks + 1);
    int64_t P[4];
    int T[4], A[4];  // A[t]: the walk t merged into (t while live)
    uint32_t C[4], D[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) P[t] = b0, T[t] = t, A[t] = t, C[t] = 0, D[t] = 0;
    int64_t cp = -1;  // the last record loaded (see k_emit_syms)
    uint64_t cr = 0;
    for (;;) {
        int w = -1;
        int64_t p = INT64_MAX;
        int tag = 0;
        uint32_t cw = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (A[t] == t && P[t] < b1 && P[t] < p) p = P[t], w = t, tag = T[t], cw = C[t];
        if (w < 0) break;
        int64_t np;
        int nt;
        const int64_t m = periodic_run(p, tag, n, nbreak);
        if (m > 0) {
            np = p + MAX_MATCH * m, nt = TAG_A, cw += (uint32_t)m;
        } else {
            const bool pending = tag == TAG_C128 || tag == TAG_C32;
            const uint64_t rpm1 = !pending || p == 0 ? 0ull : cp == p - 1 ? cr : R(p - 1);
            const uint64_t rp = cp == p ? cr : R(p);
            cp = p, cr = rp;
            const Step s = parse_step(p, tag, (int64_t)n, rp, rpm1, bytes);
            np = s.next_p, nt = s.next_tag, cw += s.emit != 0;
        }
        int u = -1;
        uint32_t cu = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (t == w) P[t] = np, T[t] = nt, C[t] = cw;
            else if (A[t] == t && P[t] == np && T[t] == nt) u = t, cu = C[t];
        }
        if (u >= 0) {  // merge the higher-numbered walk into the lower
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (t == u && u > w) A[t] = w, D[t] = cu - cw;
                if (t == w && w > u) A[t] = u, D[t] = cw - cu;
            }
        }
    }
    uint32_t ex[4], cf[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        ex[t] = (uint32_t)T[t], cf[t] = C[t];
#pragma unroll
        for (int v = 0; v < t; ++v)
            if (A[t] == v) ex[t] = ex[v], cf[t] = cf[v] + D[t];
    }
    const uint64_t o = ((uint64_t)j * nchunks + k) * 4;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        exit4[o + t] = (uint8_t)ex[t];
        cnt4[o + t] = cf[t];
    }
}

// ---------------------------------------------------------------- 6. resolve
// Two levels: threads compose the transfer maps (exit tag + symbol count per entry tag)
// of SEG consecutive chunks, one warp per stream scans the segments (k_resolve), and
// threads expand the segment entries back to per-chunk entry tags and symbol offsets.
__global__ void __launch_bounds__(256) k_seg_compose(const StreamMeta *meta, uint64_t nchunks, uint64_t nseg,
                                                    const uint8_t *exit4_all, const uint32_t *cnt4_all,
                                                    uint8_t *seg_exit4_all, uint32_t *seg_cnt4_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nseg) return;
    const uint8_t *ex = exit4_all + (uint64_t)j * nchunks * 4;
    const uint32_t *cn = cnt4_all + (uint64_t)j * nchunks * 4;
    const uint64_t k1 = min(nchunks, (g + 1) * SEG);
    uint32_t tg[4] = {0, 1, 2, 3}, c[4] = {0, 0, 0, 0};
    for (uint64_t k = g * SEG; k < k1; ++k) {
        const uint32_t e = *reinterpret_cast<const uint32_t *>(ex + k * 4);
        const uint4 cc = *reinterpret_cast<const uint4 *>(cn + k * 4);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t x = tg[t];
            c[t] += x == 0 ? cc.x : x == 1 ? cc.y : x == 2 ? cc.z : cc.w;
            tg[t] = (e >> (8 * x)) & 0xff;
        }
    }
    const uint64_t o = ((uint64_t)j * nseg + g) * 4;
#pragma unroll
    for (int t = 0; t < 4; ++t) seg_exit4_all[o + t] = (uint8_t)tg[t], seg_cnt4_all[o + t] = c[t];
}

__global__ void __launch_bounds__(256) k_seg_expand(const StreamMeta *meta, uint64_t nchunks, uint64_t nseg,
                                                   const uint8_t *exit4_all, const uint32_t *cnt4_all,
                                                   const uint8_t *seg_entry_all, const uint64_t *seg_symoff_all,
                                                   uint8_t *entry_all, uint64_t *symoff_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g > nseg) return;
    uint8_t *entry = entry_all + (uint64_t)j * (nchunks + 1);
    if (g == nseg) {
        entry[nchunks] = seg_entry_all[(uint64_t)j * (nseg + 1) + nseg];
        return;
    }
    const uint8_t *ex = exit4_all + (uint64_t)j * nchunks * 4;
    const uint32_t *cn = cnt4_all + (uint64_t)j * nchunks * 4;
    uint64_t *symoff = symoff_all + (uint64_t)j * nchunks;
    uint32_t tag = seg_entry_all[(uint64_t)j * (nseg + 1) + g];
    uint64_t sym = seg_symoff_all[(uint64_t)j * nseg + g];
    const uint64_t k1 = min(nchunks, (g + 1) * SEG);
    for (uint64_t k = g * SEG; k < k1; ++k) {
        entry[k] = (uint8_t)tag;
        symoff[k] = sym;
        sym += cn[k * 4 + tag];
        tag = ex[k * 4 + tag];
    }
}


__device__ __forceinline__ uint32_t map_apply(uint32_t m, int t) { return (m >> (2 * t)) & 3u; }
__device__ __forceinline__ uint32_t map_then(uint32_t f, uint32_t g) {  // g(f(t))
    uint32_t r = 0;
    for (int t = 0; t < 4; ++t) r |= map_apply(g, (int)map_apply(f, t)) << (2 * t);
    return r;
}

// warp scan of the items' 4->4 maps (items = segments here; `nchunks` counts items)
__global__ void k_resolve(const uint8_t *in, uint64_t in_stride, uint64_t n, StreamMeta *meta, uint64_t nchunks,
                          const uint8_t *exit4_all, const uint32_t *cnt4_all, uint8_t *entry_all, uint64_t *symoff_all,
                          uint32_t *syms_all, uint64_t maxb, uint64_t *blk_start_all) {
    const int j = blockIdx.x;
    StreamMeta &m = meta[j];
    if (!m.active || m.od) return;
    const unsigned lane = threadIdx.x;
    const uint8_t *ex = exit4_all + (uint64_t)j * nchunks * 4;
    const uint32_t *cn = cnt4_all + (uint64_t)j * nchunks * 4;
    uint8_t *entry = entry_all + (uint64_t)j * (nchunks + 1);
    uint64_t *symoff = symoff_all + (uint64_t)j * nchunks;
    int carry_tag = TAG_A;
    uint64_t carry_sym = 0;
    for (uint64_t g = 0; g < nchunks; g += 32) {
        const uint64_t k = g + lane;
        uint32_t mp = 0xE4;  // identity map (0,1,2,3)
        if (k < nchunks) mp = ex[k * 4] | (ex[k * 4 + 1] << 2) | (ex[k * 4 + 2] << 4) | (ex[k * 4 + 3] << 6);
        uint32_t incl = mp;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t other = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl = map_then(other, incl);
        }
        uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0xE4;
        const int my_entry = (int)map_apply(excl, carry_tag);
        const uint64_t c = k < nchunks ? cn[k * 4 + my_entry] : 0;
        uint64_t cs = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t other = __shfl_up_sync(0xffffffffu, cs, o);
            if ((int)lane >= o) cs += other;
        }
        if (k < nchunks) {
            entry[k] = (uint8_t)my_entry;
            symoff[k] = carry_sym + cs - c;
        }
        const uint32_t last_incl = __shfl_sync(0xffffffffu, incl, 31);
        carry_tag = (int)map_apply(last_incl, carry_tag);
        carry_sym += __shfl_sync(0xffffffffu, cs, 31);
    }
    if (lane == 0) {
        entry[nchunks] = (uint8_t)carry_tag;
        m.S_loop = carry_sym;
        m.final_tag = carry_tag;
        const bool fin = carry_tag != TAG_A && n > 0;
        m.nsyms = carry_sym + (fin ? 1 : 0);
        m.nblocks = carry_sym / BLOCK_SYMS + 1;
        uint64_t *bs = blk_start_all + (uint64_t)j * maxb;
        if (fin) {
            syms_all[(uint64_t)j * (n + 1) + carry_sym] = sym_literal(in[(uint64_t)j * in_stride + n - 1]);
            if (carry_sym % BLOCK_SYMS == 0) bs[carry_sym / BLOCK_SYMS] = n - 1;
        }
        if (m.nsyms == (m.nblocks - 1) * BLOCK_SYMS) bs[m.nblocks - 1] = n;  // empty final block
    }
}

// ------------------------------------------------------------ 7. emit symbols
// thread per chunk: re-walk it from its resolved entry tag, writing the symbols
__global__ void __launch_bounds__(256) k_emit_syms(const uint8_t *in, uint64_t in_stride, uint64_t n,
                                                  const StreamMeta *meta, const uint64_t *rec_all,
                                                  uint64_t nchunks, const uint64_t *bnd_all,
                                                  const uint32_t *nbreak_all,
                                                  const uint8_t *entry_all, const uint64_t *symoff_all,
                                                  uint32_t *syms_all, uint64_t maxb, uint64_t *blk_top_all,
                                                  uint64_t *blk_start_all, RunTask *runs,
                                                  unsigned long long *nruns) {
    const int j = blockIdx.y;
    if (!meta[j].active || meta[j].od) return;
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nchunks) return;
    const RecG R{rec_all + (uint64_t)j * n};
    const uint64_t *bnd = bnd_all + (uint64_t)j * (nchunks + 1);
    const uint64_t b0 = bnd[k], b1 = bnd[k + 1];
    if (b0 >= b1) return;
    const InBytesCached bytes{in + (uint64_t)j * in_stride};
    uint32_t *syms = syms_all + (uint64_t)j * (n + 1);
    uint64_t *btop = blk_top_all + (uint64_t)j * maxb;
    uint64_t *bstart = blk_start_all + (uint64_t)j * maxb;
    int tag = entry_all[(uint64_t)j * (nchunks + 1) + k];
    uint64_t g = symoff_all[(uint64_t)j * nchunks + k];
    uint64_t g0 = g;  // first symbol of the current stretch this thread writes itself
    const uint32_t *nbreak = nbreak_all + (uint64_t)j * (nchunks + 1);
    int64_t p = (int64_t)b0;
    // the record at p-1 is only read under a pending match (tags C*), and it is then the record
    // the previous step loaded: kept in a register (the lanes of a warp walk chunks 2 KiB apart,
    // so every record load is 32 separate L1 accesses)
    int64_t cp = -1;
    uint64_t cr = 0;
    // symbols leave in 16-byte stores: four consecutive ones gathered in registers once g is a
    // multiple of 4 (every symbol of [g0, g_end) is this thread's; the lanes' symbol ranges lie
    // ~1 KiB apart, so a 4-byte store per symbol was 32 separate L1 accesses per step)
    uint32_t sb0 = 0, sb1 = 0, sb2 = 0;
    const uint64_t ao = (reinterpret_cast<uintptr_t>(syms) >> 2) & 3;  // groups by address (a stream's symbols start at any word)
    auto flush = [&](uint64_t ge) {  // the partial group before ge, if it began in this thread's stretch
        const unsigned r = (unsigned)((ge + ao) & 3);
        const uint64_t gb = ge - r;
        if (r && ge >= g0 + r) {
            syms[gb] = sb0;
            if (r > 1) syms[gb + 1] = sb1;
            if (r > 2) syms[gb + 2] = sb2;
        }
    };
    auto put = [&](uint64_t gi, uint32_t v) {
        const unsigned r = (unsigned)((gi + ao) & 3);
        if (r == 0) sb0 = v;
        else if (r == 1) sb1 = v;
        else if (r == 2) sb2 = v;
        else if (gi >= g0 + 3) {
            *reinterpret_cast<uint4 *>(syms + gi - 3) = make_uint4(sb0, sb1, sb2, v);
            return;
        } else {
            syms[gi] = v;
            return;
        }
        if (gi < g0 + r) syms[gi] = v;  // before the stretch's first whole group: stored at once
    };
    while (p < (int64_t)b1) {
        const int64_t m = periodic_run(p, tag, n, nbreak);
        if (m > 64) {  // long stretch: hand it to k_emit_runs
            const unsigned long long t = atomicAdd(nruns, 1ull);
            runs[t] = RunTask{(uint64_t)p, g, (uint64_t)m, j};
            flush(g);  // (k_emit_runs writes the stretch's symbols: a new stretch of own symbols follows)
            g += (uint64_t)m;
            g0 = g;
            p += MAX_MATCH * m;
            continue;
        }
        if (m > 0) {
            for (int64_t i = 0; i < m; ++i, ++g) {
                const int64_t a = p + MAX_MATCH * i;
                put(g, sym_match(MAX_MATCH, mrec_d128(R(a))));
                if (g % BLOCK_SYMS == 0) bstart[g / BLOCK_SYMS] = (uint64_t)a;
                if (g % BLOCK_SYMS == BLOCK_SYMS - 1) btop[g / BLOCK_SYMS] = (uint64_t)a + 1;
            }
            p += MAX_MATCH * m;
            continue;
        }
        const bool pending = tag == TAG_C128 || tag == TAG_C32;
        const uint64_t rpm1 = !pending || p == 0 ? 0ull : cp == p - 1 ? cr : R(p - 1);
        const uint64_t rp = R(p);
        cp = p, cr = rp;
        const Step s = parse_step(p, tag, (int64_t)n, rp, rpm1, bytes);
        if (s.emit) {
            put(g, s.emit == 2 ? sym_match(s.len, s.dist) : sym_literal(s.len));
            if (g % BLOCK_SYMS == 0) bstart[g / BLOCK_SYMS] = (uint64_t)p - 1;
            if (g % BLOCK_SYMS == BLOCK_SYMS - 1) btop[g / BLOCK_SYMS] = (uint64_t)p;
            ++g;
        }
        p = s.next_p;
        tag = s.next_tag;
    }
    flush(g);  // the last, partial group
}

__global__ void __launch_bounds__(256) k_emit_runs(uint64_t n, const uint64_t *rec_all, uint32_t *syms_all,
                                                  uint64_t maxb, uint64_t *blk_top_all, uint64_t *blk_start_all,
                                                  const RunTask *runs, const unsigned long long *nruns) {
    const uint64_t nt = *nruns;
    for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const RunTask r = runs[t];
        const uint64_t *rec = rec_all + (uint64_t)r.j * n;
        uint32_t *syms = syms_all + (uint64_t)r.j * (n + 1);
        uint64_t *btop = blk_top_all + (uint64_t)r.j * maxb;
        uint64_t *bstart = blk_start_all + (uint64_t)r.j * maxb;
        for (uint64_t i = threadIdx.x; i < r.m; i += blockDim.x) {
            const uint64_t a = r.a0 + MAX_MATCH * i, g = r.g0 + i;
            syms[g] = sym_match(MAX_MATCH, mrec_d128(rec[a]));
            if (g % BLOCK_SYMS == 0) bstart[g / BLOCK_SYMS] = a;
            if (g % BLOCK_SYMS == BLOCK_SYMS - 1) btop[g / BLOCK_SYMS] = a + 1;
        }
    }
}


// ------------------------------------------------------- on-demand parse (n < 2^31)
// deflate_core.cuh's Walker: the lazy parse searches longest_match only at the loop tops it
// visits, with the one chain limit it needs.  (1) k_od_walk: a thread per chunk walks the parse
// from (chunk start, A), stamping every visited state in od_vis and buffering its symbols;
// (2) k_od_sync: a thread per chunk continues its walk past the chunk end until it reaches a
// state the walk of the chunk it is in also visited -- from there both agree; (3) k_od_chain:
// a warp per stream follows the joins from chunk 0 (the true start), giving each adopted chunk
// its output offsets; (4) k_od_place: a warp per adopted chunk copies its symbols from the join
// point and re-walks its continuation.  Pinned to zlib by tests/native/zmodel.cpp
// (zmodel_compress_od, the same functions run sequentially).
__global__ void __launch_bounds__(128) k_od_walk(const uint8_t *in, uint64_t in_stride, uint32_t n,
                                                const StreamMeta *meta, const uint16_t *prevd_all, uint32_t C,
                                                uint32_t nch, uint16_t *vis_all, uint32_t *ssym_all,
                                                uint16_t *spos_all, OdChunk *chunks_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nch) return;
    const uint8_t *inj = in + (uint64_t)j * in_stride;
    const uint16_t *pvj = prevd_all + (uint64_t)j * n;
    asm volatile("" : "+l"(inj), "+l"(pvj));
    const InWords words{inj};
    const PrevD32 prev{pvj};
    uint16_t *vis = vis_all + (uint64_t)j * n;
    uint32_t *ssym = ssym_all + (uint64_t)j * n;
    uint16_t *spos = spos_all + (uint64_t)j * n;
    const uint32_t b0 = k * C, b1 = min(n, b0 + C);
    Walker w{b0, TAG_A, 0, 0};
    uint32_t cnt = 0;
    while (w.p < b1) {
        const uint32_t p = w.p;
        vis[p] = vis_pack(w.tag, cnt);
        const uint32_t sym = walker_step(w, n, words, prev);
        if (sym != NOSYM) {
            ssym[b0 + cnt] = sym;
            spos[b0 + cnt] = (uint16_t)(p - b0);
            ++cnt;
        }
    }
    OdChunk &c = chunks_all[(uint64_t)j * nch + k];
    c.nsym = cnt;
    c.ex_p = w.p, c.ex_tag = w.tag, c.ex_pl = w.pl, c.ex_pd = w.pd;
}

// block bookkeeping of output symbol g emitted at loop top `top`: 32-bit index arithmetic (streams
// on the on-demand path are < 2^31 bytes, so symbol indices are too)
__device__ __forceinline__ void blk_mark(uint64_t g, uint64_t top, uint64_t *bstart, uint64_t *btop) {
    const uint32_t g32 = (uint32_t)g, q = g32 / (uint32_t)BLOCK_SYMS, r = g32 - q * (uint32_t)BLOCK_SYMS;
    if (r == 0) bstart[q] = top - 1;
    if (r == (uint32_t)BLOCK_SYMS - 1) btop[q] = top;
}

// Byte runs: first position y in each 64-byte group with in[y] != in[y-1] (or ~0), then the suffix
// minimum over groups, so next_change(x) -- the end of the run containing x-1 -- costs one group
// scan and one load.
__global__ void __launch_bounds__(256) k_od_chg(const uint8_t *in, uint64_t in_stride, uint32_t n, const StreamMeta *meta,
                                               uint64_t ng, uint32_t *chg_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const uint8_t *p = in + (uint64_t)j * in_stride;
    const uint32_t a = (uint32_t)g * 64, e = min(n, a + 64);
    uint32_t first = 0xffffffffu;
    for (uint32_t y = a < 1 ? 1 : a; y < e; ++y)
        if (__ldg(p + y) != __ldg(p + y - 1)) {
            first = y;
            break;
        }
    chg_all[(uint64_t)j * (ng + 1) + g] = first;
}

__global__ void __launch_bounds__(1024) k_od_chg_suffix(uint32_t n, const StreamMeta *meta, uint64_t ng,
                                                       uint32_t *chg_all) {
    const int j = blockIdx.x;
    if (!meta[j].active || !meta[j].od) return;
    uint32_t *chg = chg_all + (uint64_t)j * (ng + 1);
    __shared__ uint32_t wmin[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = n, chg[ng] = n;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t0 = ((int64_t)ng - 1) / 1024 * 1024; t0 >= 0; t0 -= 1024) {
        const uint64_t g = (uint64_t)t0 + threadIdx.x;
        uint32_t v = g < ng ? chg[g] : 0xffffffffu;
        for (int o = 1; o < 32; o <<= 1) {  // suffix min inside the warp
            const uint32_t x = __shfl_down_sync(0xffffffffu, v, o);
            if (lane + o < 32) v = min(v, x);
        }
        if (lane == 0) wmin[warp] = v;
        __syncthreads();
        uint32_t after = carry;  // minimum over later warps of this tile and later tiles
        for (unsigned w2 = warp + 1; w2 < 32; ++w2) after = min(after, wmin[w2]);
        v = min(v, after);
        if (g < ng) chg[g] = min(v, n);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t m = carry;
            for (int w2 = 0; w2 < 32; ++w2) m = min(m, wmin[w2]);
            carry = m;
        }
        __syncthreads();
    }
}

// first y >= x with in[y] != in[y-1] (n if none)
__device__ __forceinline__ uint32_t next_change(const uint8_t *p, uint32_t n, const uint32_t *chg, uint32_t x) {
    if (x >= n) return n;
    const uint32_t g = x / 64, e = min(n, g * 64 + 64);
    for (uint32_t y = x < 1 ? 1 : x; y < e; ++y)
        if (__ldg(p + y) != __ldg(p + y - 1)) return y;
    return chg[g + 1];
}

// The continuation of a chunk walk: from its exit state until a state the walk of the chunk it
// is in visited (or the stream end).  Inside a byte run the parse is periodic: at (p, A) with
// in[p-1] == in[p] and R bytes of the run left from p, the search finds (258, 1) and the next
// state emits match(258, 1) and lands on (p + 258, A) -- floor(R / 258) such cycles are taken at
// once (no sync check at the skipped states: a later join is still exact, only later).  EMIT
// places the symbols (with the block bookkeeping); a warp (LANES = 32) walks redundantly and
// writes the symbols of a jump in parallel.
template <bool EMIT, int LANES>
__device__ uint64_t od_follow(Walker w, uint32_t n, uint32_t C, uint32_t nch, const InWords &words, const PrevD32 &prev,
                              const uint16_t *vis, const uint32_t *chg, uint32_t &nxt, uint32_t &idx, uint32_t *syms,
                              uint64_t g, uint64_t *btop, uint64_t *bstart, uint64_t *cbuf = nullptr,
                              uint32_t *cbuf_ok = nullptr) {
    const unsigned lane = LANES == 1 ? 0u : (threadIdx.x & 31);
    uint64_t cnt = 0;
    bool buf_ok = cbuf != nullptr;
    for (;;) {
        if (w.p >= n) {
            nxt = nch;
            idx = w.tag;
            if (cbuf_ok) *cbuf_ok = buf_ok;
            return cnt;
        }
        const uint16_t v = vis[w.p];
        if (vis_match(v, w.tag)) {
            nxt = w.p / C;
            idx = vis_symidx(v);
            if (cbuf_ok) *cbuf_ok = buf_ok;
            return cnt;
        }
        const uint32_t p = w.p;
        if (w.tag == TAG_A && p >= 1 && p + 516 <= n && words.byte(p - 1) == words.byte(p) &&
            words.byte(p + 257) == words.byte(p) && words.byte(p + 515) == words.byte(p)) {
            const uint32_t R = next_change(words.p, n, chg, p + 1) - p;
            const uint32_t m = R / (uint32_t)MAX_MATCH;
            if (m >= 2) {
                if (EMIT) {
                    const uint32_t sym = sym_match(MAX_MATCH, 1);
                    for (uint32_t i = lane; i < m; i += LANES) {
                        syms[g + i] = sym;
                        blk_mark(g + i, (uint64_t)p + 1 + (uint64_t)MAX_MATCH * i, bstart, btop);
                    }
                    g += m;
                }
                buf_ok = false;
                cnt += m;
                w.p = p + (uint32_t)MAX_MATCH * m;  // tag stays A
                continue;
            }
        }
        const uint32_t sym = walker_step(w, n, words, prev);
        if (sym != NOSYM) {
            if (EMIT) {
                if (lane == 0) {
                    syms[g] = sym;
                    blk_mark(g, p, bstart, btop);
                }
                ++g;
            }
            if (buf_ok) {
                if (cnt < OD_CB) cbuf[cnt] = (uint64_t)sym | ((uint64_t)p << 32);
                else buf_ok = false;
            }
            ++cnt;
        }
    }
}

__global__ void __launch_bounds__(128) k_od_sync(const uint8_t *in, uint64_t in_stride, uint32_t n,
                                                const StreamMeta *meta, const uint16_t *prevd_all, uint32_t C,
                                                uint32_t nch, const uint16_t *vis_all, const uint32_t *chg_all,
                                                uint64_t ng, OdChunk *chunks_all, uint64_t *cbuf_all,
                                                uint4 *link_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nch) return;
    const uint8_t *inj = in + (uint64_t)j * in_stride;
    const uint16_t *pvj = prevd_all + (uint64_t)j * n;
    asm volatile("" : "+l"(inj), "+l"(pvj));
    const InWords words{inj};
    const PrevD32 prev{pvj};
    OdChunk &c = chunks_all[(uint64_t)j * nch + k];
    uint32_t nxt, idx;
    c.ncont = (uint32_t)od_follow<false, 1>(Walker{c.ex_p, c.ex_tag, c.ex_pl, c.ex_pd}, n, C, nch, words, prev,
                                            vis_all + (uint64_t)j * n, chg_all + (uint64_t)j * (ng + 1), nxt, idx,
                                            nullptr, 0, nullptr, nullptr,
                                            cbuf_all + ((uint64_t)j * nch + k) * OD_CB, &c.cbuf_ok);
    c.nxt = nxt, c.nidx = idx;
    link_all[(uint64_t)j * nch + k] = make_uint4(nxt, idx, c.nsym, c.ncont);  // what k_od_chain reads
}

// The true parse as a path through the chunks: chunk 0, then the chunk its continuation joins
// (nxt), and so on; an adopted chunk a contributes its own symbols from its join index (nidx of
// its predecessor) plus its continuation's.  Resolved in three steps:
//   k_od_sc_jump  a CTA per superchunk of 1024 chunks: for every possible entry chunk, by
//                 pointer doubling in shared memory, the first path node past the superchunk,
//                 the last node inside it and the symbol count along the way
//   k_od_sc_walk  a thread per stream chains the superchunk entries (1024x fewer steps)
//   k_od_sc_mark  a warp per superchunk walks its part of the path (32 chunks per step when
//                 consecutive chunks join their successors) and writes each chunk's offsets
struct OdSc {            // per superchunk entry chunk: where the path through it leads
    uint32_t exit;       // first path node past the superchunk (od_nch: the stream end)
    uint32_t exit_idx;   // nidx of the last node inside (the final tag at the stream end)
    uint64_t total;      // sum over the nodes inside of nsym + ncont - (join index), entry's excluded
};

__global__ void __launch_bounds__(OD_SC) k_od_sc_jump(const StreamMeta *meta, uint32_t nch, uint32_t nsc,
                                                     const uint4 *link_all, OdSc *sc_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint32_t s0 = blockIdx.x * OD_SC, k = s0 + threadIdx.x;
    __shared__ uint32_t J[2][OD_SC], last[2][OD_SC];
    __shared__ unsigned long long W[2][OD_SC];
    const uint4 l = k < nch ? link_all[(uint64_t)j * nch + k] : make_uint4(nch, 0, 0, 0);
    const bool inside = l.x < s0 + OD_SC && l.x < nch;
    const uint32_t t = threadIdx.x;
    J[0][t] = inside ? l.x - s0 : 0xffffffffu;
    W[0][t] = (unsigned long long)l.z + l.w - (inside ? l.y : 0u);
    last[0][t] = t;
    __syncthreads();
    int c = 0;
    for (int r = 0; r < 10; ++r) {
        const uint32_t jj = J[c][t];
        if (jj != 0xffffffffu) {
            J[c ^ 1][t] = J[c][jj];
            W[c ^ 1][t] = W[c][t] + W[c][jj];
            last[c ^ 1][t] = last[c][jj];
        } else {
            J[c ^ 1][t] = jj, W[c ^ 1][t] = W[c][t], last[c ^ 1][t] = last[c][t];
        }
        __syncthreads();
        c ^= 1;
    }
    if (k < nch) {
        const uint32_t lk = s0 + last[c][t];
        const uint4 ll = link_all[(uint64_t)j * nch + lk];
        sc_all[(uint64_t)j * nsc * OD_SC + k] = OdSc{ll.x, ll.y, W[c][t]};
    }
}

// per stream: the path's entry (chunk, join index, output offset) of every superchunk it enters
__global__ void k_od_sc_walk(const uint8_t *in, uint64_t in_stride, uint32_t n, StreamMeta *meta, int S, uint32_t nch,
                             uint32_t nsc, const OdSc *sc_all, uint4 *entry_all, uint32_t *syms_all, uint64_t maxb,
                             uint64_t *blk_start_all) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    StreamMeta &m = meta[j];
    if (!m.active || !m.od) return;
    const OdSc *sc = sc_all + (uint64_t)j * nsc * OD_SC;
    uint4 *entry = entry_all + (uint64_t)j * nsc;
    uint32_t a = 0, idx = 0, s_next = 0;
    uint64_t off = 0;
    while (a < nch) {
        const uint32_t s = a / OD_SC;
        for (; s_next < s; ++s_next) entry[s_next] = make_uint4(0xffffffffu, 0, 0, 0);  // jumped over
        entry[s] = make_uint4(a, idx, (uint32_t)off, (uint32_t)(off >> 32));
        s_next = s + 1;
        const OdSc e = sc[a];
        off += e.total - idx;
        idx = e.exit_idx;
        a = e.exit;
    }
    for (; s_next < nsc; ++s_next) entry[s_next] = make_uint4(0xffffffffu, 0, 0, 0);
    const uint32_t final_tag = idx;
    m.S_loop = off;
    m.final_tag = (int)final_tag;
    const bool fin = final_tag != TAG_A && n > 0;
    m.nsyms = off + (fin ? 1 : 0);
    m.nblocks = off / BLOCK_SYMS + 1;
    uint64_t *bs = blk_start_all + (uint64_t)j * maxb;
    if (fin) {
        syms_all[(uint64_t)j * (n + 1) + off] = sym_literal(in[(uint64_t)j * in_stride + n - 1]);
        if (off % BLOCK_SYMS == 0) bs[off / BLOCK_SYMS] = n - 1;
    }
    if (m.nsyms == (m.nblocks - 1) * BLOCK_SYMS) bs[m.nblocks - 1] = n;  // empty final block
}

// a warp per superchunk: from its entry, runs of chunks joining their successors resolve 32 at a
// time by a warp scan; a join that skips chunks starts the next run
__global__ void __launch_bounds__(128) k_od_sc_mark(const StreamMeta *meta, uint32_t nch, uint32_t nsc,
                                                   const uint4 *link_all, const uint4 *entry_all, OdChunk *chunks_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint32_t s = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (s >= nsc) return;
    const unsigned lane = threadIdx.x & 31;
    OdChunk *ch = chunks_all + (uint64_t)j * nch;
    const uint4 *link = link_all + (uint64_t)j * nch;
    const uint4 en = entry_all[(uint64_t)j * nsc + s];
    const uint32_t s0 = s * OD_SC, s1 = min(nch, s0 + OD_SC);
    uint32_t a = en.x, idx = en.y;
    uint64_t off = ((uint64_t)en.w << 32) | en.z;
    if (en.x == 0xffffffffu) a = s1;  // not on the path: every chunk is jumped over
    for (uint32_t w0 = s0; w0 < s1; w0 += 32) {
        const uint32_t k = w0 + lane;
        const bool in_range = k < s1;
        const uint4 cur = in_range ? link[k] : make_uint4(nch, 0, 0, 0);
        const uint32_t nxt = cur.x, nidx = cur.y, nsym = cur.z, ncont = cur.w;
        unsigned adopted = 0;
        while (a < w0 + 32 && a < s1) {
            const unsigned la = a - w0;
            const unsigned brk = __ballot_sync(0xffffffffu, lane >= la && in_range && (nxt != k + 1 || nxt == nch));
            const unsigned lb = brk ? (unsigned)(__ffs(brk) - 1) : 31u;
            const bool run = lane >= la && lane <= lb && in_range;
            const uint32_t prev_nidx = __shfl_up_sync(0xffffffffu, nidx, 1);
            const uint32_t my_idx = lane == la ? idx : prev_nidx;
            const uint64_t contrib = run ? (uint64_t)(nsym - my_idx) + ncont : 0;
            uint64_t incl = contrib;
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += t;
            }
            if (run) {
                OdChunk &c = ch[k];
                c.adopted = 1;
                c.aidx = my_idx;
                c.aoff = off + incl - contrib;
                c.coff = c.aoff + (nsym - my_idx);
            }
            adopted |= __ballot_sync(0xffffffffu, run);
            off += __shfl_sync(0xffffffffu, incl, 31);
            idx = __shfl_sync(0xffffffffu, nidx, lb);
            a = __shfl_sync(0xffffffffu, nxt, lb);
        }
        if (in_range && !((adopted >> lane) & 1u)) ch[k].adopted = 0;
    }
}

__global__ void __launch_bounds__(128) k_od_place(const uint8_t *in, uint64_t in_stride, uint32_t n,
                                                 const StreamMeta *meta, const uint16_t *prevd_all, uint32_t C,
                                                 uint32_t nch, const uint16_t *vis_all, const uint32_t *ssym_all,
                                                 const uint16_t *spos_all, const uint32_t *chg_all, uint64_t ng,
                                                 const OdChunk *chunks_all, const uint64_t *cbuf_all,
                                                 uint32_t *syms_all, uint64_t maxb, uint64_t *blk_top_all,
                                                 uint64_t *blk_start_all) {
    const int j = blockIdx.y;
    if (!meta[j].active || !meta[j].od) return;
    const uint32_t k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const unsigned lane = threadIdx.x & 31;
    if (k >= nch) return;
    const OdChunk c = chunks_all[(uint64_t)j * nch + k];
    if (!c.adopted) return;
    uint32_t *syms = syms_all + (uint64_t)j * (n + 1);
    uint64_t *btop = blk_top_all + (uint64_t)j * maxb, *bstart = blk_start_all + (uint64_t)j * maxb;
    const uint32_t b0 = k * C;
    const uint32_t *ssym = ssym_all + (uint64_t)j * n + b0;
    const uint16_t *spos = spos_all + (uint64_t)j * n + b0;
    for (uint32_t i = c.aidx + lane; i < c.nsym; i += 32) {
        const uint64_t g = c.aoff + (i - c.aidx);
        const uint64_t p = (uint64_t)b0 + spos[i];
        syms[g] = ssym[i];
        blk_mark(g, p, bstart, btop);
    }
    if (c.ncont && c.cbuf_ok) {
        if (lane < c.ncont) {
            const uint64_t e = cbuf_all[((uint64_t)j * nch + k) * OD_CB + lane];
            syms[c.coff + lane] = (uint32_t)e;
            blk_mark(c.coff + lane, e >> 32, bstart, btop);
        }
    } else if (c.ncont) {  // the whole warp walks the continuation (a run jump's symbols go out in parallel)
        const uint8_t *inj = in + (uint64_t)j * in_stride;
        const InWords words{inj};
        const PrevD32 prev{prevd_all + (uint64_t)j * n};
        uint32_t nxt, idx;
        od_follow<true, 32>(Walker{c.ex_p, c.ex_tag, c.ex_pl, c.ex_pd}, n, C, nch, words, prev,
                            vis_all + (uint64_t)j * n, chg_all + (uint64_t)j * (ng + 1), nxt, idx, syms, c.coff, btop,
                            bstart);
    }
}

// ------------------------------------------------------------ 8. block plans
// zlib's tree construction (build_tree/gen_bitlen/gen_codes) is a sequential chain of
// dependent shared-memory operations.  A one-warp CTA per block: the warp tallies the
// block's symbols, lane 0 builds the trees with every array (scratch and the BlockTrees
// being written) in shared memory, the warp copies the result out.  Small CTAs let 32
// independent builders share an SM and hide each other's latency.  (A thread per block
// was measured slower: the builders diverge, so a warp serialises them.)
__global__ void __launch_bounds__(32) k_plan(uint64_t n, const StreamMeta *meta, const uint32_t *syms_all,
                                            uint64_t maxb, const uint64_t *blk_top_all,
                                            const uint64_t *blk_start_all, BlockTrees *trees_all) {
    const int j = blockIdx.y;
    const StreamMeta &m = meta[j];
    const uint64_t b = blockIdx.x;
    if (!m.active || b >= m.nblocks) return;
    __shared__ uint32_t lf[L_CODES], df[D_CODES];
    __shared__ TreeScratch ts;
    __shared__ BlockTrees bt;
    const unsigned lane = threadIdx.x;
    for (int i = lane; i < L_CODES; i += 32) lf[i] = 0;
    for (int i = lane; i < D_CODES; i += 32) df[i] = 0;
    __syncwarp();
    const uint32_t *syms = syms_all + (uint64_t)j * (n + 1);
    const uint64_t s0 = b * BLOCK_SYMS, s1 = min((uint64_t)m.nsyms, (uint64_t)(s0 + BLOCK_SYMS));
    // 8 symbols per lane in flight before tallying (one dependent load per iteration left the
    // warp waiting on global latency 512 times per block); a warp-uniform code (sparse planes:
    // runs of literal 0 or of 258-byte matches) is added once instead of by 32 serialised atomics
    const uint32_t cnt = (uint32_t)(s1 - s0);
    const uint32_t *sb = syms + s0;
    for (uint32_t base = 0; base < cnt; base += 32 * 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t i = base + (uint32_t)k * 32 + lane;
            v[k] = i < cnt ? __ldg(sb + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t s = v[k];
            if (__all_sync(0xffffffffu, s == __shfl_sync(0xffffffffu, s, 0))) {
                if (lane == 0 && s != 0xFFFFFFFFu) {
                    if (sym_is_match(s)) {
                        atomicAdd(&lf[length_code(sym_lc(s)) + 257], 32u);
                        atomicAdd(&df[dist_code(sym_dist1(s))], 32u);
                    } else {
                        atomicAdd(&lf[s], 32u);
                    }
                }
                continue;
            }
            if (s == 0xFFFFFFFFu) continue;
            if (sym_is_match(s)) {
                atomicAdd(&lf[length_code(sym_lc(s)) + 257], 1u);
                atomicAdd(&df[dist_code(sym_dist1(s))], 1u);
            } else {
                atomicAdd(&lf[s], 1u);
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        lf[END_BLOCK] = 1;
        const bool last = b + 1 == m.nblocks;
        const uint64_t *bstart = blk_start_all + (uint64_t)j * maxb;
        const uint64_t start = bstart[b];
        const uint64_t stop = last ? n : bstart[b + 1];
        const uint64_t pf = last ? n : blk_top_all[(uint64_t)j * maxb + b];
        const int64_t offset = 32768 * slides_before((int64_t)pf, (int64_t)n);
        plan_block(lf, df, stop - start, (int64_t)start >= offset, last, ts, bt);
    }
    __syncwarp();
    static_assert(sizeof(BlockTrees) % 8 == 0, "BlockTrees copied as 8-byte words");
    const uint64_t *src = reinterpret_cast<const uint64_t *>(&bt);
    uint64_t *dst = reinterpret_cast<uint64_t *>(trees_all + (uint64_t)j * maxb + b);
    for (int i = lane; i < (int)(sizeof(BlockTrees) / 8); i += 32) dst[i] = src[i];
}

// --------------------------------------------------------------- 9. layout
// Bit position of every block: a stored block aligns to a byte after its 3 header bits, so
// block b maps the running position x to x + 3 + body (dynamic/static) or
// ((x + 3 + 7) & ~7) + body (stored).  Maps of the forms "x + c" and "align8(x + a) + c"
// compose within the same two forms, so one warp per stream scans them 32 blocks at a time
// (a thread walking a stream's ~900 level-1 blocks took 0.58 ms on the critical path).
struct PosMap {
    uint32_t al;  // 0: x + c, 1: ((x + a + 7) & ~7) + c
    uint64_t a, c;
};
__device__ __forceinline__ PosMap posmap_then(const PosMap &f, const PosMap &g) {  // g(f(x))
    if (!g.al) return PosMap{f.al, f.a, f.c + g.c};
    if (!f.al) return PosMap{1u, f.c + g.a, g.c};
    return PosMap{1u, f.a, ((f.c + g.a + 7) & ~7ull) + g.c};
}
__device__ __forceinline__ uint64_t posmap_apply(const PosMap &f, uint64_t x) {
    return f.al ? ((x + f.a + 7) & ~7ull) + f.c : x + f.c;
}

__global__ void __launch_bounds__(32) k_layout(uint64_t n, StreamMeta *meta, int S, uint64_t maxb,
                                              const BlockTrees *trees_all, uint64_t *bitpos_all) {
    const int j = blockIdx.x;
    StreamMeta &m = meta[j];
    if (!m.active) return;
    const unsigned lane = threadIdx.x;
    const BlockTrees *tr = trees_all + (uint64_t)j * maxb;
    uint64_t *bp = bitpos_all + (uint64_t)j * maxb;
    uint64_t pos = 16;
    for (uint64_t b0 = 0; b0 < m.nblocks; b0 += 32) {
        const uint64_t b = b0 + lane;
        PosMap f{0u, 0, 0};  // identity past the last block
        if (b < m.nblocks) f = tr[b].type == 0 ? PosMap{1u, 3, tr[b].body_bits} : PosMap{0u, 0, 3 + tr[b].body_bits};
        PosMap incl = f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            PosMap t;
            t.al = __shfl_up_sync(0xffffffffu, incl.al, o);
            t.a = __shfl_up_sync(0xffffffffu, incl.a, o);
            t.c = __shfl_up_sync(0xffffffffu, incl.c, o);
            if ((int)lane >= o) incl = posmap_then(t, incl);
        }
        const uint64_t after = posmap_apply(incl, pos);  // position after block b
        const uint64_t before = __shfl_up_sync(0xffffffffu, after, 1);
        if (b < m.nblocks) bp[b] = lane == 0 ? pos : before;
        pos = __shfl_sync(0xffffffffu, after, 31);
    }
    if (lane == 0) {
        m.total_bits = pos;
        m.comp_len = (pos + 7) / 8 + 4;
    }
}

__global__ void k_zero_out(uint64_t n, const StreamMeta *meta, uint8_t *out, uint64_t out_stride) {
    const int j = blockIdx.y;
    const StreamMeta &m = meta[j];
    if (!m.active || m.comp_len >= n) return;
    uint64_t *o = reinterpret_cast<uint64_t *>(out + (uint64_t)j * out_stride);
    const uint64_t words = (m.comp_len + 15) / 8;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        o[i] = 0;
}

// -------------------------------------------------------------- 10. emission
__device__ __forceinline__ void put_bits(unsigned long long *w, uint64_t pos, uint64_t v, uint32_t nb) {
    if (nb == 0) return;
    const uint64_t word = pos >> 6;
    const uint32_t sh = (uint32_t)(pos & 63);
    atomicOr(&w[word], (unsigned long long)(v << sh));
    if (sh + nb > 64) atomicOr(&w[word + 1], (unsigned long long)(v >> (64 - sh)));
}

__global__ void __launch_bounds__(256) k_emit(const uint8_t *in, uint64_t in_stride, uint64_t n, const StreamMeta *meta,
                                             const uint32_t *syms_all, uint64_t maxb, const uint64_t *blk_start_all,
                                             const BlockTrees *trees_all, const uint64_t *bitpos_all, uint8_t *out,
                                             uint64_t out_stride) {
    const int j = blockIdx.y;
    const StreamMeta &m = meta[j];
    const uint64_t b = blockIdx.x;
    if (!m.active || m.comp_len >= n || b >= m.nblocks) return;
    unsigned long long *w = reinterpret_cast<unsigned long long *>(out + (uint64_t)j * out_stride);
    const BlockTrees &bt = trees_all[(uint64_t)j * maxb + b];
    const bool last = b + 1 == m.nblocks;
    const uint64_t start = bitpos_all[(uint64_t)j * maxb + b];
    const uint64_t *bstart = blk_start_all + (uint64_t)j * maxb;
    const uint64_t byte0 = bstart[b], byte1 = last ? n : bstart[b + 1];
    __shared__ uint64_t hdr_end;
    if (threadIdx.x == 0) {
        if (b == 0) put_bits(w, 0, 0x9c78ull, 16);
        if (last) {
            const uint64_t tb = (m.total_bits + 7) / 8;
            const uint32_t a = m.adler;
            const uint64_t v = ((uint64_t)(a >> 24) & 0xff) | (((uint64_t)(a >> 16) & 0xff) << 8) |
                               (((uint64_t)(a >> 8) & 0xff) << 16) | (((uint64_t)a & 0xff) << 24);
            put_bits(w, tb * 8, v, 32);
        }
        uint64_t pos = start;
        const uint32_t type = bt.type == 0 ? 0u : bt.type == 1 ? 1u : 2u;
        put_bits(w, pos, type * 2 + (last ? 1 : 0), 3);
        pos += 3;
        if (bt.type == 0) {
            pos = (pos + 7) & ~7ull;
            const uint64_t len = byte1 - byte0;
            put_bits(w, pos, (len & 0xffff) | ((~len & 0xffff) << 16), 32);
            pos += 32;
        } else if (bt.type == 2) {
            const int lcodes = bt.lmax + 1, dcodes = bt.dmax + 1, blcodes = bt.max_blindex + 1;
            put_bits(w, pos, (uint64_t)(lcodes - 257) | ((uint64_t)(dcodes - 1) << 5) | ((uint64_t)(blcodes - 4) << 10), 14);
            pos += 14;
            for (int r = 0; r < blcodes; ++r, pos += 3) put_bits(w, pos, bt.bllen[bl_order(r)], 3);
            auto send = [&](int sym, int extra) {
                put_bits(w, pos, bt.blcode[sym], bt.bllen[sym]);
                pos += bt.bllen[sym];
                const int xb = extra_blbits(sym);
                if (xb) {
                    put_bits(w, pos, (uint64_t)extra, (uint32_t)xb);
                    pos += (uint32_t)xb;
                }
            };
            walk_tree_lengths(bt.llen, bt.lmax, send);
            walk_tree_lengths(bt.dlen, bt.dmax, send);
        }
        hdr_end = pos;
    }
    __syncthreads();
    if (bt.type == 0) {
        const uint8_t *src = in + (uint64_t)j * in_stride + byte0;
        uint8_t *dst = out + (uint64_t)j * out_stride + hdr_end / 8;
        for (uint64_t i = threadIdx.x; i < byte1 - byte0; i += blockDim.x) dst[i] = src[i];
        return;
    }
    // symbols: per-thread contiguous slices, block exclusive scan of their bit counts
    const uint32_t *syms = syms_all + (uint64_t)j * (n + 1);
    const uint64_t s0 = b * BLOCK_SYMS, s1 = min((uint64_t)m.nsyms, (uint64_t)(s0 + BLOCK_SYMS));
    const uint64_t cnt = s1 - s0;
    const uint64_t per = (cnt + blockDim.x - 1) / blockDim.x;
    const uint64_t t0 = s0 + threadIdx.x * per, t1 = min(s1, t0 + per);
    uint64_t mybits = 0;
    for (uint64_t i = t0; i < t1; ++i) mybits += symbol_bits(syms[i], bt);
    __shared__ uint64_t scan[256];
    scan[threadIdx.x] = mybits;
    __syncthreads();
    for (unsigned o = 1; o < blockDim.x; o <<= 1) {
        const uint64_t v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    uint64_t pos = hdr_end + scan[threadIdx.x] - mybits;
    for (uint64_t i = t0; i < t1; ++i) {
        uint32_t nb;
        const uint64_t v = symbol_code(syms[i], bt, nb);
        put_bits(w, pos, v, nb);
        pos += nb;
    }
    if (threadIdx.x == blockDim.x - 1) {
        const uint64_t e = hdr_end + scan[blockDim.x - 1];
        if (bt.type == 1) put_bits(w, e, static_lcode(END_BLOCK), 7);
        else put_bits(w, e, bt.lcode[END_BLOCK], bt.llen[END_BLOCK]);
    }
}

// -------------------------------------------------------------- 11. CRC-32
__global__ void k_crc_table(uint32_t *tab) {
    const int i = threadIdx.x;
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
    tab[i] = c;
    __syncthreads();
    for (int t = 1; t < 8; ++t) {
        const uint32_t prev = tab[(t - 1) * 256 + i];
        tab[t * 256 + i] = (prev >> 8) ^ tab[prev & 0xff];
        __syncthreads();
    }
}

__device__ uint32_t crc_bytes(const uint8_t *p, uint64_t len, const uint32_t *T) {
    uint32_t c = 0xffffffffu;
    uint64_t i = 0;
    while (i < len && (((uintptr_t)(p + i)) & 7)) c = T[(c ^ p[i++]) & 0xff] ^ (c >> 8);
    for (; i + 8 <= len; i += 8) {
        const uint64_t v = *reinterpret_cast<const uint64_t *>(p + i);
        const uint32_t lo = (uint32_t)v ^ c, hi = (uint32_t)(v >> 32);
        c = T[7 * 256 + (lo & 0xff)] ^ T[6 * 256 + ((lo >> 8) & 0xff)] ^ T[5 * 256 + ((lo >> 16) & 0xff)] ^
            T[4 * 256 + (lo >> 24)] ^ T[3 * 256 + (hi & 0xff)] ^ T[2 * 256 + ((hi >> 8) & 0xff)] ^
            T[1 * 256 + ((hi >> 16) & 0xff)] ^ T[hi >> 24];
    }
    while (i < len) c = T[(c ^ p[i++]) & 0xff] ^ (c >> 8);
    return c ^ 0xffffffffu;
}

__global__ void __launch_bounds__(128) k_crc_chunks(const uint8_t *const *ptrs, const uint64_t *lens,
                                                   const uint32_t *tab_g, uint64_t ncrc, uint32_t *part) {
    __shared__ uint32_t T[8 * 256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) T[i] = tab_g[i];
    __syncthreads();
    const int j = blockIdx.y;
    const uint64_t len = lens[j];
    const uint8_t *p = ptrs[j];
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (c >= ncrc) return;
    const uint64_t a = c * CRC_CHUNK;
    if (a >= len && !(a == 0)) return;
    const uint64_t e = min(len, a + CRC_CHUNK);
    part[(uint64_t)j * ncrc + c] = a < len ? crc_bytes(p + a, e - a, T) : 0u;
}

// crc32_combine's shift (multiply by x^(8 len) mod P) is linear: table i holds it for
// len = 2^i applied to each byte lane, so a shift costs 4 lookups per set bit of len
// (one for the power-of-two lengths the combine tree mostly uses).  Built once per
// device from crc_multmodp/crc_x8n (deflate_core.cuh, pinned to zlib by the CPU tests).
constexpr int CRC_SHIFT_BITS = 40;
__device__ uint32_t g_crc_shift[CRC_SHIFT_BITS * 1024];

__global__ void k_crc_shift_tables() {
    const int i = blockIdx.x, e = threadIdx.x;  // e: byte lane (e >> 8) and value (e & 255)
    const uint32_t op = crc_x8n(1ull << i);
    g_crc_shift[i * 1024 + e] = crc_multmodp(op, (uint32_t)(e & 255) << (8 * (e >> 8)));
}

__device__ __forceinline__ uint32_t crc_shift(uint32_t c, uint64_t len) {
    for (int i = 0; len; ++i, len >>= 1) {
        if (!(len & 1)) continue;
        const uint32_t *T = g_crc_shift + i * 1024;
        c = T[c & 0xff] ^ T[256 + ((c >> 8) & 0xff)] ^ T[512 + ((c >> 16) & 0xff)] ^ T[768 + (c >> 24)];
    }
    return c;
}

void ensure_crc_shift_tables(cudaStream_t st) {
    static bool done[64] = {false};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 64 && done[dev]) return;
    k_crc_shift_tables<<<CRC_SHIFT_BITS, 1024, 0, st>>>();
    CKL();
    if (dev < 64) done[dev] = true;
}

__global__ void __launch_bounds__(1024) k_crc_combine(const uint64_t *lens, uint64_t ncrc, uint32_t *part,
                                                     uint32_t *out) {
    const int j = blockIdx.x;
    const uint64_t len = lens[j];
    const uint64_t nc = len ? (len + CRC_CHUNK - 1) / CRC_CHUNK : 0;
    uint32_t *pp = part + (uint64_t)j * ncrc;
    // pairwise tree: chunk i covers [i*CH, min(len,(i+1)*CH)); combine right into left
    for (uint64_t stride = 1; stride < nc; stride <<= 1) {
        const uint64_t pairs = (nc + 2 * stride - 1) / (2 * stride);
        for (uint64_t q = threadIdx.x; q < pairs; q += blockDim.x) {
            const uint64_t l = q * 2 * stride, r = l + stride;
            if (r < nc) {
                const uint64_t rend = min(len, (r + stride) * (uint64_t)CRC_CHUNK);
                pp[l] = crc_shift(pp[l], rend - r * (uint64_t)CRC_CHUNK) ^ pp[r];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = nc ? pp[0] : 0u;
}

// ------------------------------------------------------------- 12. finalize
__global__ void k_results(const uint8_t *in, uint64_t in_stride, uint64_t n, const StreamMeta *meta, int S,
                          uint8_t *out, uint64_t out_stride, BackendResults res) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    const StreamMeta &m = meta[j];
    const int src = m.active ? j : m.rep;  // inactive = duplicate all-zero plane
    const StreamMeta &ms = meta[src];
    const bool defl = n > 0 && ms.comp_len < n;
    res.backend[j] = defl ? 1 : 0;
    res.length[j] = defl ? ms.comp_len : n;
    res.payload[j] = defl ? out + (uint64_t)src * out_stride : in + (uint64_t)j * in_stride;
}

__global__ void k_copy_crc(const StreamMeta *meta, int S, BackendResults res) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    if (!meta[j].active && meta[j].rep >= 0 && res.backend[j] == 1) res.crc[j] = res.crc[meta[j].rep];
}

}  // namespace

size_t DeflateBatch::workspace_bytes(int S, uint64_t n) { return carve_size(S, n); }

size_t crc32_batch_workspace(int S, uint64_t max_len) {
    const uint64_t ncrc = (max_len + 64 + CRC_CHUNK - 1) / CRC_CHUNK + 1;
    return (size_t)S * ncrc * 4 + 8 * 256 * 4 + 1024;
}

void crc32_batch(const uint8_t *const *ptrs, const uint64_t *lens, int S, uint64_t max_len, uint32_t *out,
                 void *workspace, size_t, cudaStream_t st) {
    const uint64_t ncrc = (max_len + 64 + CRC_CHUNK - 1) / CRC_CHUNK + 1;
    uint32_t *tab = reinterpret_cast<uint32_t *>(workspace);
    uint32_t *part = tab + 8 * 256;
    k_crc_table<<<1, 256, 0, st>>>(tab);
    CKL();
    ensure_crc_shift_tables(st);
    k_crc_chunks<<<dim3((unsigned)((ncrc + 127) / 128), S), 128, 0, st>>>(ptrs, lens, tab, ncrc, part);
    CKL();
    k_crc_combine<<<S, 1024, 0, st>>>(lens, ncrc, part, out);
    CKL();
}

void DeflateBatch::run(const uint8_t *in, uint64_t in_stride, int S, uint64_t n, uint8_t *out, uint64_t out_stride,
                       void *workspace, BackendResults res, cudaStream_t st, cudaEvent_t after_match,
                       cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
    if ((in_stride & 15) || (reinterpret_cast<uintptr_t>(in) & 15))
        throw Error(EINVAL_, "deflate input rows must be 16-byte aligned with a 16-byte multiple stride");
    Work w = carve(workspace, S, n);
    CK(cudaMemsetAsync(w.meta, 0, sizeof(StreamMeta) * S, st));
    CK(cudaMemsetAsync(w.nruns, 0, sizeof(unsigned long long), st));
    if (n > 0) {
        {
        ProfScope ps("deflate.scan", st, (uint64_t)S * n);
        k_scan<<<dim3(grid_for(n, 256, 256), S), 256, 0, st>>>(in, in_stride, n, w.meta);
        CKL();
        }
    }
    static const int od_mode = getenv("IPCG_OD_MODE") ? atoi(getenv("IPCG_OD_MODE")) : 0;  // dev: 1 all, 2 none
    static const int od_pct = getenv("IPCG_OD_ZEROS") ? atoi(getenv("IPCG_OD_ZEROS")) : 85;  // dev: threshold
    // the on-demand parse pays off on large sparse streams; on small ones (< 64 KiB: coarse levels,
    // small fields) its serial chunk walks and continuations are latency the all-position search
    // does not have
    static const uint64_t od_min = getenv("IPCG_OD_MIN") ? strtoull(getenv("IPCG_OD_MIN"), nullptr, 10) : (1u << 16);  // dev knob; measured 1 MiB / 256 KiB / 64 KiB / 16 KiB: cfg3 compress 5.60 / 5.36 / 5.18 / 5.10 ms, cfg1 2.72 / 2.80 / 2.71 / 4.66 ms
    const int mode = n >= (1ull << 31) ? 2 : (od_mode == 0 && n < od_min) ? 2 : od_mode;
    const bool od_possible = mode != 2;  // else no stream takes the on-demand parse: skip its launches
    k_select<<<1, 32, 0, st>>>(w.meta, S, n, mode, od_pct);
    CKL();
    if (n > 0) {
        const uint64_t nblk = (n + WSIZE - 1) / WSIZE;
        const size_t smem = (size_t)PL_WARPS * 32768 * sizeof(uint16_t);
        if (first_on_device<1>())
            CK(cudaFuncSetAttribute(k_prevlinks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        {
        ProfScope ps1("deflate.prevlinks", st, (uint64_t)S * n);
        static int span_env = getenv("IPCG_PL_SPAN") ? atoi(getenv("IPCG_PL_SPAN")) : 0;
        int span = span_env;
        if (span <= 0) {
            // waves of resident warps x per-warp windows (warm-up + span, sweeps ~0.2 window)
            const uint64_t slots = (uint64_t)num_sms() * PL_WARPS, wtot = nblk * (uint64_t)S;
            double best = 1e300;
            for (int s = 1; s <= 6; ++s) {
                const double t = (double)((wtot + slots * s - 1) / (slots * s)) * (1.0 + 1.2 * s);
                if (t < best - 1e-9) best = t, span = s;
            }
        }
        // dev A/B knob: warps per head table (0: the one-warp kernel).  Measured on cfg2, deflate.prevlinks
        // per compress: 1 warp 5.34 ms, 2 warps 3.75-3.80, 3 warps 3.58, 4 warps 6.5 (the hand-offs
        // then cost more than the overlap gains); compress 27.4 -> 25.5 ms with 2
        static const int pl_pair = getenv("IPCG_PL_PAIR") ? atoi(getenv("IPCG_PL_PAIR")) : 2;
        const dim3 plg((unsigned)((nblk + span * PL_WARPS - 1) / (span * PL_WARPS)), S);
        if (pl_pair) {
            if (first_on_device<8>()) {
                CK(cudaFuncSetAttribute(k_prevlinks_pair<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                CK(cudaFuncSetAttribute(k_prevlinks_pair<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                CK(cudaFuncSetAttribute(k_prevlinks_pair<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            }
            if (pl_pair == 3) k_prevlinks_pair<3><<<plg, PL_WARPS * 96, smem, st>>>(in, in_stride, n, w.meta, w.prevd, span);
            else if (pl_pair == 4) k_prevlinks_pair<4><<<plg, PL_WARPS * 128, smem, st>>>(in, in_stride, n, w.meta, w.prevd, span);
            else k_prevlinks_pair<2><<<plg, PL_WARPS * 64, smem, st>>>(in, in_stride, n, w.meta, w.prevd, span);
        } else {
            k_prevlinks<<<plg, PL_WARPS * 32, smem, st>>>(in, in_stride, n, w.meta, w.prevd, span);
        }
        CKL();
        }
        debug_mark("P", (int)(n >> 20), st);  // (dev timeline: hash links done; tag = stream MiB)
        // sparse streams (meta.od, k_select) take the on-demand parse, the others the all-position
        // search; each kernel below skips the streams of the other path
        const bool forked = side && fork && join && od_possible;
        const cudaStream_t ost = forked ? side : st;  // the on-demand parse's stream
        if (forked) {
            CK(cudaEventRecord(fork, st));
            CK(cudaStreamWaitEvent(side, fork, 0));
        }
        if (od_possible) {
            const uint32_t nch = (uint32_t)w.od_nch;
            {
            ProfScope ps2("deflate.walk", ost, (uint64_t)S * n);
            CK(cudaMemsetAsync(w.od_vis, 0, (size_t)S * n * sizeof(uint16_t), ost));
            k_od_chg<<<dim3((unsigned)((w.od_ng + 255) / 256), S), 256, 0, ost>>>(in, in_stride, (uint32_t)n, w.meta,
                                                                             w.od_ng, w.od_chg);
            CKL();
            k_od_chg_suffix<<<S, 1024, 0, ost>>>((uint32_t)n, w.meta, w.od_ng, w.od_chg);
            CKL();
            k_od_walk<<<dim3((nch + 127) / 128, S), 128, 0, ost>>>(in, in_stride, (uint32_t)n, w.meta, w.prevd, w.od_C,
                                                                  nch, w.od_vis, w.od_ssym, w.od_spos, w.od_chunks);
            CKL();
            }
            {
            ProfScope ps3("deflate.sync", ost, (uint64_t)S * n);
            k_od_sync<<<dim3((nch + 127) / 128, S), 128, 0, ost>>>(in, in_stride, (uint32_t)n, w.meta, w.prevd, w.od_C,
                                                                  nch, w.od_vis, w.od_chg, w.od_ng, w.od_chunks,
                                                                  w.od_cbuf, w.od_link);
            CKL();
            }
            {
            ProfScope ps3c("deflate.chain", ost, (uint64_t)S * n);
            const unsigned nsc = (unsigned)w.od_nsc;
            k_od_sc_jump<<<dim3(nsc, S), OD_SC, 0, ost>>>(w.meta, nch, nsc, w.od_link, w.od_sc);
            CKL();
            k_od_sc_walk<<<(S + 31) / 32, 32, 0, ost>>>(in, in_stride, (uint32_t)n, w.meta, S, nch, nsc, w.od_sc,
                                                      w.od_entry, w.syms, w.maxb, w.blk_start);
            CKL();
            k_od_sc_mark<<<dim3((nsc + 3) / 4, S), 128, 0, ost>>>(w.meta, nch, nsc, w.od_link, w.od_entry, w.od_chunks);
            CKL();
            }
            {
            ProfScope ps3("deflate.place", ost, (uint64_t)S * n);
            k_od_place<<<dim3((nch + 3) / 4, S), 128, 0, ost>>>(in, in_stride, (uint32_t)n, w.meta, w.prevd, w.od_C, nch,
                                                               w.od_vis, w.od_ssym, w.od_spos, w.od_chg, w.od_ng,
                                                               w.od_chunks, w.od_cbuf, w.syms, w.maxb, w.blk_top,
                                                               w.blk_start);
            CKL();
            }
        }
        {
        {
            ProfScope ps2("deflate.match", st, (uint64_t)S * n);
            static const int mblock = getenv("IPCG_MATCH_BLOCK") ? atoi(getenv("IPCG_MATCH_BLOCK")) : 512;  // dev knobs (measured on cfg2, deflate.match per compress: block x chunk 1024 x 4096 / 16384 / 65536: 8.00 / 7.29 / 7.17 ms; 512: 7.21 / 7.11 / 7.45; 256: 7.94 / 8.42 / 10.15; the grid-stride loop: 7.84)
            static const uint32_t mchunk = getenv("IPCG_MATCH_CHUNK") ? (uint32_t)atoi(getenv("IPCG_MATCH_CHUNK")) : 16384u;
            // chunks of at least a tile, and enough of them for every SM on small streams
            uint32_t chunk = mchunk;
            while (chunk > (uint32_t)mblock && (n + chunk - 1) / chunk < (uint64_t)num_sms() * 2) chunk /= 2;
            const dim3 mg((unsigned)((n + chunk - 1) / chunk), S);
            if (first_on_device<7>() && !getenv("IPCG_MATCH_NOCARVE")) {  // all of the SM's L1/shared array as L1
                CK(cudaFuncSetAttribute(k_match<false, 256>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
                CK(cudaFuncSetAttribute(k_match<false, 512>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
                CK(cudaFuncSetAttribute(k_match<false, 1024>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
            }
            if (n >= (1ull << 31))
                k_match<true, 256><<<mg, 256, 0, st>>>(in, in_stride, n, w.meta, w.prevd, w.rec, chunk);
            else if (mblock == 256)
                k_match<false, 256><<<mg, 256, 0, st>>>(in, in_stride, n, w.meta, w.prevd, w.rec, chunk);
            else if (mblock == 512)
                k_match<false, 512><<<mg, 512, 0, st>>>(in, in_stride, n, w.meta, w.prevd, w.rec, chunk);
            else
                k_match<false, 1024><<<mg, 1024, 0, st>>>(in, in_stride, n, w.meta, w.prevd, w.rec, chunk);
            CKL();
            }
            if (after_match) CK(cudaEventRecord(after_match, st));
            {
            ProfScope ps3("deflate.anchor", st, (uint64_t)S * n);
            k_anchor<<<dim3((unsigned)((n + TILE - 1) / TILE), S), 256, 0, st>>>(n, w.meta, w.rec, w.nchunks, w.first_anchor);
            CKL();
            const dim3 bg((unsigned)((w.nseg + 1 + 255) / 256), S);
            k_bounds_seg<<<bg, 256, 0, st>>>(w.meta, w.nchunks, w.nseg, w.first_anchor, w.seg_symoff, w.seg_cnt4);
            CKL();
            k_bounds_scan<<<S, 32, 0, st>>>(n, w.meta, w.nchunks, w.nseg, w.seg_symoff, w.seg_cnt4);
            CKL();
            k_bounds_expand<<<bg, 256, 0, st>>>(n, w.meta, w.nchunks, w.nseg, w.first_anchor, w.seg_symoff, w.seg_cnt4,
                                                w.bnd, w.nbreak);
            CKL();
            }
            {
            ProfScope ps3("deflate.sim", st, (uint64_t)S * n);
            k_sim<<<dim3((unsigned)((w.nchunks + 255) / 256), S), 256, 0, st>>>(n, w.meta, w.rec, w.nchunks, w.bnd,
                                                                                  w.nbreak, w.exit4, w.cnt4);
            CKL();
            }
            {
            ProfScope ps3("deflate.resolve", st, (uint64_t)S * n);
            const dim3 sg((unsigned)((w.nseg + 1 + 255) / 256), S);
            k_seg_compose<<<sg, 256, 0, st>>>(w.meta, w.nchunks, w.nseg, w.exit4, w.cnt4, w.seg_exit4, w.seg_cnt4);
            CKL();
            k_resolve<<<S, 32, 0, st>>>(in, in_stride, n, w.meta, w.nseg, w.seg_exit4, w.seg_cnt4, w.seg_entry,
                                        w.seg_symoff, w.syms, w.maxb, w.blk_start);
            CKL();
            k_seg_expand<<<sg, 256, 0, st>>>(w.meta, w.nchunks, w.nseg, w.exit4, w.cnt4, w.seg_entry, w.seg_symoff,
                                             w.entry, w.symoff);
            CKL();
            }
            {
            ProfScope ps3("deflate.emit_syms", st, (uint64_t)S * n);
            k_emit_syms<<<dim3((unsigned)((w.nchunks + 255) / 256), S), 256, 0, st>>>(in, in_stride, n, w.meta, w.rec, w.nchunks, w.bnd, w.nbreak, w.entry, w.symoff, w.syms, w.maxb, w.blk_top, w.blk_start, w.runs, w.nruns);
            CKL();
            k_emit_runs<<<148 * 4, 256, 0, st>>>(n, w.rec, w.syms, w.maxb, w.blk_top, w.blk_start, w.runs, w.nruns);
            CKL();
            }
        }
        debug_mark("S", (int)(n >> 20), st);  // dense symbols done
        if (forked) {
            debug_mark("O", (int)(n >> 20), side);  // on-demand parse done
            CK(cudaEventRecord(join, side));
            CK(cudaStreamWaitEvent(st, join, 0));
        }
        {
        ProfScope ps4("deflate.blocks", st, (uint64_t)S * n);
        k_plan<<<dim3((unsigned)w.maxb, S), 32, 0, st>>>(n, w.meta, w.syms, w.maxb, w.blk_top, w.blk_start, w.trees);
        CKL();
        k_layout<<<S, 32, 0, st>>>(n, w.meta, S, w.maxb, w.trees, w.blk_bitpos);
        CKL();
        }
        debug_mark("B", (int)(n >> 20), st);  // block plans done
        {
        ProfScope ps5("deflate.emit", st, (uint64_t)S * n);
        k_zero_out<<<dim3(grid_for(n / 8 + 2, 256, 512), S), 256, 0, st>>>(n, w.meta, out, out_stride);
        CKL();
        k_emit<<<dim3((unsigned)w.maxb, S), 256, 0, st>>>(in, in_stride, n, w.meta, w.syms, w.maxb, w.blk_start, w.trees, w.blk_bitpos, out, out_stride);
        CKL();
        }
    }
    k_results<<<(S + 31) / 32, 32, 0, st>>>(in, in_stride, n, w.meta, S, out, out_stride, res);
    CKL();
    // CRC over each payload (duplicate all-zero deflate planes reuse their representative's)
    ProfScope ps6("deflate.crc", st, (uint64_t)S * n);
    k_crc_table<<<1, 256, 0, st>>>(w.crc_tab);
    CKL();
    ensure_crc_shift_tables(st);
    k_crc_chunks<<<dim3((unsigned)((w.ncrc + 127) / 128), S), 128, 0, st>>>(res.payload, res.length, w.crc_tab, w.ncrc, w.crc_part);
    CKL();
    k_crc_combine<<<S, 1024, 0, st>>>(res.length, w.ncrc, w.crc_part, res.crc);
    CKL();
    k_copy_crc<<<(S + 31) / 32, 32, 0, st>>>(w.meta, S, res);
    CKL();
}

}  // namespace ipcg
