// assemble.cu -- the archive assembled on the device at the end of compress_field
// (pipeline.hpp:158-217, archive.cpp:31-65): block offsets by a prefix sum over the levels'
// outlier and plane blocks, the index serialized in place, the 21-byte block headers
// (backend.cpp:67-73), the payload gathered from the deflate outputs, and each level's outlier
// block compacted in ordinal order from the quantization passes' outlier bitmap (an order-
// preserving stream compaction: no sort).  The host reads the finished index back once.
#include "assemble.cuh"

namespace ipcg {
namespace {

constexpr uint64_t ASM_PIECE_H = 64 << 10;  // gather piece (k_asm_gather)

__device__ __forceinline__ void put_le(uint8_t *p, uint64_t v, int nb) {
    for (int i = 0; i < nb; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

// one warp: offsets (device prefix sum over the levels' 33 blocks, coarsest first), index,
// block headers, gather descriptors
__global__ void k_asm_layout(AsmParams P, const AsmSmall *sm, uint8_t *arch, uint64_t capacity, AsmDesc *descs,
                             AsmOut *out) {
    const unsigned lane = threadIdx.x;
    const int L = P.levels, w = P.scalar == 0 ? 4 : 8;
    // block lengths in payload order: level L..1: outlier block, planes 0..31
    __shared__ uint64_t off[IPCG_MAX_LEVELS][33];
    uint64_t carry = 0;
    for (int li = L - 1; li >= 0; --li) {
        uint64_t len = 0;
        if (lane == 0) len = sm->ocount[li] * (uint64_t)(8 + w);
        else if (lane <= 32) len = 21 + sm->length[li][lane - 1];
        uint64_t incl = len;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        // lanes 0..31 cover the outlier block and planes 0..30; plane 31 by lane 31's inclusive sum
        off[li][lane] = carry + incl - len;
        const uint64_t tot31 = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) off[li][32] = carry + tot31;
        carry += tot31 + 21 + sm->length[li][31];
    }
    __syncwarp();
    const uint64_t index_bytes = 32 + 8 * (uint64_t)P.nd + 808 * (uint64_t)L, total = index_bytes + carry;
    const bool fits = total <= capacity;
    if (lane == 0) {
        out->total = total;
        out->index_bytes = index_bytes;
        out->fits = fits ? 1 : 0;
        for (int li = 0; li < L; ++li) out->outlier_dst[li] = fits ? index_bytes + off[li][0] : 0;
    }
    if (!fits) return;
    // index (archive.cpp:36-63), written by lane 0 (a few KB)
    if (lane == 0) {
        uint8_t *q = arch;
        q[0] = 'I', q[1] = 'P', q[2] = 'C', q[3] = '1';
        put_le(q + 4, 1, 2);
        q[6] = (uint8_t)P.scalar, q[7] = (uint8_t)P.interp, q[8] = (uint8_t)P.nd, q[9] = q[10] = q[11] = 0;
        q += 12;
        for (int i = 0; i < P.nd; ++i, q += 8) put_le(q, P.dims[i], 8);
        put_le(q, (uint64_t)__double_as_longlong(P.eb), 8);
        q += 8;
        q[0] = (uint8_t)L, q[1] = (uint8_t)P.lp, q[2] = (uint8_t)P.cap, q[3] = 0;
        q += 4;
        const double range = sm->rng[1] - sm->rng[0];
        put_le(q, (uint64_t)__double_as_longlong(range), 8);
        q += 8;
        for (int li = L - 1; li >= 0; --li) {
            put_le(q, P.count[li], 8), q += 8;
            for (int d = 0; d < 33; ++d, q += 8) put_le(q, (uint64_t)__double_as_longlong(sm->delta[li][d]), 8);
            put_le(q, off[li][0], 8), q += 8;
            put_le(q, sm->ocount[li] * (uint64_t)(8 + w), 8), q += 8;
            put_le(q, sm->ocount[li], 8), q += 8;
            for (int p = 0; p < 32; ++p) {
                put_le(q, off[li][1 + p], 8), q += 8;
                put_le(q, 21 + sm->length[li][p], 8), q += 8;
            }
        }
    }
    // block headers + gather descriptors, a lane per plane
    for (int li = 0; li < L; ++li) {
        const int p = (int)lane;
        uint8_t *h = arch + index_bytes + off[li][1 + p];
        h[0] = sm->backend[li][p];
        put_le(h + 1, P.count[li], 8);
        put_le(h + 9, sm->length[li][p], 8);
        put_le(h + 17, sm->crc[li][p], 4);
        descs[li * 32 + p] = AsmDesc{sm->payload[li][p], index_bytes + off[li][1 + p] + 21, sm->length[li][p]};
    }
    // piece prefix over the descriptors (level-major, plane order) for k_asm_gather
    __syncwarp();
    if (lane == 0) {
        uint64_t acc = 0;
        for (int d = 0; d < L * 32; ++d) {
            out->pieces[d] = acc;
            acc += (sm->length[d / 32][d % 32] + ASM_PIECE_H - 1) / ASM_PIECE_H;
        }
        out->pieces[L * 32] = acc;
    }
}

// payload copies: 64 KiB pieces of all descriptors numbered consecutively (piece prefix from
// k_asm_layout), one CTA per piece in a grid-stride loop; word-aligned destination stores of
// funnel-shifted source words, as k_gather does
constexpr uint64_t ASM_PIECE = ASM_PIECE_H;
__global__ void __launch_bounds__(256) k_asm_gather(const AsmDesc *descs, int nd, const AsmOut *out, uint8_t *arch) {
    if (!out->fits) return;
    const uint64_t total = out->pieces[nd];
    for (uint64_t g = blockIdx.x; g < total; g += gridDim.x) {
        int lo = 0, hi = nd - 1;  // descriptor of piece g: last d with pieces[d] <= g
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (out->pieces[mid] <= g) lo = mid;
            else hi = mid - 1;
        }
        const AsmDesc c = descs[lo];
        const uint64_t a = (g - out->pieces[lo]) * ASM_PIECE, len = min(ASM_PIECE, c.len - a);
        uint8_t *o = arch + c.dst + a;
        const uint8_t *s = c.src + a;
        const uint64_t head = min(len, (uint64_t)((4 - ((uintptr_t)o & 3)) & 3));
        if (threadIdx.x < head) o[threadIdx.x] = s[threadIdx.x];
        const uint8_t *s2 = s + head;
        uint8_t *o2 = o + head;
        const uint64_t rem = len - head, nw = rem / 4;
        const unsigned sh = (unsigned)((uintptr_t)s2 & 3) * 8;
        const uint32_t *sw = reinterpret_cast<const uint32_t *>((uintptr_t)s2 & ~uintptr_t(3));
        uint32_t *ow = reinterpret_cast<uint32_t *>(o2);
        if (sh == 0) {
            for (uint64_t k = threadIdx.x; k < nw; k += blockDim.x) ow[k] = sw[k];
        } else {
            for (uint64_t k = threadIdx.x; k < nw; k += blockDim.x) ow[k] = __funnelshift_r(sw[k], sw[k + 1], sh);
        }
        for (uint64_t k = nw * 4 + threadIdx.x; k < rem; k += blockDim.x) o2[k] = s2[k];
    }
}

// outlier compaction: per tile of 8192 flag words the number of set bits, then each tile's
// entries (u64 ordinal, T bits) written at its exclusive prefix (tile prefixes by one CTA)
constexpr int OT_WORDS = 8192;
__global__ void __launch_bounds__(256) k_out_count(const uint32_t *flags, uint64_t words, uint32_t *tile_cnt) {
    const uint64_t t = blockIdx.x;
    uint32_t c = 0;
    for (uint64_t i = t * OT_WORDS + threadIdx.x; i < min(words, (t + 1) * OT_WORDS); i += blockDim.x) c += __popc(flags[i]);
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < 8; ++i) s += ws[i];
        tile_cnt[t] = s;
    }
}

__global__ void __launch_bounds__(1024) k_out_scan(uint32_t *tile_cnt, uint64_t ntiles) {
    __shared__ uint64_t carry_s;
    __shared__ uint64_t ws[32];
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t b = 0; b < ntiles; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        const uint64_t v = i < ntiles ? tile_cnt[i] : 0;
        uint64_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        if (lane == 31) ws[warp] = incl;
        __syncthreads();
        uint64_t before = carry_s;
        for (unsigned k = 0; k < warp; ++k) before += ws[k];
        if (i < ntiles) tile_cnt[i] = (uint32_t)(before + incl - v);
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = before + incl;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_out_write(const uint32_t *flags, uint64_t words, const uint32_t *tile_off,
                                                   const uint64_t *bits, int scalar, const AsmOut *out, int li,
                                                   uint8_t *arch) {
    if (!out->fits) return;
    const uint64_t t = blockIdx.x;
    const int w = scalar == 0 ? 4 : 8, e = 8 + w;
    uint8_t *dst = arch + out->outlier_dst[li];
    __shared__ uint32_t ws[8];
    __shared__ uint32_t base_s;
    if (threadIdx.x == 0) base_s = tile_off[t];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t i0 = t * OT_WORDS; i0 < min(words, (t + 1) * OT_WORDS); i0 += blockDim.x) {
        __syncthreads();
        const uint64_t i = i0 + threadIdx.x;
        const uint32_t f = i < words ? flags[i] : 0u;
        const uint32_t c = __popc(f);
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += v;
        }
        if (lane == 31) ws[warp] = incl;
        __syncthreads();
        uint32_t pos = base_s + incl - c;
        for (unsigned k = 0; k < warp; ++k) pos += ws[k];
        uint32_t x = f;
        while (x) {
            const int b = __ffs((int)x) - 1;
            x &= x - 1;
            const uint64_t ord = i * 32 + (uint64_t)b;
            uint8_t *q = dst + (uint64_t)pos * e;
            put_le(q, ord, 8);
            put_le(q + 8, bits[ord], w);
            ++pos;
        }
        __syncthreads();
        if (threadIdx.x == 255) {
            uint32_t tot = 0;
            for (int k = 0; k < 8; ++k) tot += ws[k];
            base_s += tot;
        }
    }
}

}  // namespace

uint64_t asm_capacity(const AsmParams &P) {
    const int w = P.scalar == 0 ? 4 : 8;
    uint64_t cap = 32 + 8 * (uint64_t)P.nd + 808 * (uint64_t)P.levels;
    for (int li = 0; li < P.levels; ++li) {
        const uint64_t pb = (P.count[li] + 7) / 8;
        // outliers are rare: room for 1/64 of a level's points (the host re-assembles exactly on overflow)
        cap += 32 * (21 + pb) + std::max<uint64_t>(64, P.count[li] / 64) * (uint64_t)(8 + w);
    }
    return cap;
}

void launch_assemble(const AsmParams &P, const AsmSmall *sm, uint8_t *arch, uint64_t capacity, AsmDesc *descs,
                     AsmOut *out, const uint32_t *const *oflags, const uint64_t *const *obits, uint32_t *tile_tmp,
                     cudaStream_t st) {
    k_asm_layout<<<1, 32, 0, st>>>(P, sm, arch, capacity, descs, out);
    CKL();
    k_asm_gather<<<(unsigned)num_sms() * 8, 256, 0, st>>>(descs, P.levels * 32, out, arch);
    CKL();
    for (int li = 0; li < P.levels; ++li) {
        const uint64_t words = (P.count[li] + 31) / 32, ntiles = (words + OT_WORDS - 1) / OT_WORDS;
        k_out_count<<<(unsigned)ntiles, 256, 0, st>>>(oflags[li], words, tile_tmp);
        CKL();
        k_out_scan<<<1, 1024, 0, st>>>(tile_tmp, ntiles);
        CKL();
        k_out_write<<<(unsigned)ntiles, 256, 0, st>>>(oflags[li], words, tile_tmp, obits[li], P.scalar, out, li, arch);
        CKL();
    }
}

}  // namespace ipcg
