// numerics.cu -- sm_100a kernels for prediction, quantization, bitplanes, loss tables,
// merge and reconstruction.  See numerics.cuh for the reference citations.
#include <type_traits>

#include "numerics.cuh"

namespace ipcg {

namespace {

constexpr unsigned kBlock = 256;

// row-major unravel of a pass-box index into (flat, coordinate along the pass axis)
template <bool Small>
__device__ __forceinline__ uint64_t pass_flat(const PassDesc &p, uint64_t i, uint64_t &axis_idx) {
    uint64_t flat = p.start_flat;
    axis_idx = 0;
    if (Small) {
        uint32_t r32 = (uint32_t)i;
        for (int d = p.nd - 1; d >= 0; --d) {
            const uint32_t c = (uint32_t)p.cnt[d];
            const uint32_t q = r32 / c, r = r32 - q * c;  // (a 64-bit reciprocal multiply measured slower)
            r32 = q;
            flat += (uint64_t)r * p.step_flat[d];
            if (d == p.axis) axis_idx = r;
        }
    } else {
        for (int d = p.nd - 1; d >= 0; --d) {
            const uint64_t c = p.cnt[d];
            const uint64_t q = i / c, r = i - q * c;
            i = q;
            flat += r * p.step_flat[d];
            if (d == p.axis) axis_idx = r;
        }
    }
    return flat;
}

// Box launch (passes of up to 3 dimensions, leading dims padded with count 1): one element
// per thread, its coordinates straight from the grid (x: blockIdx.x*blockDim.x+threadIdx.x
// along the last axis, y: blockIdx.y*blockDim.y+threadIdx.y, z: blockIdx.z), so the index
// math is multiply-adds instead of the per-axis divisions of pass_flat.
__device__ __forceinline__ bool box_index(const PassDesc &p, uint64_t &i, uint64_t &flat, uint64_t &aidx) {
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y, z = blockIdx.z;
    if (x >= p.cnt[2] || y >= p.cnt[1]) return false;
    i = ((uint64_t)z * p.cnt[1] + y) * p.cnt[2] + x;
    flat = p.start_flat + (uint64_t)z * p.step_flat[0] + (uint64_t)y * p.step_flat[1] + (uint64_t)x * p.step_flat[2];
    aidx = p.axis == 0 ? z : p.axis == 1 ? y : x;
    return true;
}

// predict_point<T>, predictor.hpp:27-38 (cubic -> linear -> copy fallback)
template <class T>
__device__ __forceinline__ T predict(const T *__restrict__ st, uint64_t flat, uint64_t coord, const PassDesc &p,
                                     bool cubic) {
    const uint64_t s = p.s, stp = p.st;
    if (cubic && coord >= 3 * s && coord + 3 * s < p.extent) {
        const T a = st[flat - 3 * stp], b = st[flat - stp], c = st[flat + stp], d = st[flat + 3 * stp];
        return ((T)9 * (b + c) - (a + d)) / (T)16;
    }
    if (coord + s < p.extent) return (st[flat - stp] + st[flat + stp]) / (T)2;
    return st[flat - stp];
}

template <class T>
__device__ __forceinline__ T reconstruct_value(T pred, double eb, int64_t code) {  // quantizer.hpp:57-60
    return (T)((double)pred + 2.0 * eb * (double)code);
}

// quantize_residual, quantizer.hpp:65-81: returns true for an outlier
template <class T>
__device__ __forceinline__ bool quantize_residual(T value, T pred, double eb, int32_t &code, T &recon) {
    const double y = (double)value - (double)pred;
    if (isfinite(y)) {
        const double q = round(y / (2.0 * eb));
        if (fabs(q) <= (double)kMaxCode) {
            const int32_t q0 = (int32_t)q;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int64_t cand = c == 0 ? (int64_t)q0 : c == 1 ? (int64_t)q0 - 1 : (int64_t)q0 + 1;
                if (cand < -kMaxCode || cand > kMaxCode) continue;
                const T r = reconstruct_value(pred, eb, cand);
                if (fabs((double)value - (double)r) <= eb) {
                    code = (int32_t)cand;
                    recon = r;
                    return false;
                }
            }
        }
    }
    code = 0;
    recon = value;
    return true;
}

template <class T>
__device__ __forceinline__ uint64_t bits_of(T v) {
    if constexpr (sizeof(T) == 4) return (uint64_t)__float_as_uint(v);
    else return (uint64_t)__double_as_longlong(v);
}

// ------------------------------------------------------------------ range scan
// std::min/std::max seeded with +/-inf: NaN never wins (pipeline.hpp:151-155)
// 16-byte vector loads; comparisons in T (float -> double is exact and order-preserving,
// and NaN loses every comparison either way), widened to double for the result
template <class T>
__global__ void k_range_partial(const T *__restrict__ v, uint64_t n, double *part) {
    constexpr int V = 16 / (int)sizeof(T);
    T lo = (T)INFINITY, hi = (T)-INFINITY;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
    uint64_t done = 0;
    if ((reinterpret_cast<uintptr_t>(v) & 15) == 0) {
        const uint64_t nv = n / V;
        const uint4 *vv = reinterpret_cast<const uint4 *>(v);
        for (uint64_t k = tid; k < nv; k += nth) {
            const uint4 q = __ldg(vv + k);
            const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                lo = (e[j] < lo) ? e[j] : lo;
                hi = (hi < e[j]) ? e[j] : hi;
            }
        }
        done = nv * V;
    }
    for (uint64_t i = done + tid; i < n; i += nth) {
        const T x = v[i];
        lo = (x < lo) ? x : lo;
        hi = (hi < x) ? x : hi;
    }
    __shared__ double slo[kBlock], shi[kBlock];
    slo[threadIdx.x] = (double)lo;
    shi[threadIdx.x] = (double)hi;
    __syncthreads();
    for (unsigned s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double a = slo[threadIdx.x + s], b = shi[threadIdx.x + s];
            slo[threadIdx.x] = (a < slo[threadIdx.x]) ? a : slo[threadIdx.x];
            shi[threadIdx.x] = (shi[threadIdx.x] < b) ? b : shi[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = slo[0];
        part[2 * blockIdx.x + 1] = shi[0];
    }
}
__global__ void k_range_final(const double *part, int nparts, double *out2) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double lo = INFINITY, hi = -INFINITY;
    for (int i = 0; i < nparts; ++i) {
        lo = (part[2 * i] < lo) ? part[2 * i] : lo;
        hi = (hi < part[2 * i + 1]) ? part[2 * i + 1] : hi;
    }
    out2[0] = lo;
    out2[1] = hi;
}

// --------------------------------------------------------- predict + quantize
// One launch per (level, axis) pass: every target reads only coarser levels and
// earlier passes, so all targets of the pass are independent (grid.hpp:40-46).
template <class T, bool Small>
__device__ __forceinline__ void quant_point(const T *__restrict__ values, T *__restrict__ state, const PassDesc &p,
                                            double eb, bool cubic, uint32_t *__restrict__ nb, uint32_t &orv,
                                            OutlierSink sink, uint64_t i, uint64_t flat, uint64_t aidx);

template <class T, bool Small, bool Box>
__global__ void __launch_bounds__(kBlock) k_quant_pass(const T *__restrict__ values, T *__restrict__ state, PassDesc p,
                                                       double eb, bool cubic, uint32_t *__restrict__ nb,
                                                       uint32_t *lowor, OutlierSink sink) {
    uint32_t orv = 0;
    if constexpr (Box) {
        uint64_t i, flat, aidx;
        if (box_index(p, i, flat, aidx)) quant_point<T, Small>(values, state, p, eb, cubic, nb, orv, sink, i, flat, aidx);
    } else {
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.size; i += (uint64_t)gridDim.x * blockDim.x) {
            uint64_t aidx;
            const uint64_t flat = pass_flat<Small>(p, i, aidx);
            quant_point<T, Small>(values, state, p, eb, cubic, nb, orv, sink, i, flat, aidx);
        }
    }
    orv = __reduce_or_sync(0xffffffffu, orv);
    // the level's OR saturates after a few warps: skip the same-address atomic when it would
    // add no bit (one atomic per warp contended heavily with one element per thread)
    if (lane_id() == 0 && (orv & ~*reinterpret_cast<volatile uint32_t *>(lowor))) atomicOr(lowor, orv);
}

// predict + quantize + write-back of one pass element (pipeline.hpp:163-180)
template <class T, bool Small>
__device__ __forceinline__ void quant_point(const T *__restrict__ values, T *__restrict__ state, const PassDesc &p,
                                            double eb, bool cubic, uint32_t *__restrict__ nb, uint32_t &orv,
                                            OutlierSink sink, uint64_t i, uint64_t flat, uint64_t aidx) {
    {
        const T v = values[flat];
        T pred = (T)0;
        if (p.axis >= 0) pred = predict<T>(state, flat, p.axis_start + aidx * p.axis_step, p, cubic);
        int32_t code;
        T recon;
        const bool outl = quantize_residual<T>(v, pred, eb, code, recon);
        state[flat] = outl ? v : recon;
        const uint32_t w = to_negabinary(code);
        nb[p.ordinal_base + i] = w;
        orv |= w;
        if (outl) {
            const uint64_t o = p.ordinal_base + i;
            atomicAdd(sink.count, 1ull);
            atomicOr(&sink.flags[o >> 5], 1u << (o & 31));
            sink.bits[o] = bits_of<T>(v);
        }
    }
}

// ------------------------------------------------------- bitplanes + XOR code
// split + xor_encode (bitplane.cpp:7-22,44-49): a warp ballot turns 32 codewords
// into one 32-bit word of plane p (bit i = codeword i, i.e. byte i/8 bit i%8 when
// stored little-endian), the 2-plane XOR runs on those words, and a shared-memory
// transpose makes every plane's store a 128-byte coalesced row.
// 32x32 bit-matrix transpose across a warp: lane r holds row r (bit c = column c) on
// entry and column r (bit c = row c) on return.  Five block-swap stages.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, unsigned lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = masks[s];  // columns c with (c & j) == 0
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
    }
    return x;
}

// bitplane.cpp:7-22 split + 44-49 xor: a warp transposes its 32 codewords (lane l: codeword
// l -> lane 31-p: plane p's word, bit l = codeword l's digit), XORs each plane word with the
// two planes above it (lanes +1, +2), and the CTA writes the 32 planes x 32 words tile.
constexpr int BP_G = 4;  // 32-codeword groups per warp (loads in flight per thread)
__global__ void __launch_bounds__(1024) k_bitplanes(const uint32_t *__restrict__ nb, uint64_t count,
                                                    uint32_t *__restrict__ planes, uint64_t stride) {
    __shared__ uint32_t tile[32][32 * BP_G + 1];
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t word0 = (uint64_t)blockIdx.x * 32 * BP_G;
    uint32_t v[BP_G];
#pragma unroll
    for (int g = 0; g < BP_G; ++g) {
        const uint64_t i = (word0 + warp + 32 * g) * 32 + lane;
        v[g] = i < count ? __ldg(nb + i) : 0u;
    }
#pragma unroll
    for (int g = 0; g < BP_G; ++g) {
        const uint32_t b = warp_transpose32(v[g], lane);  // plane 31 - lane
        const uint32_t b1 = __shfl_down_sync(0xffffffffu, b, 1), b2 = __shfl_down_sync(0xffffffffu, b, 2);
        const uint32_t e = b ^ (lane < 31 ? b1 : 0u) ^ (lane < 30 ? b2 : 0u);
        tile[31 - lane][warp + 32 * g] = e;  // tile[plane][word]
    }
    __syncthreads();
    const unsigned p = threadIdx.x >> 5, w = threadIdx.x & 31;
    const uint64_t words = (count + 31) / 32;
#pragma unroll
    for (int g = 0; g < BP_G; ++g)
        if (word0 + w + 32 * g < words) planes[(uint64_t)p * stride + word0 + w + 32 * g] = tile[p][w + 32 * g];
}

}  // namespace

namespace {
// ------------------------------------------------------------ loss table
// measure_loss_table (pipeline.hpp:85-124) for one dropped-digit count d and one
// pass: replays the level on the double deviation field `dev` (zero at coarser
// levels) and folds max|v| into rawbits[d] as an order-independent atomicMax on
// the IEEE bit patterns of non-negative doubles (exact).  d beyond the highest set
// digit of the level's OR equals d = hb+1, so those launches exit immediately.
template <bool Small, bool Cubic>
__global__ void __launch_bounds__(kBlock) k_loss_pass2(const uint32_t *__restrict__ nb, double *__restrict__ dev,
                                                       PassDesc p, double unit, int d, const uint32_t *lowor,
                                                       unsigned long long *rawbits) {
    const uint32_t lo = *lowor;
    const uint32_t mask = d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u);
    if ((lo & mask) == 0) return;
    const int hb = 31 - __clz(lo);
    if (d > hb + 1) return;
    double worst = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.size; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t aidx;
        const uint64_t flat = pass_flat<Small>(p, i, aidx);
        const uint32_t w = nb[p.ordinal_base + i];
        const int64_t truncated = from_negabinary(w & ~mask);
        const double own = unit * (double)(truncated - (int64_t)from_negabinary(w));
        const double v = p.axis < 0 ? own : predict<double>(dev, flat, p.axis_start + aidx * p.axis_step, p, Cubic) + own;
        dev[flat] = v;
        const double a = fabs(v);
        worst = (worst < a) ? a : worst;  // NaN never wins, as std::max(worst, NaN)
    }
    __shared__ double red[kBlock];
    red[threadIdx.x] = worst;
    __syncthreads();
    for (unsigned s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = (red[threadIdx.x] < red[threadIdx.x + s]) ? red[threadIdx.x + s] : red[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0 && red[0] > 0.0) atomicMax(&rawbits[d], (unsigned long long)__double_as_longlong(red[0]));
}

template <bool Small>
__global__ void k_zero_pass(double *__restrict__ dev, PassDesc p) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.size; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t aidx;
        dev[pass_flat<Small>(p, i, aidx)] = 0.0;
    }
}

__global__ void k_loss_finalize(const unsigned long long *rawbits, const uint32_t *lowor, double *delta) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t lo = *lowor;
    double raw[33];
    raw[0] = 0.0;
    const int hb = lo ? 31 - __clz(lo) : -1;
    for (int d = 1; d <= 32; ++d) {
        const uint32_t mask = d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u);
        if ((lo & mask) == 0) {
            raw[d] = 0.0;
            continue;
        }
        const int src = d > hb + 1 ? hb + 1 : d;
        raw[d] = __longlong_as_double((long long)rawbits[src]);
    }
    delta[0] = 0.0;
    for (int d = 1; d <= 32; ++d) delta[d] = (delta[d - 1] < raw[d]) ? raw[d] : delta[d - 1];
}

// ------------------------------------------------------------- outlier block
// ------------------------------------------------------------------- merge
// xor_decode + merge (bitplane.cpp:24-59), and refine's digit folding with the XOR
// prefix taken from already-merged codewords (pipeline.hpp:328-339).  A CTA takes 32
// plane words x 32 planes: warp p loads plane p's 128-byte row segment (coalesced) into
// a padded smem tile, then warp w owns word w with lane p holding plane p's bits.
// Solves b_p = e_p ^ b_{p-1} ^ b_{p-2} down a codeword (plane p at bit 31-p): over GF(2)
// B = E / (1 + S + S^2) = (1 + S) E / (1 + S^3), S = shift toward the LSB, i.e. F = E ^ (E >> 1)
// followed by a stride-3 prefix XOR.
__device__ __forceinline__ uint32_t xor_decode_word(uint32_t e) {
    uint32_t g = e ^ (e >> 1);
    g ^= g >> 3;
    g ^= g >> 6;
    g ^= g >> 12;
    g ^= g >> 24;
    return g;
}

// bitplane.cpp:24-59 (xor decode + merge) for planes [k0, k1) of one level on top of the
// codewords already merged from planes [0, k0).  Each warp works alone on 32 plane words
// (1024 codewords): lane p loads plane p's 32 words with four 16-byte loads (rows are
// 16-byte aligned and padded to a multiple of 4 words), then for each word the warp
// transposes the 32x32 bit block (lane c: codeword c's plane bits), solves the XOR recurrence
// inside the codeword and stores 32 codewords coalesced.  No shared memory, no block syncs.
__global__ void __launch_bounds__(256) k_merge(const uint32_t *const *__restrict__ rows,
                                               const uint32_t *__restrict__ merged_in,
                                               uint32_t *__restrict__ merged_out, uint64_t count, int k0, int k1) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t words = (count + 31) / 32, words4 = (words + 3) & ~3ull;
    const uint32_t pre = k0 == 0 ? 0u : ~0u << (32 - k0);                    // planes < k0
    const uint32_t keep = k1 == 0 ? 0u : k1 >= 32 ? ~0u : ~0u << (32 - k1);  // planes < k1
    const uint32_t *row = ((int)lane >= k0 && (int)lane < k1) ? rows[lane] : nullptr;
    const bool with_prefix = merged_in && k0 > 0;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; w0 < words; w0 += nwarps * 32) {
        uint32_t v[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint4 q = make_uint4(0u, 0u, 0u, 0u);
            if (row && w0 + 4 * k < words4) q = __ldg(reinterpret_cast<const uint4 *>(row + w0) + k);
            v[4 * k] = q.x, v[4 * k + 1] = q.y, v[4 * k + 2] = q.z, v[4 * k + 3] = q.w;
        }
#pragma unroll
        for (int wv = 0; wv < 32; ++wv) {
            const uint64_t w = w0 + wv;
            if (w >= words) break;  // warp-uniform
            const uint64_t i = w * 32 + lane;
            uint32_t e = __brev(warp_transpose32(v[wv], lane));
            if (with_prefix && i < count) {
                const uint32_t m = merged_in[i] & pre;
                e |= (m ^ (m >> 1) ^ (m >> 2)) & pre;
            }
            if (i < count) merged_out[i] = xor_decode_word(e) & keep;
        }
    }
}

// Refinement step adding few planes (k1 - k0 <= 8) on top of merged codewords: no transpose.
// A thread takes MF_V groups of 4 consecutive codewords (16-byte loads and stores of the merged
// codes); the 4 digits of each new plane come from one plane word shared by 8 neighbouring
// threads (an L1 broadcast).  The prefix's XOR-encoded digits are OR-ed in and the recurrence
// solved per codeword.
#ifndef IPCG_MFV
#define IPCG_MFV 4
#endif
constexpr int MF_V = IPCG_MFV;
__device__ __forceinline__ uint4 merge_few4(uint4 m, const uint32_t *const *r, int np, int k0, uint64_t w,
                                            unsigned b, uint32_t pre, uint32_t keep) {
    uint32_t e[4] = {m.x & pre, m.y & pre, m.z & pre, m.w & pre};
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = (e[j] ^ (e[j] >> 1) ^ (e[j] >> 2)) & pre;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q >= np) break;
        const uint32_t nib = (__ldg(r[q] + w) >> b) & 15u;
        const int sh = 31 - (k0 + q);
#pragma unroll
        for (int j = 0; j < 4; ++j) e[j] |= ((nib >> j) & 1u) << sh;
    }
    return make_uint4(xor_decode_word(e[0]) & keep, xor_decode_word(e[1]) & keep, xor_decode_word(e[2]) & keep,
                      xor_decode_word(e[3]) & keep);
}

__global__ void __launch_bounds__(256) k_merge_few(const uint32_t *const *__restrict__ rows,
                                                   const uint32_t *__restrict__ merged_in,
                                                   uint32_t *__restrict__ merged_out, uint64_t count, int k0, int k1) {
    const uint32_t pre = k0 == 0 ? 0u : ~0u << (32 - k0);
    const uint32_t keep = k1 >= 32 ? ~0u : ~0u << (32 - k1);
    const int np = k1 - k0;
    const uint32_t *r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = q < np ? rows[k0 + q] : nullptr;
    const uint64_t g0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * MF_V;  // first 4-codeword group
    const uint64_t full = count / 4;  // whole groups
    uint4 m[MF_V];
#pragma unroll
    for (int v = 0; v < MF_V; ++v) {
        const uint64_t g = g0 + v;
        m[v] = g < full && merged_in ? __ldg(reinterpret_cast<const uint4 *>(merged_in) + g) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int v = 0; v < MF_V; ++v) {
        const uint64_t g = g0 + v;
        if (g < full) {
            reinterpret_cast<uint4 *>(merged_out)[g] = merge_few4(m[v], r, np, k0, g / 8, (unsigned)(g % 8) * 4, pre, keep);
        } else if (g == full && count % 4) {  // tail group
            uint4 t = make_uint4(0, 0, 0, 0);
            const uint64_t i0 = g * 4;
            if (merged_in) {
                t.x = merged_in[i0];
                if (i0 + 1 < count) t.y = merged_in[i0 + 1];
                if (i0 + 2 < count) t.z = merged_in[i0 + 2];
            }
            const uint4 o = merge_few4(t, r, np, k0, g / 8, (unsigned)(g % 8) * 4, pre, keep);
            merged_out[i0] = o.x;
            if (i0 + 1 < count) merged_out[i0 + 1] = o.y;
            if (i0 + 2 < count) merged_out[i0 + 2] = o.z;
        }
    }
}

// ------------------------------------------------------------- reconstruction
// apply_level (pipeline.hpp:61-78) for one pass
template <class T, bool Small, bool Box>
__global__ void __launch_bounds__(kBlock) k_recon_pass(T *__restrict__ state, PassDesc p, double eb, bool cubic,
                                                       const uint32_t *__restrict__ merged) {
    auto point = [&](uint64_t i, uint64_t flat, uint64_t aidx) {
        T pred = (T)0;
        if (p.axis >= 0) pred = predict<T>(state, flat, p.axis_start + aidx * p.axis_step, p, cubic);
        state[flat] = reconstruct_value<T>(pred, eb, (int64_t)from_negabinary(merged[p.ordinal_base + i]));
    };
    if constexpr (Box) {
        uint64_t i, flat, aidx;
        if (box_index(p, i, flat, aidx)) point(i, flat, aidx);
    } else {
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.size; i += (uint64_t)gridDim.x * blockDim.x) {
            uint64_t aidx;
            const uint64_t flat = pass_flat<Small>(p, i, aidx);
            point(i, flat, aidx);
        }
    }
}

// Level-1 passes as whole rows of the last axis: one CTA per (row, 256*V-element chunk),
// 16-byte vector loads and stores.  Targets of a level-1 pass sit at every other element of
// a row (odd x for the last-axis pass, even x for the others); the thread rewrites the
// non-target elements of its vector with the values it loaded (no other thread of the pass
// writes them: they are stencil sources or later passes' targets), so every sector is read
// and written whole instead of half-used by one-element-per-thread accesses.  The stencil
// rows of an earlier-axis pass are vector-loaded at the same x (the cubic/linear/copy choice
// is uniform per row); the last-axis pass stages its chunk plus a 4-element halo in shared
// memory.  Arithmetic is predict()/reconstruct_value() verbatim.
constexpr int kRowThreads = 256;
// blockDim = (tx, ty): tx threads cover a chunk of tx*V elements of one row, ty rows per CTA
// (rows shorter than 256*V elements would otherwise leave threads idle).  Quant: the
// compress pass (quant_point: predict + quantize + write-back + codeword + outliers);
// otherwise the reconstruction pass (apply_level).
struct RowsQuant {
    const void *values;
    uint32_t *nb;
    uint32_t *lowor;
    OutlierSink sink;
};
template <class T, bool Last, bool Quant>
__global__ void __launch_bounds__(kRowThreads) k_rows(T *__restrict__ state, PassDesc p, uint32_t X, uint32_t x0,
                                                      double eb, bool cubic, const uint32_t *__restrict__ merged,
                                                      RowsQuant qz) {
    using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    constexpr int V = 16 / (int)sizeof(T);
    const uint32_t tx = blockDim.x, CH = tx * V;
    const uint32_t bz = blockIdx.z, by = blockIdx.y * blockDim.y + threadIdx.y;
    const bool rowok = by < p.cnt[1];  // (no early return: barrier / warp reduction below)
    const uint64_t row = p.start_flat - x0 + (uint64_t)bz * p.step_flat[0] + (uint64_t)by * p.step_flat[1];
    const uint64_t obase = p.ordinal_base + ((uint64_t)bz * p.cnt[1] + by) * p.cnt[2];
    const uint32_t xb = blockIdx.x * CH, xs = xb + threadIdx.x * V;
    const bool in = rowok && xs < X;  // X % V == 0
    auto ldv = [&](const T *src, T *o) {
        const Vec v = *reinterpret_cast<const Vec *>(src);
        const T *vv = reinterpret_cast<const T *>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) o[k] = vv[k];
    };
    T e[V], val[V];
    if (in) {
        ldv(state + row + xs, e);
        if constexpr (Quant) ldv(static_cast<const T *>(qz.values) + row + xs, val);
    }
    uint32_t orv = 0;
    // the target at element k with prediction `pred`
    auto finish = [&](int k, uint32_t x, T pred) {
        const uint64_t o = obase + (x >> 1);
        if constexpr (Quant) {
            int32_t code;
            T recon;
            const bool outl = quantize_residual<T>(val[k], pred, eb, code, recon);
            e[k] = outl ? val[k] : recon;
            const uint32_t w = to_negabinary(code);
            qz.nb[o] = w;
            orv |= w;
            if (outl) {
                atomicAdd(qz.sink.count, 1ull);
                atomicOr(&qz.sink.flags[o >> 5], 1u << (o & 31));
                qz.sink.bits[o] = bits_of<T>(val[k]);
            }
        } else {
            e[k] = reconstruct_value<T>(pred, eb, (int64_t)from_negabinary(merged[o]));
        }
    };
    if constexpr (Last) {
        extern __shared__ __align__(16) unsigned char rsm[];
        T *sm = reinterpret_cast<T *>(rsm) + (size_t)threadIdx.y * (CH + 8);
        if (rowok && threadIdx.x < 8) {  // 4-element halo on each side
            const int i = threadIdx.x < 4 ? (int)threadIdx.x - 4 : (int)CH + (int)threadIdx.x - 4;
            const int64_t x = (int64_t)xb + i;
            if (x >= 0 && x < (int64_t)X) sm[i + 4] = state[row + x];
        }
        if (in) {
#pragma unroll
            for (int k = 0; k < V; ++k) sm[threadIdx.x * V + k + 4] = e[k];
        }
        __syncthreads();
        if (in) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const uint32_t x = xs + k;
                if ((x & 1u) != x0) continue;
                const T *c = sm + (x - xb) + 4;  // c[0] = element x
                T pred;
                if (cubic && x >= 3 && x + 3 < X) pred = ((T)9 * (c[-1] + c[1]) - (c[-3] + c[3])) / (T)16;
                else if (x + 1 < X) pred = (c[-1] + c[1]) / (T)2;
                else pred = c[-1];
                finish(k, x, pred);
            }
        }
    } else if (in) {
        const uint64_t coord = p.axis_start + (uint64_t)(p.axis == 0 ? bz : by) * p.axis_step;
        const uint64_t stp = p.st;
        const bool cub = cubic && coord >= 3 * p.s && coord + 3 * p.s < p.extent;
        const bool lin = coord + p.s < p.extent;
        T a[V], b[V], c[V], d[V];
        ldv(state + row + xs - stp, b);
        if (lin) ldv(state + row + xs + stp, c);
        if (cub) ldv(state + row + xs - 3 * stp, a), ldv(state + row + xs + 3 * stp, d);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const uint32_t x = xs + k;
            if ((x & 1u) != x0) continue;
            T pred;
            if (cub) pred = ((T)9 * (b[k] + c[k]) - (a[k] + d[k])) / (T)16;
            else if (lin) pred = (b[k] + c[k]) / (T)2;
            else pred = b[k];
            finish(k, x, pred);
        }
    }
    if (in) {
        Vec v;
        T *vv = reinterpret_cast<T *>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) vv[k] = e[k];
        *reinterpret_cast<Vec *>(state + row + xs) = v;
    }
    if constexpr (Quant) {
        orv = __reduce_or_sync(0xffffffffu, orv);
        if (lane_id() == 0 && (orv & ~*reinterpret_cast<volatile uint32_t *>(qz.lowor))) atomicOr(qz.lowor, orv);
    }
}

// strictly increasing prefix of in-range ordinals = what the in-order matcher applies
__global__ void k_outlier_prefix(const uint8_t *block, uint64_t entries, int scalar, uint64_t count, uint64_t *napplied) {
    __shared__ unsigned long long first_bad;
    if (threadIdx.x == 0) first_bad = entries;
    __syncthreads();
    const int e = 8 + (scalar == 0 ? 4 : 8);
    auto ord = [&](uint64_t k) {
        uint64_t o = 0;
        for (int b = 0; b < 8; ++b) o |= (uint64_t)block[k * e + b] << (8 * b);
        return o;
    };
    for (uint64_t k = threadIdx.x; k < entries; k += blockDim.x) {
        const uint64_t o = ord(k);
        const bool bad = o >= count || (k > 0 && ord(k - 1) >= o);
        if (bad) atomicMin(&first_bad, (unsigned long long)k);
    }
    __syncthreads();
    if (threadIdx.x == 0) *napplied = first_bad;
}

template <class T, bool Small>
__global__ void k_outlier_apply(T *__restrict__ state, PassDesc p, const uint8_t *__restrict__ block,
                                const uint64_t *napplied) {
    const uint64_t n = *napplied;
    const int e = 8 + (int)sizeof(T);
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t *q = block + k * e;
        uint64_t o = 0, b = 0;
        for (int j = 0; j < 8; ++j) o |= (uint64_t)q[j] << (8 * j);
        if (o < p.ordinal_base || o >= p.ordinal_base + p.size) continue;
        for (int j = 0; j < (int)sizeof(T); ++j) b |= (uint64_t)q[8 + j] << (8 * j);
        uint64_t aidx;
        const uint64_t flat = pass_flat<Small>(p, o - p.ordinal_base, aidx);
        if constexpr (sizeof(T) == 4) state[flat] = __uint_as_float((uint32_t)b);
        else state[flat] = __longlong_as_double((long long)b);
    }
}

}  // namespace

// ============================================================= host launchers

void launch_range(const void *values, int scalar, uint64_t n, double *scratch, double *out2, cudaStream_t st) {
    const unsigned g = grid_for((n + 3) / 4, kBlock, 1024);
    if (scalar == 0) k_range_partial<float><<<g, kBlock, 0, st>>>((const float *)values, n, scratch);
    else k_range_partial<double><<<g, kBlock, 0, st>>>((const double *)values, n, scratch);
    CKL();
    k_range_final<<<1, 32, 0, st>>>(scratch, (int)g, out2);
    CKL();
}

// the pass as a 3-axis box for the Box kernels (false: more than 3 axes or grid limits)
static bool pass_box(const PassDesc &pd, PassDesc &q, dim3 &grid, dim3 &block) {
    if (pd.nd > 3 || pd.size == 0) return false;
    q = pd;
    const int pad = 3 - pd.nd;
    for (int d = 2; d >= 0; --d) {
        const int sd = d - pad;
        q.cnt[d] = sd >= 0 ? pd.cnt[sd] : 1;
        q.step_flat[d] = sd >= 0 ? pd.step_flat[sd] : 0;
    }
    q.nd = 3;
    q.axis = pd.axis >= 0 ? pd.axis + pad : -1;
    if (q.cnt[2] >= (1ull << 31)) return false;
    const unsigned bx = (unsigned)std::min<uint64_t>(kBlock, (q.cnt[2] + 31) / 32 * 32);
    const unsigned by = kBlock / bx;
    const uint64_t gy = (q.cnt[1] + by - 1) / by;
    if (gy > 65535 || q.cnt[0] > 65535) return false;
    block = dim3(bx, by, 1);
    grid = dim3((unsigned)((q.cnt[2] + bx - 1) / bx), (unsigned)gy, (unsigned)q.cnt[0]);
    return true;
}

template <bool Quant>
static void launch_rows(void *state, int scalar, const PassDesc &q, uint32_t X, uint32_t x0, double eb, bool cubic,
                        const uint32_t *merged, RowsQuant qz, cudaStream_t st) {
    const int w = scalar == 0 ? 4 : 8, V = 16 / w;
    const unsigned tx = (unsigned)std::min<uint64_t>(kRowThreads, ((uint64_t)X / V + 31) / 32 * 32);
    const unsigned ty = kRowThreads / tx;
    const dim3 blk(tx, ty, 1);
    const dim3 g((X + tx * V - 1) / (tx * V), (unsigned)((q.cnt[1] + ty - 1) / ty), (unsigned)q.cnt[0]);
    const size_t smem = q.axis == 2 ? (size_t)ty * (tx * V + 8) * w : 0;
    if (scalar == 0) {
        if (q.axis == 2) k_rows<float, true, Quant><<<g, blk, smem, st>>>((float *)state, q, X, x0, eb, cubic, merged, qz);
        else k_rows<float, false, Quant><<<g, blk, 0, st>>>((float *)state, q, X, x0, eb, cubic, merged, qz);
    } else {
        if (q.axis == 2) k_rows<double, true, Quant><<<g, blk, smem, st>>>((double *)state, q, X, x0, eb, cubic, merged, qz);
        else k_rows<double, false, Quant><<<g, blk, 0, st>>>((double *)state, q, X, x0, eb, cubic, merged, qz);
    }
    CKL();
}

// a level-1 pass whose targets are every other element of whole rows of the last axis
static bool rows_applicable(const PassDesc &q, uint64_t X, int w, const void *state, uint32_t &x0) {
    if (q.s != 1 || q.axis < 0 || X < 2 || X % (16 / w) != 0 || (reinterpret_cast<uintptr_t>(state) & 15)) return false;
    if (q.step_flat[2] != 2 || q.cnt[1] > 65535 || q.cnt[0] > 65535 || X >= (1u << 31)) return false;
    x0 = (uint32_t)(q.start_flat % X);
    if (x0 > 1 || q.cnt[2] != (X - x0 + 1) / 2) return false;
    if (q.axis == 2) return x0 == 1 && q.st == 1;
    return x0 == 0 && q.st % (16 / w) == 0;  // stencil rows stay 16-byte aligned
}

void launch_quant_pass(const void *values, void *state, int scalar, bool cubic, const PassDesc &pd, double eb,
                       uint32_t *nb, uint32_t *lowor, OutlierSink sink, uint64_t row_len, cudaStream_t st) {
    PassDesc q;
    dim3 grid, block;
    uint32_t x0 = 0;
    if (pass_box(pd, q, grid, block) && (reinterpret_cast<uintptr_t>(values) & 15) == 0 &&
        rows_applicable(q, row_len, scalar == 0 ? 4 : 8, state, x0)) {
        launch_rows<true>(state, scalar, q, (uint32_t)row_len, x0, eb, cubic, nullptr, RowsQuant{values, nb, lowor, sink}, st);
        return;
    }
    if (pass_box(pd, q, grid, block)) {
        if (scalar == 0)
            k_quant_pass<float, true, true><<<grid, block, 0, st>>>((const float *)values, (float *)state, q, eb, cubic, nb, lowor, sink);
        else
            k_quant_pass<double, true, true><<<grid, block, 0, st>>>((const double *)values, (double *)state, q, eb, cubic, nb, lowor, sink);
        CKL();
        return;
    }
    const unsigned g = grid_for(pd.size, kBlock);
    const bool small = pd.size < (uint64_t(1) << 32);
    if (scalar == 0) {
        if (small) k_quant_pass<float, true, false><<<g, kBlock, 0, st>>>((const float *)values, (float *)state, pd, eb, cubic, nb, lowor, sink);
        else k_quant_pass<float, false, false><<<g, kBlock, 0, st>>>((const float *)values, (float *)state, pd, eb, cubic, nb, lowor, sink);
    } else {
        if (small) k_quant_pass<double, true, false><<<g, kBlock, 0, st>>>((const double *)values, (double *)state, pd, eb, cubic, nb, lowor, sink);
        else k_quant_pass<double, false, false><<<g, kBlock, 0, st>>>((const double *)values, (double *)state, pd, eb, cubic, nb, lowor, sink);
    }
    CKL();
}

void launch_bitplanes(const uint32_t *nb, uint64_t count, uint32_t *planes, uint64_t stride, cudaStream_t st) {
    const uint64_t words = (count + 31) / 32;
    if (words == 0) return;
    const uint64_t blocks = (words + 32 * BP_G - 1) / (32 * BP_G);
    k_bitplanes<<<(unsigned)blocks, 1024, 0, st>>>(nb, count, planes, stride);
    CKL();
}

void launch_loss_pass(const uint32_t *nb, double *dev, const PassDesc &pd, bool cubic, double u, int d,
                      const uint32_t *lowor, unsigned long long *rawbits, cudaStream_t st) {
    const unsigned g = grid_for(pd.size, kBlock);
    const bool small = pd.size < (uint64_t(1) << 32);
    if (small) {
        if (cubic) k_loss_pass2<true, true><<<g, kBlock, 0, st>>>(nb, dev, pd, u, d, lowor, rawbits);
        else k_loss_pass2<true, false><<<g, kBlock, 0, st>>>(nb, dev, pd, u, d, lowor, rawbits);
    } else {
        if (cubic) k_loss_pass2<false, true><<<g, kBlock, 0, st>>>(nb, dev, pd, u, d, lowor, rawbits);
        else k_loss_pass2<false, false><<<g, kBlock, 0, st>>>(nb, dev, pd, u, d, lowor, rawbits);
    }
    CKL();
}

void launch_zero_pass(double *dev, const PassDesc &pd, cudaStream_t st) {
    const unsigned g = grid_for(pd.size, kBlock);
    if (pd.size < (uint64_t(1) << 32)) k_zero_pass<true><<<g, kBlock, 0, st>>>(dev, pd);
    else k_zero_pass<false><<<g, kBlock, 0, st>>>(dev, pd);
    CKL();
}

void launch_loss_finalize(const unsigned long long *rawbits, const uint32_t *lowor, double *delta, cudaStream_t st) {
    k_loss_finalize<<<1, 32, 0, st>>>(rawbits, lowor, delta);
    CKL();
}

void launch_merge(const uint32_t *const *rows, const uint32_t *merged_in, uint32_t *merged_out, uint64_t count, int k0,
                  int k1, cudaStream_t st) {
    const uint64_t words = (count + 31) / 32;
    if (words == 0) return;
    // few planes -- a refinement step on merged codewords, or a fresh merge of a coarse plan (k0 = 0,
    // no prefix to read) -- skip the 32 x 32 bit transpose
    if (k1 - k0 <= 8 && ((merged_in && k0 > 0) || (!merged_in && k0 == 0))) {
        const uint64_t groups = count / 4 + 1;  // + the tail group
        const unsigned g = (unsigned)((groups + 256 * MF_V - 1) / (256 * MF_V));
        k_merge_few<<<g, 256, 0, st>>>(rows, merged_in, merged_out, count, k0, k1);
    } else {
        // a warp per 32 plane words, no grid-stride loop: the scheduler keeps replacing finished
        // warps, so loads stay in flight (a capped grid serialised load -> transpose -> store per warp)
        const unsigned g = (unsigned)(((words + 31) / 32 + 7) / 8);
        k_merge<<<g, 256, 0, st>>>(rows, merged_in, merged_out, count, k0, k1);
    }
    CKL();
}

void launch_recon_pass(void *state, int scalar, bool cubic, const PassDesc &pd, double eb, const uint32_t *merged,
                       uint64_t row_len, cudaStream_t st) {
    PassDesc q;
    dim3 grid, block;
    uint32_t x0 = 0;
    if (pass_box(pd, q, grid, block) && rows_applicable(q, row_len, scalar == 0 ? 4 : 8, state, x0)) {
        launch_rows<false>(state, scalar, q, (uint32_t)row_len, x0, eb, cubic, merged, RowsQuant{}, st);
        return;
    }
    if (pass_box(pd, q, grid, block)) {
        if (scalar == 0) k_recon_pass<float, true, true><<<grid, block, 0, st>>>((float *)state, q, eb, cubic, merged);
        else k_recon_pass<double, true, true><<<grid, block, 0, st>>>((double *)state, q, eb, cubic, merged);
        CKL();
        return;
    }
    const unsigned g = grid_for(pd.size, kBlock);
    const bool small = pd.size < (uint64_t(1) << 32);
    if (scalar == 0) {
        if (small) k_recon_pass<float, true, false><<<g, kBlock, 0, st>>>((float *)state, pd, eb, cubic, merged);
        else k_recon_pass<float, false, false><<<g, kBlock, 0, st>>>((float *)state, pd, eb, cubic, merged);
    } else {
        if (small) k_recon_pass<double, true, false><<<g, kBlock, 0, st>>>((double *)state, pd, eb, cubic, merged);
        else k_recon_pass<double, false, false><<<g, kBlock, 0, st>>>((double *)state, pd, eb, cubic, merged);
    }
    CKL();
}

void launch_outlier_prefix(const uint8_t *block, uint64_t entries, int scalar, uint64_t count, uint64_t *napplied,
                           cudaStream_t st) {
    k_outlier_prefix<<<1, 1024, 0, st>>>(block, entries, scalar, count, napplied);
    CKL();
}

void launch_outlier_apply(void *state, int scalar, const PassDesc &pd, const uint8_t *block, const uint64_t *napplied,
                          uint64_t max_entries, cudaStream_t st) {
    if (max_entries == 0) return;
    const unsigned g = grid_for(max_entries, 256, 1024);
    const bool small = pd.size < (uint64_t(1) << 32);
    if (scalar == 0) {
        if (small) k_outlier_apply<float, true><<<g, 256, 0, st>>>((float *)state, pd, block, napplied);
        else k_outlier_apply<float, false><<<g, 256, 0, st>>>((float *)state, pd, block, napplied);
    } else {
        if (small) k_outlier_apply<double, true><<<g, 256, 0, st>>>((double *)state, pd, block, napplied);
        else k_outlier_apply<double, false><<<g, 256, 0, st>>>((double *)state, pd, block, napplied);
    }
    CKL();
}

}  // namespace ipcg
