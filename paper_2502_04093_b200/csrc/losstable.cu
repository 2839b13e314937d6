// losstable.cu -- fused per-level loss table (detail::measure_loss_table,
// proj/include/ipcomp/pipeline.hpp:85-124) for every level below the coarsest.
//
// The reference replays a whole level once per dropped-digit count d on a double
// deviation field.  Here one CTA owns a box of the level's lattice (coordinates in
// units of the level stride s): it stages the level's codewords for the box plus a
// 3-point halo along every later axis in shared memory, and then, for each d, replays
// the passes in order entirely in shared memory.  Pass j's value at x needs pass<j values
// at x +- {1,3} e_j, so pass j is evaluated on the box widened by 3 along the axes > j;
// every level point is counted in exactly one box.  max|v| per d is folded with an
// atomicMax on the IEEE bits of a non-negative double (exact, order-free).
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "numerics.cuh"
#include "tiles.cuh"

namespace ipcg {

namespace {

constexpr int LT_THREADS = 256;



__device__ __forceinline__ int32_t from_nb(uint32_t w) { return (int32_t)((w ^ kNbMask) - kNbMask); }

// Per CTA: (1) enumerate each pass's evaluation points directly from its sub-lattice
// (axes < j: the box; axis j: odd coordinates in the box; axes > j: even coordinates in the
// box widened by the halo), storing (staged position, edge class, interior flag) and the
// point's codeword; (2) replay the valid d (a contiguous range) two at a time, one
// deviation array each, so list/code/address work and barriers are shared by the pair.
template <bool Cubic>
__global__ void __launch_bounds__(LT_THREADS) k_loss_fused(const uint32_t *__restrict__ nb, TileGeom g, double unit,
                                                          const uint32_t *lowor, unsigned long long *raw) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lo = *lowor;
    if (lo == 0) return;
    double *dev0 = reinterpret_cast<double *>(smem);
    double *dev1 = dev0 + g.region;
    uint32_t *codes = reinterpret_cast<uint32_t *>(dev1 + g.region);
    uint16_t *list = reinterpret_cast<uint16_t *>(codes + g.region);  // u | edge << 13 | interior << 15
    __shared__ int off[5];
    __shared__ int first[4][4], cnt[4][4];
    __shared__ uint64_t mag[4][4];  // ceil(2^32 / cnt)
    __shared__ double red[2][LT_THREADS / 32];
    int tile = blockIdx.x, t0[4];
    for (int i = g.nd - 1; i >= 0; --i) {
        t0[i] = (tile % g.NT[i]) * g.T[i];
        tile /= g.NT[i];
    }
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int p = 0; p < g.npass; ++p) {
            const int j = g.paxis[p];
            int total = 1;
            for (int i = 0; i < g.nd; ++i) {
                int a0, a1, step;
                if (i < j) a0 = t0[i], a1 = min(t0[i] + g.T[i], g.M[i]), step = 1;
                else if (i == j) a0 = t0[i] | 1, a1 = min(t0[i] + g.T[i], g.M[i]), step = 2;
                else a0 = max(t0[i] - g.H[i], 0), a0 += a0 & 1, a1 = min(t0[i] + g.T[i] + g.H[i], g.M[i]), step = 2;
                const int c = a1 > a0 ? (a1 - a0 + step - 1) / step : 0;
                first[p][i] = a0;
                cnt[p][i] = c;
                mag[p][i] = c ? ((1ull << 32) + (uint64_t)c - 1) / (uint64_t)c : 0;
                total *= c;
            }
            off[p + 1] = off[p] + total;
        }
    }
    for (int u = threadIdx.x; u < 2 * g.region; u += blockDim.x) dev0[u] = 0.0;
    __syncthreads();
    const int nent = off[g.npass];
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
        int p = 0;
        while (e >= off[p + 1]) ++p;
        const int j = g.paxis[p];
        int rem = e - off[p], u = 0, mj = 0;
        uint64_t ord = 0;
        bool interior = true;
        int m[4];
        for (int i = g.nd - 1; i >= 0; --i) {
            const int q = (int)(((uint64_t)rem * mag[p][i]) >> 32);
            const int k = rem - q * cnt[p][i];
            rem = q;
            m[i] = first[p][i] + (i < j ? k : 2 * k);
        }
        for (int i = 0; i < g.nd; ++i) {
            u += (m[i] - t0[i] + g.H[i]) * g.S[i];
            if (m[i] < t0[i] || m[i] >= t0[i] + g.T[i]) interior = false;
            const uint32_t idx = i < j ? (uint32_t)m[i] : i == j ? (uint32_t)(m[i] - 1) / 2 : (uint32_t)m[i] / 2;
            ord = ord * g.pcnt[p][i] + idx;
            if (i == j) mj = m[i];
        }
        const int edge = (Cubic && mj >= 3 && mj + 3 < g.M[j]) ? 0 : (mj + 1 < g.M[j]) ? 1 : 2;
        codes[e] = __ldg(nb + g.pbase[p] + ord);
        list[e] = (uint16_t)(u | (edge << 13) | ((interior ? 1 : 0) << 15));
    }
    __syncthreads();
    const int d0 = __ffs((int)lo);  // first d whose mask reaches a set bit
    const int hb = 31 - __clz(lo);
    const int dmax = hb + 1 < 32 ? hb + 1 : 32;
    for (int da = d0; da <= dmax; da += 2) {
        const int db = da + 1 <= dmax ? da + 1 : da;  // a lone last d is computed twice
        const uint32_t ma = da == 32 ? 0xFFFFFFFFu : ((1u << da) - 1u);
        const uint32_t mb = db == 32 ? 0xFFFFFFFFu : ((1u << db) - 1u);
        double wa = 0.0, wb = 0.0;
        for (int pi = 0; pi < g.npass; ++pi) {
            const int stp = g.S[g.paxis[pi]];
            // without a halo along the pass axis (the first axis) every source is a coarser
            // point, whose deviation is zero
            const bool zero_src = g.H[g.paxis[pi]] == 0;
            for (int e = off[pi] + threadIdx.x; e < off[pi + 1]; e += blockDim.x) {
                const uint32_t ent = list[e];
                const int u = (int)(ent & 0x1fff), edge = (int)((ent >> 13) & 3);
                const uint32_t w = codes[e];
                const int64_t full = (int64_t)from_nb(w);
                const double oa = unit * (double)((int64_t)from_nb(w & ~ma) - full);
                const double ob = unit * (double)((int64_t)from_nb(w & ~mb) - full);
                double pa, pb;
                if (zero_src) {
                    const double z = edge == 0 ? (9.0 * (0.0 + 0.0) - (0.0 + 0.0)) / 16.0 : edge == 1 ? (0.0 + 0.0) / 2.0 : 0.0;
                    pa = z, pb = z;
                } else if (edge == 0) {
                    pa = (9.0 * (dev0[u - stp] + dev0[u + stp]) - (dev0[u - 3 * stp] + dev0[u + 3 * stp])) / 16.0;
                    pb = (9.0 * (dev1[u - stp] + dev1[u + stp]) - (dev1[u - 3 * stp] + dev1[u + 3 * stp])) / 16.0;
                } else if (edge == 1) {
                    pa = (dev0[u - stp] + dev0[u + stp]) / 2.0;
                    pb = (dev1[u - stp] + dev1[u + stp]) / 2.0;
                } else {
                    pa = dev0[u - stp];
                    pb = dev1[u - stp];
                }
                const double va = pa + oa, vb = pb + ob;
                dev0[u] = va;
                dev1[u] = vb;
                if (ent >> 15) {
                    const double xa = fabs(va), xb = fabs(vb);
                    wa = (wa < xa) ? xa : wa;
                    wb = (wb < xb) ? xb : wb;
                }
            }
            __syncthreads();
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double xa = __shfl_down_sync(0xffffffffu, wa, o), xb = __shfl_down_sync(0xffffffffu, wb, o);
            wa = (wa < xa) ? xa : wa;
            wb = (wb < xb) ? xb : wb;
        }
        if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = wa, red[1][threadIdx.x >> 5] = wb;
        __syncthreads();
        if (threadIdx.x < 2) {
            double mx = 0.0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = (mx < red[threadIdx.x][i]) ? red[threadIdx.x][i] : mx;
            if (mx > 0.0) atomicMax(&raw[threadIdx.x ? db : da], (unsigned long long)__double_as_longlong(mx));
        }
        __syncthreads();
    }
}


}  // namespace

bool launch_loss_fused(const uint32_t *nb, const Geometry &G, int level, bool cubic, double unit,
                       const uint32_t *lowor, unsigned long long *raw, cudaStream_t st) {
    static const int tiles[5][4] = {{0, 0, 0, 0}, {2048, 1, 1, 1}, {32, 64, 1, 1}, {4, 16, 32, 1}, {1, 4, 8, 16}};
    TileGeom g;
    uint64_t ntiles, region;
    if (!tile_geom(G, level, tiles, g, ntiles, region)) return false;
    const size_t smem = region * (2 * 8 + 4 + 2) + 64;
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(k_loss_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k_loss_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    if (cubic) k_loss_fused<true><<<(unsigned)ntiles, LT_THREADS, smem, st>>>(nb, g, unit, lowor, raw);
    else k_loss_fused<false><<<(unsigned)ntiles, LT_THREADS, smem, st>>>(nb, g, unit, lowor, raw);
    CKL();
    return true;
}

}  // namespace ipcg
