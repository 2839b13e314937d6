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

#include "numerics.cuh"

namespace ipcg {

namespace {

constexpr int LT_THREADS = 256;

struct LossGeom {
    int nd, npass;
    int M[4];      // lattice extents ceil(dims/s)
    int T[4];      // box extents
    int H[4];      // halo (0 or 3)
    int R[4];      // staged region extents T + 2H
    int NT[4];     // boxes per axis
    int S[4];      // row-major strides of the staged region
    int region;
    int paxis[4];
    uint64_t pbase[4];
    uint32_t pcnt[4][4];
};

__device__ __forceinline__ int32_t from_nb(uint32_t w) { return (int32_t)((w ^ kNbMask) - kNbMask); }

template <bool Cubic>
__global__ void __launch_bounds__(LT_THREADS) k_loss_fused(const uint32_t *__restrict__ nb, LossGeom g, double unit,
                                                          const uint32_t *lowor, unsigned long long *raw) {
    extern __shared__ unsigned char smem[];
    double *dev = reinterpret_cast<double *>(smem);
    uint32_t *code = reinterpret_cast<uint32_t *>(dev + g.region);
    uint16_t *list = reinterpret_cast<uint16_t *>(code + g.region);  // per-pass work lists
    __shared__ int cnt[4], off[5];
    __shared__ double red[LT_THREADS / 32];
    const uint32_t lo = *lowor;
    if (lo == 0) return;
    // box origin
    int tile = blockIdx.x, t0[4];
    for (int i = g.nd - 1; i >= 0; --i) {
        t0[i] = (tile % g.NT[i]) * g.T[i];
        tile /= g.NT[i];
    }
    if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
    __syncthreads();
    // stage codewords, classify every staged position, count per-pass work
    for (int u = threadIdx.x; u < g.region; u += blockDim.x) {
        dev[u] = 0.0;
        int lu[4], m[4], rem = u;
        for (int i = g.nd - 1; i >= 0; --i) {
            lu[i] = rem % g.R[i];
            rem /= g.R[i];
            m[i] = t0[i] - g.H[i] + lu[i];
        }
        bool in = true;
        int j = -1;
        for (int i = 0; i < g.nd; ++i) {
            if (m[i] < 0 || m[i] >= g.M[i]) in = false;
            if (m[i] & 1) j = i;
        }
        uint32_t w = 0;
        if (in && j >= 0) {
            int pi = 0;
            while (g.paxis[pi] != j) ++pi;
            uint64_t ord = 0;
            for (int i = 0; i < g.nd; ++i) {
                const uint32_t idx = i < j ? (uint32_t)m[i] : i == j ? (uint32_t)(m[i] - 1) / 2 : (uint32_t)m[i] / 2;
                ord = ord * g.pcnt[pi][i] + idx;
            }
            w = nb[g.pbase[pi] + ord];
            // member of pass j's evaluation region: inside the box on axes <= j
            bool member = true;
            for (int i = 0; i <= j; ++i)
                if (lu[i] < g.H[i] || lu[i] >= g.H[i] + g.T[i]) member = false;
            if (member) atomicAdd(&cnt[pi], 1);
        }
        code[u] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int p = 0; p < g.npass; ++p) off[p + 1] = off[p] + cnt[p];
        for (int p = 0; p < 4; ++p) cnt[p] = 0;
    }
    __syncthreads();
    // build the lists: entry = position (13 bits) | edge class << 13 | interior << 15
    for (int u = threadIdx.x; u < g.region; u += blockDim.x) {
        int lu[4], m[4], rem = u;
        for (int i = g.nd - 1; i >= 0; --i) {
            lu[i] = rem % g.R[i];
            rem /= g.R[i];
            m[i] = t0[i] - g.H[i] + lu[i];
        }
        bool in = true;
        int j = -1;
        for (int i = 0; i < g.nd; ++i) {
            if (m[i] < 0 || m[i] >= g.M[i]) in = false;
            if (m[i] & 1) j = i;
        }
        if (!in || j < 0) continue;
        bool member = true, interior = true;
        for (int i = 0; i < g.nd; ++i) {
            const bool inbox = lu[i] >= g.H[i] && lu[i] < g.H[i] + g.T[i];
            if (i <= j && !inbox) member = false;
            if (!inbox) interior = false;
        }
        if (!member) continue;
        int pi = 0;
        while (g.paxis[pi] != j) ++pi;
        const int mj = m[j];
        const int edge = (Cubic && mj >= 3 && mj + 3 < g.M[j]) ? 0 : (mj + 1 < g.M[j]) ? 1 : 2;
        const int slot = off[pi] + atomicAdd(&cnt[pi], 1);
        list[slot] = (uint16_t)(u | (edge << 13) | ((interior ? 1 : 0) << 15));
    }
    __syncthreads();
    const int hb = 31 - __clz(lo);
    const int dmax = hb + 1 < 32 ? hb + 1 : 32;
    for (int d = 1; d <= dmax; ++d) {
        const uint32_t mask = d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u);
        if ((lo & mask) == 0) continue;
        double worst = 0.0;
        for (int pi = 0; pi < g.npass; ++pi) {
            const int stp = g.S[g.paxis[pi]];
            // without a halo along the pass axis (the first axis) every source is a coarser
            // point, whose deviation is zero
            const bool zero_src = g.H[g.paxis[pi]] == 0;
            for (int e = off[pi] + threadIdx.x; e < off[pi + 1]; e += blockDim.x) {
                const uint32_t ent = list[e];
                const int u = (int)(ent & 0x1fff), edge = (int)((ent >> 13) & 3);
                const uint32_t w = code[u];
                const double own = unit * (double)((int64_t)from_nb(w & ~mask) - (int64_t)from_nb(w));
                double pred;
                if (zero_src) {
                    pred = edge == 0 ? (9.0 * (0.0 + 0.0) - (0.0 + 0.0)) / 16.0 : edge == 1 ? (0.0 + 0.0) / 2.0 : 0.0;
                } else if (edge == 0) {
                    const double a = dev[u - 3 * stp], b = dev[u - stp], c = dev[u + stp], dd = dev[u + 3 * stp];
                    pred = (9.0 * (b + c) - (a + dd)) / 16.0;
                } else if (edge == 1) {
                    pred = (dev[u - stp] + dev[u + stp]) / 2.0;
                } else {
                    pred = dev[u - stp];
                }
                const double v = pred + own;
                dev[u] = v;
                if (ent >> 15) {
                    const double a = fabs(v);
                    worst = (worst < a) ? a : worst;
                }
            }
            __syncthreads();
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double x = __shfl_down_sync(0xffffffffu, worst, o);
            worst = (worst < x) ? x : worst;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = 0.0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = (m < red[i]) ? red[i] : m;
            if (m > 0.0) atomicMax(&raw[d], (unsigned long long)__double_as_longlong(m));
        }
        __syncthreads();
    }
}

}  // namespace

bool launch_loss_fused(const uint32_t *nb, const Geometry &G, int level, bool cubic, double unit,
                       const uint32_t *lowor, unsigned long long *raw, cudaStream_t st) {
    const LevelGeom &lg = G.level[level - 1];
    if (level == G.levels || lg.passes.empty()) return false;
    const uint64_t s = uint64_t(1) << (level - 1);
    LossGeom g{};
    g.nd = G.nd;
    static const int tiles[5][4] = {{0, 0, 0, 0}, {4096, 1, 1, 1}, {32, 128, 1, 1}, {4, 16, 64, 1}, {1, 4, 8, 32}};
    uint64_t region = 1, ntiles = 1;
    for (int i = 0; i < g.nd; ++i) {
        const uint64_t M = (G.dims[i] + s - 1) / s;
        if (M > (1u << 30)) return false;
        g.M[i] = (int)M;
        g.T[i] = (int)std::min<uint64_t>(tiles[g.nd][i], M);
        g.H[i] = (i >= 1 && M > 1) ? 3 : 0;
        g.R[i] = g.T[i] + 2 * g.H[i];
        g.NT[i] = (int)((M + g.T[i] - 1) / g.T[i]);
        region *= (uint64_t)g.R[i];
        ntiles *= (uint64_t)g.NT[i];
    }
    if (region >= 8192 || ntiles > 0x7fffffff) return false;  // 13-bit list entries
    g.region = (int)region;
    int acc = 1;
    for (int i = g.nd - 1; i >= 0; --i) {
        g.S[i] = acc;
        acc *= g.R[i];
    }
    g.npass = (int)lg.passes.size();
    for (int p = 0; p < g.npass; ++p) {
        g.paxis[p] = lg.passes[p].axis;
        g.pbase[p] = lg.passes[p].ordinal_base;
        for (int i = 0; i < g.nd; ++i) g.pcnt[p][i] = (uint32_t)lg.passes[p].cnt[i];
    }
    const size_t smem = region * (8 + 4 + 2) + 64;
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
