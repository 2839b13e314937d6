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
#include <cstdlib>
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


// ---------------------------------------------------------------------------------------
// k_loss_lines: the same replay for levels of 1-3 dimensions (leading axes padded with extent
// 1), with every deviation value in registers.  On a level's lattice (coordinates in units of
// the level stride) the passes are: over x (x odd, y, z even), over y (y odd, z even), over z
// (z odd).  Their sources are always points of coarser levels or of EARLIER passes, so:
//   pass-x value  v0 = 0 + own                      (its sources are coarser: deviation 0)
//   pass-y value  v1 = pred_y(v0 at y+-1, y+-3) + own  (v0 = 0 at even x)
//   pass-z value  v2 = pred_z(E at z+-1, z+-3) + own   (E = v1 / v0 / 0 at even z)
// i.e. every value is a 2-deep stencil of codewords.  A warp owns one x, a segment of z and a
// range of y rows: lane l holds the even-z indices S+2l, S+2l+1 (E values) and the odd-z
// targets of the same indices; pass-z sources of the neighbours come by shuffle, pass-y sources
// from a 4-row register window of v0 walked down the y rows.  Dropped-digit counts go two at a
// time; the codewords of a task are re-read per pair (L2-resident).  No shared memory, no
// barriers.  Owned indices per segment: [S+1, S+62) (61 of the 64 held), S = 61k - 1.
struct LossLines {
    int Mx, My, Mz;                  // lattice extents
    uint32_t cey, coy, cez, coz;     // even / odd lattice counts along y, z
    uint32_t cox;                    // odd count along x
    uint64_t b0, b1, b2;             // ordinal bases of the passes over x, y, z
    uint32_t nseg, rows_per_task, nyr;
    uint64_t ntasks;
};

constexpr int LL_WARPS = 8;

// (double)v for |v| < 2^51 by the 2^52 + 2^51 bias: an integer add and one DADD on the FP64 pipe
// instead of an I2F.F64 on the conversion unit (same value: both are exact)
__device__ __forceinline__ double i2d_exact(int64_t v) {
    return __longlong_as_double(v + 0x4338000000000000ll) - 6755399441055744.0;
}
// own = unit * (double)(from_negabinary(w & ~m) - from_negabinary(w)) (pipeline.hpp:104-106)
__device__ __forceinline__ double own_dev(uint32_t w, uint32_t m, double unit) {
    return unit * i2d_exact((int64_t)from_nb(w & ~m) - (int64_t)from_nb(w));
}

template <bool Cubic>
__device__ __forceinline__ double pred4(double a, double b, double c, double d, int cls) {
    // predict_cubic / predict_linear / copy (predictor.hpp:16-38); x/16 and x/2 are exact scalings
    return cls == 0 ? (9.0 * (b + c) - (a + d)) * 0.0625 : cls == 1 ? (b + c) * 0.5 : b;
}

__device__ __forceinline__ int edge_class(bool cubic, int c, int M) {
    return (cubic && c >= 3 && c + 3 < M) ? 0 : (c + 1 < M) ? 1 : 2;
}

__device__ __forceinline__ void fold_max(double v, double &m) { m = (m < v) ? v : m; }

// u64 max of a non-negative double across the warp (bit patterns order like the values)
__device__ __forceinline__ unsigned long long warp_max_bits(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// one task of k_loss_lines for one pair of dropped-digit counts (masks ma, mb); XODD: the
// task's x is odd (pass-x points exist in it), ZCUBIC: every target of the warp has the
// interior (cubic) class along z.  Returns the lane's running maxima in mxa / mxb.
struct LaneCtx {
    const uint32_t *r0, *r1, *r2;  // this x's rows of the pass-x / pass-y / pass-z boxes, + e0
    int e0;                        // first E index held by the lane
    bool eok0, eok1, own0, own1, tok0, tok1;
    int zc0, zc1;                  // z edge classes of the lane's two targets
};

template <bool Cubic, bool ZCUBIC>
__device__ __forceinline__ void pass_z(const LaneCtx &L, double E0, double E1, uint32_t c20, uint32_t c21, uint32_t m,
                                       double unit, double &mx) {
    // target e reads E at e-1, e, e+1, e+2 (lane-1's second, own two, lane+1's two)
    const double left = __shfl_up_sync(0xffffffffu, E1, 1);
    const double r0 = __shfl_down_sync(0xffffffffu, E0, 1);
    const double r1 = __shfl_down_sync(0xffffffffu, E1, 1);
    double p0, p1;
    if (ZCUBIC) {
        p0 = (9.0 * (E0 + E1) - (left + r0)) * 0.0625;
        p1 = (9.0 * (E1 + r0) - (E0 + r1)) * 0.0625;
    } else {
        p0 = pred4<Cubic>(left, E0, E1, r0, L.zc0);
        p1 = pred4<Cubic>(E0, E1, r0, r1, L.zc1);
    }
    const double va = p0 + own_dev(c20, m, unit), vb = p1 + own_dev(c21, m, unit);
    if (L.tok0) fold_max(fabs(va), mx);
    if (L.tok1) fold_max(fabs(vb), mx);
}

template <bool Cubic, bool XODD, bool ZCUBIC>
__device__ void loss_task(const LaneCtx &L, const LossLines &g, uint32_t p0, uint32_t p1, uint32_t ma, uint32_t mb,
                          bool two, double unit, double &mxa, double &mxb) {
    const uint32_t cez = g.cez, coz = g.coz;
    // v0 window over even rows q-1 .. q+2 of pair q: [row][z][d]
    double w[4][2][2];
    auto v0 = [&](int q, double (&o)[2][2]) {
        uint32_t c[2] = {0u, 0u};
        const bool rq = XODD && q >= 0 && (uint32_t)q < g.cey;
        if (rq && L.eok0) c[0] = __ldg(L.r0 + (uint64_t)q * cez);
        if (rq && L.eok1) c[1] = __ldg(L.r0 + (uint64_t)q * cez + 1);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const bool ok = rq && (k ? L.eok1 : L.eok0);
            o[k][0] = ok ? own_dev(c[k], ma, unit) : 0.0;
            o[k][1] = ok ? own_dev(c[k], mb, unit) : 0.0;
        }
    };
    if (XODD) {
        v0((int)p0 - 1, w[0]);
        v0((int)p0, w[1]);
        v0((int)p0 + 1, w[2]);
    }
    for (uint32_t p = p0; p < p1; ++p) {
        const int yo = 2 * (int)p + 1;
        const bool has_odd = yo < g.My;
        uint32_t c1[2] = {0u, 0u}, c2e[2] = {0u, 0u}, c2o[2] = {0u, 0u};
        const uint32_t *q1 = L.r1 + (uint64_t)p * cez, *q2 = L.r2 + (uint64_t)(2 * p) * coz;
        if (has_odd && L.eok0) c1[0] = __ldg(q1);
        if (has_odd && L.eok1) c1[1] = __ldg(q1 + 1);
        if (L.tok0) c2e[0] = __ldg(q2);
        if (L.tok1) c2e[1] = __ldg(q2 + 1);
        if (has_odd && L.tok0) c2o[0] = __ldg(q2 + coz);
        if (has_odd && L.tok1) c2o[1] = __ldg(q2 + coz + 1);
        if (XODD) v0((int)p + 2, w[3]);
        // row y = 2p: E = v0 (pass-x points at odd x, coarser points at even x)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (!two && t) break;
            double &mx = t ? mxb : mxa;
            const uint32_t m = t ? mb : ma;
            const double E0 = XODD ? w[1][0][t] : 0.0, E1 = XODD ? w[1][1][t] : 0.0;
            if (XODD) {
                if (L.eok0 && L.own0) fold_max(fabs(E0), mx);
                if (L.eok1 && L.own1) fold_max(fabs(E1), mx);
            }
            pass_z<Cubic, ZCUBIC>(L, E0, E1, c2e[0], c2e[1], m, unit, mx);
        }
        // row y = 2p + 1: E = v1 = pred_y(v0 window) + own (at even x the window is all zero:
        // pred = +0 exactly, and +0 + own == own)
        if (has_odd) {
            const int ycls = edge_class(Cubic, yo, g.My);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (!two && t) break;
                double &mx = t ? mxb : mxa;
                const uint32_t m = t ? mb : ma;
                double E0 = own_dev(c1[0], m, unit), E1 = own_dev(c1[1], m, unit);
                if (XODD) {
                    double p0v, p1v;
                    if (ycls == 0) {
                        p0v = (9.0 * (w[1][0][t] + w[2][0][t]) - (w[0][0][t] + w[3][0][t])) * 0.0625;
                        p1v = (9.0 * (w[1][1][t] + w[2][1][t]) - (w[0][1][t] + w[3][1][t])) * 0.0625;
                    } else {
                        p0v = pred4<Cubic>(w[0][0][t], w[1][0][t], w[2][0][t], w[3][0][t], ycls);
                        p1v = pred4<Cubic>(w[0][1][t], w[1][1][t], w[2][1][t], w[3][1][t], ycls);
                    }
                    E0 = p0v + E0;
                    E1 = p1v + E1;
                }
                if (L.eok0 && L.own0) fold_max(fabs(E0), mx);
                if (L.eok1 && L.own1) fold_max(fabs(E1), mx);
                pass_z<Cubic, ZCUBIC>(L, E0, E1, c2o[0], c2o[1], m, unit, mx);
            }
        }
        if (XODD) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int t = 0; t < 2; ++t) w[0][k][t] = w[1][k][t], w[1][k][t] = w[2][k][t], w[2][k][t] = w[3][k][t];
        }
    }
}

template <bool Cubic>
__global__ void __launch_bounds__(LL_WARPS * 32, 3) k_loss_lines(const uint32_t *__restrict__ nb, LossLines g,
                                                              double unit, const uint32_t *lowor,
                                                              unsigned long long *raw) {
    const uint32_t lo = *lowor;
    if (lo == 0) return;
    const int d0 = __ffs((int)lo), hb = 31 - __clz(lo), dmax = hb + 1 < 32 ? hb + 1 : 32;
    const unsigned lane = threadIdx.x & 31;
    for (uint64_t task = (uint64_t)blockIdx.x * LL_WARPS + (threadIdx.x >> 5); task < g.ntasks;
         task += (uint64_t)gridDim.x * LL_WARPS) {
        const uint32_t yr = (uint32_t)(task % g.nyr);
        const uint32_t seg = (uint32_t)((task / g.nyr) % g.nseg);
        const int x = (int)(task / ((uint64_t)g.nyr * g.nseg));
        const uint32_t p0 = yr * g.rows_per_task, p1 = min(p0 + g.rows_per_task, g.cey);  // row pairs
        const int S = (int)seg * 61 - 1;
        LaneCtx L;
        L.e0 = S + 2 * (int)lane;
        const int e1 = L.e0 + 1;
        L.eok0 = L.e0 >= 0 && (uint32_t)L.e0 < g.cez;
        L.eok1 = (uint32_t)e1 < g.cez;
        L.own0 = L.e0 >= S + 1 && L.e0 < S + 62;
        L.own1 = e1 < S + 62;
        L.tok0 = L.own0 && L.e0 >= 0 && (uint32_t)L.e0 < g.coz;
        L.tok1 = L.own1 && (uint32_t)e1 < g.coz;
        L.zc0 = edge_class(Cubic, 2 * L.e0 + 1, g.Mz);
        L.zc1 = edge_class(Cubic, 2 * e1 + 1, g.Mz);
        const int eb = L.e0 < 0 ? 0 : L.e0;  // row pointers are only dereferenced where e0 >= 0
        L.r0 = nb + g.b0 + (uint64_t)(x >> 1) * g.cey * g.cez + eb;
        L.r1 = nb + g.b1 + (uint64_t)x * g.coy * g.cez + eb;
        L.r2 = nb + g.b2 + (uint64_t)x * g.My * g.coz + eb;
        if (L.e0 < 0) {  // (lane 0 of the first segment: its e0 = -1 holds nothing, e1 = 0 sits at +0)
            L.r0 -= 1, L.r1 -= 1, L.r2 -= 1;
        }
        const bool zcubic = __all_sync(0xffffffffu, !(L.tok0 || L.tok1) || ((!L.tok0 || L.zc0 == 0) && (!L.tok1 || L.zc1 == 0)));
        const bool xodd = x & 1;
        for (int da = d0; da <= dmax; da += 2) {
            const int db = da + 1 <= dmax ? da + 1 : da;
            const uint32_t ma = da == 32 ? 0xFFFFFFFFu : ((1u << da) - 1u);
            const uint32_t mb = db == 32 ? 0xFFFFFFFFu : ((1u << db) - 1u);
            const bool two = db != da;
            double mxa = 0.0, mxb = 0.0;
            if (xodd) {
                if (zcubic) loss_task<Cubic, true, true>(L, g, p0, p1, ma, mb, two, unit, mxa, mxb);
                else loss_task<Cubic, true, false>(L, g, p0, p1, ma, mb, two, unit, mxa, mxb);
            } else {
                if (zcubic) loss_task<Cubic, false, true>(L, g, p0, p1, ma, mb, two, unit, mxa, mxb);
                else loss_task<Cubic, false, false>(L, g, p0, p1, ma, mb, two, unit, mxa, mxb);
            }
            const unsigned long long ba = warp_max_bits(mxa), bb = warp_max_bits(mxb);
            if (lane == 0) {
                if (ba) atomicMax(&raw[da], ba);
                if (bb && two) atomicMax(&raw[db], bb);
            }
        }
    }
}

// the level as a padded 3-D lattice, or false (4-D grids, the coarsest level)
bool loss_lines_geom(const Geometry &G, int level, LossLines &g) {
    if (level == G.levels || G.nd > 3) return false;
    const LevelGeom &lg = G.level[level - 1];
    const uint64_t s = uint64_t(1) << (level - 1);
    int M[3] = {1, 1, 1};
    for (int i = 0; i < G.nd; ++i) {
        const uint64_t m = (G.dims[i] + s - 1) / s;
        if (m > (1u << 30)) return false;
        M[3 - G.nd + i] = (int)m;
    }
    g = LossLines{};
    g.Mx = M[0], g.My = M[1], g.Mz = M[2];
    g.cox = (uint32_t)(M[0] / 2);
    g.cey = (uint32_t)((M[1] + 1) / 2), g.coy = (uint32_t)(M[1] / 2);
    g.cez = (uint32_t)((M[2] + 1) / 2), g.coz = (uint32_t)(M[2] / 2);
    for (const PassDesc &pd : lg.passes) {
        const int a = pd.axis + (3 - G.nd);
        if (a == 0) g.b0 = pd.ordinal_base;
        else if (a == 1) g.b1 = pd.ordinal_base;
        else if (a == 2) g.b2 = pd.ordinal_base;
    }
    g.nseg = (std::max(g.cez, g.coz) + 60) / 61;
    // rows per task: enough tasks to fill the GPU a few times over, at least 16 row pairs each
    const uint64_t lines = (uint64_t)g.Mx * g.nseg;
    const uint64_t want = (uint64_t)num_sms() * 64 * 4;
    uint32_t nyr = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((want + lines - 1) / lines, (g.cey + 15) / 16));
    g.rows_per_task = (g.cey + nyr - 1) / nyr;
    g.nyr = (g.cey + g.rows_per_task - 1) / g.rows_per_task;
    g.ntasks = lines * g.nyr;
    return true;
}

}  // namespace

bool launch_loss_fused(const uint32_t *nb, const Geometry &G, int level, bool cubic, double unit,
                       const uint32_t *lowor, unsigned long long *raw, cudaStream_t st) {
    static const bool lines_off = getenv("IPCG_LOSS_TILES") != nullptr;  // dev: the smem-tile kernel
    LossLines ll;
    if (!lines_off && loss_lines_geom(G, level, ll)) {
        const unsigned grid = (unsigned)std::min<uint64_t>((ll.ntasks + LL_WARPS - 1) / LL_WARPS, (uint64_t)num_sms() * 16);
        if (cubic) k_loss_lines<true><<<grid, LL_WARPS * 32, 0, st>>>(nb, ll, unit, lowor, raw);
        else k_loss_lines<false><<<grid, LL_WARPS * 32, 0, st>>>(nb, ll, unit, lowor, raw);
        CKL();
        return true;
    }
    static const int tiles[5][4] = {{0, 0, 0, 0}, {2048, 1, 1, 1}, {32, 64, 1, 1}, {4, 16, 32, 1}, {1, 4, 8, 16}};
    TileGeom g;
    uint64_t ntiles, region;
    if (!tile_geom(G, level, tiles, g, ntiles, region)) return false;
    const size_t smem = region * (2 * 8 + 4 + 2) + 64;
    if (first_on_device<2>()) {
        CK(cudaFuncSetAttribute(k_loss_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k_loss_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    if (cubic) k_loss_fused<true><<<(unsigned)ntiles, LT_THREADS, smem, st>>>(nb, g, unit, lowor, raw);
    else k_loss_fused<false><<<(unsigned)ntiles, LT_THREADS, smem, st>>>(nb, g, unit, lowor, raw);
    CKL();
    return true;
}

}  // namespace ipcg
