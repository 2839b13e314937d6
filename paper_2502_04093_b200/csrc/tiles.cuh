// tiles.cuh -- box-plus-halo tiling of one level's lattice, shared by the fused loss-table
// kernel (losstable.cu, 4-D grids and the smem-tile variant).  A CTA owns a box of the
// level's lattice (coordinates in units of the level stride s) plus a 3-point halo along
// every axis after the first; pass j is evaluated on the box widened by the halo along the
// axes > j, so every level point is produced by exactly one box.
#pragma once
#include <algorithm>

#include "grid.h"
#include "util.cuh"

namespace ipcg {

struct TileGeom {
    int nd, npass;
    int M[4];      // lattice extents ceil(dims/s)
    int T[4];      // box extents
    int H[4];      // halo (0 or 3)
    int R[4];      // staged region extents T + 2H
    int NT[4];     // boxes per axis
    int S[4];      // row-major strides of the staged region
    uint64_t Rm[4];  // ceil(2^32 / R[i]): x / R[i] == (x * Rm[i]) >> 32 for x, R[i] < 2^16
    uint64_t Tm[4];  // the same for T[i]
    uint64_t gstride[4];  // flat grid distance of one lattice step along axis i (level stride s)
    int region;
    int paxis[4];
    uint64_t pbase[4];
    uint32_t pcnt[4][4];
};

// tile geometry of `level` for the fused kernels; false when the level does not fit the
// 13-bit staged-position encoding (callers fall back to per-pass kernels)
inline bool tile_geom(const Geometry &G, int level, const int (*tiles)[4], TileGeom &g, uint64_t &ntiles,
                      uint64_t &region) {
    const LevelGeom &lg = G.level[level - 1];
    if (level == G.levels || lg.passes.empty()) return false;
    const uint64_t s = uint64_t(1) << (level - 1);
    g = TileGeom{};
    g.nd = G.nd;
    region = 1, ntiles = 1;
    for (int i = 0; i < g.nd; ++i) {
        const uint64_t M = (G.dims[i] + s - 1) / s;
        if (M > (1u << 30)) return false;
        g.M[i] = (int)M;
        g.T[i] = (int)std::min<uint64_t>(tiles[g.nd][i], M);
        g.H[i] = (i >= 1 && M > 1) ? 3 : 0;
        g.R[i] = g.T[i] + 2 * g.H[i];
        g.Rm[i] = ((1ull << 32) + (uint64_t)g.R[i] - 1) / (uint64_t)g.R[i];
        g.Tm[i] = ((1ull << 32) + (uint64_t)g.T[i] - 1) / (uint64_t)g.T[i];
        g.gstride[i] = s * G.strides[i];
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
    return true;
}


}  // namespace ipcg
