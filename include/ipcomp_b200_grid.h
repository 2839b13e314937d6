// ipcomp_b200_grid.h -- level/pass geometry of the reference's LevelTraversal (grid.hpp:14-161),
// expressed as per-pass box descriptors the sm_100a kernels index directly.
#pragma once
#include <stdint.h>

#include <vector>

namespace ipcg {

constexpr int kMaxDims = 4;

// One interpolation pass: a row-major box of targets.  The ordinal of the box's
// row-major index i is ordinal_base + i (grid.hpp:124-156 defines the order).
struct PassDesc {
    int nd;
    int axis;                  // -1 for the coarsest level (predicts 0)
    uint64_t cnt[kMaxDims];    // box extent per axis
    uint64_t step_flat[kMaxDims];
    uint64_t start_flat;
    uint64_t axis_start, axis_step;  // coordinate along `axis`: axis_start + idx[axis]*axis_step
    uint64_t extent;           // dims[axis]
    uint64_t s;                // level stride
    uint64_t st;               // flat distance of one stride step along axis
    uint64_t size;
    uint64_t ordinal_base;
};

struct LevelGeom {
    int level;
    uint64_t count;
    std::vector<PassDesc> passes;
};

struct Geometry {
    int nd = 0, levels = 0;
    uint64_t dims[kMaxDims] = {0, 0, 0, 0}, strides[kMaxDims] = {0, 0, 0, 0}, n = 0;
    std::vector<LevelGeom> level;  // [l-1]
};

inline int max_levels_for_cap(uint64_t cap) {  // grid.hpp:14-18
    int l = 1;
    while (l < 63 && (uint64_t(1) << l) <= cap) ++l;
    return l;
}

inline int level_count(const uint64_t *dims, int nd, int max_levels) {  // grid.hpp:21-28
    uint64_t m = 1;
    for (int i = 0; i < nd; ++i)
        if (dims[i] > m) m = dims[i];
    int l = 1;
    while ((uint64_t(1) << l) < m && l < max_levels) ++l;
    return l;
}

inline uint64_t lattice_count(uint64_t extent, uint64_t start, uint64_t step) {
    return start >= extent ? 0 : (extent - 1 - start) / step + 1;
}

inline Geometry make_geometry(const uint64_t *dims, int nd, int max_levels) {
    Geometry g;
    g.nd = nd;
    uint64_t acc = 1;
    for (int i = nd - 1; i >= 0; --i) {
        g.dims[i] = dims[i];
        g.strides[i] = acc;
        acc *= dims[i];
    }
    g.n = acc;
    g.levels = level_count(dims, nd, max_levels);
    g.level.resize(g.levels);
    for (int level = 1; level <= g.levels; ++level) {
        LevelGeom &lg = g.level[level - 1];
        lg.level = level;
        lg.count = 0;
        const uint64_t s = uint64_t(1) << (level - 1);
        auto add_pass = [&](int axis, const uint64_t *start, const uint64_t *step) {
            PassDesc p{};
            p.nd = nd;
            p.axis = axis;
            p.size = 1;
            p.start_flat = 0;
            for (int i = 0; i < nd; ++i) {
                p.cnt[i] = lattice_count(dims[i], start[i], step[i]);
                p.size *= p.cnt[i];
                p.step_flat[i] = step[i] * g.strides[i];
                p.start_flat += start[i] * g.strides[i];
            }
            if (p.size == 0) return;
            p.s = s;
            if (axis >= 0) {
                p.axis_start = start[axis];
                p.axis_step = step[axis];
                p.extent = dims[axis];
                p.st = s * g.strides[axis];
            }
            p.ordinal_base = lg.count;
            lg.count += p.size;
            lg.passes.push_back(p);
        };
        uint64_t start[kMaxDims], step[kMaxDims];
        if (level == g.levels) {
            for (int i = 0; i < nd; ++i) start[i] = 0, step[i] = s;
            add_pass(-1, start, step);
            continue;
        }
        for (int axis = 0; axis < nd; ++axis) {
            if (dims[axis] <= s) continue;
            for (int i = 0; i < nd; ++i) {
                if (i < axis) start[i] = 0, step[i] = s;
                else if (i == axis) start[i] = s, step[i] = 2 * s;
                else start[i] = 0, step[i] = 2 * s;
            }
            add_pass(axis, start, step);
        }
    }
    return g;
}

}  // namespace ipcg
