// ipcomp/grid.hpp -- the level partition of the reference's proj/include/ipcomp/grid.hpp
// (LevelTraversal, LevelPoint, level_count, max_levels_for_cap), host-side.  It walks the same
// pass boxes (include/ipcomp_b200_grid.h) the device kernels index, so the traversal order a
// caller sees is the one codes, outliers and plane bits are stored in.
#ifndef IPCOMP_GRID_HPP
#define IPCOMP_GRID_HPP

#include <cstdint>
#include <stdexcept>
#include <utility>

#include "ipcomp/common.hpp"
#include "ipcomp_b200_grid.h"

namespace ipcomp {

inline constexpr std::size_t kDefaultAnchorStrideCap = 64;  // grid.hpp:12

inline int max_levels_for_cap(std::size_t cap) { return ipcg::max_levels_for_cap(cap); }

inline int level_count(const Dims &dims, int max_levels = 7) {
    validate_dims(dims);
    std::uint64_t d[4] = {1, 1, 1, 1};
    for (std::size_t i = 0; i < dims.size(); ++i) d[i] = dims[i];
    return ipcg::level_count(d, static_cast<int>(dims.size()), max_levels);
}

struct LevelPoint {
    std::size_t flat;       // row-major element index
    int axis;               // interpolation axis of the pass (-1 on the coarsest level)
    std::size_t coord;      // coordinate along that axis
    std::size_t extent;     // grid extent along that axis
    std::size_t axis_step;  // flat distance of one stride step along the axis
};

class LevelTraversal {
   public:
    explicit LevelTraversal(Dims dims, int max_levels = 7) : dims_(std::move(dims)) {
        validate_dims(dims_);
        std::uint64_t d[4] = {1, 1, 1, 1};
        for (std::size_t i = 0; i < dims_.size(); ++i) d[i] = dims_[i];
        g_ = ipcg::make_geometry(d, static_cast<int>(dims_.size()), max_levels);
    }

    const Dims &dims() const { return dims_; }
    int levels() const { return g_.levels; }
    std::size_t size() const { return static_cast<std::size_t>(g_.n); }
    std::size_t stride(int level) const { return std::size_t{1} << (level - 1); }
    std::size_t anchor_stride() const { return stride(g_.levels); }
    std::size_t level_size(int level) const {
        check(level);
        return static_cast<std::size_t>(g_.level[static_cast<std::size_t>(level - 1)].count);
    }

    // the level's points in ordinal order: pass by pass, row-major inside each pass box
    template <class F>
    void for_each(int level, F &&fn) const {
        check(level);
        for (const ipcg::PassDesc &p : g_.level[static_cast<std::size_t>(level - 1)].passes) {
            std::uint64_t idx[4] = {0, 0, 0, 0};
            std::uint64_t flat = p.start_flat;
            const std::size_t ext = p.axis >= 0 ? static_cast<std::size_t>(p.extent) : 0;
            const std::size_t st = p.axis >= 0 ? static_cast<std::size_t>(p.st) : 0;
            for (std::uint64_t i = 0; i < p.size; ++i) {
                const std::size_t coord = p.axis >= 0 ? static_cast<std::size_t>(p.axis_start + idx[p.axis] * p.axis_step) : 0;
                fn(LevelPoint{static_cast<std::size_t>(flat), p.axis, coord, ext, st});
                for (int d = p.nd - 1; d >= 0; --d) {  // odometer step
                    flat += p.step_flat[d];
                    if (++idx[d] < p.cnt[d]) break;
                    flat -= idx[d] * p.step_flat[d];
                    idx[d] = 0;
                }
            }
        }
    }

   private:
    void check(int level) const {
        if (level < 1 || level > g_.levels) throw std::invalid_argument("level index out of range");
    }
    Dims dims_;
    ipcg::Geometry g_;
};

}  // namespace ipcomp

#endif
