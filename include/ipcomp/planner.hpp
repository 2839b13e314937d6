// ipcomp/planner.hpp -- the retrieval planner of the reference's proj/include/ipcomp/planner.hpp
// (src/planner.cpp): a knapsack over per-level plane drops on 1024 ceiling buckets.  It reads
// only the index, so it stays host C++ inside the library (ipcg_model_*), on the plain
// ErrorModel a caller may also build by hand.
#ifndef IPCOMP_PLANNER_HPP
#define IPCOMP_PLANNER_HPP

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "ipcomp/archive.hpp"
#include "ipcomp/common.hpp"

namespace ipcomp {

struct LevelCosts {
    std::array<double, 33> delta{};               // measured loss for d dropped planes
    std::array<std::uint64_t, 32> plane_bytes{};  // serialized block size per plane
    std::uint64_t outlier_bytes = 0;
    bool progressive = false;
};

struct ErrorModel {
    int levels = 0;
    int progressive_levels = 0;
    double eb = 0.0;
    double amplification = 1.0;
    std::vector<LevelCosts> level;  // [l-1]

    const LevelCosts &at(int l) const { return level[static_cast<std::size_t>(l - 1)]; }
};

namespace b200 {
inline ipcg_error_model to_model(const ErrorModel &m) {
    if (m.levels < 0 || m.levels > IPCG_MAX_LEVELS || m.level.size() < static_cast<std::size_t>(m.levels))
        throw std::invalid_argument("error model level count out of range");
    ipcg_error_model o{};
    o.levels = m.levels;
    o.progressive_levels = m.progressive_levels;
    o.eb = m.eb;
    o.amplification = m.amplification;
    for (int l = 0; l < m.levels; ++l) {
        const LevelCosts &lc = m.level[static_cast<std::size_t>(l)];
        for (int d = 0; d < 33; ++d) o.level[l].delta[d] = lc.delta[static_cast<std::size_t>(d)];
        for (int p = 0; p < 32; ++p) o.level[l].plane_bytes[p] = lc.plane_bytes[static_cast<std::size_t>(p)];
        o.level[l].outlier_bytes = lc.outlier_bytes;
        o.level[l].progressive = lc.progressive ? 1 : 0;
    }
    return o;
}
inline const int *plan_for(const ErrorModel &m, const RetrievalPlan &plan) {
    if (plan.k.size() < static_cast<std::size_t>(m.levels))
        throw std::invalid_argument("plan level count does not match archive");
    return plan.k.data();
}
}  // namespace b200

inline ErrorModel build_error_model(const ArchiveHeader &header, std::span<const LevelRecord> records) {
    const ipcg_index ix = b200::to_index(header, records);
    ipcg_error_model cm{};
    b200::check(ipcg_build_error_model(&ix, &cm), nullptr);
    ErrorModel m;
    m.levels = cm.levels;
    m.progressive_levels = cm.progressive_levels;
    m.eb = cm.eb;
    m.amplification = cm.amplification;
    m.level.resize(static_cast<std::size_t>(cm.levels));
    for (int l = 0; l < cm.levels; ++l) {
        LevelCosts &lc = m.level[static_cast<std::size_t>(l)];
        for (int d = 0; d < 33; ++d) lc.delta[static_cast<std::size_t>(d)] = cm.level[l].delta[d];
        for (int p = 0; p < 32; ++p) lc.plane_bytes[static_cast<std::size_t>(p)] = cm.level[l].plane_bytes[p];
        lc.outlier_bytes = cm.level[l].outlier_bytes;
        lc.progressive = cm.level[l].progressive != 0;
    }
    return m;
}

inline RetrievalPlan full_plan(const ErrorModel &model) {
    return RetrievalPlan{std::vector<int>(static_cast<std::size_t>(model.levels), 32)};
}

inline double bound_for_plan(const ErrorModel &model, const RetrievalPlan &plan) {
    const ipcg_error_model m = b200::to_model(model);
    return ipcg_model_bound_for_plan(&m, b200::plan_for(model, plan));
}
inline std::uint64_t plan_payload_bytes(const ErrorModel &model, const RetrievalPlan &plan) {
    const ipcg_error_model m = b200::to_model(model);
    return ipcg_model_plan_payload_bytes(&m, b200::plan_for(model, plan));
}
inline std::uint64_t mandatory_payload_bytes(const ErrorModel &model) {
    const ipcg_error_model m = b200::to_model(model);
    return ipcg_model_mandatory_payload_bytes(&m);
}
inline std::uint64_t total_payload_bytes(const ErrorModel &model) {
    const ipcg_error_model m = b200::to_model(model);
    return ipcg_model_total_payload_bytes(&m);
}
inline RetrievalPlan plan_for_error(const ErrorModel &model, double max_error) {
    const ipcg_error_model m = b200::to_model(model);
    RetrievalPlan plan{std::vector<int>(static_cast<std::size_t>(model.levels), 32)};
    b200::check(ipcg_model_plan_for_error(&m, max_error, plan.k.data()), nullptr);
    return plan;
}
inline RetrievalPlan plan_for_size(const ErrorModel &model, std::uint64_t byte_budget) {
    const ipcg_error_model m = b200::to_model(model);
    RetrievalPlan plan{std::vector<int>(static_cast<std::size_t>(model.levels), 32)};
    b200::check(ipcg_model_plan_for_size(&m, byte_budget, plan.k.data()), nullptr);
    return plan;
}

}  // namespace ipcomp

#endif
