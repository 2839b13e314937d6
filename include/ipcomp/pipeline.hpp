// ipcomp/pipeline.hpp -- the public compress / retrieve API of the reference's
// proj/include/ipcomp/pipeline.hpp, source-compatible, on the B200 library:
//   compress_field<T>    (pipeline.hpp:140-223)  -> ipcg_compress: every pass, the loss tables,
//                         the bitplanes and the zlib-exact deflate run as sm_100a kernels
//   reconstruct_field<T> (pipeline.hpp:260-287)  -> ipcg_reconstruct: partial-bitplane fetch of
//                         the planned blocks only, device inflate, merge, reconstruction
//   refine_field<T>      (pipeline.hpp:294-352)  -> ipcg_refine
//   compute_metrics<T>   (pipeline.hpp:354-372)  -> ipcg_compute_metrics
// Types, argument meanings, results and exception types/messages are the reference's; results
// are bit-identical to it (archive bytes, reconstructed values, session codewords).
#ifndef IPCOMP_PIPELINE_HPP
#define IPCOMP_PIPELINE_HPP

#include <cmath>
#include <cstdint>
#include <limits>
#include <span>
#include <utility>
#include <vector>

#include "ipcomp/archive.hpp"
#include "ipcomp/backend.hpp"
#include "ipcomp/bitplane.hpp"
#include "ipcomp/grid.hpp"
#include "ipcomp/planner.hpp"
#include "ipcomp/predictor.hpp"
#include "ipcomp/quantizer.hpp"
#include "ipcomp/session.hpp"

namespace ipcomp {

template <class T>
constexpr ScalarKind scalar_kind_of() {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "field scalars must be f32 or f64");
    return sizeof(T) == 4 ? ScalarKind::f32 : ScalarKind::f64;
}

struct CompressOptions {
    double eb = 0.0;
    InterpKind interp = InterpKind::cubic;
    int progressive_levels = 0;  // 0 selects every level
    std::size_t anchor_cap = kDefaultAnchorStrideCap;
};

struct ReconstructStats {
    std::vector<int> level_visits;
    std::uint64_t payload_bytes_loaded = 0;
};

template <class T>
struct Retrieved {
    std::vector<T> values;
    RetrievalSession session;
    ReconstructStats stats;
};

struct FieldMetrics {
    double max_error = 0.0;
    double mse = 0.0;
    double psnr = 0.0;
};

namespace b200 {

struct SessionFree {
    void operator()(ipcg_session *s) const { ipcg_session_free(s); }
};
using SessionHandle = std::unique_ptr<ipcg_session, SessionFree>;

// host copies of a device session's codewords, for the progressive levels the call touched
inline void fetch_session(ipcg_ctx *c, const ipcg_session *s, const ArchiveHeader &h, const std::vector<int> &k,
                          RetrievalSession &out, bool only_progressive_update) {
    for (int level = 1; level <= h.levels; ++level) {
        RetrievalSession::LevelState &ls = out.level[static_cast<std::size_t>(level - 1)];
        if (level > h.progressive_levels) {
            if (!only_progressive_update) ls.planes_loaded = k[static_cast<std::size_t>(level - 1)], ls.merged.clear();
            continue;
        }
        ls.planes_loaded = k[static_cast<std::size_t>(level - 1)];
        ls.merged.resize(static_cast<std::size_t>(ipcg_session_count(s, level)));
        if (!ls.merged.empty()) check(ipcg_session_merged(c, s, level, ls.merged.data(), 0), c);
    }
}

template <class T>
ScalarKind require_scalar(const ArchiveHeader &h) {
    if (h.scalar != scalar_kind_of<T>()) throw std::invalid_argument("scalar kind does not match archive");
    return h.scalar;
}

}  // namespace b200

template <class T>
ArchiveData compress_field(std::span<const T> values, const Dims &dims, const CompressOptions &opt) {
    validate_dims(dims);
    if (values.size() != element_count(dims)) throw std::invalid_argument("value count does not match dimensions");
    if (!(opt.eb > 0.0) || !std::isfinite(opt.eb)) throw std::invalid_argument("error bound must be positive and finite");
    std::uint64_t d[4] = {0, 0, 0, 0};
    for (std::size_t i = 0; i < dims.size(); ++i) d[i] = dims[i];
    ArchiveData out;
    b200::call([&](ipcg_ctx *c) {
        ipcg_archive *raw = nullptr;
        b200::check(ipcg_compress(c, static_cast<int>(scalar_kind_of<T>()), values.data(), 0, d,
                                  static_cast<int>(dims.size()), opt.eb, static_cast<int>(opt.interp),
                                  opt.progressive_levels, static_cast<std::uint64_t>(opt.anchor_cap), &raw),
                    c);
        b200::ArchiveHandle a(raw);
        ipcg_index ix{};
        ipcg_archive_index(a.get(), &ix);
        b200::from_index(ix, out.header, out.records);
        out.payload.resize(static_cast<std::size_t>(ix.payload_bytes));
        b200::check(ipcg_archive_copy(c, a.get(), ix.index_bytes, ix.payload_bytes, out.payload.data(), 0), c);
    });
    return out;
}

template <class T>
Retrieved<T> reconstruct_field(ArchiveReader &archive, const RetrievalPlan &plan) {
    const ArchiveHeader &h = archive.header();
    const ScalarKind sk = b200::require_scalar<T>(h);
    validate_plan(h, plan);
    Retrieved<T> out;
    out.values.resize(element_count(h.dims));
    out.session.archive_crc = archive.identity();
    out.session.level.resize(h.levels);
    b200::call([&](ipcg_ctx *c) {
        ipcg_session *raw = nullptr;
        ipcg_retrieve_stats st{};
        b200::check(ipcg_reconstruct(c, archive.handle(), static_cast<int>(sk), plan.k.data(), out.values.data(), 0,
                                     out.values.size(), &raw, &st),
                    c);
        b200::SessionHandle s(raw);
        b200::fetch_session(c, s.get(), h, plan.k, out.session, false);
        out.stats.level_visits.assign(st.level_visits, st.level_visits + h.levels);
        out.stats.payload_bytes_loaded = st.payload_bytes_loaded;
    });
    return out;
}

template <class T>
Retrieved<T> refine_field(ArchiveReader &archive, const RetrievalSession &session, std::span<const T> previous,
                          const RetrievalPlan &target) {
    const ArchiveHeader &h = archive.header();
    const ScalarKind sk = b200::require_scalar<T>(h);
    validate_plan(h, target);
    if (session.archive_crc != archive.identity()) throw std::runtime_error("session does not belong to this archive");
    if (session.level.size() != h.levels) throw std::runtime_error("session level count does not match archive");
    if (previous.size() != element_count(h.dims)) throw std::invalid_argument("previous reconstruction has wrong size");
    for (int level = 1; level <= h.levels; ++level)
        if (target.k[static_cast<std::size_t>(level - 1)] < session.level[static_cast<std::size_t>(level - 1)].planes_loaded)
            throw std::invalid_argument("refinement plan must not drop planes the session already loaded");
    // the session's codewords go back to the device (sessions are plain values in this API)
    std::vector<int> k0(h.levels, 32);
    std::vector<const std::uint32_t *> merged(h.levels, nullptr);
    for (int level = h.levels; level >= 1; --level) {
        if (level > h.progressive_levels) continue;
        const RetrievalSession::LevelState &ls = session.level[static_cast<std::size_t>(level - 1)];
        if (ls.merged.size() != archive.record(level).count)
            throw std::runtime_error("session codeword array has wrong length");
        if (ls.planes_loaded < 0) throw std::invalid_argument("plane index out of range");
        k0[static_cast<std::size_t>(level - 1)] = ls.planes_loaded;
        merged[static_cast<std::size_t>(level - 1)] = ls.merged.data();
    }
    Retrieved<T> out;
    out.values.resize(previous.size());
    out.session = session;
    b200::call([&](ipcg_ctx *c) {
        ipcg_session *prev = nullptr;
        b200::check(ipcg_session_create(c, archive.handle(), k0.data(), merged.data(), &prev), c);
        b200::SessionHandle ps(prev);
        ipcg_session *raw = nullptr;
        ipcg_retrieve_stats st{};
        b200::check(ipcg_refine(c, archive.handle(), static_cast<int>(sk), ps.get(), previous.data(), 0, previous.size(),
                                target.k.data(), out.values.data(), 0, out.values.size(), &raw, &st),
                    c);
        b200::SessionHandle s(raw);
        b200::fetch_session(c, s.get(), h, target.k, out.session, true);
        out.stats.level_visits.assign(st.level_visits, st.level_visits + h.levels);
        out.stats.payload_bytes_loaded = st.payload_bytes_loaded;
    });
    return out;
}

template <class T>
FieldMetrics compute_metrics(std::span<const T> original, std::span<const T> decoded) {
    if (original.size() != decoded.size()) throw std::invalid_argument("metrics inputs differ in size");
    FieldMetrics m;
    b200::call([&](ipcg_ctx *c) {
        b200::check(ipcg_compute_metrics(c, static_cast<int>(scalar_kind_of<T>()), original.data(), 0, original.size(),
                                         decoded.data(), 0, decoded.size(), &m.max_error, &m.mse, &m.psnr),
                    c);
    });
    return m;
}

}  // namespace ipcomp

#endif
