// ipcomp_b200.hpp -- the DEVICE-RESIDENT extension API (namespace ipcomp_b200), header-only
// over the C-ABI in ipcomp_b200.h.  The source-compatible drop-in for the reference's public
// API is include/ipcomp/*.hpp (namespace ipcomp; the reference's own acceptance.cpp and unit
// tests compile against it unchanged).  This header is for callers who keep archives,
// sessions and fields in HBM across calls: compress_field returns the device-resident archive,
// sessions keep their merged codewords on the device, and every call takes an explicit
// Context (one CUDA device + stream).  Names and exception types follow the reference.
#ifndef IPCOMP_B200_HPP
#define IPCOMP_B200_HPP

#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "ipcomp_b200.h"

namespace ipcomp_b200 {

enum class ScalarKind : std::uint8_t { f32 = 0, f64 = 1 };       // common.hpp:14
enum class InterpKind : std::uint8_t { linear = 0, cubic = 1 };  // common.hpp:15
using Dims = std::vector<std::size_t>;                           // common.hpp:28
inline constexpr std::size_t kDefaultAnchorStrideCap = 64;       // grid.hpp:12

// common.hpp:23-25
struct InfeasibleRequest : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// device failures (no reference counterpart)
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
[[noreturn]] inline void raise(int code, const char *msg) {
    const std::string m = msg ? msg : "ipcomp_b200 error";
    switch (code) {
        case IPCG_EINVAL: throw std::invalid_argument(m);
        case IPCG_EDOMAIN: throw std::domain_error(m);
        case IPCG_EINFEASIBLE: throw InfeasibleRequest(m);
        case IPCG_ECUDA: throw CudaError(m);
        default: throw std::runtime_error(m);
    }
}
inline void check_plan_size(const ipcg_index &h, const std::vector<int> &k) {  // archive.cpp:203
    if (k.size() != h.levels) throw std::invalid_argument("plan level count does not match archive");
}
template <class T>
constexpr int scalar_of() {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "field must be float or double");
    return std::is_same_v<T, float> ? 0 : 1;
}
}  // namespace detail

class Context {
   public:
    explicit Context(int device = 0) {
        ipcg_ctx *c = nullptr;
        const int rc = ipcg_ctx_create(device, &c);
        if (rc) detail::raise(rc, "cannot create an ipcomp_b200 context (no CUDA device?)");
        c_.reset(c);
    }
    static Context &default_context() {
        static Context ctx(0);
        return ctx;
    }
    ipcg_ctx *get() const { return c_.get(); }
    void check(int rc) const {
        if (rc) detail::raise(rc, ipcg_last_error(c_.get()));
    }
    void set_stream(void *cuda_stream) { check(ipcg_set_stream(get(), cuda_stream)); }
    void synchronize() { check(ipcg_synchronize(get())); }
    void set_host_async(bool enable) { check(ipcg_set_host_async(get(), enable ? 1 : 0)); }

   private:
    struct Del {
        void operator()(ipcg_ctx *c) const { ipcg_ctx_destroy(c); }
    };
    std::unique_ptr<ipcg_ctx, Del> c_;
};

// pipeline.hpp:30-35
struct CompressOptions {
    double eb = 0.0;
    InterpKind interp = InterpKind::cubic;
    int progressive_levels = 0;  // 0 selects every level
    std::size_t anchor_cap = kDefaultAnchorStrideCap;
};

// archive.hpp:59-61
struct RetrievalPlan {
    std::vector<int> k;
};

// The archive: ArchiveData (archive.hpp:49-53) and ArchiveReader (archive.hpp:67-114) in
// one handle.  compress_field returns it device-resident; the istream constructor reads a
// serialized archive into host memory like the reference reader.
class ArchiveReader {
   public:
    explicit ArchiveReader(std::istream &in, Context &ctx = Context::default_context()) : ctx_(&ctx) {
        host_.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
        open(host_.data(), host_.size(), 0);
    }
    // borrow serialized bytes in caller memory (host or device); they must outlive the reader
    ArchiveReader(const void *bytes, std::uint64_t size, bool on_device, Context &ctx = Context::default_context())
        : ctx_(&ctx) {
        open(bytes, size, on_device ? 1 : 0);
    }
    ArchiveReader(ipcg_archive *owned, Context &ctx) : ctx_(&ctx), a_(owned) { load_index(); }

    const ipcg_index &header() const { return ix_; }  // header + records (archive.hpp:19-46)
    const ipcg_level_record &record(int level) const {
        if (level < 1 || level > ix_.levels) throw std::out_of_range("level out of range");
        return ix_.records[level - 1];
    }
    std::uint32_t identity() const { return ix_.identity; }
    std::uint64_t index_bytes() const { return ix_.index_bytes; }
    std::uint64_t payload_bytes_read() const { return ipcg_archive_payload_bytes_read(a_.get()); }
    std::uint64_t size() const { return ipcg_archive_size(a_.get()); }
    ipcg_archive *get() const { return a_.get(); }
    Context &context() const { return *ctx_; }

    // write_archive (archive.cpp:72-81)
    void write(std::ostream &out) const {
        std::vector<char> buf(size());
        ctx_->check(ipcg_archive_write(ctx_->get(), a_.get(), buf.data(), 0, buf.size()));
        out.write(buf.data(), (std::streamsize)buf.size());
        if (!out) throw std::runtime_error("failed to write archive");
    }
    std::vector<std::uint8_t> bytes() const {
        std::vector<std::uint8_t> buf(size());
        ctx_->check(ipcg_archive_write(ctx_->get(), a_.get(), buf.data(), 0, buf.size()));
        return buf;
    }

   private:
    void open(const void *bytes, std::uint64_t size, int on_device) {
        ipcg_archive *a = nullptr;
        ctx_->check(ipcg_archive_open(ctx_->get(), bytes, size, on_device, &a));
        a_.reset(a);
        load_index();
    }
    void load_index() { ctx_->check(ipcg_archive_index(a_.get(), &ix_)); }
    struct Del {
        void operator()(ipcg_archive *a) const { ipcg_archive_free(a); }
    };
    Context *ctx_;
    std::vector<char> host_;
    std::unique_ptr<ipcg_archive, Del> a_;
    ipcg_index ix_{};
};

inline void write_archive(std::ostream &out, const ArchiveReader &archive) { archive.write(out); }

// session.hpp:19-34: merged codewords stay device-resident
class RetrievalSession {
   public:
    RetrievalSession() = default;
    explicit RetrievalSession(ipcg_session *s) : s_(s, Del{}) {}
    bool valid() const { return (bool)s_; }
    std::uint32_t archive_crc() const { return s_ ? ipcg_session_archive_crc(s_.get()) : 0u; }
    RetrievalPlan plan() const {
        RetrievalPlan p;
        if (!s_) return p;
        p.k.resize((std::size_t)ipcg_session_levels(s_.get()));
        ipcg_session_planes_loaded(s_.get(), p.k.data());
        return p;
    }
    ipcg_session *get() const { return s_.get(); }

   private:
    struct Del {
        void operator()(ipcg_session *s) const { ipcg_session_free(s); }
    };
    std::shared_ptr<ipcg_session> s_{nullptr, Del{}};
};

// pipeline.hpp:37-47
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

// compress_field<T> (pipeline.hpp:140-223); `values` in host memory
template <class T>
ArchiveReader compress_field(std::span<const T> values, const Dims &dims, const CompressOptions &opt,
                             Context &ctx = Context::default_context()) {
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    std::uint64_t count = 1;
    for (auto x : dims) count *= x;
    if (!dims.empty() && dims.size() <= 4 && count != values.size())
        throw std::invalid_argument("value count does not match the grid");
    ipcg_archive *a = nullptr;
    ctx.check(ipcg_compress(ctx.get(), detail::scalar_of<T>(), values.data(), 0, d.data(), (int)d.size(), opt.eb,
                            (int)opt.interp, opt.progressive_levels, opt.anchor_cap, &a));
    return ArchiveReader(a, ctx);
}

// reconstruct_field<T> (pipeline.hpp:260-287)
template <class T>
Retrieved<T> reconstruct_field(ArchiveReader &archive, const RetrievalPlan &plan) {
    Context &ctx = archive.context();
    detail::check_plan_size(archive.header(), plan.k);
    std::uint64_t count = 1;
    for (int i = 0; i < archive.header().ndims; ++i) count *= archive.header().dims[i];
    Retrieved<T> out;
    out.values.resize(count);
    ipcg_session *s = nullptr;
    ipcg_retrieve_stats st{};
    ctx.check(ipcg_reconstruct(ctx.get(), archive.get(), detail::scalar_of<T>(), plan.k.data(), out.values.data(), 0,
                               out.values.size(), &s, &st));
    out.stats.payload_bytes_loaded = st.payload_bytes_loaded;
    out.stats.level_visits.assign(st.level_visits, st.level_visits + archive.header().levels);
    out.session = RetrievalSession(s);
    return out;
}

// refine_field<T> (pipeline.hpp:294-352)
template <class T>
Retrieved<T> refine_field(ArchiveReader &archive, const RetrievalSession &session, std::span<const T> previous,
                          const RetrievalPlan &target) {
    Context &ctx = archive.context();
    detail::check_plan_size(archive.header(), target.k);
    Retrieved<T> out;
    out.values.resize(previous.size());
    ipcg_session *s = nullptr;
    ipcg_retrieve_stats st{};
    ctx.check(ipcg_refine(ctx.get(), archive.get(), detail::scalar_of<T>(), session.get(), previous.data(), 0,
                          previous.size(), target.k.data(), out.values.data(), 0, out.values.size(), &s, &st));
    out.stats.payload_bytes_loaded = st.payload_bytes_loaded;
    out.stats.level_visits.assign(st.level_visits, st.level_visits + archive.header().levels);
    out.session = RetrievalSession(s);
    return out;
}

// write_session / read_session (session.hpp:36-40, session.cpp:8-61): the merged codewords
// are deflated / inflated on the device
inline void write_session(std::ostream &out, const RetrievalSession &session,
                          Context &ctx = Context::default_context()) {
    std::vector<char> buf(ipcg_session_write_bound(session.get()));
    std::uint64_t size = 0;
    ctx.check(ipcg_session_write(ctx.get(), session.get(), buf.data(), 0, buf.size(), &size));
    out.write(buf.data(), (std::streamsize)size);
    if (!out) throw std::runtime_error("failed to write session stream");
}
inline RetrievalSession read_session(std::istream &in, const ArchiveReader &archive) {
    std::vector<char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    ipcg_session *s = nullptr;
    archive.context().check(
        ipcg_session_read(archive.context().get(), archive.get(), bytes.data(), bytes.size(), 0, &s));
    return RetrievalSession(s);
}

// FieldMetrics / compute_metrics<T> (pipeline.hpp:49-53,354-372), one pass on the device
struct FieldMetrics {
    double max_error = 0.0;
    double mse = 0.0;
    double psnr = 0.0;
};
template <class T>
FieldMetrics compute_metrics(std::span<const T> original, std::span<const T> decoded,
                             Context &ctx = Context::default_context()) {
    FieldMetrics m;
    ctx.check(ipcg_compute_metrics(ctx.get(), detail::scalar_of<T>(), original.data(), 0, original.size(),
                                   decoded.data(), 0, decoded.size(), &m.max_error, &m.mse, &m.psnr));
    return m;
}

// planner.hpp:15-55 over the archive's index (the ErrorModel is the index itself)
inline const ArchiveReader &build_error_model(const ArchiveReader &a) { return a; }
inline RetrievalPlan full_plan(const ArchiveReader &a) {
    RetrievalPlan p;
    p.k.assign((std::size_t)a.header().levels, 32);
    return p;
}
inline RetrievalPlan plan_for_error(const ArchiveReader &a, double max_error) {
    RetrievalPlan p;
    p.k.resize((std::size_t)a.header().levels);
    a.context().check(ipcg_plan_for_error(a.context().get(), a.get(), max_error, p.k.data()));
    return p;
}
inline RetrievalPlan plan_for_size(const ArchiveReader &a, std::uint64_t byte_budget) {
    RetrievalPlan p;
    p.k.resize((std::size_t)a.header().levels);
    a.context().check(ipcg_plan_for_size(a.context().get(), a.get(), byte_budget, p.k.data()));
    return p;
}
inline double bound_for_plan(const ArchiveReader &a, const RetrievalPlan &plan) {
    detail::check_plan_size(a.header(), plan.k);
    return ipcg_bound_for_plan(a.get(), plan.k.data());
}
inline std::uint64_t plan_payload_bytes(const ArchiveReader &a, const RetrievalPlan &plan) {
    detail::check_plan_size(a.header(), plan.k);
    return ipcg_plan_payload_bytes(a.get(), plan.k.data());
}

}  // namespace ipcomp_b200

#endif
