// ref_shim.cpp -- CPU ORACLE (test infrastructure only).
//
// Exposes the UNMODIFIED reference (compiled from /root/reference/proj/src/*.cpp
// by oracle/Makefile target `ref`, output oracle/_ref/libipcomp_ref.so) through
// a plain C surface with the same signatures as ipcomp_oracle.h, prefixed ref_.
// It is used to pin the C restatement (oracle/ipcomp_oracle.c), to generate the
// golden fixtures in tests/golden/, and as bench.py's `--impl reference` /
// cpu_baseline arm (the reference's own multi-threaded CPU code path).
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "ipcomp/pipeline.hpp"
#include "ipcomp/session.hpp"

using namespace ipcomp;

namespace {

int set_err(char *err, int errlen, const char *msg) {
    if (err && errlen > 0) std::snprintf(err, static_cast<size_t>(errlen), "%s", msg);
    return 0;
}

template <class F>
int guarded(char *err, int errlen, F &&f) {
    try {
        f();
        return 0;
    } catch (const InfeasibleRequest &e) {
        set_err(err, errlen, e.what());
        return 4;
    } catch (const std::invalid_argument &e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const std::domain_error &e) {
        set_err(err, errlen, e.what());
        return 3;
    } catch (const std::exception &e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

struct MemArchive {
    std::string bytes;
    std::istringstream in;
    ArchiveReader reader;
    MemArchive(const uint8_t *p, uint64_t n)
        : bytes(reinterpret_cast<const char *>(p), n), in(bytes, std::ios::binary), reader(in) {}
};

}  // namespace

extern "C" {

int ref_compress(int scalar, const void *values, const uint64_t *dims, int nd, double eb, int interp,
                 int progressive_levels, uint64_t anchor_cap, uint8_t **out, uint64_t *out_size, char *err,
                 int errlen) {
    return guarded(err, errlen, [&] {
        Dims d(dims, dims + nd);
        std::size_t n = 1;
        for (auto x : d) n *= x;
        CompressOptions opt;
        opt.eb = eb;
        opt.interp = interp == 1 ? InterpKind::cubic : InterpKind::linear;
        opt.progressive_levels = progressive_levels;
        opt.anchor_cap = anchor_cap;
        ArchiveData a = scalar == 0
                            ? compress_field<float>(std::span<const float>(static_cast<const float *>(values), n), d, opt)
                            : compress_field<double>(std::span<const double>(static_cast<const double *>(values), n), d, opt);
        std::ostringstream os(std::ios::binary);
        write_archive(os, a);
        const std::string s = os.str();
        *out = static_cast<uint8_t *>(std::malloc(s.size() ? s.size() : 1));
        std::memcpy(*out, s.data(), s.size());
        *out_size = s.size();
    });
}

void ref_free(void *p) { std::free(p); }

int ref_reconstruct(const uint8_t *archive, uint64_t size, int scalar, const int *k, void *out_values,
                    uint32_t **merged, uint64_t *payload_bytes_loaded, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        RetrievalPlan plan;
        plan.k.assign(k, k + m.reader.header().levels);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            auto r = reconstruct_field<T>(m.reader, plan);
            std::memcpy(out_values, r.values.data(), r.values.size() * sizeof(T));
            if (payload_bytes_loaded) *payload_bytes_loaded = r.stats.payload_bytes_loaded;
            if (merged) {
                for (std::size_t l = 0; l < r.session.level.size(); ++l) {
                    const auto &mm = r.session.level[l].merged;
                    if (l + 1 > m.reader.header().progressive_levels) {
                        merged[l] = nullptr;
                        continue;
                    }
                    merged[l] = static_cast<uint32_t *>(std::malloc(mm.size() * 4 + 4));
                    std::memcpy(merged[l], mm.data(), mm.size() * 4);
                }
            }
        };
        if (scalar == 0) run(float{});
        else run(double{});
    });
}

int ref_refine(const uint8_t *archive, uint64_t size, int scalar, const int *session_k, uint32_t *const *session_merged,
               const void *previous, const int *target_k, void *out_values, uint32_t **merged_out,
               uint64_t *payload_bytes_loaded, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        const auto &h = m.reader.header();
        RetrievalSession sess;
        sess.archive_crc = m.reader.identity();
        sess.level.resize(h.levels);
        for (int l = 0; l < h.levels; ++l) {
            sess.level[l].planes_loaded = session_k[l];
            if (l + 1 <= h.progressive_levels) {
                const auto cnt = m.reader.record(l + 1).count;
                sess.level[l].merged.assign(session_merged[l], session_merged[l] + cnt);
            }
        }
        RetrievalPlan plan;
        plan.k.assign(target_k, target_k + h.levels);
        std::size_t n = 1;
        for (auto x : h.dims) n *= x;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            auto r = refine_field<T>(m.reader, sess, std::span<const T>(static_cast<const T *>(previous), n), plan);
            std::memcpy(out_values, r.values.data(), r.values.size() * sizeof(T));
            if (payload_bytes_loaded) *payload_bytes_loaded = r.stats.payload_bytes_loaded;
            for (int l = 0; l < h.levels; ++l) {
                const auto &mm = r.session.level[l].merged;
                if (l + 1 > h.progressive_levels) {
                    merged_out[l] = nullptr;
                    continue;
                }
                merged_out[l] = static_cast<uint32_t *>(std::malloc(mm.size() * 4 + 4));
                std::memcpy(merged_out[l], mm.data(), mm.size() * 4);
            }
        };
        if (scalar == 0) run(float{});
        else run(double{});
    });
}

// write_session (session.cpp:8-24) of the session {k, merged} bound to `archive`
int ref_write_session(const uint8_t *archive, uint64_t size, const int *session_k, uint32_t *const *session_merged,
                      uint8_t **out, uint64_t *out_size, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        const auto &h = m.reader.header();
        RetrievalSession sess;
        sess.archive_crc = m.reader.identity();
        sess.level.resize(h.levels);
        for (int l = 0; l < h.levels; ++l) {
            sess.level[l].planes_loaded = session_k[l];
            if (l + 1 <= h.progressive_levels && session_merged[l]) {
                const auto cnt = m.reader.record(l + 1).count;
                sess.level[l].merged.assign(session_merged[l], session_merged[l] + cnt);
            }
        }
        std::ostringstream os(std::ios::binary);
        write_session(os, sess);
        const std::string b = os.str();
        *out = static_cast<uint8_t *>(std::malloc(b.size() + 1));
        std::memcpy(*out, b.data(), b.size());
        *out_size = b.size();
    });
}

// read_session (session.cpp:26-61); merged_out[l] malloc'd for progressive levels
int ref_read_session(const uint8_t *archive, uint64_t size, const uint8_t *bytes, uint64_t n, int *k_out,
                     uint32_t **merged_out, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        std::string b(reinterpret_cast<const char *>(bytes), n);
        std::istringstream is(b, std::ios::binary);
        const RetrievalSession sess = read_session(is, m.reader);
        for (std::size_t l = 0; l < sess.level.size(); ++l) {
            k_out[l] = sess.level[l].planes_loaded;
            const auto &mm = sess.level[l].merged;
            if (l + 1 > (std::size_t)m.reader.header().progressive_levels) {
                merged_out[l] = nullptr;
                continue;
            }
            merged_out[l] = static_cast<uint32_t *>(std::malloc(mm.size() * 4 + 4));
            std::memcpy(merged_out[l], mm.data(), mm.size() * 4);
        }
    });
}

// compute_metrics<T> (pipeline.hpp:354-372)
int ref_compute_metrics(int scalar, const void *original, const void *decoded, uint64_t n, double *out) {
    auto run = [&](auto tag) {
        using T = decltype(tag);
        const auto m = compute_metrics<T>(std::span<const T>(static_cast<const T *>(original), n),
                                          std::span<const T>(static_cast<const T *>(decoded), n));
        out[0] = m.max_error;
        out[1] = m.mse;
        out[2] = m.psnr;
    };
    if (scalar == 0) run(float{});
    else run(double{});
    return 0;
}

int ref_plan_for_error(const uint8_t *archive, uint64_t size, double max_error, int *k_out, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        auto model = build_error_model(m.reader.header(), m.reader.records());
        auto plan = plan_for_error(model, max_error);
        std::copy(plan.k.begin(), plan.k.end(), k_out);
    });
}

int ref_plan_for_size(const uint8_t *archive, uint64_t size, uint64_t budget, int *k_out, char *err, int errlen) {
    return guarded(err, errlen, [&] {
        MemArchive m(archive, size);
        auto model = build_error_model(m.reader.header(), m.reader.records());
        auto plan = plan_for_size(model, budget);
        std::copy(plan.k.begin(), plan.k.end(), k_out);
    });
}

double ref_bound_for_plan(const uint8_t *archive, uint64_t size, const int *k) {
    MemArchive m(archive, size);
    auto model = build_error_model(m.reader.header(), m.reader.records());
    RetrievalPlan plan;
    plan.k.assign(k, k + m.reader.header().levels);
    return bound_for_plan(model, plan);
}

uint64_t ref_plan_payload_bytes(const uint8_t *archive, uint64_t size, const int *k) {
    MemArchive m(archive, size);
    auto model = build_error_model(m.reader.header(), m.reader.records());
    RetrievalPlan plan;
    plan.k.assign(k, k + m.reader.header().levels);
    return plan_payload_bytes(model, plan);
}

int ref_backend_encode(const uint8_t *raw, uint64_t n, int preferred, uint8_t **payload, uint64_t *payload_len,
                       int *backend, uint32_t *crc) {
    auto b = backend_encode(std::span<const uint8_t>(raw, n), preferred ? Backend::deflate : Backend::identity, n * 8);
    *payload = static_cast<uint8_t *>(std::malloc(b.payload.size() + 1));
    std::memcpy(*payload, b.payload.data(), b.payload.size());
    *payload_len = b.payload.size();
    *backend = static_cast<int>(b.backend);
    *crc = b.checksum;
    return 0;
}

}  // extern "C"
