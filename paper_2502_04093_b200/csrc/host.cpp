// host.cpp -- index format and retrieval planner of the reference, host C++.
//   serialize/parse: proj/src/archive.cpp:12-170, format proj/README.md:87-106
//   planner:         proj/src/planner.cpp:30-290 (1024 ceiling buckets, knapsack DP)
#include "host.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "util.cuh"

namespace ipcg {

namespace {

uint32_t crc_table[256];
bool crc_init = false;

void put(std::vector<uint8_t> &w, uint64_t v, int nb) {
    for (int i = 0; i < nb; ++i) w.push_back((uint8_t)(v >> (8 * i)));
}
uint64_t f2u(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}
double u2f(uint64_t u) {
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}

void check_header(const ipcg_index &h) {  // archive.cpp:12-21
    if (h.version != 1) throw Error(ERUNTIME, "unsupported archive version");
    if (h.ndims < 1 || h.ndims > 4) throw Error(EINVAL_, "grid must have between 1 and 4 dimensions");
    for (int i = 0; i < h.ndims; ++i)
        if (h.dims[i] < 1) throw Error(EINVAL_, "grid extents must be positive");
    if (h.levels < 1) throw Error(ERUNTIME, "archive has no levels");
    if (h.progressive_levels < 1 || h.progressive_levels > h.levels)
        throw Error(ERUNTIME, "progressive level bound out of range");
    if (!(h.eb > 0.0) || !std::isfinite(h.eb)) throw Error(ERUNTIME, "archive error bound is not positive");
}

void check_record(const ipcg_level_record &r) {  // archive.cpp:23-28
    if (r.delta[0] != 0.0) throw Error(ERUNTIME, "loss table must start at zero");
    for (int d = 1; d <= 32; ++d)
        if (!(r.delta[d] >= r.delta[d - 1])) throw Error(ERUNTIME, "loss table must be non-decreasing");
}

// The reference's IndexParser (archive.cpp:87-113) takes one field at a time from its stream;
// `more` (optional) appends the next `need` bytes of a seekable source to `buf`, so the index
// is read field by field and never past its end.
struct Reader {
    const uint8_t *p;
    uint64_t n, pos = 0;
    std::vector<uint8_t> *buf = nullptr;
    const IndexSource *more = nullptr;
    uint64_t get(int nb) {
        if (n - pos < (uint64_t)nb && more) {
            const uint64_t need = pos + (uint64_t)nb - n;
            buf->resize(n + need);
            const int64_t got = more->read(more->user, n, buf->data() + n, need);
            n += got > 0 ? std::min<uint64_t>((uint64_t)got, need) : 0;
            buf->resize(n);
            p = buf->data();
        }
        if (n - pos < (uint64_t)nb) throw Error(ERUNTIME, "truncated archive index");
        uint64_t v = 0;
        for (int i = 0; i < nb; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
        pos += (uint64_t)nb;
        return v;
    }
};

}  // namespace

uint32_t crc32_host(const uint8_t *p, size_t n, uint32_t crc) {
    if (!crc_init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
            crc_table[i] = c;
        }
        crc_init = true;
    }
    uint32_t c = crc ^ 0xffffffffu;
    for (size_t i = 0; i < n; ++i) c = crc_table[(c ^ p[i]) & 0xff] ^ (c >> 8);
    return c ^ 0xffffffffu;
}

std::vector<uint8_t> serialize_index(const ipcg_index &h) {
    check_header(h);
    std::vector<uint8_t> w;
    w.reserve(64 + 808 * h.levels);
    w.insert(w.end(), {'I', 'P', 'C', '1'});
    put(w, h.version, 2);
    put(w, h.scalar, 1);
    put(w, h.interp, 1);
    put(w, h.ndims, 1);
    put(w, 0, 3);
    for (int i = 0; i < h.ndims; ++i) put(w, h.dims[i], 8);
    put(w, f2u(h.eb), 8);
    put(w, h.levels, 1);
    put(w, h.progressive_levels, 1);
    put(w, h.anchor_cap, 1);
    put(w, 0, 1);
    put(w, f2u(h.range), 8);
    for (int level = h.levels; level >= 1; --level) {
        const ipcg_level_record &r = h.records[level - 1];
        check_record(r);
        put(w, r.count, 8);
        for (int d = 0; d < 33; ++d) put(w, f2u(r.delta[d]), 8);
        put(w, r.outlier_offset, 8);
        put(w, r.outlier_length, 8);
        put(w, r.outlier_count, 8);
        for (int p = 0; p < 32; ++p) {
            put(w, r.plane_offset[p], 8);
            put(w, r.plane_length[p], 8);
        }
    }
    return w;
}

namespace {
void parse_index_impl(Reader &r, ipcg_index &h) {
    std::memset(&h, 0, sizeof h);
    const uint64_t magic = r.get(4);
    if (magic != 0x31435049ull) throw Error(ERUNTIME, "not an archive: bad magic");  // "IPC1"
    h.version = (uint16_t)r.get(2);
    if (h.version != 1) throw Error(ERUNTIME, "unsupported archive version");
    h.scalar = (uint8_t)r.get(1);
    if (h.scalar > 1) throw Error(ERUNTIME, "unknown scalar kind");
    h.interp = (uint8_t)r.get(1);
    if (h.interp > 1) throw Error(ERUNTIME, "unknown interpolation kind");
    h.ndims = (uint8_t)r.get(1);
    r.get(1);
    r.get(1);
    r.get(1);
    if (h.ndims < 1 || h.ndims > 4) throw Error(ERUNTIME, "dimension count out of range");
    for (int i = 0; i < h.ndims; ++i) h.dims[i] = r.get(8);
    h.eb = u2f(r.get(8));
    h.levels = (uint8_t)r.get(1);
    h.progressive_levels = (uint8_t)r.get(1);
    h.anchor_cap = (uint8_t)r.get(1);
    r.get(1);
    h.range = u2f(r.get(8));
    check_header(h);
    if (h.levels > IPCG_MAX_LEVELS) throw Error(ERUNTIME, "archive has more levels than supported");
    for (int level = h.levels; level >= 1; --level) {
        ipcg_level_record &rec = h.records[level - 1];
        rec.count = r.get(8);
        for (int d = 0; d < 33; ++d) rec.delta[d] = u2f(r.get(8));
        rec.outlier_offset = r.get(8);
        rec.outlier_length = r.get(8);
        rec.outlier_count = r.get(8);
        for (int p = 0; p < 32; ++p) {
            rec.plane_offset[p] = r.get(8);
            rec.plane_length[p] = r.get(8);
        }
        check_record(rec);
    }
    h.index_bytes = r.pos;
    h.identity = crc32_host(r.p, r.pos);
    // archive.cpp:164-169 (the same wrapping u64 sums as the reference)
    uint64_t end = 0;
    for (int l = 0; l < h.levels; ++l) {
        const ipcg_level_record &rec = h.records[l];
        end = std::max(end, rec.outlier_offset + rec.outlier_length);
        for (int p = 0; p < 32; ++p) end = std::max(end, rec.plane_offset[p] + rec.plane_length[p]);
    }
    h.payload_bytes = end;
}
}  // namespace

void parse_index(const uint8_t *bytes, uint64_t avail, ipcg_index &h) {
    Reader r{bytes, avail};
    parse_index_impl(r, h);
}

void parse_index(const IndexSource &src, ipcg_index &h) {
    std::vector<uint8_t> buf;
    Reader r{nullptr, 0, 0, &buf, &src};
    parse_index_impl(r, h);
}

void validate_plan(const ipcg_index &h, const int *k) {
    for (int level = 1; level <= h.levels; ++level) {
        const int kk = k[level - 1];
        if (kk < 0 || kk > 32) throw Error(EINVAL_, "plan plane count out of range");
        if (level > h.progressive_levels && kk != 32) throw Error(EINVAL_, "non-progressive levels must load all planes");
    }
}

// ------------------------------------------------------------------ planner
// planner.cpp:30-290 over the plain model (planner.hpp:13-32); the index-based entry points
// build the model first, as build_error_model does.
namespace {

constexpr int kBuckets = 1024;
constexpr int kInfCost = kBuckets + 1;

double weight(const ipcg_error_model &m, int level) { return std::pow(m.amplification, level - 1); }
const ipcg_level_costs &at(const ipcg_error_model &m, int level) { return m.level[level - 1]; }
uint64_t optional_bytes(const ipcg_level_costs &lc, int dropped) {
    uint64_t s = 0;
    for (int p = 0; p < 32 - dropped; ++p) s += lc.plane_bytes[p];
    return s;
}

struct Choice {
    int dropped, cost;
    uint64_t bytes;
    double err;
};

}  // namespace

void check_model(const ipcg_error_model &m) {
    if (m.levels < 0 || m.levels > IPCG_MAX_LEVELS) throw Error(EINVAL_, "error model level count out of range");
    if (m.progressive_levels < 0 || m.progressive_levels > m.levels)
        throw Error(EINVAL_, "error model progressive level count out of range");
}

void build_error_model(const ipcg_index &h, ipcg_error_model &m) {  // planner.cpp:30-45
    std::memset(&m, 0, sizeof m);
    m.levels = h.levels;
    m.progressive_levels = h.progressive_levels;
    m.eb = h.eb;
    m.amplification = h.interp == 1 ? 1.25 : 1.0;  // predictor.hpp:12 amplification()
    for (int l = 0; l < h.levels; ++l) {
        ipcg_level_costs &lc = m.level[l];
        std::memcpy(lc.delta, h.records[l].delta, sizeof lc.delta);
        for (int p = 0; p < 32; ++p) lc.plane_bytes[p] = h.records[l].plane_length[p];
        lc.outlier_bytes = h.records[l].outlier_length;
        lc.progressive = l + 1 <= h.progressive_levels;
    }
}

double bound_for_plan(const ipcg_error_model &m, const int *k) {
    double sum = 0.0;
    for (int l = 1; l <= m.levels; ++l) sum += weight(m, l) * at(m, l).delta[32 - k[l - 1]];
    return sum + m.eb;
}

uint64_t mandatory_payload_bytes(const ipcg_error_model &m) {
    uint64_t s = 0;
    for (int l = 1; l <= m.levels; ++l) {
        s += at(m, l).outlier_bytes;
        if (!at(m, l).progressive) s += optional_bytes(at(m, l), 0);
    }
    return s;
}

uint64_t total_payload_bytes(const ipcg_error_model &m) {
    uint64_t s = 0;
    for (int l = 1; l <= m.levels; ++l) s += at(m, l).outlier_bytes + optional_bytes(at(m, l), 0);
    return s;
}

uint64_t plan_payload_bytes(const ipcg_error_model &m, const int *k) {
    uint64_t s = mandatory_payload_bytes(m);
    for (int l = 1; l <= m.progressive_levels; ++l) s += optional_bytes(at(m, l), 32 - k[l - 1]);
    return s;
}

void plan_for_error(const ipcg_error_model &m, double max_error, int *k) {
    if (std::isnan(max_error) || max_error < m.eb)
        throw Error(EINFEASIBLE, "requested error bound is below the archive's compression bound");
    const double slack = max_error - m.eb;
    for (int l = 0; l < m.levels; ++l) k[l] = 32;
    const int lp = m.progressive_levels;
    if (lp == 0) return;
    std::vector<std::vector<Choice>> cs(lp);
    for (int l = 1; l <= lp; ++l) {
        const double w = weight(m, l);
        for (int d = 0; d <= 32; ++d) {
            const double e = w * at(m, l).delta[d];
            int cost;
            if (e <= 0.0 || std::isinf(slack)) cost = 0;
            else if (slack <= 0.0) cost = kInfCost;
            else {
                const double units = std::ceil(e * (double)kBuckets / slack);
                cost = units > (double)kInfCost ? kInfCost : (int)units;
            }
            if (cost > kBuckets) continue;
            const Choice c{d, cost, optional_bytes(at(m, l), d), e};
            if (!cs[l - 1].empty() && cs[l - 1].back().cost == cost) cs[l - 1].back() = c;
            else cs[l - 1].push_back(c);
        }
    }
    std::vector<std::vector<uint64_t>> best(lp + 1, std::vector<uint64_t>(kBuckets + 1, 0));
    for (int i = 1; i <= lp; ++i) {
        const uint64_t base = optional_bytes(at(m, i), 0);
        for (int e = 0; e <= kBuckets; ++e) {
            uint64_t v = 0;
            bool any = false;
            for (const Choice &c : cs[i - 1]) {
                if (c.cost > e) continue;
                const uint64_t cand = best[i - 1][e - c.cost] + (base - c.bytes);
                if (!any || cand > v) v = cand, any = true;
            }
            best[i][e] = v;
        }
    }
    int e = kBuckets;
    for (int i = lp; i >= 1; --i) {
        const uint64_t base = optional_bytes(at(m, i), 0), want = best[i][e];
        bool found = false;
        for (auto it = cs[i - 1].rbegin(); it != cs[i - 1].rend(); ++it) {
            if (it->cost > e) continue;
            if (best[i - 1][e - it->cost] + (base - it->bytes) == want) {
                k[i - 1] = 32 - it->dropped;
                e -= it->cost;
                found = true;
                break;
            }
        }
        if (!found) throw Error(ERUNTIME, "plan reconstruction lost the optimum");
    }
    while (bound_for_plan(m, k) > max_error) {
        int worst = -1;
        double worst_err = 0.0;
        for (int l = 1; l <= lp; ++l) {
            const int d = 32 - k[l - 1];
            const double er = weight(m, l) * at(m, l).delta[d];
            if (d > 0 && er > worst_err) worst_err = er, worst = l;
        }
        if (worst < 0) break;
        k[worst - 1] += 1;
    }
}

void plan_for_size(const ipcg_error_model &m, uint64_t byte_budget, int *k) {
    const uint64_t mandatory = mandatory_payload_bytes(m);
    if (byte_budget < mandatory)
        throw Error(EINFEASIBLE, "byte budget is below the mandatory payload (outliers and non-progressive levels)");
    const uint64_t budget = byte_budget - mandatory;
    for (int l = 0; l < m.levels; ++l) k[l] = 32;
    const int lp = m.progressive_levels;
    if (lp == 0) return;
    auto cost_of = [&](uint64_t bytes) -> int {
        if (bytes == 0) return 0;
        if (budget == 0) return kInfCost;
        const uint64_t units = (bytes * kBuckets + budget - 1) / budget;
        return units > (uint64_t)kBuckets ? kInfCost : (int)units;
    };
    std::vector<std::vector<Choice>> cs(lp);
    for (int l = 1; l <= lp; ++l) {
        const double w = weight(m, l);
        for (int d = 32; d >= 0; --d) {
            const uint64_t bytes = optional_bytes(at(m, l), d);
            const int cost = cost_of(bytes);
            if (cost > kBuckets) continue;
            const double e = w * at(m, l).delta[d];
            if (!cs[l - 1].empty() && cs[l - 1].back().cost == cost) {
                if (e < cs[l - 1].back().err) cs[l - 1].back() = Choice{d, cost, bytes, e};
            } else {
                cs[l - 1].push_back(Choice{d, cost, bytes, e});
            }
        }
        if (cs[l - 1].empty()) throw Error(EINFEASIBLE, "no loadable configuration fits the byte budget");
    }
    struct Value {
        double err;
        uint64_t bytes;
    };
    auto lt = [](const Value &a, const Value &b) { return a.err < b.err || (a.err == b.err && a.bytes < b.bytes); };
    const double inf = std::numeric_limits<double>::infinity();
    std::vector<std::vector<Value>> best(lp + 1, std::vector<Value>(kBuckets + 1, Value{inf, 0}));
    for (int e = 0; e <= kBuckets; ++e) best[0][e] = Value{0.0, 0};
    for (int i = 1; i <= lp; ++i) {
        for (int e = 0; e <= kBuckets; ++e) {
            Value v{inf, 0};
            for (const Choice &c : cs[i - 1]) {
                if (c.cost > e) continue;
                const Value &prev = best[i - 1][e - c.cost];
                if (std::isinf(prev.err)) continue;
                const Value cand{prev.err + c.err, prev.bytes + c.bytes};
                if (lt(cand, v)) v = cand;
            }
            best[i][e] = v;
        }
    }
    if (std::isinf(best[lp][kBuckets].err)) throw Error(EINFEASIBLE, "no loadable configuration fits the byte budget");
    int e = kBuckets;
    for (int i = lp; i >= 1; --i) {
        const Value want = best[i][e];
        bool found = false;
        for (const Choice &c : cs[i - 1]) {
            if (c.cost > e) continue;
            const Value &prev = best[i - 1][e - c.cost];
            if (std::isinf(prev.err)) continue;
            if (prev.err + c.err == want.err && prev.bytes + c.bytes == want.bytes) {
                k[i - 1] = 32 - c.dropped;
                e -= c.cost;
                found = true;
                break;
            }
        }
        if (!found) throw Error(ERUNTIME, "plan reconstruction lost the optimum");
    }
}

// index-based entry points
namespace {
ipcg_error_model model_of(const ipcg_index &h) {
    ipcg_error_model m;
    build_error_model(h, m);
    return m;
}
}  // namespace
double bound_for_plan(const ipcg_index &h, const int *k) { return bound_for_plan(model_of(h), k); }
uint64_t plan_payload_bytes(const ipcg_index &h, const int *k) { return plan_payload_bytes(model_of(h), k); }
uint64_t mandatory_payload_bytes(const ipcg_index &h) { return mandatory_payload_bytes(model_of(h)); }
void plan_for_error(const ipcg_index &h, double max_error, int *k) { plan_for_error(model_of(h), max_error, k); }
void plan_for_size(const ipcg_index &h, uint64_t budget, int *k) { plan_for_size(model_of(h), budget, k); }

}  // namespace ipcg
