// ipcomp/archive.hpp -- archive types and the stream reader of the reference's
// proj/include/ipcomp/archive.hpp (src/archive.cpp).  The index format and its checks are the
// library's host layer (ipcg_index_*); ArchiveReader reads the index from the caller's stream
// field by field and afterwards only the blocks a retrieval plans (ipcg_archive_open_source),
// so progressive retrievals fetch only their planned bytes, as the reference's reader does.
#ifndef IPCOMP_ARCHIVE_HPP
#define IPCOMP_ARCHIVE_HPP

#include <array>
#include <cstdint>
#include <istream>
#include <memory>
#include <ostream>
#include <span>
#include <utility>
#include <vector>

#include "ipcomp/backend.hpp"
#include "ipcomp/common.hpp"

namespace ipcomp {

inline constexpr char kArchiveMagic[4] = {'I', 'P', 'C', '1'};
inline constexpr std::uint16_t kArchiveVersion = 1;

struct ArchiveHeader {
    std::uint16_t version = kArchiveVersion;
    ScalarKind scalar = ScalarKind::f64;
    InterpKind interp = InterpKind::cubic;
    Dims dims;
    double eb = 0.0;
    double range = 0.0;  // max - min of the original
    std::uint8_t levels = 0;
    std::uint8_t progressive_levels = 0;
    std::uint8_t anchor_cap = 64;
    std::uint64_t payload_bytes = 0;  // derived from the block index, not serialized
};

struct PlaneEntry {
    std::uint64_t offset = 0;  // relative to the payload start
    std::uint64_t length = 0;
};

struct LevelRecord {
    std::uint64_t count = 0;
    std::array<double, 33> delta{};  // loss with d low digits dropped; delta[0] = 0, non-decreasing
    std::uint64_t outlier_offset = 0;
    std::uint64_t outlier_length = 0;
    std::uint64_t outlier_count = 0;
    std::array<PlaneEntry, 32> planes{};
};

// records[l-1] describes level l (level 1 finest); serialized coarsest first
struct ArchiveData {
    ArchiveHeader header;
    std::vector<LevelRecord> records;
    std::vector<std::uint8_t> payload;
};

struct RetrievalPlan {
    std::vector<int> k;  // k[l-1]: MSB-first planes of level l to load
};

namespace b200 {

inline ipcg_index to_index(const ArchiveHeader &h, std::span<const LevelRecord> records) {
    if (records.size() != h.levels) throw std::invalid_argument("record count does not match level count");
    if (h.levels > IPCG_MAX_LEVELS) throw std::invalid_argument("archive has more levels than supported");
    ipcg_index ix{};
    ix.version = h.version;
    ix.scalar = static_cast<std::uint8_t>(h.scalar);
    ix.interp = static_cast<std::uint8_t>(h.interp);
    ix.ndims = static_cast<std::uint8_t>(h.dims.size() <= 4 ? h.dims.size() : 0);  // 0: rejected as the reference does
    for (std::size_t i = 0; i < h.dims.size() && i < 4; ++i) ix.dims[i] = h.dims[i];
    ix.eb = h.eb;
    ix.range = h.range;
    ix.levels = h.levels;
    ix.progressive_levels = h.progressive_levels;
    ix.anchor_cap = h.anchor_cap;
    for (std::size_t l = 0; l < records.size(); ++l) {
        const LevelRecord &r = records[l];
        ipcg_level_record &o = ix.records[l];
        o.count = r.count;
        for (int d = 0; d < 33; ++d) o.delta[d] = r.delta[static_cast<std::size_t>(d)];
        o.outlier_offset = r.outlier_offset;
        o.outlier_length = r.outlier_length;
        o.outlier_count = r.outlier_count;
        for (int p = 0; p < 32; ++p) {
            o.plane_offset[p] = r.planes[static_cast<std::size_t>(p)].offset;
            o.plane_length[p] = r.planes[static_cast<std::size_t>(p)].length;
        }
    }
    return ix;
}

inline void from_index(const ipcg_index &ix, ArchiveHeader &h, std::vector<LevelRecord> &records) {
    h.version = ix.version;
    h.scalar = static_cast<ScalarKind>(ix.scalar);
    h.interp = static_cast<InterpKind>(ix.interp);
    h.dims.assign(ix.dims, ix.dims + ix.ndims);
    h.eb = ix.eb;
    h.range = ix.range;
    h.levels = ix.levels;
    h.progressive_levels = ix.progressive_levels;
    h.anchor_cap = ix.anchor_cap;
    h.payload_bytes = ix.payload_bytes;
    records.assign(ix.levels, LevelRecord{});
    for (int l = 0; l < ix.levels; ++l) {
        const ipcg_level_record &r = ix.records[l];
        LevelRecord &o = records[static_cast<std::size_t>(l)];
        o.count = r.count;
        for (int d = 0; d < 33; ++d) o.delta[static_cast<std::size_t>(d)] = r.delta[d];
        o.outlier_offset = r.outlier_offset;
        o.outlier_length = r.outlier_length;
        o.outlier_count = r.outlier_count;
        for (int p = 0; p < 32; ++p) o.planes[static_cast<std::size_t>(p)] = PlaneEntry{r.plane_offset[p], r.plane_length[p]};
    }
}

// the archive handle of the C-ABI, released with the reader
struct ArchiveFree {
    void operator()(ipcg_archive *a) const { ipcg_archive_free(a); }
};
using ArchiveHandle = std::unique_ptr<ipcg_archive, ArchiveFree>;

}  // namespace b200

// header + records exactly as they precede the payload (archive.cpp:31-65)
inline std::vector<std::uint8_t> serialize_index(const ArchiveHeader &header, std::span<const LevelRecord> records) {
    const ipcg_index ix = b200::to_index(header, records);
    std::uint64_t size = 0;
    ipcg_index_serialize(&ix, nullptr, 0, &size);  // size query (also validates)
    std::vector<std::uint8_t> out(static_cast<std::size_t>(size));
    b200::check(ipcg_index_serialize(&ix, out.data(), out.size(), &size), nullptr);
    return out;
}

inline std::uint32_t archive_identity(const ArchiveData &archive) {
    const auto index = serialize_index(archive.header, archive.records);
    return crc32_bytes(index);
}

// archive.cpp:72-84
inline void write_archive(std::ostream &out, const ArchiveData &archive) {
    const std::uint64_t size = archive.payload.size();
    auto inside = [&](std::uint64_t off, std::uint64_t len) {
        if (len > size || off > size - len) throw std::invalid_argument("block offset outside payload");
    };
    for (const LevelRecord &r : archive.records) {
        inside(r.outlier_offset, r.outlier_length);
        for (const PlaneEntry &p : r.planes) inside(p.offset, p.length);
    }
    const auto index = serialize_index(archive.header, archive.records);
    out.write(reinterpret_cast<const char *>(index.data()), static_cast<std::streamsize>(index.size()));
    out.write(reinterpret_cast<const char *>(archive.payload.data()), static_cast<std::streamsize>(archive.payload.size()));
    if (!out) throw std::runtime_error("failed to write archive stream");
}

// archive.cpp:202-211
inline void validate_plan(const ArchiveHeader &header, const RetrievalPlan &plan) {
    if (plan.k.size() != header.levels) throw std::invalid_argument("plan level count does not match archive");
    for (int level = 1; level <= header.levels; ++level) {
        const int k = plan.k[static_cast<std::size_t>(level - 1)];
        if (k < 0 || k > 32) throw std::invalid_argument("plan plane count out of range");
        if (level > header.progressive_levels && k != 32)
            throw std::invalid_argument("non-progressive levels must load all planes");
    }
}

// Parses the index without touching payload bytes; blocks are read on demand (by load_* here,
// or by reconstruct_field / refine_field for a plan's blocks) and accounted.
class ArchiveReader {
   public:
    explicit ArchiveReader(std::istream &in) : in_(&in) {
        ipcg_archive *a = nullptr;
        b200::call([&](ipcg_ctx *c) { b200::check(ipcg_archive_open_source(c, &ArchiveReader::read_at, in_, &a), c); });
        a_.reset(a);
        ipcg_index ix{};
        ipcg_archive_index(a, &ix);
        b200::from_index(ix, header_, records_);
        identity_ = ix.identity;
        index_bytes_ = ix.index_bytes;
    }
    ArchiveReader(const ArchiveReader &) = delete;
    ArchiveReader &operator=(const ArchiveReader &) = delete;

    const ArchiveHeader &header() const { return header_; }
    const LevelRecord &record(int level) const { return records_.at(static_cast<std::size_t>(level - 1)); }
    std::span<const LevelRecord> records() const { return records_; }
    std::uint32_t identity() const { return identity_; }
    std::uint64_t index_bytes() const { return index_bytes_; }
    std::uint64_t payload_bytes_read() const { return ipcg_archive_payload_bytes_read(a_.get()); }

    EncodedBlock load_plane(int level, int plane) {
        if (plane < 0 || plane > 31) throw std::invalid_argument("plane index out of range");
        const PlaneEntry &e = record(level).planes[static_cast<std::size_t>(plane)];
        const auto bytes = read_range(e.offset, e.length);
        ByteReader br(bytes.data(), bytes.size());
        EncodedBlock block = read_block(br);
        if (br.remaining() != 0) throw std::runtime_error("plane block has trailing bytes");
        return block;
    }

    std::vector<std::uint8_t> load_outlier_bytes(int level) {
        const LevelRecord &r = record(level);
        const std::uint64_t e = 8 + scalar_width(header_.scalar);
        if (r.outlier_length % e != 0 || r.outlier_length / e != r.outlier_count)
            throw std::runtime_error("outlier block length does not match its count");
        return read_range(r.outlier_offset, r.outlier_length);
    }

    template <class T>
    std::vector<std::pair<std::uint64_t, T>> load_outliers(int level) {
        const auto raw = load_outlier_bytes(level);
        ByteReader br(raw.data(), raw.size());
        std::vector<std::pair<std::uint64_t, T>> out;
        out.reserve(static_cast<std::size_t>(record(level).outlier_count));
        for (std::uint64_t i = 0; i < record(level).outlier_count; ++i) {
            const std::uint64_t ordinal = br.u64();
            const T v = sizeof(T) == 4 ? static_cast<T>(br.f32()) : static_cast<T>(br.f64());
            out.emplace_back(ordinal, v);
        }
        return out;
    }

    // the library handle (reconstruct_field / refine_field run on it)
    ipcg_archive *handle() const { return a_.get(); }

   private:
    std::vector<std::uint8_t> read_range(std::uint64_t offset, std::uint64_t length) {
        std::vector<std::uint8_t> bytes(static_cast<std::size_t>(length));
        b200::call([&](ipcg_ctx *c) { b200::check(ipcg_archive_read_range(c, a_.get(), offset, length, bytes.data()), c); });
        return bytes;
    }
    // ipcg_read_fn over the caller's stream: absolute offsets, as the reference's seekg
    static std::int64_t read_at(void *user, std::uint64_t offset, void *dst, std::uint64_t len) {
        auto *in = static_cast<std::istream *>(user);
        in->clear();
        in->seekg(static_cast<std::streamoff>(offset));
        if (!*in) return -1;
        in->read(static_cast<char *>(dst), static_cast<std::streamsize>(len));
        return static_cast<std::int64_t>(in->gcount());
    }

    std::istream *in_;
    b200::ArchiveHandle a_;
    ArchiveHeader header_;
    std::vector<LevelRecord> records_;
    std::uint32_t identity_ = 0;
    std::uint64_t index_bytes_ = 0;
};

}  // namespace ipcomp

#endif
