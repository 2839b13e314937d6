// ipcomp/backend.hpp -- the lossless block stage of the reference's
// proj/include/ipcomp/backend.hpp / src/backend.cpp.  backend_encode / backend_decode run on the
// GPU (the zlib-1.3-exact deflate and the block-parallel inflate of
// paper_2502_04093_b200/csrc/deflate.cu, inflate.cu); the 21-byte block wire format is the
// reference's.
#ifndef IPCOMP_BACKEND_HPP
#define IPCOMP_BACKEND_HPP

#include <cstdint>
#include <span>
#include <vector>

#include "ipcomp/common.hpp"

namespace ipcomp {

enum class Backend : std::uint8_t { identity = 0, deflate = 1 };
inline constexpr Backend kDefaultBackend = Backend::deflate;

struct EncodedBlock {
    Backend backend = Backend::identity;
    std::uint64_t raw_bits = 0;
    std::uint32_t checksum = 0;  // CRC-32 of the payload
    std::vector<std::uint8_t> payload;

    std::size_t raw_bytes() const { return static_cast<std::size_t>((raw_bits + 7) / 8); }
    std::size_t wire_size() const { return 21 + payload.size(); }
};

inline std::uint32_t crc32_bytes(std::span<const std::uint8_t> bytes) { return ipcg_crc32(bytes.data(), bytes.size()); }

// zlib compress2(level 6) on the device, kept only when strictly shorter (backend.cpp:34-53)
inline EncodedBlock backend_encode(std::span<const std::uint8_t> raw, Backend preferred, std::uint64_t raw_bits) {
    if (raw.size() != static_cast<std::size_t>((raw_bits + 7) / 8))
        throw std::invalid_argument("raw byte length does not match bit count");
    EncodedBlock b;
    b.raw_bits = raw_bits;
    if (preferred == Backend::deflate && !raw.empty()) {
        std::vector<std::uint8_t> out(raw.size());
        std::uint8_t be = 0;
        std::uint64_t len = 0;
        std::uint32_t crc = 0;
        b200::call([&](ipcg_ctx *c) {
            b200::check(ipcg_backend_encode(c, raw.data(), 0, raw.size(), raw.size(), 1, &be, &len, &crc, out.data(),
                                            out.size()),
                        c);
        });
        b.backend = be ? Backend::deflate : Backend::identity;
        b.checksum = crc;
        out.resize(len);
        b.payload = std::move(out);
        return b;
    }
    b.payload.assign(raw.begin(), raw.end());
    b.checksum = crc32_bytes(b.payload);
    return b;
}

// CRC check, then inflate on the device or the identity length check (backend.cpp:55-65)
inline std::vector<std::uint8_t> backend_decode(const EncodedBlock &block) {
    if (static_cast<std::uint8_t>(block.backend) > 1) {
        if (crc32_bytes(block.payload) != block.checksum) throw std::runtime_error("block checksum mismatch");
        throw std::runtime_error("unknown backend id");
    }
    const std::uint64_t plen = block.payload.size(), raw = block.raw_bytes();
    const std::uint8_t be = static_cast<std::uint8_t>(block.backend);
    std::vector<std::uint8_t> out(raw + 1);
    int status = 0;
    b200::call([&](ipcg_ctx *c) {
        static const std::uint8_t none = 0;
        b200::check(ipcg_backend_decode(c, plen ? block.payload.data() : &none, &plen, &be, &block.checksum, &raw, 1,
                                        out.data(), &status),
                    c);
    });
    switch (status) {
        case 0: break;
        case 1: throw std::runtime_error("block checksum mismatch");
        case 3: throw std::runtime_error("identity block has wrong length");
        default: throw std::runtime_error("deflate backend failed to decompress block");
    }
    out.resize(raw);
    return out;
}

// backend u8 | raw bit count u64 | payload length u64 | crc32(payload) u32 | payload
inline void write_block(ByteWriter &out, const EncodedBlock &block) {
    out.u8(static_cast<std::uint8_t>(block.backend));
    out.u64(block.raw_bits);
    out.u64(block.payload.size());
    out.u32(block.checksum);
    out.raw(block.payload.data(), block.payload.size());
}

inline EncodedBlock read_block(ByteReader &in) {
    EncodedBlock b;
    const std::uint8_t id = in.u8();
    if (id > 1) throw std::runtime_error("unknown backend id");
    b.backend = static_cast<Backend>(id);
    b.raw_bits = in.u64();
    const std::uint64_t len = in.u64();
    b.checksum = in.u32();
    if (len > in.remaining()) throw std::runtime_error("truncated input while parsing");
    b.payload.resize(static_cast<std::size_t>(len));
    in.raw(b.payload.data(), b.payload.size());
    return b;
}

}  // namespace ipcomp

#endif
