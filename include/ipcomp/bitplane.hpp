// ipcomp/bitplane.hpp -- the bitplane API of the reference's proj/include/ipcomp/bitplane.hpp
// (src/bitplane.cpp), each operation one device pass (paper_2502_04093_b200/csrc/bitops.cu):
// plane p holds negabinary digit 31-p of every codeword, bit i at byte i/8, bit i%8.
#ifndef IPCOMP_BITPLANE_HPP
#define IPCOMP_BITPLANE_HPP

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "ipcomp/common.hpp"

namespace ipcomp {

struct BitplaneSet {
    std::size_t count = 0;
    std::array<std::vector<std::uint8_t>, 32> planes;
};

inline std::size_t plane_bytes(std::size_t count) { return (count + 7) / 8; }

namespace b200 {
inline BitplaneSet split_coded(std::span<const std::uint32_t> codewords, bool xor_code) {
    BitplaneSet set;
    set.count = codewords.size();
    std::uint8_t *rows[32];
    for (int p = 0; p < 32; ++p) {
        set.planes[static_cast<std::size_t>(p)].assign(plane_bytes(set.count), 0);
        rows[p] = set.planes[static_cast<std::size_t>(p)].data();
    }
    call([&](ipcg_ctx *c) { check(ipcg_split(c, codewords.data(), codewords.size(), xor_code ? 1 : 0, rows), c); });
    return set;
}
}  // namespace b200

inline BitplaneSet split(std::span<const std::uint32_t> codewords) { return b200::split_coded(codewords, false); }

inline std::vector<std::uint32_t> merge(const BitplaneSet &set, int planes_loaded) {
    if (planes_loaded < 0 || planes_loaded > 32) throw std::invalid_argument("plane count out of range");
    const std::uint8_t *rows[32] = {};
    for (int p = 0; p < planes_loaded; ++p) {
        if (set.planes[static_cast<std::size_t>(p)].size() < plane_bytes(set.count))
            throw std::invalid_argument("plane missing from set");
        rows[p] = set.planes[static_cast<std::size_t>(p)].data();
    }
    std::vector<std::uint32_t> codes(set.count, 0);
    b200::call([&](ipcg_ctx *c) { b200::check(ipcg_merge(c, rows, set.count, planes_loaded, codes.data()), c); });
    return codes;
}

// e_p = b_p ^ b_{p-1} ^ b_{p-2} over all 32 planes, in place
inline void xor_encode(BitplaneSet &set) {
    std::uint8_t *rows[32];
    for (int p = 0; p < 32; ++p) {
        auto &pl = set.planes[static_cast<std::size_t>(p)];
        if (pl.size() < plane_bytes(set.count)) pl.resize(plane_bytes(set.count), 0);
        rows[p] = pl.data();
    }
    b200::call([&](ipcg_ctx *c) { b200::check(ipcg_plane_xor(c, rows, set.count, 32, 0), c); });
}

// inverse of xor_encode over the first planes_present planes, in place
inline void xor_decode(BitplaneSet &set, int planes_present) {
    if (planes_present < 0 || planes_present > 32) throw std::invalid_argument("plane count out of range");
    std::uint8_t *rows[32] = {};
    for (int p = 0; p < planes_present; ++p) {
        auto &pl = set.planes[static_cast<std::size_t>(p)];
        if (pl.size() < plane_bytes(set.count)) throw std::invalid_argument("plane missing while decoding prefix");
        rows[p] = pl.data();
    }
    b200::call([&](ipcg_ctx *c) { b200::check(ipcg_plane_xor(c, rows, set.count, planes_present, 1), c); });
}

inline std::vector<std::uint8_t> extract_digit_plane(std::span<const std::uint32_t> codewords, int plane) {
    if (plane < 0 || plane > 31) throw std::invalid_argument("plane index out of range");
    BitplaneSet set = split(codewords);
    return std::move(set.planes[static_cast<std::size_t>(plane)]);
}

}  // namespace ipcomp

#endif
