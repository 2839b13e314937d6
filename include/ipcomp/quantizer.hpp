// ipcomp/quantizer.hpp -- the quantization-code contract of the reference's
// proj/include/ipcomp/quantizer.hpp (code range, negabinary codewords, suffix uncertainty,
// dequantization).  Quantization itself runs inside the device passes of compress_field
// (paper_2502_04093_b200/csrc/numerics.cu, quantize_residual); these are the scalar helpers
// callers use to interpret codes.
#ifndef IPCOMP_QUANTIZER_HPP
#define IPCOMP_QUANTIZER_HPP

#include <cstdint>
#include <stdexcept>

namespace ipcomp {

inline constexpr std::int32_t kMaxCode = std::int32_t{1} << 30;  // quantizer.hpp:11
inline constexpr std::uint32_t kNegabinaryMask = 0xAAAAAAAAu;     // quantizer.hpp:12

inline double dequantize(std::int64_t code, double eb) { return 2.0 * eb * static_cast<double>(code); }

// base -2 digits of q: (q + M) ^ M with M the alternating mask (quantizer.hpp:29-37)
inline std::uint32_t to_negabinary(std::int32_t q) {
    if (q < -kMaxCode || q > kMaxCode) throw std::domain_error("quantization code out of negabinary range");
    return static_cast<std::uint32_t>(std::int64_t{q} + std::int64_t{kNegabinaryMask}) ^ kNegabinaryMask;
}
inline std::int32_t from_negabinary(std::uint32_t w) {
    return static_cast<std::int32_t>((w ^ kNegabinaryMask) - kNegabinaryMask);
}

// largest |value| a dropped d-digit negabinary suffix can carry, in code units
// ((2^(d+1) - 1)/3 for odd d, (2^(d+1) - 2)/3 for even d; quantizer.hpp:39-46)
inline std::int64_t suffix_uncertainty(int d) {
    if (d < 0 || d > 32) throw std::domain_error("discarded digit count out of range");
    if (d == 0) return 0;
    const std::int64_t two = std::int64_t{1} << (d + 1);
    return (d & 1) ? (two - 1) / 3 : (two - 2) / 3;
}

}  // namespace ipcomp

#endif
