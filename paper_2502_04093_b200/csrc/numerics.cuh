// numerics.cuh -- sm_100a kernels for the interpolation/quantization hot path
// (reference: predictor.hpp:14-38, quantizer.hpp:29-81, bitplane.cpp:7-59,
// pipeline.hpp:61-124,172-193).  All floating point follows the reference's
// operation order; the build uses -fmad=false -prec-div=true -ftz=false so every
// operation rounds exactly like the -ffp-contract=off CPU build.
#pragma once
#include <stdint.h>

#include "grid.h"
#include "util.cuh"

namespace ipcg {

constexpr int32_t kMaxCode = int32_t(1) << 30;  // quantizer.hpp:11
constexpr uint32_t kNbMask = 0xAAAAAAAAu;       // quantizer.hpp:12

__host__ __device__ __forceinline__ uint32_t to_negabinary(int32_t q) {
    return (uint32_t)((int64_t)q + (int64_t)kNbMask) ^ kNbMask;
}
__host__ __device__ __forceinline__ int32_t from_negabinary(uint32_t w) { return (int32_t)((w ^ kNbMask) - kNbMask); }

// a level's escaped points (pipeline.hpp:184-188): flags bit o = the point of ordinal o is an
// outlier, bits[o] = its exact value's bit pattern; count totals them.  The outlier block is
// compacted in ordinal order from the bitmap (assemble.cu), so no sort is needed.
struct OutlierSink {
    unsigned long long *count;
    uint32_t *flags;
    uint64_t *bits;
};

// ---- host launchers (numerics.cu) ----
void launch_range(const void *values, int scalar, uint64_t n, double *scratch /*2*1024*/, double *out2,
                  cudaStream_t st);
void launch_quant_pass(const void *values, void *state, int scalar, bool cubic, const PassDesc &pd, double eb,
                       uint32_t *nb, uint32_t *lowor, OutlierSink sink, uint64_t row_len, cudaStream_t st);
void launch_bitplanes(const uint32_t *nb, uint64_t count, uint32_t *planes, uint64_t plane_stride_words,
                      cudaStream_t st);
void launch_loss_pass(const uint32_t *nb, double *dev, const PassDesc &pd, bool cubic, double unit, int d,
                      const uint32_t *lowor, unsigned long long *rawbits, cudaStream_t st);
void launch_zero_pass(double *dev, const PassDesc &pd, cudaStream_t st);
// one launch per level (levels below the coarsest): all d replayed in shared-memory tiles;
// returns false when the level's geometry needs the per-pass path
bool launch_loss_fused(const uint32_t *nb, const Geometry &G, int level, bool cubic, double unit,
                       const uint32_t *lowor, unsigned long long *raw, cudaStream_t st);
void launch_loss_finalize(const unsigned long long *rawbits, const uint32_t *lowor, double *delta, cudaStream_t st);

// rows: device array of 32 plane-row pointers (rows[p] used for k0 <= p < k1)
void launch_merge(const uint32_t *const *rows, const uint32_t *merged_in, uint32_t *merged_out, uint64_t count, int k0,
                  int k1, cudaStream_t st);
void launch_recon_pass(void *state, int scalar, bool cubic, const PassDesc &pd, double eb, const uint32_t *merged,
                       uint64_t row_len, cudaStream_t st);
// outlier block bytes (u64 ordinal, T) -> overwrite inside one pass's ordinal range
void launch_outlier_apply(void *state, int scalar, const PassDesc &pd, const uint8_t *block, const uint64_t *napplied,
                          uint64_t max_entries, cudaStream_t st);
// number of leading entries the reference's in-order matcher applies (pipeline.hpp:71-75)
void launch_outlier_prefix(const uint8_t *block, uint64_t entries, int scalar, uint64_t count, uint64_t *napplied,
                           cudaStream_t st);

// bitplane.cpp:7-59 as standalone operations on 32 word rows (bitops.cu)
void launch_split(const uint32_t *codes, uint64_t count, uint32_t *rows, uint64_t stride, bool xor_encode,
                  cudaStream_t st);
void launch_plane_xor(uint32_t *rows, uint64_t stride, uint64_t count, int np, bool decode, cudaStream_t st);
void launch_merge_raw(const uint32_t *rows, uint64_t stride, uint64_t count, int k, uint32_t *out, cudaStream_t st);

}  // namespace ipcg
