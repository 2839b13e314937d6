// assemble.cuh -- device-side archive assembly (assemble.cu)
#pragma once
#include <stdint.h>

#include <algorithm>

#include "../../include/ipcomp_b200.h"
#include "util.cuh"

namespace ipcg {

// per-call device results of compress_field's level loop, read by the assembly
struct AsmSmall {
    double rng[2];
    uint32_t lowor[IPCG_MAX_LEVELS];
    unsigned long long raw[IPCG_MAX_LEVELS][33];
    double delta[IPCG_MAX_LEVELS][33];
    unsigned long long ocount[IPCG_MAX_LEVELS];
    uint8_t backend[IPCG_MAX_LEVELS][32];
    uint64_t length[IPCG_MAX_LEVELS][32];
    uint32_t crc[IPCG_MAX_LEVELS][32];
    const uint8_t *payload[IPCG_MAX_LEVELS][32];
    double range_part[2 * 1024];
};

struct AsmParams {  // host-known header fields
    int scalar, interp, nd, levels, lp, cap;
    uint64_t dims[4];
    double eb;
    uint64_t count[IPCG_MAX_LEVELS];
};

struct AsmDesc {
    const uint8_t *src;
    uint64_t dst, len;
};

struct AsmOut {
    uint64_t total, index_bytes;
    uint64_t outlier_dst[IPCG_MAX_LEVELS];
    int fits;
    uint64_t pieces[IPCG_MAX_LEVELS * 32 + 1];  // gather pieces before each descriptor
};

// worst-case archive size for the device assembly (outliers capped at 1/64 of each level)
uint64_t asm_capacity(const AsmParams &P);

// oflags[l] / obits[l]: level l+1's outlier bitmap (one bit per ordinal) and values by ordinal;
// tile_tmp: (count/32 + 8191) / 8192 words per level
void launch_assemble(const AsmParams &P, const AsmSmall *sm, uint8_t *arch, uint64_t capacity, AsmDesc *descs,
                     AsmOut *out, const uint32_t *const *oflags, const uint64_t *const *obits, uint32_t *tile_tmp,
                     cudaStream_t st);

}  // namespace ipcg
