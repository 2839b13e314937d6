// inflate.cuh -- GPU `uncompress` for the reference's backend_decode
// (proj/src/backend.cpp:24-30,55-65): zlib wrapper, stored/fixed/dynamic blocks,
// Adler-32 trailer, exact-length check.
#pragma once
#include <stdint.h>

#include "util.cuh"

namespace ipcg {

struct InflateJob {
    const uint8_t *src;
    uint64_t src_len;
    uint8_t *dst;
    uint64_t dst_len;  // expected output length (uncompress destLen)
};

// status[i] = 0 on success, 1 on any zlib error (uncompress != Z_OK or length mismatch)
void inflate_batch(const InflateJob *jobs_dev, int count, int *status_dev, cudaStream_t st);

}  // namespace ipcg
