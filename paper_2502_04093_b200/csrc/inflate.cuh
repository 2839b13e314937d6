// inflate.cuh -- GPU `uncompress` for the reference's backend_decode
// (proj/src/backend.cpp:24-30,55-65): zlib wrapper, stored/fixed/dynamic blocks,
// Adler-32 trailer, exact-length check.
#pragma once
#include <stdint.h>

#include <vector>

#include "util.cuh"

namespace ipcg {

struct InflateJob {
    const uint8_t *src;
    uint64_t src_len;
    uint8_t *dst;
    uint64_t dst_len;  // expected output length (uncompress destLen)
};

// status_dev[i] = 0 on success, 1 on any zlib error (uncompress != Z_OK or length
// mismatch).  Temporaries come from `alloc` (stream-ordered, released by its owner).
// check: optional side stream for the Adler-32 / final status kernels (they then run after
// `fork` is recorded on st and `done` is recorded on check; the caller waits on `done` before
// reading the status and keeps `alloc` alive until then)
void inflate_batch_host(const std::vector<InflateJob> &jobs, int *status_dev, DevAlloc &alloc, cudaStream_t st,
                        cudaStream_t check = nullptr, cudaEvent_t fork = nullptr, cudaEvent_t done = nullptr);

}  // namespace ipcg
