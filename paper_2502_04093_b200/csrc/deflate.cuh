// deflate.cuh -- batched, zlib-1.3-exact `compress2(level 6)` on the GPU for the
// reference's lossless stage (backend_encode, proj/src/backend.cpp:34-53).
#pragma once
#include <stdint.h>

#include "util.cuh"

namespace ipcg {

// results of backend_encode for S streams (device arrays of S entries)
struct BackendResults {
    uint8_t *backend;          // 0 identity, 1 deflate
    uint64_t *length;          // payload bytes
    uint32_t *crc;             // crc32(payload)
    const uint8_t **payload;   // device address of the payload bytes
};

// S equal-length streams in[j*in_stride .. +n) (in 16-byte aligned, in_stride a multiple
// of 16: the match search reads whole aligned words of the padded rows); outputs land in out[j*out_stride ..],
// out_stride >= n + 16.  Workspace from DeflateBatch::workspace_bytes.
struct DeflateBatch {
    static constexpr int CH = 256;  // nominal parse chunk (boundaries snap to anchors)
    static size_t workspace_bytes(int S, uint64_t n);
    // after_match (optional): recorded on `st` once the match search is enqueued, so a caller
    // can start other work when the throughput-bound phases are over
    // side (optional): a second stream the on-demand parse of the sparse streams runs on, concurrent
    // with the all-position search of the others on `st` (joined before the block plans); fork/join
    // are two caller-owned events
    static void run(const uint8_t *in, uint64_t in_stride, int S, uint64_t n, uint8_t *out, uint64_t out_stride,
                    void *workspace, BackendResults res, cudaStream_t st, cudaEvent_t after_match = nullptr,
                    cudaStream_t side = nullptr, cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);
};

// standalone CRC-32 (zlib polynomial) of S (ptr, len) device ranges
void crc32_batch(const uint8_t *const *ptrs, const uint64_t *lens, int S, uint64_t max_len, uint32_t *out,
                 void *workspace, size_t workspace_bytes, cudaStream_t st);
size_t crc32_batch_workspace(int S, uint64_t max_len);

}  // namespace ipcg
