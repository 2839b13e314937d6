// bitops.cu -- bitplane.cpp:7-68 as standalone device operations on 32 plane rows, for the
// reference's public BitplaneSet API (split / xor_encode / xor_decode / merge).  The
// compress and retrieval paths use the fused forms in numerics.cu (k_bitplanes, k_merge);
// these serve callers of the bitplane API directly.  Rows are 32-bit words: bit l of word g
// is codeword 32g + l, i.e. the reference's byte i/8, bit i%8 packing read little-endian.
#include "numerics.cuh"

namespace ipcg {
namespace {

// split (+ xor_encode): one warp per 32 codewords; 32 ballots give the 32 plane words, lane p
// keeps plane p's, and the 2-plane XOR takes planes p-1, p-2 from lanes p-1, p-2
__global__ void __launch_bounds__(256) k_split(const uint32_t *__restrict__ codes, uint64_t count,
                                               uint32_t *__restrict__ rows, uint64_t stride, int xor_encode) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t words = (count + 31) / 32;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < words; g += nwarps) {
        const uint64_t i = g * 32 + lane;
        const uint32_t c = i < count ? codes[i] : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            const uint32_t wp = __ballot_sync(0xffffffffu, (c >> (31 - p)) & 1u);
            if ((int)lane == p) mine = wp;
        }
        if (xor_encode) {
            const uint32_t u1 = __shfl_up_sync(0xffffffffu, mine, 1), u2 = __shfl_up_sync(0xffffffffu, mine, 2);
            mine ^= (lane >= 1 ? u1 : 0u) ^ (lane >= 2 ? u2 : 0u);
        }
        rows[(uint64_t)lane * stride + g] = mine;
    }
}

// xor_encode over all 32 planes (bitplane.cpp:44-49) or xor_decode of the first np planes
// (bitplane.cpp:51-59): a thread per word, planes walked in the reference's order
__global__ void __launch_bounds__(256) k_plane_xor(uint32_t *__restrict__ rows, uint64_t stride, uint64_t words,
                                                   int np, int decode) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < words; g += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t b[32];
#pragma unroll
        for (int p = 0; p < 32; ++p) b[p] = p < np ? rows[(uint64_t)p * stride + g] : 0u;
        if (decode) {
#pragma unroll
            for (int p = 1; p < 32; ++p) b[p] ^= b[p - 1] ^ (p >= 2 ? b[p - 2] : 0u);  // b_p = e_p ^ b_{p-1} ^ b_{p-2}
        } else {
#pragma unroll
            for (int p = 31; p >= 1; --p) b[p] ^= b[p - 1] ^ (p >= 2 ? b[p - 2] : 0u);  // from the originals
        }
#pragma unroll
        for (int p = 0; p < 32; ++p)
            if (p < np) rows[(uint64_t)p * stride + g] = b[p];
    }
}

// merge of raw planes 0..k-1 (bitplane.cpp:24-38): a thread per codeword
__global__ void __launch_bounds__(256) k_merge_raw(const uint32_t *__restrict__ rows, uint64_t stride, uint64_t count,
                                                   int k, uint32_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i >> 5;
        const unsigned bit = (unsigned)(i & 31);
        uint32_t c = 0;
        for (int p = 0; p < k; ++p) c |= ((rows[(uint64_t)p * stride + g] >> bit) & 1u) << (31 - p);
        out[i] = c;
    }
}

}  // namespace

void launch_split(const uint32_t *codes, uint64_t count, uint32_t *rows, uint64_t stride, bool xor_encode,
                  cudaStream_t st) {
    if (!count) return;
    k_split<<<grid_for((count + 31) / 32 * 32, 256, 148 * 16), 256, 0, st>>>(codes, count, rows, stride, xor_encode ? 1 : 0);
    CKL();
}
void launch_plane_xor(uint32_t *rows, uint64_t stride, uint64_t count, int np, bool decode, cudaStream_t st) {
    const uint64_t words = (count + 31) / 32;
    if (!words || np <= 0) return;
    k_plane_xor<<<grid_for(words, 256, 148 * 8), 256, 0, st>>>(rows, stride, words, np, decode ? 1 : 0);
    CKL();
}
void launch_merge_raw(const uint32_t *rows, uint64_t stride, uint64_t count, int k, uint32_t *out, cudaStream_t st) {
    if (!count) return;
    k_merge_raw<<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(rows, stride, count, k, out);
    CKL();
}

}  // namespace ipcg
