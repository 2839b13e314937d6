// inflate.cu -- GPU uncompress (RFC 1950/1951) for backend_decode
// (proj/src/backend.cpp:24-30).  One warp per stream: the Huffman decode runs
// warp-uniformly (every lane decodes the same symbol, so control flow never
// diverges and table reads broadcast), lane 0 stores literals and the whole warp
// performs match and stored-block copies.  Error behaviour follows zlib's
// inflate/inflate_table: over-subscribed or incomplete codes, missing end-of-block,
// distances too far back, bad header, Adler-32 mismatch and output-size mismatch
// all fail the stream, as uncompress() would.
#include "inflate.cuh"

namespace ipcg {

namespace {

constexpr int WARPS = 4;
constexpr int FASTBITS = 9;

struct Huff {
    uint16_t count[16];
    uint16_t first[16];   // canonical first code per length
    uint16_t offs[16];    // index of the first symbol of each length in sym[]
    uint16_t sym[320];
    uint16_t fast[1 << FASTBITS];  // (len << 12) | symbol, 0 = slow path
    int max;
};

struct Bits {
    const uint8_t *src;
    uint64_t len, pos;  // next byte to load
    uint64_t buf;
    int cnt;
    uint64_t used;      // bits consumed
    __device__ __forceinline__ void refill() {
        while (cnt <= 56) {
            const uint64_t b = pos < len ? src[pos] : 0u;
            ++pos;
            buf |= b << cnt;
            cnt += 8;
        }
    }
    __device__ __forceinline__ uint32_t peek(int k) {
        if (cnt < k) refill();
        return (uint32_t)(buf & ((1ull << k) - 1));
    }
    __device__ __forceinline__ void drop(int k) {
        buf >>= k;
        cnt -= k;
        used += (uint64_t)k;
    }
    __device__ __forceinline__ uint32_t get(int k) {
        if (k == 0) return 0;
        const uint32_t v = peek(k);
        drop(k);
        return v;
    }
    __device__ __forceinline__ bool overrun() const { return used > 8 * len; }
    __device__ __forceinline__ void align() {
        const int r = (int)(used & 7);
        if (r) drop(8 - r);
    }
    __device__ __forceinline__ uint64_t byte_pos() const { return used >> 3; }
    __device__ __forceinline__ void seek_byte(uint64_t p) {
        pos = p;
        buf = 0;
        cnt = 0;
        used = p * 8;
    }
};

// inflate_table semantics: returns false on over-subscribed / disallowed incomplete sets.
// type 0 = code lengths, 1 = literal/length, 2 = distance.  Runs on the whole warp.
__device__ bool build(Huff &h, const uint8_t *lens, int n, int type, unsigned lane) {
    __shared__ int ok_s[WARPS];
    const unsigned w = threadIdx.x >> 5;
    if (lane == 0) {
        for (int i = 0; i < 16; ++i) h.count[i] = 0;
        for (int i = 0; i < n; ++i) h.count[lens[i]]++;
        int max = 15;
        while (max >= 1 && h.count[max] == 0) --max;
        h.max = max;
        int left = 1;
        bool ok = true;
        for (int l = 1; l <= 15; ++l) {
            left <<= 1;
            left -= h.count[l];
            if (left < 0) ok = false;
        }
        if (ok && max > 0 && left > 0 && (type == 0 || max != 1)) ok = false;
        h.offs[1] = 0;
        for (int l = 1; l < 15; ++l) h.offs[l + 1] = (uint16_t)(h.offs[l] + h.count[l]);
        uint16_t code = 0;
        h.count[0] = 0;
        for (int l = 1; l <= 15; ++l) {
            code = (uint16_t)((code + h.count[l - 1]) << 1);
            h.first[l] = code;
        }
        uint16_t o[16];
        for (int l = 0; l < 16; ++l) o[l] = h.offs[l];
        for (int i = 0; i < n; ++i)
            if (lens[i]) h.sym[o[lens[i]]++] = (uint16_t)i;
        ok_s[w] = ok;
    }
    __syncwarp();
    for (int i = lane; i < (1 << FASTBITS); i += 32) h.fast[i] = 0;
    __syncwarp();
    // fill the fast table: symbol index t of length L has code first[L] + (t - offs[L])
    int total = 0;
    for (int l = 1; l <= 15; ++l) total += h.count[l];
    for (int t = lane; t < total; t += 32) {
        int L = 1;
        while (L < 15 && !(t >= h.offs[L] && t < h.offs[L] + h.count[L])) ++L;
        if (L > FASTBITS) continue;
        const uint32_t code = h.first[L] + (uint32_t)(t - h.offs[L]);
        const uint32_t rev = __brev(code) >> (32 - L);
        for (uint32_t e = 0; e < (1u << (FASTBITS - L)); ++e)
            h.fast[rev | (e << L)] = (uint16_t)((L << 12) | h.sym[t]);
    }
    __syncwarp();
    return ok_s[w] != 0;
}

// returns symbol or -1 (invalid code)
__device__ __forceinline__ int decode(const Huff &h, Bits &b) {
    const uint32_t e = h.fast[b.peek(FASTBITS)];
    if (e) {
        b.drop((int)(e >> 12));
        return (int)(e & 0xfff);
    }
    // canonical slow path (puff)
    int code = 0, first = 0, index = 0;
    for (int len = 1; len <= 15; ++len) {
        code |= (int)b.get(1);
        const int count = h.count[len];
        if (code - count < first) return h.sym[index + (code - first)];
        index += count;
        first += count;
        first <<= 1;
        code <<= 1;
    }
    return -1;
}

__constant__ uint16_t kLBase[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                    35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t kLExt[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t kDBase[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                                    257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t kDExt[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t kOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

__global__ void __launch_bounds__(WARPS * 32) k_inflate(const InflateJob *jobs, int count, int *status) {
    __shared__ Huff lit_s[WARPS], dist_s[WARPS], cl_s[WARPS];
    __shared__ uint8_t lens_s[WARPS][320];
    const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jid = blockIdx.x * WARPS + (int)w;
    if (jid >= count) return;
    const InflateJob job = jobs[jid];
    Huff &lit = lit_s[w], &dist = dist_s[w], &cl = cl_s[w];
    uint8_t *lens = lens_s[w];
    Bits b{job.src, job.src_len, 0, 0, 0, 0};
    uint8_t *dst = job.dst;
    const uint64_t outcap = job.dst_len;
    uint64_t out = 0;
    bool err = false;
    // zlib header (inflate.c HEAD state)
    {
        const uint32_t cmf = b.get(8), flg = b.get(8);
        if (((cmf << 8) | flg) % 31 != 0 || (cmf & 15) != 8 || (cmf >> 4) + 8 > 15 || (flg & 0x20)) err = true;
    }
    int last = 0;
    while (!err && !last) {
        last = (int)b.get(1);
        const uint32_t type = b.get(2);
        if (type == 0) {
            b.align();
            const uint64_t bp = b.byte_pos();
            b.seek_byte(bp);
            if (bp + 4 > job.src_len) {
                err = true;
                break;
            }
            const uint32_t L = job.src[bp] | (job.src[bp + 1] << 8), NL = job.src[bp + 2] | (job.src[bp + 3] << 8);
            if (L != (~NL & 0xffff) || bp + 4 + L > job.src_len || out + L > outcap) {
                err = true;
                break;
            }
            for (uint32_t i = lane; i < L; i += 32) dst[out + i] = job.src[bp + 4 + i];
            out += L;
            b.seek_byte(bp + 4 + L);
            continue;
        }
        if (type == 3) {
            err = true;
            break;
        }
        if (type == 1) {
            if (lane == 0) {
                for (int i = 0; i < 144; ++i) lens[i] = 8;
                for (int i = 144; i < 256; ++i) lens[i] = 9;
                for (int i = 256; i < 280; ++i) lens[i] = 7;
                for (int i = 280; i < 288; ++i) lens[i] = 8;
                for (int i = 0; i < 30; ++i) lens[288 + i] = 5;
            }
            __syncwarp();
            build(lit, lens, 288, 1, lane);
            build(dist, lens + 288, 30, 2, lane);
        } else {
            const int nlen = (int)b.get(5) + 257, ndist = (int)b.get(5) + 1, ncode = (int)b.get(4) + 4;
            if (nlen > 286 || ndist > 30) {
                err = true;
                break;
            }
            uint8_t cll[19];
            for (int i = 0; i < 19; ++i) cll[i] = 0;
            for (int i = 0; i < ncode; ++i) cll[kOrder[i]] = (uint8_t)b.get(3);
            if (lane == 0)
                for (int i = 0; i < 19; ++i) lens[i] = cll[i];
            __syncwarp();
            if (!build(cl, lens, 19, 0, lane)) {
                err = true;
                break;
            }
            uint8_t *ll = lens;  // reuse: cl table already built from lens[0..18]
            __syncwarp();
            int idx = 0;
            uint8_t prev = 0;
            bool bad = false;
            while (idx < nlen + ndist) {
                const int sym = decode(cl, b);
                if (sym < 0) {
                    bad = true;
                    break;
                }
                if (sym < 16) {
                    if (lane == 0) ll[idx] = (uint8_t)sym;
                    prev = (uint8_t)sym;
                    ++idx;
                    continue;
                }
                int rep;
                uint8_t v = 0;
                if (sym == 16) {
                    if (idx == 0) {
                        bad = true;
                        break;
                    }
                    v = prev;
                    rep = 3 + (int)b.get(2);
                } else if (sym == 17) {
                    rep = 3 + (int)b.get(3);
                } else {
                    rep = 11 + (int)b.get(7);
                }
                if (idx + rep > nlen + ndist) {
                    bad = true;
                    break;
                }
                if (lane == 0)
                    for (int r = 0; r < rep; ++r) ll[idx + r] = v;
                prev = v;
                idx += rep;
            }
            __syncwarp();
            if (bad || ll[256] == 0) {
                err = true;
                break;
            }
            if (!build(lit, ll, nlen, 1, lane) || !build(dist, ll + nlen, ndist, 2, lane)) {
                err = true;
                break;
            }
        }
        // symbols
        for (;;) {
            const int sym = decode(lit, b);
            if (sym < 0 || b.overrun()) {
                err = true;
                break;
            }
            if (sym < 256) {
                if (out >= outcap) {
                    err = true;
                    break;
                }
                if (lane == 0) dst[out] = (uint8_t)sym;
                ++out;
                continue;
            }
            if (sym == 256) break;
            const int li = sym - 257;
            if (li >= 29) {
                err = true;
                break;
            }
            const uint32_t len = kLBase[li] + b.get(kLExt[li]);
            const int ds = decode(dist, b);
            if (ds < 0 || ds >= 30) {
                err = true;
                break;
            }
            const uint32_t d = kDBase[ds] + b.get(kDExt[ds]);
            if (d > out || out + len > outcap) {
                err = true;
                break;
            }
            __syncwarp();
            if (d >= len) {
                for (uint32_t i = lane; i < len; i += 32) dst[out + i] = dst[out - d + i];
            } else {
                for (uint32_t i = lane; i < len; i += 32) dst[out + i] = dst[out - d + (i % d)];
            }
            __syncwarp();
            out += len;
        }
        if (b.overrun()) err = true;
    }
    if (!err) {
        b.align();
        const uint64_t bp = b.byte_pos();
        if (bp + 4 > job.src_len || out != outcap) {
            err = true;
        } else {
            const uint32_t want = ((uint32_t)job.src[bp] << 24) | ((uint32_t)job.src[bp + 1] << 16) |
                                  ((uint32_t)job.src[bp + 2] << 8) | job.src[bp + 3];
            __syncwarp();
            unsigned long long A = 0, B = 0;
            for (uint64_t i = lane; i < out; i += 32) {
                const uint32_t v = dst[i];
                A += v;
                B += (unsigned long long)((out - i) % 65521u) * v;
            }
            B %= 65521u;
            for (int o = 16; o > 0; o >>= 1) {
                A += __shfl_down_sync(0xffffffffu, A, o);
                B += __shfl_down_sync(0xffffffffu, B, o);
            }
            const uint32_t a = (uint32_t)((1 + A) % 65521u), bb = (uint32_t)((B + out) % 65521u);
            if (((bb << 16) | a) != want) err = true;
        }
    }
    if (lane == 0) status[jid] = err ? 1 : 0;
}

}  // namespace

void inflate_batch(const InflateJob *jobs_dev, int count, int *status_dev, cudaStream_t st) {
    if (count <= 0) return;
    k_inflate<<<(count + WARPS - 1) / WARPS, WARPS * 32, 0, st>>>(jobs_dev, count, status_dev);
    CKL();
}

}  // namespace ipcg
