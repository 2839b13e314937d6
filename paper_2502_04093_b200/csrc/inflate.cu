// inflate.cu -- block-parallel GPU `uncompress` (RFC 1950/1951) for backend_decode
// (proj/src/backend.cpp:24-30,55-65).
//
// A deflate stream is a chain of blocks whose boundaries are only known after
// decoding.  To decode the blocks of one stream in parallel:
//   1. scan     every bit offset of every stream for a *dynamic block header* that is
//               valid the way zlib's inflate/inflate_table check it (complete code-length
//               code, decodable length sequence, complete lit/len code with an end-of-block
//               code, admissible distance code); hits go into a per-stream hash table.
//   2. decode   every candidate block, one warp each (warp-uniform Huffman decode, tables
//               in shared memory), to its end-of-block: symbols, end bit, output size.
//   3. chain    one thread per stream walks the real block sequence from the zlib header:
//               stored blocks are parsed in place, dynamic blocks are looked up among the
//               candidates, fixed (and any unmatched) blocks are decoded on the spot.
//   4. emit     one warp per real block writes literals and intra-block copies; bytes whose
//               copy source lies in an earlier block get a pointer to that source instead.
//   5. resolve  follow those pointers (they always point into earlier blocks) to bytes
//               that hold values.
//   6. check    Adler-32 trailer and exact output length, as uncompress() does.
// Any stream that fails any zlib rule is reported, like uncompress() != Z_OK.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "inflate.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#ifndef IPCG_SUBB
#define IPCG_SUBB 512
#endif
#ifndef IPCG_NPH
#define IPCG_NPH 2
#endif
#ifndef IPCG_SEG
#define IPCG_SEG 512
#endif
#ifndef IPCG_CPW
#define IPCG_CPW 1
#endif
namespace ipcg {

namespace {

constexpr int FASTBITS = 9;
constexpr int MAXSYM = 16400;  // symbols stored per candidate block (zlib blocks: <= 16383)
constexpr int WARPS = 4;
constexpr int SEG = IPCG_SEG;             // symbols per emit segment
constexpr int NCKPT = MAXSYM / SEG + 2;   // output-offset checkpoints per candidate

// ------------------------------------------------------------------ bit reader
struct Bits {
    const uint8_t *src;
    uint64_t len, pos;  // next byte to load
    uint64_t buf;
    int cnt;
    uint64_t used;  // absolute bit position of the next unread bit
    __device__ __forceinline__ void init(const uint8_t *s, uint64_t l, uint64_t bit) {
        src = s;
        len = l;
        pos = bit >> 3;
        buf = 0;
        cnt = 0;
        used = bit & ~7ull;
        const int r = (int)(bit & 7);
        if (r) {
            refill();
            drop(r);
        }
    }
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
};

__constant__ uint16_t kLBase[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                    35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t kLExt[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t kDBase[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                                    257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t kDExt[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t kOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// ------------------------------------------------------------ canonical codes
struct Canon {  // puff-style: count per length + symbols in canonical order
    uint16_t count[16];
    uint16_t sym[320];
};

// inflate_table's acceptance rule: no over-subscription; incomplete only when allowed
// (never for code lengths; lit/len and dist only with a single 1-bit code).  max==0 is
// accepted (zlib builds an all-invalid table).  type 0 = code lengths, 1 = lit/len, 2 = dist.
__device__ bool canon_build(Canon &h, const uint8_t *lens, int n, int type) {
    for (int i = 0; i < 16; ++i) h.count[i] = 0;
    for (int i = 0; i < n; ++i) h.count[lens[i]]++;
    h.count[0] = 0;
    int max = 15;
    while (max >= 1 && h.count[max] == 0) --max;
    int left = 1;
    for (int l = 1; l <= 15; ++l) {
        left <<= 1;
        left -= h.count[l];
        if (left < 0) return false;
    }
    if (max > 0 && left > 0 && (type == 0 || max != 1)) return false;
    uint16_t offs[16];
    offs[1] = 0;
    for (int l = 1; l < 15; ++l) offs[l + 1] = (uint16_t)(offs[l] + h.count[l]);
    for (int i = 0; i < n; ++i)
        if (lens[i]) h.sym[offs[lens[i]]++] = (uint16_t)i;
    return true;
}

__device__ __forceinline__ int canon_decode(const Canon &h, Bits &b) {
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

// read a dynamic header at the bit reader's position into lens (lit/len then dist);
// returns false on any zlib rejection.  Leaves b after the header.
__device__ bool read_dynamic_header(Bits &b, uint8_t *lens, int &nlen, int &ndist, Canon &scratch) {
    nlen = (int)b.get(5) + 257;
    ndist = (int)b.get(5) + 1;
    const int ncode = (int)b.get(4) + 4;
    if (nlen > 286 || ndist > 30) return false;
    uint8_t cll[19];
    for (int i = 0; i < 19; ++i) cll[i] = 0;
    for (int i = 0; i < ncode; ++i) cll[kOrder[i]] = (uint8_t)b.get(3);
    if (!canon_build(scratch, cll, 19, 0)) return false;
    int idx = 0;
    uint8_t prev = 0;
    // Kraft sums of the two codes so far (units of 2^-15): an over-subscribed code is rejected by
    // inflate_table anyway (canon_build below), so stop reading at once -- random bit offsets
    // that pass the scan's filters mostly fail here, about halfway through their lengths
    uint32_t kl = 0, kd = 0;
    while (idx < nlen + ndist) {
        const int sym = canon_decode(scratch, b);
        if (sym < 0) return false;
        if (sym < 16) {
            if (sym) {
                if (idx < nlen) kl += 32768u >> sym;
                else kd += 32768u >> sym;
                if (kl > 32768u || kd > 32768u) return false;
            }
            lens[idx++] = (uint8_t)sym;
            prev = (uint8_t)sym;
            continue;
        }
        int rep;
        uint8_t v = 0;
        if (sym == 16) {
            if (idx == 0) return false;
            v = prev;
            rep = 3 + (int)b.get(2);
        } else if (sym == 17) {
            rep = 3 + (int)b.get(3);
        } else {
            rep = 11 + (int)b.get(7);
        }
        if (idx + rep > nlen + ndist) return false;
        if (v) {
            const int inl = idx < nlen ? min(rep, nlen - idx) : 0;
            kl += (uint32_t)inl * (32768u >> v);
            kd += (uint32_t)(rep - inl) * (32768u >> v);
            if (kl > 32768u || kd > 32768u) return false;
        }
        for (int r = 0; r < rep; ++r) lens[idx + r] = v;
        prev = v;
        idx += rep;
    }
    if (lens[256] == 0) return false;
    if (b.overrun()) return false;
    return true;
}

// ----------------------------------------------------------- fast warp tables
// k_decode_cands' tables: canonical counts/symbols (codes longer than the table) plus a
// resolved table indexed by the next BITS stream bits: code length (0 = longer code) |
// kind << 4 | extra bits << 6 | value << 16.  kind 0 literal (value = byte), 1 length or
// distance (value = base), 2 end of block, 3 invalid symbol.  A literal/length table of
// 11 bits leaves almost no code to the canonical loop (which diverges a lane-parallel warp).
#ifndef IPCG_DISTBITS
#define IPCG_DISTBITS 8
#endif
#ifndef IPCG_STAGE
#define IPCG_STAGE 1
#endif
#ifndef IPCG_LITBITS
#define IPCG_LITBITS 11
#endif
constexpr int LITBITS = IPCG_LITBITS, DISTBITS = IPCG_DISTBITS;
template <int BITS>
struct Huff {
    uint16_t count[16];
    uint16_t first[16];
    uint16_t offs[16];
    uint16_t sym[BITS == LITBITS ? 320 : 32];  // canonical symbol order (lit/len: 288 + slack; distance: 30 + slack)
    uint32_t fx[1 << BITS];
};

__device__ __forceinline__ uint32_t fx_entry(uint32_t L, uint32_t sym, bool dist) {
    uint32_t kind = 3, ext = 0, val = 0;
    if (dist) {
        if (sym < 30) kind = 1, ext = kDExt[sym], val = kDBase[sym];
    } else if (sym < 256) {
        kind = 0, val = sym;
    } else if (sym == 256) {
        kind = 2;
    } else if (sym < 286) {
        kind = 1, ext = kLExt[sym - 257], val = kLBase[sym - 257];
    }
    return L | kind << 4 | ext << 6 | val << 16;
}

// built by a group of G lanes (gl = lane within the group); every lane of the warp calls it
// (inactive groups pass active = false) so the warp-wide syncs line up
template <int BITS>
__device__ void huff_build_group(Huff<BITS> &h, const uint8_t *lens, int n, unsigned gl, unsigned G, bool active,
                                 bool dist) {
    if (active && gl == 0) {
        for (int i = 0; i < 16; ++i) h.count[i] = 0;
        for (int i = 0; i < n; ++i) h.count[lens[i]]++;
        h.count[0] = 0;
        h.offs[1] = 0;
        for (int l = 1; l < 15; ++l) h.offs[l + 1] = (uint16_t)(h.offs[l] + h.count[l]);
        uint16_t code = 0;
        for (int l = 1; l <= 15; ++l) {
            code = (uint16_t)((code + h.count[l - 1]) << 1);
            h.first[l] = code;
        }
        uint16_t o[16];
        for (int l = 0; l < 16; ++l) o[l] = h.offs[l];
        for (int i = 0; i < n; ++i)
            if (lens[i]) h.sym[o[lens[i]]++] = (uint16_t)i;
    }
    __syncwarp();
    if (active)
        for (int i = gl; i < (1 << BITS); i += G) h.fx[i] = 0;
    __syncwarp();
    if (active) {
        int total = 0;
        for (int l = 1; l <= 15; ++l) total += h.count[l];
        for (int t = gl; t < total; t += G) {
            int L = 1;
            while (L < 15 && !(t >= h.offs[L] && t < h.offs[L] + h.count[L])) ++L;
            if (L > BITS) continue;
            const uint32_t code = h.first[L] + (uint32_t)(t - h.offs[L]);
            const uint32_t rev = __brev(code) >> (32 - L);
            const uint32_t fx = fx_entry((uint32_t)L, h.sym[t], dist);
            for (uint32_t e = 0; e < (1u << (BITS - L)); ++e) h.fx[rev | (e << L)] = fx;
        }
    }
    __syncwarp();
}

// the table entry for the code at the start of bb, the canonical loop for a longer code
template <int BITS>
__device__ __forceinline__ uint32_t huff_entry(const Huff<BITS> &h, uint64_t bb, bool dist) {
    const uint32_t e = h.fx[(uint32_t)bb & ((1u << BITS) - 1)];
    if (e & 15u) return e;
    int code = 0, first = 0, index = 0;
    for (int l = 1; l <= 15; ++l) {
        code |= (int)(bb & 1);
        bb >>= 1;
        const int count = h.count[l];
        if (code - count < first) return fx_entry((uint32_t)l, h.sym[index + (code - first)], dist);
        index += count;
        first += count;
        first <<= 1;
        code <<= 1;
    }
    return 0u;  // no code: invalid
}

// symbol words: literal = byte; match = 1<<31 | len << 16 | dist  (len <= 258, dist <= 32768)
__device__ __forceinline__ uint32_t sym_lit(uint32_t c) { return c; }
__device__ __forceinline__ uint32_t sym_match(uint32_t len, uint32_t dist) {
    return 0x80000000u | (len << 16) | (dist - 1);
}

// One whole deflate symbol (literal, or length + distance with their extra bits) at the start
// of a 64-bit window.  kind: 0 literal, 1 match, 2 end of block, 3 invalid; nbits = bits used.
__device__ __forceinline__ uint32_t decode_symbol(const Huff<LITBITS> &lit, const Huff<DISTBITS> &dist, uint64_t bb,
                                                  uint32_t &kind, uint32_t &nbits, uint32_t &blen) {
    const uint32_t e = huff_entry(lit, bb, false);
    const uint32_t k = (e >> 4) & 3u, cl = e & 15u;
    if (cl == 0u || k >= 2u) {
        kind = cl == 0u ? 3u : k;
        nbits = cl;
        return 0;
    }
    if (k == 0u) {
        kind = 0, nbits = cl, blen = 1;
        return sym_lit(e >> 16);
    }
    const uint32_t ext = (e >> 6) & 15u;
    const uint32_t len = (e >> 16) + ((uint32_t)(bb >> cl) & ((1u << ext) - 1u));
    const uint64_t rest = bb >> (cl + ext);
    const uint32_t ed = huff_entry(dist, rest, true);
    const uint32_t dcl = ed & 15u;
    if (dcl == 0u || ((ed >> 4) & 3u) != 1u) {
        kind = 3;
        return 0;
    }
    const uint32_t dext = (ed >> 6) & 15u;
    const uint32_t d = (ed >> 16) + ((uint32_t)(rest >> dcl) & ((1u << dext) - 1u));
    kind = 1, nbits = cl + ext + dcl + dext, blen = len;
    return sym_match(len, d);
}

// ------------------------------------------------------------------ state
struct JobMeta {
    int status;          // 0 ok, 1 error
    int overflow;        // candidate table overflowed -> chain uses the slow path
    uint32_t adler_want;
    uint32_t nblocks;
    unsigned long long ncand;
    int allzero;         // every literal of every block is 0 -> output is all zero
    uint32_t nseg;       // emit segments over all blocks
    uint32_t nfallback;  // blocks the chain decoded itself (fixed, stored excluded, unmatched dynamic)
    uint64_t fb_syms;    // their symbols
    int bad;             // a match reached before the start of the output (k_emit)
    int ranked;          // block table built by k_rank (k_chain skips the job)
};

struct Cand {
    uint64_t hdr_bit;
    uint64_t end_bit;
    uint64_t out_bytes;
    uint32_t nsyms;
    int job;
    int ok;
    int nzlit;   // some literal is non-zero
    int bfinal;  // BFINAL bit of this block's header
    int rounds;  // lane-parallel decode rounds (diagnostics)
    int next;    // candidate starting at end_bit, -1 if none (set by k_decode_cands)
    uint32_t t_hdr, t_tab, t_dec;  // ns: header read, table build, symbol decode (diagnostics)
    uint32_t t_ph[6];              // IPCG_DTIME builds: ns in stage, P1, P2, range resolve, P3, P4
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct Blk {
    int type;        // 0 stored, 1 symbols (candidate or fallback)
    uint32_t nsyms;
    uint64_t src;    // stored: byte offset in src;  symbols: index into the symbol pool
    uint64_t out_off;
    uint64_t out_len;
    uint32_t seg_base, nseg;  // emit segments (SEG symbols each) of this block
    uint64_t ckpt;            // candidate index for output checkpoints, ~0 = none (one segment)
};

struct Tables {  // per-job device pointers
    unsigned long long *hash;  // key = bit+1 (high 40) | cand index (low 24) ... stored as two arrays
    uint32_t *hval;
    uint64_t hcap;
    Blk *blocks;
    uint64_t bcap;
    uint32_t *fallback;  // symbols decoded by the chain itself
    uint64_t fcap;
    uint32_t *flags;     // unresolved-byte bitmap
    uint32_t *mark;      // unresolved bytes that some pointer targets (resolve)
    uint32_t *ptr;       // source pointer of unresolved bytes
};

__device__ __forceinline__ uint64_t hslot(uint64_t key, uint64_t cap) {
    key ^= key >> 33;
    key *= 0xff51afd7ed558ccdull;
    key ^= key >> 33;
    return key & (cap - 1);
}

// ------------------------------------------------------------------ 1. scan
// A CTA stages a tile of the stream in shared memory; each thread tests 32 consecutive bit
// offsets from four aligned words (funnel shifts), rejecting on BTYPE/HLIT/HDIST and then on
// the code-length code's Kraft sum, looked up 4 fields (12 bits) at a time.  Survivors
// (rare) get the full zlib header validation.
constexpr int SCAN_TILE = 256 * 4;  // bytes per tile: 4 per thread = 32 bit offsets
constexpr int SCAN_HALO = 16;       // a header's fixed part spans < 80 bits

__device__ __forceinline__ void list_candidate(const InflateJob &job, const Tables &T, JobMeta *meta, int j,
                                            Cand *cands, unsigned long long *ncand_total, uint64_t cand_cap,
                                            uint64_t bit) {
    const unsigned long long ci = atomicAdd(ncand_total, 1ull);
    if (ci >= cand_cap) {
        meta[j].overflow = 1;
        return;
    }
    Cand c;
    c.hdr_bit = bit;
    c.end_bit = 0;
    c.out_bytes = 0;
    c.nsyms = 0;
    c.job = j;
    c.ok = 0;
    c.nzlit = 0;
    c.bfinal = (job.src[bit >> 3] >> (bit & 7)) & 1;
    c.next = -1;
    cands[ci] = c;
    // insert into the job's hash table
    const unsigned long long key = bit + 1;
    uint64_t sl = hslot(key, T.hcap);
    for (uint64_t probe = 0; probe < T.hcap; ++probe, sl = (sl + 1) & (T.hcap - 1)) {
        const unsigned long long prev = atomicCAS(&T.hash[sl], 0ull, key);
        if (prev == 0ull || prev == key) {
            T.hval[sl] = (uint32_t)ci;
            return;
        }
    }
    meta[j].overflow = 1;
}

// zlib's acceptance of a dynamic header at `bit` (BFINAL at bit), as a filter in front of
// scan_offset: the same rules as read_dynamic_header + canon_build (complete code-length code,
// repeat and length-count rules, end-of-block code present, no over-subscribed lit/len or
// distance code, incomplete only as a single 1-bit code, no read past the stream end), but on
// Kraft sums and maximum lengths instead of length arrays, with the code-length code decoded
// through a 128-entry table (`tab`, this thread's slice of shared memory) and the bits read from
// aligned words.  Rejects only what the full check rejects; the ~1% that pass are re-read in full.
__device__ bool quick_header_ok(const InflateJob &job, uint64_t bit, uint8_t *tab) {
    const uintptr_t sa = reinterpret_cast<uintptr_t>(job.src);
    const uint64_t off = (uint64_t)(sa & 3) * 8;
    const uint32_t *W = reinterpret_cast<const uint32_t *>(sa & ~uintptr_t(3));
    const uint64_t nwords = (off / 8 + job.src_len + 3) / 4;
    auto window = [&](uint64_t P) {  // 64 stream bits from absolute (word-aligned-base) bit P
        const uint64_t k = P >> 5;
        const uint32_t sh = (uint32_t)(P & 31);
        const uint32_t w0 = k < nwords ? __ldg(W + k) : 0u, w1 = k + 1 < nwords ? __ldg(W + k + 1) : 0u,
                       w2 = k + 2 < nwords ? __ldg(W + k + 2) : 0u;
        return (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
    };
    uint64_t p = off + bit + 3;
    uint64_t v = window(p);
    const int nlen = (int)(v & 31) + 257, ndist = (int)((v >> 5) & 31) + 1, ncode = (int)((v >> 10) & 15) + 4;
    if (nlen > 286 || ndist > 30) return false;
    p += 14;
    v = window(p);
    uint8_t cll[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) cll[i] = 0;
    for (int i = 0; i < ncode; ++i) cll[kOrder[i]] = (uint8_t)((v >> (3 * i)) & 7);
    p += 3 * (uint64_t)ncode;
    uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 19; ++i) cnt[cll[i]]++;
    int left = 1;
#pragma unroll
    for (int l = 1; l <= 7; ++l) {
        left = (left << 1) - (int)cnt[l];
        if (left < 0) return false;
    }
    if (left != 0) return false;  // incomplete (or empty) code-length code
    // canonical codes -> reversed-bit table of (symbol | length << 5)
    uint32_t next[8];
    next[1] = 0;
#pragma unroll
    for (int l = 1; l < 7; ++l) next[l + 1] = (next[l] + cnt[l]) << 1;
    for (int sym = 0; sym < 19; ++sym) {
        const int L = cll[sym];
        if (!L) continue;
        const uint32_t code = next[L]++;
        const uint32_t rev = __brev(code) >> (32 - L);
        for (uint32_t e = 0; e < (1u << (7 - L)); ++e) tab[rev | (e << L)] = (uint8_t)(sym | L << 5);
    }
    const int total = nlen + ndist;
    int idx = 0, prevl = 0, maxl = 0, maxd = 0;
    uint32_t kl = 0, kd = 0;
    bool eob = false;
    while (idx < total) {
        v = window(p);
        const uint32_t e = tab[v & 127];
        const int L = e >> 5, sym = e & 31;
        v >>= L;
        p += (uint64_t)L;
        int rep, val;
        if (sym < 16) {
            rep = 1, val = sym;
        } else if (sym == 16) {
            if (idx == 0) return false;
            rep = 3 + (int)(v & 3), val = prevl, p += 2;
        } else if (sym == 17) {
            rep = 3 + (int)(v & 7), val = 0, p += 3;
        } else {
            rep = 11 + (int)(v & 127), val = 0, p += 7;
        }
        if (idx + rep > total) return false;
        if (val) {
            const int inl = idx < nlen ? min(rep, nlen - idx) : 0;
            if (inl) {
                kl += (uint32_t)inl * (32768u >> val), maxl = max(maxl, val);
                if (idx <= 256 && 256 < idx + inl) eob = true;
            }
            if (rep - inl) kd += (uint32_t)(rep - inl) * (32768u >> val), maxd = max(maxd, val);
            if (kl > 32768u || kd > 32768u) return false;
        }
        prevl = val;
        idx += rep;
    }
    if (!eob) return false;
    if (p - off > 8 * job.src_len) return false;  // read past the stream end
    if (kl < 32768u && maxl != 1) return false;    // incomplete lit/len code
    if (kd < 32768u && maxd > 1) return false;     // incomplete distance code (none at all is accepted)
    return true;
}

// survivors of the cheap filters, validated by k_validate with every lane busy (validating
// in place left 31 lanes waiting on the one running zlib's header decode)
struct Survivor {
    uint64_t bit;
    int job;
};

__global__ void __launch_bounds__(256) k_validate(const InflateJob *jobs, const Tables *tabs, JobMeta *meta,
                                                 const Survivor *surv, const unsigned long long *nsurv,
                                                 uint64_t surv_cap, Cand *cands, unsigned long long *ncand_total,
                                                 uint64_t cand_cap) {
    __shared__ uint8_t qtab[256][128];
    const uint64_t ns = min((unsigned long long)surv_cap, *nsurv);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x) {
        const Survivor sv = surv[i];
        // quick_header_ok is zlib's acceptance rule itself (same predicate as read_dynamic_header +
        // canon_build), so an accepted header is listed directly; k_decode_cands reads it in full
        // again and would still reject it (ok = 0).  (The full read here was a one-thread serial
        // tail: ~0.4 ms per retrieval for the ~2000 real block headers.)
        if (!quick_header_ok(jobs[sv.job], sv.bit, qtab[threadIdx.x])) continue;
        list_candidate(jobs[sv.job], tabs[sv.job], meta, sv.job, cands, ncand_total, cand_cap, sv.bit);
    }
}

__global__ void __launch_bounds__(256) k_scan(const InflateJob *jobs, int njobs, const uint64_t *tile_off,
                                             const Tables *tabs, JobMeta *meta, Survivor *surv,
                                             unsigned long long *nsurv, uint64_t surv_cap) {
    // persistent CTAs over every (job, tile): the 4096-entry Kraft table is built once per CTA
    __shared__ uint16_t kraft4[4096];  // sum of 128 >> l over four 3-bit lengths (0 = unused)
    __shared__ __align__(16) uint8_t tile[SCAN_TILE + SCAN_HALO];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        uint32_t k = 0;
        for (int q = 0; q < 4; ++q) {
            const int l = (i >> (3 * q)) & 7;
            if (l) k += 128u >> l;
        }
        kraft4[i] = (uint16_t)k;
    }
    const uint64_t total = tile_off[njobs];
    const uint32_t *tw = reinterpret_cast<const uint32_t *>(tile);
    for (uint64_t g = blockIdx.x; g < total; g += gridDim.x) {
        int lo = 0, hi = njobs - 1;  // job of tile g: last j with tile_off[j] <= g
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (tile_off[mid] <= g) lo = mid;
            else hi = mid - 1;
        }
        const int j = lo;
        const InflateJob job = jobs[j];
        const uint64_t t0 = (g - tile_off[j]) * SCAN_TILE;
        __syncthreads();
        for (int i = threadIdx.x; i < SCAN_TILE + SCAN_HALO; i += blockDim.x)
            tile[i] = t0 + i < job.src_len ? job.src[t0 + i] : 0;
        __syncthreads();
        const uint64_t byte0 = t0 + 4 * threadIdx.x;
        const uint32_t W0 = tw[threadIdx.x], W1 = tw[threadIdx.x + 1], W2 = tw[threadIdx.x + 2],
                       W3 = tw[threadIdx.x + 3];
        // the fixed-position filters for all 32 offsets at once (bit k of each mask is offset k):
        // BTYPE = 2 (bit k+1 clear, bit k+2 set), HLIT <= 29 and HDIST <= 29 (not bits k+4..k+7,
        // resp. k+9..k+12, all set); the Kraft sum of the code-length code only for the ~22% left
        // (the per-offset test made this kernel issue-bound)
        const uint64_t X = (uint64_t)W0 | ((uint64_t)W1 << 32);
        uint32_t m = (uint32_t)((~(X >> 1)) & (X >> 2) & ~((X >> 4) & (X >> 5) & (X >> 6) & (X >> 7)) &
                                ~((X >> 9) & (X >> 10) & (X >> 11) & (X >> 12)));
        const uint64_t bit0 = byte0 * 8, nbits = job.src_len * 8;
        if (bit0 < 16) m &= 0xffffffffu << (uint32_t)(16 - bit0);  // offsets >= 16 (after the zlib header)
        if (bit0 + 32 > nbits) m &= nbits <= bit0 ? 0u : (1u << (uint32_t)(nbits - bit0)) - 1u;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t f0 = __funnelshift_r(W0, W1, k), f1 = __funnelshift_r(W1, W2, k),
                           f2 = __funnelshift_r(W2, W3, k);
            // code-length lengths: bits 17 .. 17 + 3*ncode of the window; complete code only
            const int ncode = (int)((f0 >> 13) & 15) + 4;
            const uint64_t lo2 = (uint64_t)f0 | ((uint64_t)f1 << 32);
            uint64_t cl = (lo2 >> 17) | ((uint64_t)f2 << 47);  // 57 bits = 19 fields
            cl &= (1ull << (3 * ncode)) - 1;
            const uint32_t kraft = (uint32_t)kraft4[cl & 4095] + kraft4[(cl >> 12) & 4095] +
                                   kraft4[(cl >> 24) & 4095] + kraft4[(cl >> 36) & 4095] +
                                   kraft4[(cl >> 48) & 511];
            if (kraft == 128) {  // rare (~1 in 1100 offsets): one atomic each
                const unsigned long long si = atomicAdd(nsurv, 1ull);
                if (si < surv_cap) surv[si] = Survivor{bit0 + (uint64_t)k, j};
                else meta[j].overflow = 1;
            }
        }
    }
}

// read_dynamic_header for k_decode_cands: the same acceptance rules and the same lens[], but the
// header's words staged in shared memory by the warp first (one coalesced load instead of a byte
// refill every few symbols) and the code-length code decoded through a 128-entry table instead of
// zlib's bit-at-a-time canonical loop (20-135 us -> a few us per block on the retrievals' critical
// path).  Every lane runs it on the same block (uniform; shared-memory writes are the same value
// from every lane).  hw: HDRW words, tab: 128 bytes, lens: >= 320 bytes, all shared and warp-private.
// `used` returns the bit position after the header, relative to the stream's first byte.
constexpr int HDRW = 160;  // 14 + 57 + 316 symbols x (7 + 7) bits = 4495 bits at most, + alignment + window reach
__device__ bool read_dynamic_header_warp(const InflateJob &job, uint64_t bit, uint32_t *hw, uint8_t *tab, uint8_t *lens,
                                         int &nlen, int &ndist, uint64_t &used, unsigned lane) {
    const uintptr_t sa = reinterpret_cast<uintptr_t>(job.src);
    const uint64_t off = (uint64_t)(sa & 3) * 8;
    const uint32_t *W = reinterpret_cast<const uint32_t *>(sa & ~uintptr_t(3));
    const uint64_t nwords = (off / 8 + job.src_len + 3) / 4;
    const uint64_t p0 = off + bit, k0 = p0 >> 5;
    __syncwarp();
    for (int i = (int)lane; i < HDRW; i += 32) hw[i] = k0 + i < nwords ? __ldg(W + k0 + i) : 0u;
    __syncwarp();
    uint32_t r = (uint32_t)(p0 & 31);  // bit position relative to the first staged word
    auto window = [&](uint32_t q) {
        const uint32_t k = q >> 5, sh = q & 31;
        return (uint64_t)__funnelshift_r(hw[k], hw[k + 1], sh) | ((uint64_t)__funnelshift_r(hw[k + 1], hw[k + 2], sh) << 32);
    };
    uint64_t v = window(r);
    nlen = (int)(v & 31) + 257, ndist = (int)((v >> 5) & 31) + 1;
    const int ncode = (int)((v >> 10) & 15) + 4;
    if (nlen > 286 || ndist > 30) return false;
    r += 14;
    v = window(r);
    uint8_t cll[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) cll[i] = 0;
    for (int i = 0; i < ncode; ++i) cll[kOrder[i]] = (uint8_t)((v >> (3 * i)) & 7);
    r += 3 * (uint32_t)ncode;
    uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 19; ++i) cnt[cll[i]]++;
    int left = 1;
#pragma unroll
    for (int l = 1; l <= 7; ++l) {
        left = (left << 1) - (int)cnt[l];
        if (left < 0) return false;
    }
    if (left != 0) return false;  // incomplete or empty code-length code (inflate_table rejects both here)
    uint32_t next[8];
    next[1] = 0;
#pragma unroll
    for (int l = 1; l < 7; ++l) next[l + 1] = (next[l] + cnt[l]) << 1;
    for (int sym = 0; sym < 19; ++sym) {
        const int L = cll[sym];
        if (!L) continue;
        const uint32_t code = next[L]++;
        const uint32_t rev = __brev(code) >> (32 - L);
        for (uint32_t e = 0; e < (1u << (7 - L)); ++e) tab[rev | (e << L)] = (uint8_t)(sym | L << 5);
    }
    __syncwarp();
    const int total = nlen + ndist;
    int idx = 0;
    uint8_t prev = 0;
    uint32_t kl = 0, kd = 0;  // Kraft sums (units of 2^-15): an over-subscribed code is rejected at once
    while (idx < total) {
        v = window(r);
        const uint32_t e = tab[v & 127];
        const int L = e >> 5, sym = e & 31;
        v >>= L;
        r += (uint32_t)L;
        if (sym < 16) {
            if (sym) {
                if (idx < nlen) kl += 32768u >> sym;
                else kd += 32768u >> sym;
                if (kl > 32768u || kd > 32768u) return false;
            }
            lens[idx++] = (uint8_t)sym;
            prev = (uint8_t)sym;
            continue;
        }
        int rep;
        uint8_t val = 0;
        if (sym == 16) {
            if (idx == 0) return false;
            val = prev;
            rep = 3 + (int)(v & 3), r += 2;
        } else if (sym == 17) {
            rep = 3 + (int)(v & 7), r += 3;
        } else {
            rep = 11 + (int)(v & 127), r += 7;
        }
        if (idx + rep > total) return false;
        if (val) {
            const int inl = idx < nlen ? min(rep, nlen - idx) : 0;
            kl += (uint32_t)inl * (32768u >> val);
            kd += (uint32_t)(rep - inl) * (32768u >> val);
            if (kl > 32768u || kd > 32768u) return false;
        }
        for (int q = 0; q < rep; ++q) lens[idx + q] = val;
        prev = val;
        idx += rep;
    }
    __syncwarp();
    if (lens[256] == 0) return false;
    used = (k0 << 5) + r - off;
    if (used > 8 * job.src_len) return false;  // read past the stream end
    return true;
}

// ------------------------------------------------------------ 2. candidates
// CPW candidates per warp, one per group of 32/CPW lanes: the decode is inherently
// sequential per block and every lane of a group does the same work, so packing several
// blocks into a warp divides the (issue-bound) warp-instruction count.
constexpr int SUBB = IPCG_SUBB;      // bits per lane subsequence (lane-parallel candidate decode)
constexpr int MARKW = SUBB / 32;     // its symbol-start bitmap words
constexpr int NPH = IPCG_NPH;         // speculative start phases after a loss of synchronisation
#ifdef IPCG_DTIME
#define DT_MARK(i) do { const unsigned long long t_ = gtimer(); dt[i] += (uint32_t)(t_ - dtl); dtl = t_; } while (0)
#else
#define DT_MARK(i) do { } while (0)
#endif
constexpr int DWARPS = 2;  // warps per k_decode_cands CTA (static smem: ~16 KB of tables + bitmaps per warp)

template <int CPW>
__global__ void __launch_bounds__(DWARPS * 32) k_decode_cands(const InflateJob *jobs, const Tables *tabs, Cand *cands,
                                                           const unsigned long long *ncand_total, uint64_t cand_cap,
                                                           uint32_t *pool, uint32_t *ckpt_pool) {
    static_assert(CPW == 1, "the speculative decode runs all 32 lanes of a warp on one candidate");
    constexpr unsigned G = 32 / CPW;
    __shared__ Huff<LITBITS> lit_s[DWARPS * CPW];
    __shared__ Huff<DISTBITS> dist_s[DWARPS * CPW];
    __shared__ uint32_t marks_s[DWARPS][NPH * 32 * MARKW];
    __shared__ uint32_t li_e1[DWARPS][NPH][32], li_x[DWARPS][NPH][32];  // per lane and phase
    __shared__ int8_t li_sync[DWARPS][NPH][32];
    __shared__ int8_t li_skip[DWARPS][NPH][32];    // 1: the continuation met lane gl+2's path (gl+1 covered)
    __shared__ uint32_t li_x1[DWARPS][NPH][32];    // its first symbol start in lane gl+2's subsequence
    // symbol counts and output bytes: of the P1 path (n1, b1), of the whole continuation (nc, bc)
    // and of its part before lane gl+2's subsequence (nx, bx) -- P3 counts a lane's true range
    // from these instead of decoding it again
    __shared__ uint16_t li_n1[DWARPS][NPH][32], li_nc[DWARPS][NPH][32], li_nx[DWARPS][NPH][32];
    __shared__ uint32_t li_b1[DWARPS][NPH][32], li_bc[DWARPS][NPH][32], li_bx[DWARPS][NPH][32];
    __shared__ uint8_t li_fl[DWARPS][NPH][32];  // 1: path ends in own subsequence, 2: in the next  // symbol-start bitmaps of the lane subsequences
    // the round's bits (32 subsequences + the reach of the last symbols), staged once per round:
    // the per-symbol window loads were the decode's top stall (L1 misses on the critical path)
    constexpr int STG = IPCG_STAGE ? 32 * SUBB / 32 + 8 : 80;  // (>= 80 words: the code lengths live here first)
    __shared__ uint32_t stg_s[DWARPS][STG];
    const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned sub = lane / G, gl = lane % G, slot = w * CPW + sub;
    const uint64_t n = min((unsigned long long)cand_cap, *ncand_total);
    for (uint64_t bw = blockIdx.x * (uint64_t)DWARPS + w; bw * CPW < n; bw += (uint64_t)gridDim.x * DWARPS) {
        const uint64_t ci = bw * CPW + sub;
        bool act = ci < n;
        Cand dummy;
        Cand &c = act ? cands[ci] : dummy;
        const InflateJob job = jobs[act ? c.job : 0];
        int nlen = 0, ndist = 0;
        uint64_t used = 0;  // bits of the stream consumed so far (from its first byte)
        const unsigned long long tm0 = gtimer();
        {
            // the header's code lengths land in the staging buffer (the tables are built from
            // there); the header words and the code-length table borrow the mark bitmaps
            uint32_t *hw = marks_s[w];
            const bool ok = act && read_dynamic_header_warp(job, c.hdr_bit + 3, hw, reinterpret_cast<uint8_t *>(hw + HDRW),
                                                            reinterpret_cast<uint8_t *>(stg_s[slot]), nlen, ndist, used, lane);
            if (act && !ok) {
                if (gl == 0) c.ok = 0;
                act = false;
            }
        }
        __syncwarp();
        const unsigned long long tm1 = gtimer();
        // (the code lengths sit in the staging buffer until the tables are built)
        huff_build_group(lit_s[slot], reinterpret_cast<const uint8_t *>(stg_s[slot]), nlen, gl, G, act, false);
        huff_build_group(dist_s[slot], reinterpret_cast<const uint8_t *>(stg_s[slot]) + nlen, ndist, gl, G, act, true);
        __syncwarp();
        const unsigned long long tm2 = gtimer();
        if (act) {  // (no early exits: every lane reaches the syncs below)
        uint32_t *out = pool + ci * (uint64_t)MAXSYM;
        uint32_t ns = 0, nz = 0;
        uint32_t bytes = 0;  // <= 16383 symbols x 258 bytes
        bool good = true;
        // Lane-parallel decode with self-synchronisation.  A round covers 32 subsequences of
        // SUBB bits from the round's (true) start: lane i decodes subsequence i speculatively
        // from its first bit, marking its symbol starts in shared memory (P1), then continues
        // into subsequence i+1 until it meets a start lane i+1 marked (P2: from there the two
        // paths coincide).  Lane 0 starts on the true path, so by induction every lane whose
        // left neighbour synchronised is on the true path from its sync point; the round covers
        // lanes up to the first one without a sync (its true exit is its left neighbour's
        // continued exit) or the end of block.  P3 decodes each lane's true range counting
        // symbols and bytes, a warp scan places them, P4 decodes again and writes them (with the
        // SEG checkpoints).  Canonical Huffman codes resynchronise within a few symbols; a block
        // that never does still advances >= 2 subsequences per round.
        const uintptr_t sa = reinterpret_cast<uintptr_t>(job.src);
        const uint64_t off = (uint64_t)(sa & 3) * 8;
        const uint32_t *W = reinterpret_cast<const uint32_t *>(sa & ~uintptr_t(3));
        const uint64_t nwords = (off / 8 + job.src_len + 3) / 4, endbit = off + 8 * job.src_len;
        uint32_t *stg = stg_s[w];
        uint64_t k0 = 0;  // first staged word
        // 64 stream bits from absolute bit P >= the round's first staged bit: the position relative
        // to the staged words in 32-bit arithmetic (a round spans < 2^16 bits; the 64-bit word
        // index, bounds and shifts were ~20 of the ~45 instructions before each table lookup)
        uint32_t kb32 = 0;  // low word of the first staged bit's position (k0 << 5)
        auto window = [&](uint64_t P) {
            const uint32_t q = (uint32_t)P - kb32, k = q >> 5, sh = q & 31;
            uint32_t w0, w1, w2;
            if (IPCG_STAGE && k < (uint32_t)(STG - 2)) {
                w0 = stg[k], w1 = stg[k + 1], w2 = stg[k + 2];
            } else {
                const uint64_t kk = k0 + k;
                w0 = kk < nwords ? __ldg(W + kk) : 0u, w1 = kk + 1 < nwords ? __ldg(W + kk + 1) : 0u,
                w2 = kk + 2 < nwords ? __ldg(W + kk + 2) : 0u;
            }
            return (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
        };
        uint32_t *marks = marks_s[w];  // [32 lanes][MARKW words]
        const uint32_t subb = SUBB;
        // Periodic streams can keep an off-phase path off-phase forever (a run of one 2-bit
        // match symbol: a path started one bit late decodes the same symbols shifted).  After a
        // round that lost synchronisation every lane also runs its subsequence from the next
        // NPH-1 bit offsets, and a left neighbour may synchronise with any of those paths.
        int nph = 1;
        uint64_t base = off + used;
        bool eob = false;
        int nrounds = 0;
#ifdef IPCG_DTIME
        uint32_t dt[6] = {0, 0, 0, 0, 0, 0};
        unsigned long long dtl = gtimer();
#endif
        while (good && !eob) {
            ++nrounds;
            if (base > endbit) {  // overrun (the stream reads as zeros past its end)
                good = false;
                break;
            }
            const uint64_t g = base + (uint64_t)gl * subb, gn = g + subb;
            k0 = base >> 5;
            kb32 = (uint32_t)(k0 << 5);
            if (IPCG_STAGE) {
                __syncwarp();  // the previous round's readers are done
                for (int i = (int)gl; i < STG; i += 32) stg[i] = k0 + i < nwords ? __ldg(W + k0 + i) : 0u;
                __syncwarp();
            }
            DT_MARK(0);
            // P1: speculative decode of my subsequence from nph bit offsets, marking symbol starts;
            // per phase the exit (or the position of a path-ending symbol) goes to shared memory
            // relative to `base` (per-phase registers cost the kernel 40 registers)
            uint32_t nb, bl;
            for (int ph = 0; ph < nph; ++ph) {
                uint32_t *mk = marks + (ph * 32 + gl) * MARKW;
                for (int q = 0; q < MARKW; ++q) mk[q] = 0u;
                uint64_t p = g + ph;
                uint32_t k1 = 0, c1 = 0, b1 = 0;
                while (p < gn) {
                    const uint32_t r = (uint32_t)(p - g);
                    mk[r >> 5] |= 1u << (r & 31);
                    decode_symbol(lit_s[slot], dist_s[slot], window(p), k1, nb, bl);
                    if (k1 >= 2u) break;  // this path ends (end of block or invalid code) at p
                    ++c1, b1 += bl;
                    p += nb;
                }
                li_e1[w][ph][gl] = (uint32_t)(p - base);
                li_fl[w][ph][gl] = k1 >= 2u ? 1 : 0;
                li_n1[w][ph][gl] = (uint16_t)c1;
                li_b1[w][ph][gl] = b1;
            }
            __syncwarp();
            DT_MARK(1);
            // P2: each phase's path continues into subsequence gl+1 until it meets a symbol start
            // of one of lane gl+1's paths (from there the two coincide)
            // (a path that has not met lane gl+1's within its subsequence goes on through lane
            // gl+2's: blocks of long match symbols -- extra bits resynchronise slowly -- lost the
            // round at such lanes and took ~2x the rounds of their bit length)
            for (int ph = 0; ph < nph; ++ph) {
                int hit = -1, skip = 0;
                uint64_t x1 = 0;
                uint32_t cc = 0, cb = 0, cx = 0, bx = 0;
                uint8_t fl = li_fl[w][ph][gl];
                uint64_t x = base + li_e1[w][ph][gl];
                if (gl < 31 && !(fl & 1)) {
                    const uint64_t g2 = gn + subb, g3 = gl < 30 ? g2 + subb : g2;
                    while (x < g3) {
                        if (x < g2) {
                            const uint32_t r = (uint32_t)(x - gn);
                            for (int q = 0; q < nph && hit < 0; ++q)
                                if ((marks[(q * 32 + gl + 1) * MARKW + (r >> 5)] >> (r & 31)) & 1u) hit = q;
                        } else {
                            if (!x1) x1 = x, cx = cc, bx = cb;
                            const uint32_t r = (uint32_t)(x - g2);
                            for (int q = 0; q < nph && hit < 0; ++q)
                                if ((marks[(q * 32 + gl + 2) * MARKW + (r >> 5)] >> (r & 31)) & 1u) hit = q, skip = 1;
                        }
                        if (hit >= 0) break;
                        uint32_t k2;
                        decode_symbol(lit_s[slot], dist_s[slot], window(x), k2, nb, bl);
                        if (k2 >= 2u) {
                            fl |= 2;
                            break;
                        }
                        ++cc, cb += bl;
                        x += nb;
                    }
                }
                li_x[w][ph][gl] = (uint32_t)(x - base);
                li_sync[w][ph][gl] = (int8_t)hit;
                li_skip[w][ph][gl] = (int8_t)skip;
                li_x1[w][ph][gl] = (uint32_t)((x1 ? x1 : x) - base);
                li_fl[w][ph][gl] = fl;
                li_nc[w][ph][gl] = (uint16_t)cc, li_bc[w][ph][gl] = cb;
                li_nx[w][ph][gl] = (uint16_t)(x1 ? cx : cc), li_bx[w][ph][gl] = x1 ? bx : cb;
            }
            __syncwarp();
            DT_MARK(2);
            // resolve the true range [t_i, t_i+1) of every covered lane (uniform loop over shared
            // memory): lane 0's phase 0 is the true path; lane i+1's true phase is the one lane
            // i's true path met; a lane whose left neighbour met none is covered by that
            // neighbour's continuation, and the round ends there
            uint64_t my_t = 0, my_e = 0;
            // how P3 counts my range: on my P1 path of phase my_ph from my_sp (continuation symbols
            // my_pc/my_pb before it), or (my_ph < 0) wholly the left neighbour's continuation
            int my_ph = -1;
            uint64_t my_sp = 0;
            uint32_t my_pc = 0, my_pb = 0;
            int last = -1;
            bool lost = false, other = false;
            {
                uint64_t t = base;
                int cur = 0;          // true phase of lane i, or -1: covered by lane i-1's continuation
                int next_phase = -1;  // for a covered lane: the phase of lane i+1 its coverer met (-1: none)
                uint64_t prev_x = 0;
                bool prev_end2 = false;
                uint64_t sp = base;      // lane i's sync point on its P1 path (cur >= 0)
                uint32_t pc = 0, pb = 0;  // true symbols/bytes of lane i before sp (cur >= 0), or all of
                                         // its range (cur < 0)
                uint64_t nsp = 0;        // after a covered lane: the sync point / counts of the next
                uint32_t npc = 0, npb = 0;
                for (int i = 0; i < 32; ++i) {
                    uint64_t E;
                    bool stop;
                    if (cur >= 0) {
                        E = base + li_e1[w][cur][i];
                        stop = li_fl[w][cur][i] & 1;
                        other |= cur != 0;
                    } else {
                        E = prev_x;
                        stop = prev_end2;
                    }
                    if (gl == (unsigned)i) my_t = t, my_e = E, my_ph = cur, my_sp = sp, my_pc = pc, my_pb = pb;
                    last = i;
                    t = E;
                    if (stop) break;  // end of block / invalid code inside lane i
                    if (cur < 0) {
                        if (next_phase < 0) {
                            lost = true;
                            break;
                        }
                        cur = next_phase;  // lane i+1 on the path lane i-1's continuation met
                        next_phase = -1;
                        sp = nsp, pc = npc, pb = npb;
                        continue;
                    }
                    if (i == 31) break;
                    const int hit = li_sync[w][cur][i];
                    const bool sk = hit >= 0 && li_skip[w][cur][i];
                    if (sk) {
                        // lane i+1 is covered up to the continuation's first symbol in lane i+2's
                        // subsequence, where lane i+2's path `hit` takes over
                        prev_x = base + li_x1[w][cur][i];
                        prev_end2 = false;
                        next_phase = hit;
                        nsp = base + li_x[w][cur][i];
                        npc = li_nc[w][cur][i] - li_nx[w][cur][i], npb = li_bc[w][cur][i] - li_bx[w][cur][i];
                        pc = li_nx[w][cur][i], pb = li_bx[w][cur][i];
                    } else {
                        prev_x = base + li_x[w][cur][i];
                        prev_end2 = (li_fl[w][cur][i] & 2) != 0;
                        next_phase = -1;
                        sp = prev_x;  // (hit: lane i+1's sync point; none: lane i+1 is covered)
                        pc = li_nc[w][cur][i], pb = li_bc[w][cur][i];
                    }
                    cur = hit >= 0 && !sk ? hit : -1;
                }
            }
            // speculate the other phases after a round that lost synchronisation within its first
            // lanes (a phase-locked stream: the round covered almost nothing), and keep doing so
            // while some lane's true path is one of them; a loss further on costs little
            nph = ((lost && last < 4) || (nph > 1 && other)) ? NPH : 1;
            DT_MARK(3);
            // P3: count my true range (the range of the last covered lane may end at the block's
            // end-of-block or at an invalid code).  From the counts P1/P2 kept: a lane on its P1
            // path takes the continuation symbols before its sync point plus its P1 symbols from
            // there (P1's prefix before the sync point -- a few symbols -- decoded again); a
            // covered lane takes its coverer's continuation counts.  An empty last range (an
            // end-of-block right at its start) is decoded as before.
            const bool mine = (int)gl <= last;
            uint32_t cnt = 0, byt = 0, kend = 0;
            uint64_t q = my_t;
            bool counted = false;
            if (mine && !(my_t == my_e && (int)gl == last)) {
                if (my_ph < 0) {
                    cnt = my_pc, byt = my_pb, q = my_e, counted = true;
                } else {
                    uint64_t pp = g + (uint64_t)my_ph;
                    uint32_t c0 = 0, b0c = 0;
                    while (pp < my_sp) {
                        uint32_t kk;
                        decode_symbol(lit_s[slot], dist_s[slot], window(pp), kk, nb, bl);
                        if (kk >= 2u) break;
                        ++c0, b0c += bl;
                        pp += nb;
                    }
                    if (pp == my_sp) {
                        cnt = my_pc + li_n1[w][my_ph][gl] - c0;
                        byt = my_pb + li_b1[w][my_ph][gl] - b0c;
                        q = my_e, counted = true;
                    }
                }
            }
            if (mine && !counted) {
                cnt = 0, byt = 0, q = my_t;
                while (q < my_e || (q == my_e && (int)gl == last)) {
                    decode_symbol(lit_s[slot], dist_s[slot], window(q), kend, nb, bl);
                    if (kend >= 2u) {
                        q += kend == 2u ? nb : 0;
                        break;
                    }
                    ++cnt;
                    byt += bl;
                    q += nb;
                    if (q >= my_e && (int)gl != last) break;
                    if (q >= my_e) break;
                }
            }
            __syncwarp();
            DT_MARK(4);
            // the last covered lane tells how the round ended
            const uint32_t kl = __shfl_sync(0xffffffffu, kend, last);
            const uint64_t ql = __shfl_sync(0xffffffffu, q, last);
            uint32_t ci_ = cnt, cb_ = byt;  // exclusive scans of counts and bytes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t a1 = __shfl_up_sync(0xffffffffu, ci_, o), a2 = __shfl_up_sync(0xffffffffu, cb_, o);
                if ((int)gl >= o) ci_ += a1, cb_ += a2;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, ci_, 31), totb = __shfl_sync(0xffffffffu, cb_, 31);
            const uint32_t sbase = ns + ci_ - cnt, bbase = bytes + cb_ - byt;
            // P4: write my symbols (indices past MAXSYM are not stored: the block fails below)
            if (mine && cnt) {
                uint64_t r = my_t;
                uint32_t bsum = bbase;
                for (uint32_t m = 0; m < cnt; ++m) {
                    uint32_t kk;
                    const uint32_t sym = decode_symbol(lit_s[slot], dist_s[slot], window(r), kk, nb, bl);
                    const uint32_t idx = sbase + m;
                    if (idx < MAXSYM) {
                        if (idx % SEG == 0) ckpt_pool[ci * NCKPT + idx / SEG] = bsum;
                        out[idx] = sym;
                    }
                    if (kk == 0u) nz |= sym;
                    bsum += bl;
                    r += nb;
                }
            }
            ns += tot;
            bytes += totb;
            if (ns > MAXSYM) good = false;  // only an end-of-block may follow MAXSYM symbols
            if (kl == 3u) good = false;
            if (kl == 2u) {
                eob = true;
                if (ns % SEG == 0 && ns < MAXSYM && gl == 0) ckpt_pool[ci * NCKPT + ns / SEG] = bytes;
            }
            base = (kl == 2u) ? ql : __shfl_sync(0xffffffffu, my_e, last);
            __syncwarp();
            DT_MARK(5);
        }
        const uint64_t pos = base;
        nz = __reduce_or_sync(0xffffffffu, nz);
        if (pos > endbit) good = false;
        used = pos - off;
        if (gl == 0) {
            c.ok = good ? 1 : 0;
            c.nzlit = nz != 0;
            c.end_bit = used;
            c.nsyms = ns;
            c.out_bytes = bytes;
            c.rounds = nrounds;
            c.t_hdr = (uint32_t)(tm1 - tm0), c.t_tab = (uint32_t)(tm2 - tm1), c.t_dec = (uint32_t)(gtimer() - tm2);
#ifdef IPCG_DTIME
            for (int i = 0; i < 6; ++i) c.t_ph[i] = dt[i];
#endif
            // link to the candidate that starts where this block ends (the chain follows it)
            int nx = -1;
            const Tables T = tabs[c.job];
            const unsigned long long key = used + 1;
            uint64_t sl = hslot(key, T.hcap);
            for (uint64_t probe = 0; probe < T.hcap; ++probe, sl = (sl + 1) & (T.hcap - 1)) {
                const unsigned long long k = T.hash[sl];
                if (k == 0ull) break;
                if (k == key) {
                    nx = (int)T.hval[sl];
                    break;
                }
            }
            c.next = nx;
        }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------- 3. chain
// decode one block at `b` into fallback symbols (slow path, one thread)
__device__ bool chain_decode_block(Bits &b, int type, uint32_t *fb, uint64_t fcap, uint64_t &fused, uint32_t &nsyms,
                                   uint64_t &bytes) {
    uint8_t lens[320];
    Canon lit, dist, cs;
    int nlen, ndist;
    if (type == 1) {
        for (int i = 0; i < 144; ++i) lens[i] = 8;
        for (int i = 144; i < 256; ++i) lens[i] = 9;
        for (int i = 256; i < 280; ++i) lens[i] = 7;
        for (int i = 280; i < 288; ++i) lens[i] = 8;
        for (int i = 0; i < 32; ++i) lens[288 + i] = 5;  // zlib's fixed distance table has 32 codes
        nlen = 288;
        ndist = 32;
    } else {
        if (!read_dynamic_header(b, lens, nlen, ndist, cs)) return false;
    }
    nsyms = 0;
    bytes = 0;
    if (type == 1) {
        // the fixed codes by arithmetic on the bit-reversed next 7/8/9 bits (the canonical
        // bit-at-a-time loop cost ~1 us per symbol here, on small fields' critical path)
        for (;;) {
            const uint32_t v = b.peek(9);
            const uint32_t c7 = __brev(v) >> 25, c8 = __brev(v) >> 24, c9 = __brev(v) >> 23;
            int sym;
            if (c7 <= 23u) sym = 256 + (int)c7, b.drop(7);
            else if (c8 >= 48u && c8 <= 191u) sym = (int)c8 - 48, b.drop(8);
            else if (c8 >= 192u && c8 <= 199u) sym = 280 + (int)c8 - 192, b.drop(8);
            else sym = 144 + (int)c9 - 400, b.drop(9);
            if (b.overrun()) return false;
            if (sym == 256) return true;
            if (fused >= fcap) return false;
            if (sym < 256) {
                fb[fused++] = sym_lit((uint32_t)sym);
                ++nsyms;
                ++bytes;
                continue;
            }
            const int li = sym - 257;
            if (li >= 29) return false;
            const uint32_t len = kLBase[li] + b.get(kLExt[li]);
            const int ds = (int)(__brev(b.peek(5)) >> 27);
            b.drop(5);
            if (ds >= 30) return false;
            const uint32_t d = kDBase[ds] + b.get(kDExt[ds]);
            fb[fused++] = sym_match(len, d);
            ++nsyms;
            bytes += len;
        }
    }
    if (!canon_build(lit, lens, nlen, 1) || !canon_build(dist, lens + nlen, ndist, 2)) return false;
    for (;;) {
        const int sym = canon_decode(lit, b);
        if (sym < 0 || b.overrun()) return false;
        if (sym == 256) return true;
        if (fused >= fcap) return false;
        if (sym < 256) {
            fb[fused++] = sym_lit((uint32_t)sym);
            ++nsyms;
            ++bytes;
            continue;
        }
        const int li = sym - 257;
        if (li >= 29) return false;
        const uint32_t len = kLBase[li] + b.get(kLExt[li]);
        const int ds = canon_decode(dist, b);
        if (ds < 0 || ds >= 30) return false;
        const uint32_t d = kDBase[ds] + b.get(kDExt[ds]);
        fb[fused++] = sym_match(len, d);
        ++nsyms;
        bytes += len;
    }
}

// The common case of the chain, in parallel: every block of every stream is a dynamic block
// whose candidate decoded ok, so a stream's blocks are the candidate list from the one at bit 16
// (after the zlib header) along `next` to a BFINAL candidate.  One CTA ranks all candidates by
// pointer jumping (suffix sums of output bytes, emit segments, block counts; the 2^l-th
// successors kept per level), then a thread per block of each complete stream finds its node by
// the binary expansion of its rank and writes its Blk; k_chain walks only the streams left over
// (stored/fixed/unmatched blocks, or chains of 2^RANK_L blocks or more).  The walk this replaces
// cost ~0.45 ms for a 900-block stream: one dependent L2 round trip per block.
constexpr int RANK_L = 16;
struct RankWs {
    int *nx[2];
    int *tm[2];
    uint64_t *sb[2];
    uint32_t *ss[2], *sn[2];
    uint8_t *sz[2];
    int *jump;  // [RANK_L][nc]
    int *jhead;         // [njobs]: head candidate of a ranked stream, -1 otherwise
    uint64_t *jpre;     // [njobs + 1]: prefix sums of the ranked streams' block counts
};

__global__ void __launch_bounds__(1024) k_rank(const InflateJob *jobs, int njobs, const Tables *tabs, JobMeta *meta,
                                              const Cand *cands, uint32_t nc, RankWs W) {
    const unsigned tid = threadIdx.x, nth = blockDim.x;
    for (uint32_t c = tid; c < nc; c += nth) {
        const Cand &k = cands[c];
        const int nx = (k.ok && !k.bfinal && k.next >= 0 && (uint32_t)k.next < nc && cands[k.next].ok) ? k.next : -1;
        W.nx[0][c] = nx;
        W.tm[0][c] = (int)c;
        W.sb[0][c] = k.ok ? k.out_bytes : 0;
        W.ss[0][c] = k.nsyms > 0 ? (k.nsyms + SEG - 1) / SEG : 1;
        W.sn[0][c] = 1;
        W.sz[0][c] = k.nzlit ? 1 : 0;
    }
    __shared__ int more;
    int cur = 0;
    for (int l = 0; l < RANK_L; ++l) {
        if (tid == 0) more = 0;
        __syncthreads();
        const int o = cur ^ 1;
        for (uint32_t c = tid; c < nc; c += nth) {
            const int nx = W.nx[cur][c];
            W.jump[(size_t)l * nc + c] = nx;
            if (nx >= 0) {
                W.nx[o][c] = W.nx[cur][nx];
                W.tm[o][c] = W.tm[cur][nx];
                W.sb[o][c] = W.sb[cur][c] + W.sb[cur][nx];
                W.ss[o][c] = W.ss[cur][c] + W.ss[cur][nx];
                W.sn[o][c] = W.sn[cur][c] + W.sn[cur][nx];
                W.sz[o][c] = W.sz[cur][c] | W.sz[cur][nx];
                more = 1;
            } else {
                W.nx[o][c] = -1;
                W.tm[o][c] = W.tm[cur][c];
                W.sb[o][c] = W.sb[cur][c];
                W.ss[o][c] = W.ss[cur][c];
                W.sn[o][c] = W.sn[cur][c];
                W.sz[o][c] = W.sz[cur][c];
            }
        }
        __syncthreads();
        cur = o;
        if (!more) {
            for (int l2 = l + 1; l2 < RANK_L; ++l2)
                for (uint32_t c = tid; c < nc; c += nth) W.jump[(size_t)l2 * nc + c] = -1;
            break;
        }
        __syncthreads();  // `more` is reset only after every thread read it
    }
    __syncthreads();
    // per stream (a thread each): its head, and whether the ranked list is the whole stream
    for (int j = (int)tid; j < njobs; j += (int)nth) {
        int head = -1;
        bool ok = false;
        const InflateJob job = jobs[j];
        const Tables T = tabs[j];
        bool hdr = job.src_len >= 2 && !meta[j].overflow;
        if (hdr) {
            const uint32_t cmf = job.src[0], flg = job.src[1];
            hdr = ((cmf << 8) | flg) % 31 == 0 && (cmf & 15) == 8 && (cmf >> 4) + 8 <= 15 && !(flg & 0x20);
        }
        if (hdr) {
            const unsigned long long key = 16 + 1;
            uint64_t sl = hslot(key, T.hcap);
            for (uint64_t probe = 0; probe < T.hcap; ++probe, sl = (sl + 1) & (T.hcap - 1)) {
                const unsigned long long kk = T.hash[sl];
                if (kk == 0ull) break;
                if (kk == key) {
                    head = (int)T.hval[sl];
                    break;
                }
            }
        }
        if (head >= 0 && (uint32_t)head < nc && cands[head].ok && W.nx[cur][head] < 0) {
            const int term = W.tm[cur][head];
            const Cand &tc = cands[term];
            const uint64_t e = tc.end_bit, bp = (e + 7) >> 3;
            if (tc.bfinal && W.sn[cur][head] <= T.bcap && W.sb[cur][head] == job.dst_len && bp + 4 <= job.src_len) {
                ok = true;
                JobMeta &m = meta[j];
                m.adler_want = ((uint32_t)job.src[bp] << 24) | ((uint32_t)job.src[bp + 1] << 16) |
                               ((uint32_t)job.src[bp + 2] << 8) | job.src[bp + 3];
                m.nblocks = W.sn[cur][head];
                m.allzero = !W.sz[cur][head];
                m.nseg = W.ss[cur][head];
                m.ranked = 1;
            }
        }
        W.jhead[j] = ok ? head : -1;
    }
    __syncthreads();
    if (tid == 0) {  // (streams are few: a serial prefix)
        uint64_t acc = 0;
        for (int j = 0; j < njobs; ++j) {
            W.jpre[j] = acc;
            if (W.jhead[j] >= 0) acc += W.sn[cur][W.jhead[j]];
        }
        W.jpre[njobs] = acc;
    }
    __syncthreads();
    // a thread per block of every ranked stream: its node by the binary expansion of its rank
    const uint64_t total = W.jpre[njobs];
    for (uint64_t idx = tid; idx < total; idx += nth) {
        int jl = 0, jh = njobs - 1;  // last stream with jpre <= idx
        while (jl < jh) {
            const int mid = (jl + jh + 1) / 2;
            if (W.jpre[mid] <= idx) jl = mid;
            else jh = mid - 1;
        }
        const int head = W.jhead[jl];
        const uint32_t r = (uint32_t)(idx - W.jpre[jl]);
        const Tables T = tabs[jl];
        const uint64_t B = W.sb[cur][head];
        const uint32_t SS = W.ss[cur][head];
        int node = head;
        for (int l = 0; l < RANK_L && node >= 0; ++l)
            if ((r >> l) & 1u) node = W.jump[(size_t)l * nc + node];
        const Cand &c = cands[node];
        Blk blk;
        blk.type = 1;
        blk.nsyms = c.nsyms;
        blk.src = (uint64_t)node * MAXSYM;
        blk.out_off = B - W.sb[cur][node];
        blk.out_len = c.out_bytes;
        blk.nseg = c.nsyms > 0 ? (c.nsyms + SEG - 1) / SEG : 1;
        blk.seg_base = SS - W.ss[cur][node];
        blk.ckpt = (uint64_t)node;
        T.blocks[r] = blk;
    }
}

__global__ void k_chain(const InflateJob *jobs, int njobs, const Tables *tabs, JobMeta *meta, const Cand *cands) {
    // a warp per stream (lane 0): the serial walks and fallback decodes of different streams must
    // not share a warp, where their divergent loops would run one after another
    const int j = blockIdx.x;
    if (threadIdx.x != 0 || j >= njobs || meta[j].ranked) return;
    const InflateJob job = jobs[j];
    const Tables T = tabs[j];
    JobMeta &m = meta[j];
    bool err = false;
    uint64_t out = 0, nb = 0, fused = 0;
    bool nonzero = false;
    uint32_t segs = 0;
    if (job.src_len < 2) err = true;
    if (!err) {
        const uint32_t cmf = job.src[0], flg = job.src[1];
        if (((cmf << 8) | flg) % 31 != 0 || (cmf & 15) != 8 || (cmf >> 4) + 8 > 15 || (flg & 0x20)) err = true;
    }
    uint64_t e = 16;
    int last = 0;
    int pending = -1;  // candidate known (linked by k_decode_cands) to start at e
    while (!err && !last) {
        if (nb >= T.bcap) {
            err = true;
            break;
        }
        Blk blk;
        blk.out_off = out;
        if (pending >= 0 && cands[pending].ok) {  // fast path: no header read, no hash probe
            const Cand &c = cands[pending];
            last = c.bfinal;
            blk.type = 1;
            blk.ckpt = (uint64_t)pending;
            blk.src = (uint64_t)pending * MAXSYM;
            blk.nsyms = c.nsyms;
            blk.out_len = c.out_bytes;
            e = c.end_bit;
            if (c.nzlit) nonzero = true;
            pending = c.next;
            out += blk.out_len;
            if (out > job.dst_len) {
                err = true;
                break;
            }
            blk.nseg = blk.nsyms > 0 ? (blk.nsyms + SEG - 1) / SEG : 1;
            blk.seg_base = segs;
            segs += blk.nseg;
            T.blocks[nb++] = blk;
            continue;
        }
        pending = -1;
        Bits b;
        b.init(job.src, job.src_len, e);
        last = (int)b.get(1);
        const uint32_t type = b.get(2);
        if (type == 0) {
            const uint64_t bp = (b.used + 7) >> 3;
            if (bp + 4 > job.src_len) {
                err = true;
                break;
            }
            const uint32_t L = job.src[bp] | (job.src[bp + 1] << 8), NL = job.src[bp + 2] | (job.src[bp + 3] << 8);
            if (L != (~NL & 0xffff) || bp + 4 + L > job.src_len) {
                err = true;
                break;
            }
            blk.type = 0;
            blk.ckpt = ~0ull;
            blk.src = bp + 4;
            blk.out_len = L;
            blk.nsyms = 0;
            e = (bp + 4 + L) * 8;
            if (L) nonzero = true;  // conservative
        } else if (type == 3) {
            err = true;
            break;
        } else {
            bool found = false;
            if (type == 2 && !m.overflow) {
                const unsigned long long key = e + 1;
                uint64_t s = hslot(key, T.hcap);
                for (uint64_t probe = 0; probe < T.hcap; ++probe, s = (s + 1) & (T.hcap - 1)) {
                    const unsigned long long k = T.hash[s];
                    if (k == 0ull) break;
                    if (k == key) {
                        const Cand &c = cands[T.hval[s]];
                        if (c.ok) {
                            blk.type = 1;
                            blk.ckpt = T.hval[s];
                            blk.src = (uint64_t)T.hval[s] * MAXSYM;
                            blk.nsyms = c.nsyms;
                            blk.out_len = c.out_bytes;
                            e = c.end_bit;
                            found = true;
                            pending = c.next;
                            if (c.nzlit) nonzero = true;
                        }
                        break;
                    }
                }
            }
            if (!found) {
                uint32_t ns;
                uint64_t bytes;
                const uint64_t f0 = fused;
                if (!chain_decode_block(b, (int)type, T.fallback, T.fcap, fused, ns, bytes)) {
                    err = true;
                    break;
                }
                blk.type = 2;  // symbols in the job's fallback buffer
                ++m.nfallback;
                m.fb_syms += ns;
                blk.ckpt = ~0ull;
                blk.src = f0;
                blk.nsyms = ns;
                blk.out_len = bytes;
                e = b.used;
                nonzero = true;  // conservative
            }
        }
        out += blk.out_len;
        if (out > job.dst_len) {
            err = true;
            break;
        }
        blk.nseg = (blk.type == 1 && blk.nsyms > 0) ? (blk.nsyms + SEG - 1) / SEG : 1;
        blk.seg_base = segs;
        segs += blk.nseg;
        T.blocks[nb++] = blk;
    }
    if (!err) {
        const uint64_t bp = (e + 7) >> 3;
        if (bp + 4 > job.src_len || out != job.dst_len) err = true;
        else
            m.adler_want = ((uint32_t)job.src[bp] << 24) | ((uint32_t)job.src[bp + 1] << 16) |
                           ((uint32_t)job.src[bp + 2] << 8) | job.src[bp + 3];
    }
    m.nblocks = err ? 0 : (uint32_t)nb;
    m.allzero = !nonzero;
    m.nseg = err ? 0 : segs;
    if (err) m.status = 1;
}

__global__ void k_fill_zero(const InflateJob *jobs, const JobMeta *meta) {
    const int j = blockIdx.y;
    if (meta[j].status || !meta[j].allzero) return;
    const InflateJob job = jobs[j];
    const uint64_t v = (reinterpret_cast<uintptr_t>(job.dst) & 15) ? 0 : job.dst_len / 16;
    uint4 *d4 = reinterpret_cast<uint4 *>(job.dst);  // plane rows are 16-byte aligned
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < v; i += (uint64_t)gridDim.x * blockDim.x)
        d4[i] = make_uint4(0, 0, 0, 0);
    for (uint64_t i = v * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < job.dst_len;
         i += (uint64_t)gridDim.x * blockDim.x)
        job.dst[i] = 0;
}

// -------------------------------------------------------------------- 4. emit
__device__ __forceinline__ bool flag_get(const uint32_t *f, uint64_t i) { return (f[i >> 5] >> (i & 31)) & 1u; }

// bytes [mo, tend) all repeat byte mo-1 (distance-1 matches); every lane calls it
__device__ __forceinline__ void emit_run(const Tables &T, uint8_t *dst, uint64_t mo, uint64_t tend, uint64_t b0,
                                         unsigned lane) {
    const uint64_t s = mo - 1;
    bool unres = true;
    uint32_t P = (uint32_t)s;
    uint8_t val = 0;
    if (s >= b0) {
        if (flag_get(T.flags, s)) P = T.ptr[s];
        else unres = false, val = dst[s];
    }
    if (unres) {
        // 16-byte stores from the first index whose address is 16-byte aligned
        const uint64_t pb = reinterpret_cast<uintptr_t>(T.ptr) / 4;  // ptr is 4-byte aligned
        const uint64_t a = min(tend, ((pb + mo + 3) & ~(uint64_t)3) - pb), be = (pb + tend) & ~(uint64_t)3;
        const uint64_t b = be > pb + a ? be - pb : a;
        for (uint64_t x = mo + lane; x < a; x += 32) T.ptr[x] = P;
        const uint4 PP = make_uint4(P, P, P, P);
        uint4 *p4 = reinterpret_cast<uint4 *>(T.ptr + a);
        for (uint64_t x = lane; x < (b - a) / 4; x += 32) p4[x] = PP;
        for (uint64_t x = b + lane; x < tend; x += 32) T.ptr[x] = P;
        // flag bits: partial words at the ends by atomics (their other bits belong to other
        // symbols, possibly other warps' segments), whole words stored
        const uint64_t fa = min(tend, (mo + 31) & ~(uint64_t)31), fb = max(fa, tend & ~(uint64_t)31);
        if (lane == 0 && mo < fa) atomicOr(&T.flags[mo >> 5], ((1u << (uint32_t)(fa - mo)) - 1u) << (mo & 31));
        for (uint64_t w = fa / 32 + lane; w < fb / 32; w += 32) T.flags[w] = 0xffffffffu;
        if (lane == 1 && fb < tend) atomicOr(&T.flags[fb >> 5], (1u << (uint32_t)(tend - fb)) - 1u);
    } else {
        const uint64_t db = reinterpret_cast<uintptr_t>(dst);
        const uint64_t a = min(tend, ((db + mo + 15) & ~(uint64_t)15) - db), be = (db + tend) & ~(uint64_t)15;
        const uint64_t b = be > db + a ? be - db : a;
        for (uint64_t x = mo + lane; x < a; x += 32) dst[x] = val;
        const uint32_t w4 = (uint32_t)val * 0x01010101u;
        const uint4 VV = make_uint4(w4, w4, w4, w4);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst + a);
        for (uint64_t x = lane; x < (b - a) / 16; x += 32) d4[x] = VV;
        for (uint64_t x = b + lane; x < tend; x += 32) dst[x] = val;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(WARPS * 32) k_emit(const InflateJob *jobs, const Tables *tabs, JobMeta *meta,
                                                   const uint32_t *pool, const uint32_t *ckpt_pool, const uint64_t *segoff,
                                                   int njobs) {
    // one warp per emit segment (SEG symbols of one block, output offset from the
    // candidate's checkpoints); copies reaching before the segment become pointers.
    // A match whose distance exceeds the bytes written before it is zlib's "invalid distance
    // too far back": the job fails (meta.bad) and nothing is written for it.  All-zero jobs
    // (filled by k_fill_zero) still run their first 32 KiB of output here, check only.
    // the grid covers the segments of every job back to back (segoff: their prefix sums; a
    // (segment, job) grid left ~95% of a cfg2 retrieval's CTAs with nothing to do)
    const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gg = (uint64_t)blockIdx.x * WARPS + w;
    if (gg >= segoff[njobs]) return;
    int jl = 0, jh = njobs - 1;  // last job with segoff[j] <= gg
    while (jl < jh) {
        const int mid = (jl + jh + 1) / 2;
        if (segoff[mid] <= gg) jl = mid;
        else jh = mid - 1;
    }
    const int j = jl;
    JobMeta &jm = meta[j];
    if (jm.status) return;
    const bool check_only = jm.allzero != 0;
    const uint64_t gs = gg - segoff[j];
    if (gs >= jm.nseg) return;
    const InflateJob job = jobs[j];
    const Tables T = tabs[j];
    uint32_t lo = 0, hi = jm.nblocks - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (T.blocks[mid].seg_base <= gs) lo = mid;
        else hi = mid - 1;
    }
    const Blk blk = T.blocks[lo];
    const uint32_t seg = (uint32_t)(gs - blk.seg_base);
    uint8_t *dst = job.dst;
    if (check_only && blk.type == 0) return;
    if (blk.type == 0) {
        for (uint64_t i = lane; i < blk.out_len; i += 32) dst[blk.out_off + i] = job.src[blk.src + i];
        return;
    }
    // a block without checkpoints (decoded by the chain itself) is one segment of any length
    const uint32_t s_begin = seg * SEG, s_end = blk.nseg == 1 ? blk.nsyms : min(blk.nsyms, s_begin + SEG);
    const uint64_t b0 = blk.out_off + (seg ? ckpt_pool[blk.ckpt * NCKPT + seg] : 0);
    if (check_only && b0 >= 32768) return;  // no distance reaches past 32 KiB of output
    const uint32_t *syms = blk.type == 1 ? pool + blk.src : T.fallback + blk.src;
    uint64_t o = b0;
    // 32 symbols per step: output offsets by a warp prefix sum, literals written in parallel,
    // then the step's matches in order (a match may read bytes of earlier ones)
    for (uint32_t sb = s_begin; sb < s_end; sb += 32) {
        const uint32_t s = sb + lane;
        const bool valid = s < s_end;
        const uint32_t v = valid ? syms[s] : 0u;
        const bool ismatch = valid && (v & 0x80000000u);
        const uint32_t mylen = !valid ? 0u : ismatch ? ((v >> 16) & 0x1ff) : 1u;
        uint32_t incl = mylen;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
            if ((int)lane >= off) incl += t;
        }
        const uint32_t my_rel = incl - mylen;
        if (valid && !ismatch && !check_only) dst[o + my_rel] = (uint8_t)v;
        __syncwarp();
        unsigned mm = __ballot_sync(0xffffffffu, ismatch);
        const unsigned r1 = __ballot_sync(0xffffffffu, ismatch && (v & 0xffffu) == 0u);  // distance-1 matches
        while (mm) {
            const int l = __ffs(mm) - 1;
            const uint32_t mv = __shfl_sync(0xffffffffu, v, l);
            const uint64_t mo = o + __shfl_sync(0xffffffffu, my_rel, l);
            const uint32_t len = (mv >> 16) & 0x1ff, d = (mv & 0xffff) + 1;
            if (d == 1u && mo >= 1 && !check_only) {
                // a run: consecutive distance-1 matches (lanes l .. e-1) all repeat the byte before
                // the first, so the whole run is one fill -- of its value when that byte is
                // resolved, else of its pointer with the flag bits set -- in 16-byte stores (the
                // per-match byte loop was the emit's latency on run-heavy planes)
                const unsigned above = ~r1 & (0xffffffffu << l);
                const int e = above ? __ffs(above) - 1 : 32;
                mm &= e == 32 ? 0u : (0xffffffffu << e);
                const uint64_t tend = o + __shfl_sync(0xffffffffu, incl, e - 1);
                emit_run(T, dst, mo, tend, b0, lane);
                continue;
            }
            mm &= mm - 1;
            if ((uint64_t)d > mo) {  // warp-uniform
                if (lane == 0) atomicOr(&jm.bad, 1);
                continue;
            }
            if (check_only) continue;
            // i % d by a reciprocal multiply (exact for i < 2^16: i < len <= 258; d = 1 apart,
            // whose reciprocal 2^32 does not fit)
            const uint32_t rcp = (d > 1u && d < len) ? 0xffffffffu / d + 1u : 0u;  // (an integer division: only when used)
            // every source byte precedes mo, so the lanes of one match never depend on each other;
            // unresolved bytes (sources in earlier segments) get a pointer, and their flag bits
            // are set with one ballot-aggregated atomic per 32 bytes
            for (uint32_t base = 0; base < len; base += 32) {
                const uint32_t i = base + lane;
                const bool act = i < len;
                bool unres = false;
                if (act) {
                    const uint64_t src = mo - d + (d < len ? (d == 1u ? 0u : i - d * __umulhi(i, rcp)) : i);
                    const uint64_t t = mo + i;
                    if (src >= b0) {
                        if (flag_get(T.flags, src)) {
                            T.ptr[t] = T.ptr[src];
                            unres = true;
                        } else {
                            dst[t] = dst[src];
                        }
                    } else {
                        T.ptr[t] = (uint32_t)src;
                        unres = true;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, unres);
                if (m) {
                    const uint64_t t0 = mo + base;
                    const unsigned sh = (unsigned)(t0 & 31);
                    if (lane == 0) atomicOr(&T.flags[t0 >> 5], m << sh);
                    if (lane == 1 && sh) atomicOr(&T.flags[(t0 >> 5) + 1], m >> (32 - sh));
                }
                __syncwarp();
            }
        }
        o += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// ------------------------------------------------------------------ 5. resolve
// Every unresolved byte t points (ptr[t]) to an earlier byte with the same final value.  In
// run-heavy planes nearly every byte of every segment after the first is unresolved and the
// chains cross all segments, but they funnel through few distinct bytes (the tails of
// earlier segments).  So, in one cooperative launch:
//   A. mark every unresolved byte that some pointer targets (the marked set is closed under
//      ptr: a marked byte's own target is marked by it);
//   B. pointer-jump on the marked bytes only, until none targets an unresolved byte;
//   C. resolve every unresolved byte in one step (its target is resolved or marked).
// (Jumping on all unresolved bytes cost ~8 rounds x 40 M random updates.)
template <class F>
__device__ __forceinline__ void for_each_set(const uint32_t *bits, uint64_t words, uint64_t tid, uint64_t nth, F &&f) {
    for (uint64_t wi = tid; wi < words; wi += nth) {
        uint32_t x = bits[wi];
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            f(wi * 32 + (uint64_t)b);
        }
    }
}

// every set flag, one thread per BYTE: the flag word is a warp broadcast, ptr/dst accesses of a
// warp are 32 consecutive bytes (a thread per flag WORD made every lane's accesses 32 bytes
// apart: one sector per lane per access, and run-heavy planes are almost all unresolved)
// (a warp loads 32 flag words at once and skips the zero ones with a ballot; every thread of
// the grid must call it: nth is a multiple of 32)
template <class F>
__device__ __forceinline__ void for_each_flagged(const uint32_t *bits, uint64_t nbytes, uint64_t tid, uint64_t nth,
                                                 F &&f) {
    const uint64_t nwords = (nbytes + 31) / 32;
    const unsigned lane = (unsigned)(tid & 31);
    for (uint64_t w0 = (tid >> 5) * 32; w0 < nwords; w0 += (nth >> 5) * 32) {
        const uint32_t mine = w0 + lane < nwords ? bits[w0 + lane] : 0u;
        unsigned nz = __ballot_sync(0xffffffffu, mine != 0u);
        while (nz) {
            const int k = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t word = __shfl_sync(0xffffffffu, mine, k);
            const uint64_t t = (w0 + (uint64_t)k) * 32 + lane;
            if ((word >> lane) & 1u) f(t);
        }
    }
}

// CTA-aggregated append: returns the first of `n` list slots claimed for this thread (one global
// atomic per CTA; every thread of the CTA must call it)
__device__ __forceinline__ unsigned long long cta_append(unsigned n, unsigned long long *ctr, unsigned *s_cnt,
                                                        unsigned long long *s_base) {
    const unsigned lane = threadIdx.x & 31;
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += v;
    }
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    unsigned woff = 0;
    if (lane == 31 && incl) woff = atomicAdd(s_cnt, incl);
    woff = __shfl_sync(0xffffffffu, woff, 31);
    __syncthreads();
    if (threadIdx.x == 0) *s_base = *s_cnt ? atomicAdd(ctr, (unsigned long long)*s_cnt) : 0ull;
    __syncthreads();
    return *s_base + woff + (incl - n);
}

__global__ void __launch_bounds__(256) k_resolve_all(const InflateJob *jobs, const Tables *tabs, const JobMeta *meta,
                                                    int njobs, unsigned *changed, uint64_t *mlist, uint64_t mcap,
                                                    unsigned long long *mcount) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    if (tid == 0) mcount[7] = gtimer();
    // A1: mark every unresolved byte some pointer targets (lanes of a warp that point at the byte
    // the previous lane points at -- the bytes of one run -- leave the atomic to that lane)
    const unsigned lane = threadIdx.x & 31;
    __shared__ unsigned s_cnt;
    __shared__ unsigned long long s_base;
    for (int j = 0; j < njobs; ++j) {
        if (meta[j].status || meta[j].allzero) continue;
        const Tables T = tabs[j];
        const uint64_t nwords = (jobs[j].dst_len + 31) / 32;
        for (uint64_t w0 = (tid >> 5) * 32; w0 < nwords; w0 += (nth >> 5) * 32) {
            const uint32_t mine = w0 + lane < nwords ? T.flags[w0 + lane] : 0u;
            unsigned nz = __ballot_sync(0xffffffffu, mine != 0u);
            while (nz) {  // four flag words per step, loads interleaved (see C)
                constexpr int U = 4;
                uint32_t sp[U];
                bool f[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = nz ? __ffs(nz) - 1 : 0;
                    const uint32_t word = __shfl_sync(0xffffffffu, mine, k);
                    f[u] = nz && ((word >> lane) & 1u);
                    nz &= nz - 1;
                    sp[u] = f[u] ? T.ptr[(w0 + (uint64_t)k) * 32 + lane] : ~0u;
                }
                bool c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t up = __shfl_up_sync(0xffffffffu, sp[u], 1);
                    c[u] = f[u] && (lane == 0 || up != sp[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) c[u] = c[u] && flag_get(T.flags, sp[u]) && !flag_get(T.mark, sp[u]);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (c[u]) atomicOr(&T.mark[sp[u] >> 5], 1u << (sp[u] & 31));
            }
        }
    }
    grid.sync();
    // A2: list the marked bytes (job << 40 | byte): a CTA-uniform pass over the mark words, one
    // list atomic per CTA step (one per warp, or per byte, serialised on the counter)
    for (int j = 0; j < njobs; ++j) {
        if (meta[j].status || meta[j].allzero) continue;
        const Tables T = tabs[j];
        const uint64_t nwords = (jobs[j].dst_len + 31) / 32;
        for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < nwords; b0 += nth) {
            const uint64_t wi = b0 + threadIdx.x;
            const uint32_t mw = wi < nwords ? T.mark[wi] : 0u;
            const unsigned long long at = cta_append(__popc(mw), mcount, &s_cnt, &s_base);
            uint32_t x = mw;
            for (unsigned long long i = at; x; ++i) {
                const int b = __ffs(x) - 1;
                x &= x - 1;
                if (i < mcap) mlist[i] = ((uint64_t)j << 40) | (wi * 32 + (uint64_t)b);
            }
        }
    }
    grid.sync();
    const unsigned long long M0 = *(volatile unsigned long long *)mcount;
    unsigned long long *stamp = mcount + 4;  // diagnostics: globaltimer after A, B, C
    if (tid == 0) stamp[0] = gtimer();
    if (M0 <= mcap) {
        unsigned long long *cnt = mcount + 1;  // three rotating survivor counters
        uint64_t *cur = mlist, *nxt = mlist + mcap;
        unsigned long long M = M0;
        for (int round = 0; M; ++round) {
            if (tid == 0) cnt[(round + 1) % 3] = 0;  // its last reader finished before the previous sync
            for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < M; b0 += nth) {
                const uint64_t i = b0 + threadIdx.x;
                bool keep = false;
                uint64_t e = 0;
                if (i < M) {
                    e = cur[i];
                    const Tables T = tabs[e >> 40];
                    const uint32_t t = (uint32_t)(e & 0xffffffffffull);
                    const uint32_t sp = T.ptr[t];
                    if (flag_get(T.flags, sp)) {
                        const uint32_t np = T.ptr[sp];
                        T.ptr[t] = np;
                        keep = flag_get(T.flags, np);
                    }
                }
                const unsigned long long at = cta_append(keep ? 1u : 0u, &cnt[round % 3], &s_cnt, &s_base);
                if (keep) nxt[at] = e;
            }
            grid.sync();
            M = *(volatile unsigned long long *)&cnt[round % 3];
            uint64_t *tmp = cur;
            cur = nxt, nxt = tmp;
            if (M == 0 && tid == 0) changed[3] = (unsigned)round + 1;  // rounds run (diagnostics)
        }
    } else {
        for (int round = 0;; ++round) {
            if (tid == 0) changed[(round + 1) % 3] = 0;  // its last reader finished before the previous sync
            bool any = false;
            for (int j = 0; j < njobs; ++j) {
                if (meta[j].status || meta[j].allzero) continue;
                const Tables T = tabs[j];
                for_each_set(T.mark, (jobs[j].dst_len + 31) / 32, tid, nth, [&](uint64_t t) {
                    const uint32_t sp = T.ptr[t];
                    if (flag_get(T.flags, sp)) {
                        T.ptr[t] = T.ptr[sp];
                        any = true;
                    }
                });
            }
            if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(&changed[round % 3], 1u);
            grid.sync();
            if (*(volatile unsigned *)&changed[round % 3] == 0) {
                if (tid == 0) changed[3] = (unsigned)round + 1;  // rounds run (diagnostics)
                break;
            }
        }
    }
    grid.sync();
    if (tid == 0) stamp[1] = gtimer();
    // C: resolve every unresolved byte in one step (its target is resolved or listed); four flag
    // words per step with their loads interleaved (the chain ptr -> flag -> ptr -> value is
    // latency-bound one word at a time)
    for (int j = 0; j < njobs; ++j) {
        if (meta[j].status || meta[j].allzero) continue;
        const InflateJob job = jobs[j];
        const Tables T = tabs[j];
        const uint64_t nwords = (job.dst_len + 31) / 32;
        for (uint64_t w0 = (tid >> 5) * 32; w0 < nwords; w0 += (nth >> 5) * 32) {
            const uint32_t mine = w0 + lane < nwords ? T.flags[w0 + lane] : 0u;
            unsigned nz = __ballot_sync(0xffffffffu, mine != 0u);
            while (nz) {
                constexpr int U = 4;
                uint64_t t[U];
                uint32_t sp[U];
                bool f[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = nz ? __ffs(nz) - 1 : 0;
                    const uint32_t word = __shfl_sync(0xffffffffu, mine, k);
                    f[u] = nz && ((word >> lane) & 1u);
                    nz &= nz - 1;
                    t[u] = (w0 + (uint64_t)k) * 32 + lane;
                    sp[u] = f[u] ? T.ptr[t[u]] : 0u;
                }
                bool g[U];
#pragma unroll
                for (int u = 0; u < U; ++u) g[u] = f[u] && flag_get(T.flags, sp[u]);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (g[u]) sp[u] = T.ptr[sp[u]];
                uint8_t v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = f[u] ? job.dst[sp[u]] : 0;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (f[u]) job.dst[t[u]] = v[u];
            }
        }
    }
    grid.sync();
    if (tid == 0) stamp[2] = gtimer();
}

// --------------------------------------------------------------- 6. checks
// Adler-32 of the output: B = sum_i (n - i) b_i = n A - sum_i i b_i (mod 65521), 16-byte loads
// from the first 16-byte boundary, dp4a sums and index-weighted sums, one modulo per thread
__global__ void k_adler(const InflateJob *jobs, JobMeta *meta, unsigned long long *acc) {
    const int j = blockIdx.y;
    if (meta[j].status) return;
    const InflateJob job = jobs[j];
    const uint64_t n = job.dst_len;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t head0 = (16 - (reinterpret_cast<uintptr_t>(job.dst) & 15)) & 15, head = head0 < n ? head0 : n;
    const uint64_t nv = (n - head) / 16;
    unsigned long long A = 0, W = 0;
    const uint4 *pv = reinterpret_cast<const uint4 *>(job.dst + head);
    for (uint64_t v = tid; v < nv; v += nth) {
        const uint4 q = pv[v];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t s = 0, ws = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t sk = __dp4a(w[k], 0x01010101u, 0u);
            s += sk;
            ws += __dp4a(w[k], 0x03020100u, 0u) + 4u * k * sk;
        }
        A += s;
        W += (unsigned long long)(head + 16 * v) * s + ws;
    }
    for (uint64_t i = tid; i < n; i += nth) {  // the unaligned head and the tail
        if (i >= head && i < head + 16 * nv) continue;
        const uint32_t b = job.dst[i];
        A += b;
        W += (unsigned long long)i * b;
    }
    const unsigned long long M = 65521;
    unsigned long long B = ((n % M) * (A % M) + M - W % M) % M;
    for (int o = 16; o > 0; o >>= 1) {
        A += __shfl_down_sync(0xffffffffu, A, o);
        B += __shfl_down_sync(0xffffffffu, B, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc[2 * j], A);
        atomicAdd(&acc[2 * j + 1], B % 65521u);
    }
}
__global__ void k_finish(const InflateJob *jobs, int njobs, JobMeta *meta, const unsigned long long *acc, int *status) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= njobs) return;
    JobMeta &m = meta[j];
    if (m.bad) m.status = 1;
    if (!m.status) {
        const uint64_t n = jobs[j].dst_len;
        const uint32_t a = (uint32_t)((1 + acc[2 * j]) % 65521u), b = (uint32_t)((acc[2 * j + 1] + n) % 65521u);
        if (((b << 16) | a) != m.adler_want) m.status = 1;
    }
    status[j] = m.status;
}

// per-job arena: [hash keys | flags | mark] (zeroed) then [hash values | blocks | fallback | ptr]
__global__ void k_setup(const InflateJob *jobs, int njobs, Tables *tabs, uint8_t *arena, const uint64_t *offs,
                        const uint64_t *caps) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= njobs) return;
    uint8_t *a = arena + offs[j];
    Tables T;
    T.hcap = caps[4 * j];
    T.bcap = caps[4 * j + 1];
    T.fcap = caps[4 * j + 2];
    const uint64_t n = jobs[j].dst_len;
    T.hash = reinterpret_cast<unsigned long long *>(a);
    a += T.hcap * 8;
    T.flags = reinterpret_cast<uint32_t *>(a);
    a += ((n + 31) / 32) * 4 + 16;
    T.mark = reinterpret_cast<uint32_t *>(a);
    a += ((n + 31) / 32) * 4 + 16;
    a = reinterpret_cast<uint8_t *>(((uintptr_t)a + 15) & ~uintptr_t(15));
    T.hval = reinterpret_cast<uint32_t *>(a);
    a += T.hcap * 4;
    a = reinterpret_cast<uint8_t *>(((uintptr_t)a + 15) & ~uintptr_t(15));
    T.blocks = reinterpret_cast<Blk *>(a);
    a += T.bcap * sizeof(Blk);
    T.fallback = reinterpret_cast<uint32_t *>(a);
    a += T.fcap * 4;
    a = reinterpret_cast<uint8_t *>(((uintptr_t)a + 15) & ~uintptr_t(15));  // k_emit's run fills store 16 bytes
    T.ptr = reinterpret_cast<uint32_t *>(a);
    tabs[j] = T;
}

__global__ void k_zero(const InflateJob *jobs, const Tables *tabs) {
    const int j = blockIdx.y;
    const Tables T = tabs[j];
    const uint64_t words = (T.hcap * 8 + 2 * (((jobs[j].dst_len + 31) / 32) * 4 + 16)) / 4;
    uint32_t *z = reinterpret_cast<uint32_t *>(T.hash);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        z[i] = 0;
}

}  // namespace

// per-job arena layout (host mirror of k_setup)
static uint64_t pow2_at_least(uint64_t v) {
    uint64_t p = 64;
    while (p < v) p <<= 1;
    return p;
}

struct InflatePlan {
    std::vector<uint64_t> offs, caps;
    uint64_t arena = 0;
};

static InflatePlan plan_jobs(const std::vector<InflateJob> &jobs) {
    InflatePlan p;
    for (const InflateJob &j : jobs) {
        const uint64_t hcap = pow2_at_least(2 * (j.src_len / 512 + 64));
        const uint64_t bcap = j.src_len / 16 + 64;  // zlib blocks are >= 2 KiB compressed
        const uint64_t fcap = j.dst_len + 16;
        const uint64_t bytes = hcap * 12 + 64 + bcap * sizeof(Blk) + fcap * 4 + 2 * (((j.dst_len + 31) / 32) * 4 + 16) +
                               (j.dst_len + 4) * 4 + 64;
        p.offs.push_back(p.arena);
        p.caps.insert(p.caps.end(), {hcap, bcap, fcap, 0});
        p.arena += (bytes + 255) & ~uint64_t(255);
    }
    return p;
}

void inflate_batch_host(const std::vector<InflateJob> &jobs, int *status_dev, DevAlloc &alloc, cudaStream_t st,
                        cudaStream_t check, cudaEvent_t fork, cudaEvent_t done) {
    const int n = (int)jobs.size();
    if (n == 0) return;
    const InflatePlan P = plan_jobs(jobs);
    uint64_t max_src = 0, max_dst = 0, total_src = 0;
    for (const InflateJob &j : jobs) {
        max_src = std::max(max_src, j.src_len);
        max_dst = std::max(max_dst, j.dst_len);
        total_src += j.src_len;
    }
    const uint64_t cand_cap = total_src / 256 + 64 * (uint64_t)n;
    // small tables: jobs, offs, caps, tabs, meta, counters
    const size_t jb = n * sizeof(InflateJob), ob = n * 8, cb = n * 4 * 8, tb = n * sizeof(Tables),
                 mb = n * sizeof(JobMeta), sb = (n + 1) * 8;
    uint8_t *small = static_cast<uint8_t *>(alloc.get(jb + ob + cb + sb + tb + mb + 16 * n + 64 + 1024, st));
    InflateJob *jd = reinterpret_cast<InflateJob *>(small);
    uint64_t *od = reinterpret_cast<uint64_t *>(small + jb);
    uint64_t *cd = reinterpret_cast<uint64_t *>(small + jb + ob);
    uint64_t *tiles_d = reinterpret_cast<uint64_t *>(small + jb + ob + cb);  // scan tiles: prefix per job
    Tables *td = reinterpret_cast<Tables *>(((uintptr_t)(small + jb + ob + cb + sb) + 15) & ~uintptr_t(15));
    JobMeta *md = reinterpret_cast<JobMeta *>(((uintptr_t)(td + n) + 15) & ~uintptr_t(15));
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(((uintptr_t)(md + n) + 15) & ~uintptr_t(15));
    unsigned long long *ncand = acc + 2 * n;
    std::vector<uint8_t> host(jb + ob + cb + sb);
    std::memcpy(host.data(), jobs.data(), jb);
    std::memcpy(host.data() + jb, P.offs.data(), ob);
    std::memcpy(host.data() + jb + ob, P.caps.data(), cb);
    std::vector<uint64_t> tiles(n + 1, 0);
    for (int q = 0; q < n; ++q) tiles[q + 1] = tiles[q] + (jobs[q].src_len + SCAN_TILE - 1) / SCAN_TILE;
    std::memcpy(host.data() + jb + ob + cb, tiles.data(), sb);
    CK(cudaMemcpyAsync(small, host.data(), host.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(md, 0, (uint8_t *)(ncand + 1) - (uint8_t *)md, st));
    uint8_t *arena = static_cast<uint8_t *>(alloc.get(P.arena + 256, st));
    Cand *cands = static_cast<Cand *>(alloc.get(cand_cap * sizeof(Cand) + 64, st));
    const uint64_t surv_cap = total_src / 32 + 4096;  // measured: ~1 in 1100 bit offsets survives (overflow -> slow chain path)
    Survivor *surv = static_cast<Survivor *>(alloc.get(surv_cap * sizeof(Survivor), st));
    unsigned long long *nsurv = static_cast<unsigned long long *>(alloc.get(8, st));
    CK(cudaMemsetAsync(nsurv, 0, 8, st));
    k_setup<<<(n + 63) / 64, 64, 0, st>>>(jd, n, td, arena, od, cd);
    CKL();
    k_zero<<<dim3(grid_for(max_dst / 32 + 1024, 256, 512), n), 256, 0, st>>>(jd, td);
    CKL();
    {
        ProfScope ps("inflate.scan", st, total_src);
        k_scan<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles[n], (uint64_t)num_sms() * 8)), 256, 0, st>>>(
            jd, n, tiles_d, td, md, surv, nsurv, surv_cap);
        CKL();
        k_validate<<<148 * 8, 256, 0, st>>>(jd, td, md, surv, nsurv, surv_cap, cands, ncand, cand_cap);
        CKL();
    }
    unsigned long long hc = 0;
    readback(&hc, ncand, 8, st);
    const uint64_t nc = std::min<uint64_t>(hc, cand_cap);
    uint32_t *pool = static_cast<uint32_t *>(alloc.get(std::max<uint64_t>(nc, 1) * MAXSYM * 4, st));
    uint32_t *ckpt = static_cast<uint32_t *>(alloc.get(std::max<uint64_t>(nc, 1) * NCKPT * 4, st));
    {
        ProfScope ps("inflate.decode", st, total_src);
        if (nc) {
            constexpr int CPW = IPCG_CPW;  // measured: 2 or 4 per warp diverge (literal vs match paths) and lose
            const unsigned g = (unsigned)std::min<uint64_t>((nc + DWARPS * CPW - 1) / (DWARPS * CPW), 148ull * 32);
            k_decode_cands<CPW><<<g, DWARPS * 32, 0, st>>>(jd, td, cands, ncand, cand_cap, pool, ckpt);
            CKL();
        }
        if (nc && nc <= (1u << 20)) {
            RankWs W;
            uint8_t *rw = static_cast<uint8_t *>(alloc.get(nc * (2 * (4 + 4 + 8 + 4 + 4 + 1) + 4 * RANK_L) + (size_t)n * 12 + 512, st));
            auto take = [&](size_t b) { uint8_t *q = rw; rw += (b + 15) & ~size_t(15); return q; };
            for (int h = 0; h < 2; ++h) {
                W.nx[h] = reinterpret_cast<int *>(take(nc * 4));
                W.tm[h] = reinterpret_cast<int *>(take(nc * 4));
                W.sb[h] = reinterpret_cast<uint64_t *>(take(nc * 8));
                W.ss[h] = reinterpret_cast<uint32_t *>(take(nc * 4));
                W.sn[h] = reinterpret_cast<uint32_t *>(take(nc * 4));
                W.sz[h] = take(nc);
            }
            W.jump = reinterpret_cast<int *>(take(nc * 4 * RANK_L));
            W.jhead = reinterpret_cast<int *>(take((size_t)n * 4));
            W.jpre = reinterpret_cast<uint64_t *>(take((size_t)(n + 1) * 8));
            k_rank<<<1, 1024, 0, st>>>(jd, n, td, md, cands, (uint32_t)nc, W);
            CKL();
        }
        k_chain<<<n, 32, 0, st>>>(jd, n, td, md, cands);
        CKL();
    }
    {
        ProfScope ps("inflate.emit", st, max_dst * n);
        std::vector<JobMeta> hm(n);
        readback(hm.data(), md, n * sizeof(JobMeta), st);
        uint64_t maxseg = 1;
        for (const JobMeta &m : hm) maxseg = std::max<uint64_t>(maxseg, m.nseg);
        if (getenv("IPCG_DEBUG_INFLATE")) {
            std::vector<Cand> hcands(nc);
            CK(cudaMemcpy(hcands.data(), cands, nc * sizeof(Cand), cudaMemcpyDeviceToHost));
            uint64_t ok = 0, okn = 0, badn = 0, hist[6] = {0, 0, 0, 0, 0, 0};
            uint64_t rsum = 0, rmax = 0, bits_sum = 0;
            for (const Cand &cc : hcands) {
                rsum += cc.rounds, rmax = std::max<uint64_t>(rmax, cc.rounds);
                bits_sum += cc.end_bit > cc.hdr_bit ? cc.end_bit - cc.hdr_bit : 0;
                if (cc.ok) ++ok, okn += cc.nsyms;
                else badn += cc.nsyms;
                const uint32_t v = cc.nsyms;
                hist[v == 0 ? 0 : v < 16 ? 1 : v < 256 ? 2 : v < 4096 ? 3 : v < 16000 ? 4 : 5]++;
            }
            unsigned long long hs = 0;
            CK(cudaMemcpy(&hs, nsurv, 8, cudaMemcpyDeviceToHost));
            {
                std::vector<std::pair<int, uint64_t>> rb;
                for (const Cand &cc : hcands) rb.push_back({cc.rounds, cc.end_bit > cc.hdr_bit ? cc.end_bit - cc.hdr_bit : 0});
                std::sort(rb.begin(), rb.end());
                fprintf(stderr, "inflate: slowest candidates (rounds, bits, syms):");
                for (size_t q = rb.size() > 8 ? rb.size() - 8 : 0; q < rb.size(); ++q) fprintf(stderr, " (%d, %llu)", rb[q].first, (unsigned long long)rb[q].second);
                fprintf(stderr, "\n");
                std::vector<const Cand *> byt;
                for (const Cand &cc : hcands) byt.push_back(&cc);
                std::sort(byt.begin(), byt.end(), [](const Cand *a, const Cand *b) { return a->t_hdr + a->t_tab + a->t_dec > b->t_hdr + b->t_tab + b->t_dec; });
                fprintf(stderr, "inflate: slowest candidates by time (hdr us, tables us, decode us, rounds, syms):");
                for (size_t q = 0; q < byt.size() && q < 6; ++q)
                    fprintf(stderr, " (%.1f, %.1f, %.1f, %d, %u)", byt[q]->t_hdr * 1e-3, byt[q]->t_tab * 1e-3, byt[q]->t_dec * 1e-3, byt[q]->rounds, byt[q]->nsyms);
#ifdef IPCG_DTIME
                fprintf(stderr, "\ninflate: their decode phases (stage, P1, P2, ranges, P3, P4 us):");
                for (size_t q = 0; q < byt.size() && q < 6; ++q)
                    fprintf(stderr, " (%.1f, %.1f, %.1f, %.1f, %.1f, %.1f)", byt[q]->t_ph[0] * 1e-3, byt[q]->t_ph[1] * 1e-3, byt[q]->t_ph[2] * 1e-3, byt[q]->t_ph[3] * 1e-3, byt[q]->t_ph[4] * 1e-3, byt[q]->t_ph[5] * 1e-3);
#endif
                double sh = 0, stb = 0, sd = 0;
                for (const Cand &cc : hcands) sh += cc.t_hdr, stb += cc.t_tab, sd += cc.t_dec;
                fprintf(stderr, "\ninflate: candidate time sums: hdr %.3f ms, tables %.3f ms, decode %.3f ms\n", sh * 1e-6, stb * 1e-6, sd * 1e-6);
            }
            fprintf(stderr, "inflate: %llu survivors of %llu bit offsets; decode rounds mean %.1f max %llu, bits/cand %.0f\n", hs,
                    (unsigned long long)total_src * 8, nc ? (double)rsum / nc : 0.0, (unsigned long long)rmax,
                    nc ? (double)bits_sum / nc : 0.0);
            fprintf(stderr, "inflate: %d jobs, %llu candidates (%llu ok, syms ok %llu bad %llu) nsyms hist 0:%llu <16:%llu <256:%llu <4k:%llu <16k:%llu >=16k:%llu\n",
                    n, (unsigned long long)nc, (unsigned long long)ok, (unsigned long long)okn, (unsigned long long)badn,
                    (unsigned long long)hist[0], (unsigned long long)hist[1], (unsigned long long)hist[2],
                    (unsigned long long)hist[3], (unsigned long long)hist[4], (unsigned long long)hist[5]);
            for (int q = 0; q < n; ++q)
                fprintf(stderr, "inflate job %d: src %llu dst %llu blocks %u allzero %d status %d fallback %u (%llu syms)\n", q,
                        (unsigned long long)jobs[q].src_len, (unsigned long long)jobs[q].dst_len, hm[q].nblocks,
                        hm[q].allzero, hm[q].status, hm[q].nfallback, (unsigned long long)hm[q].fb_syms);
        }
        {
            ProfScope ps2("inflate.emit_blocks", st, max_dst * n);
            std::vector<uint64_t> so(n + 1, 0);
            for (int q = 0; q < n; ++q) so[q + 1] = so[q] + (hm[q].status ? 0 : hm[q].nseg);
            uint64_t *sod = static_cast<uint64_t *>(alloc.get((n + 1) * 8, st));
            CK(cudaMemcpyAsync(sod, so.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
            if (so[n])
                k_emit<<<(unsigned)((so[n] + WARPS - 1) / WARPS), WARPS * 32, 0, st>>>(jd, td, md, pool, ckpt, sod, n);
            CKL();
            k_fill_zero<<<dim3(grid_for(max_dst / 16 + 1, 256, 512), n), 256, 0, st>>>(jd, md);
            CKL();
        }
        {
            ProfScope ps3("inflate.resolve", st, max_dst * n / 8);
            unsigned *changed = static_cast<unsigned *>(alloc.get(4 * sizeof(unsigned) + 8 * 8, st));
            unsigned long long *mcount = reinterpret_cast<unsigned long long *>(changed + 4);  // + 3 round counters
            CK(cudaMemsetAsync(changed, 0, 4 * sizeof(unsigned) + 8 * 8, st));
            uint64_t mcap = std::max<uint64_t>(1 << 20, max_dst * (uint64_t)n / 32);  // marked bytes listed
            uint64_t *mlist = static_cast<uint64_t *>(alloc.get(2 * mcap * 8, st));  // two halves (compaction)
            static int coop_cache[64] = {0};  // per device
            int &coop_blocks = coop_cache[current_device() & 63];
            if (!coop_blocks) {
                int per = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_resolve_all, 256, 0));
                coop_blocks = num_sms() * std::max(1, std::min(per, getenv("IPCG_RES_CTAS") ? atoi(getenv("IPCG_RES_CTAS")) : 8));
            }
            int nj = n;
            void *args[] = {(void *)&jd, (void *)&td, (void *)&md, (void *)&nj, (void *)&changed, (void *)&mlist,
                            (void *)&mcap, (void *)&mcount};
            CK(cudaLaunchCooperativeKernel((const void *)k_resolve_all, dim3(coop_blocks), dim3(256), args, 0, st));
            CKL();
            if (getenv("IPCG_DEBUG_INFLATE")) {
                unsigned hr[4];
                unsigned long long hm = 0;
                CK(cudaStreamSynchronize(st));
                CK(cudaMemcpy(hr, changed, sizeof(hr), cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(&hm, mcount, 8, cudaMemcpyDeviceToHost));
                unsigned long long stp[4];
                CK(cudaMemcpy(stp, mcount + 4, sizeof(stp), cudaMemcpyDeviceToHost));
                fprintf(stderr, "inflate: %llu listed (marked) bytes; resolve A %.3f B %.3f C %.3f ms\n", hm,
                        (stp[0] - stp[3]) * 1e-6, (stp[1] - stp[0]) * 1e-6, (stp[2] - stp[1]) * 1e-6);
                uint64_t unres = 0;
                std::vector<Tables> ht(n);
                CK(cudaMemcpy(ht.data(), td, n * sizeof(Tables), cudaMemcpyDeviceToHost));
                for (int q = 0; q < n; ++q) {
                    std::vector<uint32_t> fl((jobs[q].dst_len + 31) / 32);
                    CK(cudaMemcpy(fl.data(), ht[q].flags, fl.size() * 4, cudaMemcpyDeviceToHost));
                    for (uint32_t x : fl) unres += __builtin_popcount(x);
                }
                fprintf(stderr, "inflate: resolve rounds %u, unresolved bytes %llu of %llu\n", hr[3],
                        (unsigned long long)unres, (unsigned long long)(max_dst * n));
            }
        }
        // the checksum and final status: on `check` (when given) alongside the caller's next work
        const cudaStream_t cs = check ? check : st;
        if (check) {
            CK(cudaEventRecord(fork, st));
            CK(cudaStreamWaitEvent(check, fork, 0));
        }
        ProfScope ps4("inflate.adler", cs, max_dst * n);
        k_adler<<<dim3(grid_for(max_dst, 256, 256), n), 256, 0, cs>>>(jd, md, acc);
        CKL();
        k_finish<<<(n + 63) / 64, 64, 0, cs>>>(jd, n, md, acc, status_dev);
        CKL();
        if (check) CK(cudaEventRecord(done, check));
    }
}

}  // namespace ipcg
