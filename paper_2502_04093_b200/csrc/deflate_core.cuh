// deflate_core.cuh -- the zlib-1.3 `compress2(level 6)` semantics the reference's
// lossless stage produces (proj/src/backend.cpp:15-22), restated as position-
// parallel pieces so the GPU can produce the identical byte stream.
//
// The sequential algorithm (deflate_slow + longest_match + trees.c) is split into
//   1. per-position hash-chain links           (prev distance, u16)
//   2. per-position longest-match results      for chain limits 128 and 32
//   3. a lazy-parse *tag graph*: the parser state at a loop top is one of 4 tags
//      {A: after a match, B: literal pending, C128/C32: match pending, found with
//      chain 128/32}, so the parse is a functional graph over (position, tag);
//      "anchor" positions no match can jump over split it into chunks whose 4-entry
//      transfer maps compose associatively (parallel scan), then every chunk re-runs
//      from its true entry tag and emits its symbols
//   4. blocks of 16383 symbols, zlib's Huffman construction (build_tree/gen_bitlen/
//      gen_codes, build_bl_tree/scan_tree/send_tree), the stored/static/dynamic
//      choice including window-slide limits on stored blocks, bit emission.
// Everything here is __host__ __device__ so tests/native/zmodel.cpp can run the
// same code on the CPU and diff it against the system libz.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace ipz {

constexpr int WSIZE = 32768;
constexpr int MIN_LOOKAHEAD = 262;
constexpr int MAX_DIST = WSIZE - MIN_LOOKAHEAD;  // 32506
constexpr int MIN_MATCH = 3, MAX_MATCH = 258;
constexpr int GOOD_LENGTH = 8, MAX_LAZY = 16, NICE_LENGTH = 128, MAX_CHAIN = 128;  // configuration_table[6]
constexpr int TOO_FAR = 4096;
constexpr int BLOCK_SYMS = 16383;  // lit_bufsize - 1 (memLevel 8)
constexpr int L_CODES = 286, D_CODES = 30, BL_CODES = 19, END_BLOCK = 256;
constexpr int HEAP_SIZE = 2 * L_CODES + 1;
constexpr int MAX_BITS = 15, MAX_BL_BITS = 7;

enum Tag : int { TAG_A = 0, TAG_B = 1, TAG_C128 = 2, TAG_C32 = 3 };

HD uint32_t hash3(uint32_t a, uint32_t b, uint32_t c) { return ((a << 10) ^ (b << 5) ^ c) & 0x7fffu; }

// ----------------------------------------------------------------- match record
// bits 0-8 L128 | 9-23 D128 | 24-32 L32 | 33-47 D32 | 48 head at exactly MAX_DIST
HD uint64_t mrec_pack(uint32_t l128, uint32_t d128, uint32_t l32, uint32_t d32, uint32_t flag) {
    return (uint64_t)l128 | ((uint64_t)d128 << 9) | ((uint64_t)l32 << 24) | ((uint64_t)d32 << 33) | ((uint64_t)flag << 48);
}
HD uint32_t mrec_l128(uint64_t r) { return (uint32_t)(r & 0x1ff); }
HD uint32_t mrec_d128(uint64_t r) { return (uint32_t)((r >> 9) & 0x7fff); }
HD uint32_t mrec_l32(uint64_t r) { return (uint32_t)((r >> 24) & 0x1ff); }
HD uint32_t mrec_d32(uint64_t r) { return (uint32_t)((r >> 33) & 0x7fff); }
HD uint32_t mrec_flag(uint64_t r) { return (uint32_t)((r >> 48) & 1); }

// longest_match (deflate.c) for chain limits 128 and 32 at once.  `prevd[q]` is the
// distance from q to the previous position with the same hash (0 = none).  Lengths
// are capped at the lookahead, which is equivalent to zlib's garbage-tolerant scan
// because nice_match is capped at the lookahead too (the first candidate reaching
// the data end always terminates the search).
// The search is a small state machine (init + one candidate per step) so a GPU lane can
// interleave many positions and never idle behind a neighbour's long chain.
struct MatchState {
    int64_t p, q, maxlen, nice, limit;
    uint32_t best, bestd, l32, d32, flag;
    int i;     // index of the candidate q (1-based)
    int done;  // 1 once the search has terminated
};

template <class Bytes, class Prev>
HD void match_init(MatchState &s, int64_t p, int64_t n, const Bytes &, const Prev &prevd) {
    s.p = p;
    s.best = s.bestd = s.l32 = s.d32 = s.flag = 0;
    s.i = 1;
    s.done = 1;
    if (p + MIN_MATCH > n) return;  // not inserted: hash_head = NIL
    const uint32_t d0 = prevd(p);
    if (d0 == 0) return;
    s.q = p - (int64_t)d0;
    if (s.q == 0 || d0 > (uint32_t)MAX_DIST) return;  // NIL / too far for the head check
    s.flag = d0 == (uint32_t)MAX_DIST;
    s.maxlen = (n - p) < MAX_MATCH ? (n - p) : MAX_MATCH;
    s.nice = (n - p) < NICE_LENGTH ? (n - p) : NICE_LENGTH;
    s.limit = p - MAX_DIST > 0 ? p - MAX_DIST : 0;
    s.done = 0;
}

// evaluate candidate s.i at s.q, then move to the next candidate (or finish)
template <class Bytes, class Prev>
HD void match_step(MatchState &s, const Bytes &bytes, const Prev &prevd) {
    const int64_t p = s.p, q = s.q;
    // zlib's quick reject: a candidate that differs at best or best-1 cannot beat best
    const bool reject = s.best >= MIN_MATCH && (int64_t)s.best < s.maxlen &&
                        (bytes(q + s.best) != bytes(p + s.best) || bytes(q + s.best - 1) != bytes(p + s.best - 1));
    int64_t next_from = q;
    if (!reject) {
        // match length between p and q (>= 3 only when bytes 0,1 agree: hash implies byte 2)
        const int64_t len0 = bytes.match_len(p, q, s.maxlen);
        const int64_t len = len0 < MIN_MATCH ? 0 : len0;
        if ((uint32_t)len > s.best) {
            s.best = (uint32_t)len;
            s.bestd = (uint32_t)(p - q);
            if (len >= s.nice) {
                if (s.i <= 32) s.l32 = s.best, s.d32 = s.bestd;
                s.done = 1;
                return;
            }
        }
        if (s.i == 1 && q == p - 1 && len >= MIN_MATCH) {
            // p-1 starts a run of one byte value v covering [p-1, p-1+best].  The chain
            // continues p-2, p-3, ... down to the run start r (all hash(v,v,v)), and each of
            // those candidates fails the quick reject (its byte at +best is still v, the byte
            // at p+best is not).  Consume them in one step; results are unchanged.
            if (s.i <= 32) s.l32 = s.best, s.d32 = s.bestd;
            const uint32_t v = bytes(p - 1);
            const int64_t lo = p - (int64_t)MAX_CHAIN;
            const int64_t floor_ = (s.limit + 1) > lo ? (s.limit + 1) : lo;
            int64_t r = p - 1;
            while (r - 1 >= floor_ && bytes(r - 1) == v) --r;
            s.i += (int)(p - 1 - r);  // candidates p-2 .. r consumed
            if (s.i >= MAX_CHAIN) {
                s.done = 1;
                return;
            }
            next_from = r;
        }
    }
    if (s.i <= 32) s.l32 = s.best, s.d32 = s.bestd;
    const uint32_t dq = prevd(next_from);
    const int64_t q2 = next_from - (int64_t)dq;
    if (dq == 0 || !(q2 > s.limit) || s.i >= MAX_CHAIN) {
        s.done = 1;
        return;
    }
    s.q = q2;
    s.i += 1;
}

HD uint64_t match_result(const MatchState &s) { return mrec_pack(s.best, s.bestd, s.l32, s.d32, s.flag); }

template <class Bytes, class Prev>
HD uint64_t match_search(int64_t p, int64_t n, const Bytes &bytes, const Prev &prevd) {
    MatchState s;
    match_init(s, p, n, bytes, prevd);
    while (!s.done) match_step(s, bytes, prevd);
    return match_result(s);
}

// ---------------------------------------------------- match_search, fast form
// Same candidates in the same order and the same record as match_search, for streams
// shorter than 2^31 bytes.  Differences are only in how the work is spent:
//  * 32-bit positions;
//  * zlib's scan_end1/scan_end bytes of p live in registers (longest_match keeps them
//    in locals too), so a quick reject loads two bytes of q only;
//  * the run skip can only fire on candidate 1, which is peeled; in the loop the next
//    link prevd(q) does not depend on the compare and is loaded alongside it;
//  * common-prefix lengths compare 4 bytes per step from 4-byte-aligned words
//    (Words::word(k) = bytes 4k..4k+3, little-endian; Words::word is only called for
//    words whose first byte is < n).
HD uint32_t ldg_byte(const uint8_t *a) {
#if defined(__CUDA_ARCH__)
    return __ldg(a);
#else
    return *a;
#endif
}
// bytes a[0] | a[1] << 8 from the aligned word holding a[0] (and the next one when a[0] is its
// last byte): the chain walk's two quick-reject bytes in ~1.25 loads instead of 2 -- k_match is
// bound by L1 accesses of scattered lanes.  (Stream rows are 16-byte aligned and padded, and
// a[1] is a byte the walk reads anyway.)
HD uint32_t ldg_pair(const uint8_t *a) {
#if defined(__CUDA_ARCH__)
    const uintptr_t u = reinterpret_cast<uintptr_t>(a);
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(u & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(u & 3) * 8;
    uint32_t v = __ldg(wp) >> sh;
    if (sh == 24) v |= __ldg(wp + 1) << 8;
    return v & 0xffffu;
#else
    return (uint32_t)a[0] | (uint32_t)a[1] << 8;
#endif
}
HD uint32_t funnel_r(uint32_t lo, uint32_t hi, uint32_t sh) {
#if defined(__CUDA_ARCH__)
    return __funnelshift_r(lo, hi, sh);
#else
    return (uint32_t)((((uint64_t)hi << 32) | lo) >> sh);
#endif
}
HD uint32_t first_set_byte(uint32_t x) {  // x != 0
#if defined(__CUDA_ARCH__)
    return (uint32_t)(__ffs((int)x) - 1) >> 3;
#else
    return (uint32_t)__builtin_ctz(x) >> 3;
#endif
}

template <class Words>
HD uint32_t match_len32(const Words &w, uint32_t n, uint32_t a, uint32_t b, uint32_t maxlen) {
    const uint32_t sa = (a & 3) * 8, sb = (b & 3) * 8;
    uint32_t ka = a >> 2, kb = b >> 2;
    uint32_t a0 = w.word(ka), b0 = w.word(kb);
    for (uint32_t len = 0;; len += 4) {
        const uint32_t a1 = 4 * (ka + 1) < n ? w.word(ka + 1) : 0u;
        const uint32_t b1 = 4 * (kb + 1) < n ? w.word(kb + 1) : 0u;
        uint32_t x = funnel_r(a0, a1, sa) ^ funnel_r(b0, b1, sb);
        if (len + 4 >= maxlen) {
            const uint32_t r = maxlen - len;  // 1..4
            if (r < 4) x &= (1u << (8 * r)) - 1u;
            return x ? len + first_set_byte(x) : maxlen;
        }
        if (x) return len + first_set_byte(x);
        ++ka, ++kb;
        a0 = a1, b0 = b1;
    }
}

// The walk is resumable: walk32_start examines candidate 1 (and its run skip) and
// positions the walk on candidate 2; walk32_run examines up to `budget` candidates and
// either finishes (returns true, record in `rec`) or stops at the top of the next
// candidate with the state in `s` (tests/native/zmodel.cpp pins stop/resume at every
// budget).  A k_match that gave every position a short budget and resumed the unfinished
// walks from a compacted queue was measured slower (25.8 vs 22.1 ms): ncu showed the same
// 11 active lanes per instruction in the resume pass, so the divergence is within a chain
// step (quick reject vs. compare), not between chain lengths.
struct Walk32 {
    uint32_t p, q, best, bestd, l32, d32, flag;
    int i;  // index of candidate q
};

template <class Words, class Prev>
HD bool walk32_start(uint32_t p, uint32_t n, const Words &w, const Prev &prevd, Walk32 &s, uint64_t &rec,
                     int max_chain = MAX_CHAIN) {
    rec = 0;
    if (p + MIN_MATCH > n) return true;
    const uint32_t d0 = prevd(p);
    if (d0 == 0 || d0 == p || d0 > (uint32_t)MAX_DIST) return true;
    const uint32_t flag = d0 == (uint32_t)MAX_DIST;
    const uint32_t maxlen = n - p < (uint32_t)MAX_MATCH ? n - p : (uint32_t)MAX_MATCH;
    const uint32_t nice = n - p < (uint32_t)NICE_LENGTH ? n - p : (uint32_t)NICE_LENGTH;
    const uint32_t limit = p > (uint32_t)MAX_DIST ? p - (uint32_t)MAX_DIST : 0u;
    uint32_t best = 0, bestd = 0;
    uint32_t q = p - d0, from = q;
    int i = 1;
    {  // candidate 1: no quick reject (best == 0); may start a same-byte run
       // (a pair-load reject of candidates whose first two bytes differ from p's was measured:
       // no change -- the compare's first words are L1 hits next to the link loads)
        const uint32_t len = match_len32(w, n, p, q, maxlen);
        if (len >= (uint32_t)MIN_MATCH) {
            best = len, bestd = p - q;
            if (len >= nice) {
                rec = mrec_pack(best, bestd, best, bestd, flag);
                return true;
            }
            if (q == p - 1) {  // see match_step: candidates p-2 .. r all fail the quick reject
                const uint32_t v = w.byte(p - 1);
                const uint32_t lo = p > (uint32_t)MAX_CHAIN ? p - (uint32_t)MAX_CHAIN : 0u;
                const uint32_t floor_ = limit + 1 > lo ? limit + 1 : lo;
                uint32_t r = p - 1;
                while (r >= floor_ + 1 && w.byte(r - 1) == v) --r;
                i += (int)(p - 1 - r);
                if (i >= max_chain) {
                    rec = mrec_pack(best, bestd, best, bestd, flag);
                    return true;
                }
                from = r;
            }
        }
    }
    const uint32_t dq = prevd(from);
    // (from == limit is possible here: the head candidate may sit at exactly MAX_DIST)
    if (dq == 0 || from - dq <= limit || i >= max_chain) {
        rec = mrec_pack(best, bestd, best, bestd, flag);
        return true;
    }
    s = Walk32{p, from - dq, best, bestd, best, bestd, flag, i + 1};
    return false;
}

// scan_end1 / scan_end (only meaningful while MIN_MATCH <= best; best < nice <= maxlen holds
// in the loop).  Both quick-reject bytes of q are loaded unconditionally through
// qb = stream + best - 1.  While best == 0 they are q, q+1, checked against p, p+1: a chained
// candidate has p's hash, and hash3 keeps all 8 bits of the third byte once the first two are
// fixed, so equal first two bytes mean a match of >= MIN_MATCH, and any other candidate's
// compare could not set best (it would be < MIN_MATCH).  (Comparing every candidate while
// best == 0 made the compare loop, run by ~5 lanes of 32, 45% of k_match's instructions.)
// The chain ends when the link is NIL or leaves the window: dq - 1 >= q - lim1 (unsigned;
// dq <= q and q >= lim1 for every chained candidate).  Candidates up to 32 and beyond run as
// two phases so the chain-32 snapshot is taken once instead of every step.  BUDGETED: stop
// after `budget` candidates (resumable walks); the one-pass search compiles the check out.
template <bool BUDGETED = true, class Words, class Prev>
HD bool walk32_run(uint32_t n, const Words &w, const Prev &prevd, Walk32 &s, int budget, uint64_t &rec,
                   int max_chain = MAX_CHAIN) {
    const uint32_t p = s.p;
    const uint32_t maxlen = n - p < (uint32_t)MAX_MATCH ? n - p : (uint32_t)MAX_MATCH;
    const uint32_t nice = n - p < (uint32_t)NICE_LENGTH ? n - p : (uint32_t)NICE_LENGTH;
    const uint32_t lim1 = (p > (uint32_t)MAX_DIST ? p - (uint32_t)MAX_DIST : 0u) + 1u;
    uint32_t q = s.q, best = s.best, bestd = s.bestd, l32 = s.l32, d32 = s.d32;
    int i = s.i;
    uint32_t e01 = w.byte(p + (best ? best - 1 : 0u)) | w.byte(p + (best ? best : 1u)) << 8;
    const uint8_t *qb = w.at(best ? best - 1 : 0u);
    int stop = i <= 32 ? 32 : MAX_CHAIN;
    for (;;) {
        if (BUDGETED && budget-- <= 0) {
            s.q = q, s.best = best, s.bestd = bestd, s.l32 = l32, s.d32 = d32, s.i = i;
            return false;
        }
        const uint32_t dq = prevd(q);
        if (ldg_pair(qb + q) == e01) {
            const uint32_t len = match_len32(w, n, p, q, maxlen);
            if (len >= (uint32_t)MIN_MATCH && len > best) {
                best = len, bestd = p - q;
                if (len >= nice) {
                    if (i <= 32) l32 = best, d32 = bestd;
                    break;
                }
                e01 = w.byte(p + best - 1) | w.byte(p + best) << 8;
                qb = w.at(best - 1);
            }
        }
        if (dq - 1u >= q - lim1 || i >= stop) {
            if (stop == 32) {
                l32 = best, d32 = bestd;
                if (max_chain > 32 && i == 32 && dq - 1u < q - lim1) {  // phase 2: candidates 33..MAX_CHAIN
                    stop = MAX_CHAIN;
                    q -= dq;
                    ++i;
                    continue;
                }
            }
            break;
        }
        q -= dq;
        ++i;
    }
    rec = mrec_pack(best, bestd, l32, d32, s.flag);
    return true;
}

template <class Words, class Prev>
HD uint64_t match_search32(uint32_t p, uint32_t n, const Words &w, const Prev &prevd) {
    Walk32 s;
    uint64_t rec;
    if (walk32_start(p, n, w, prevd, s, rec)) return rec;
    walk32_run<false>(n, w, prevd, s, 0, rec);
    return rec;
}

// ------------------------------------------------------------- window slides
// fill_window slides the 64 KiB window by WSIZE at loop tops; with the whole input
// available, the k-th slide happens at the first loop top >= slide_threshold(k).
HD int64_t tail_slide_index(int64_t n) { return n >= 65536 ? (n - 65536) / 32768 + 1 : 0; }
HD int64_t slides_before(int64_t p, int64_t n) {  // slides done by the loop top at p (inclusive)
    const int64_t kt = tail_slide_index(n);
    int64_t c = 0;
    if (p >= 65275) {
        c = (p - 65275) / 32768 + 1;
        if (c > kt) c = kt;
    }
    if (p >= n - 261 && p >= 32768 * kt + 65274) c = kt + 1;
    return c;
}
// the head candidate at window index 0 is NIL: only reachable right after a tail slide
HD bool tail_slide_nil(int64_t p, int64_t n) {
    const int64_t kt = tail_slide_index(n);
    return p == 32768 * kt + 65274 && p >= n - 261;
}

// -------------------------------------------------------------- parse step
struct Step {
    int64_t next_p;
    int next_tag;
    int emit;          // 0 none, 1 literal, 2 match
    uint32_t len, dist;  // match length / distance, or literal byte in len
};

// One iteration of deflate_slow's loop at loop top p entered with `tag`.
// rp = match record at p, rpm1 = match record at p-1 (only read for tags C*).
template <class Bytes>
HD Step parse_step(int64_t p, int tag, int64_t n, uint64_t rp, uint64_t rpm1, const Bytes &bytes) {
    Step s;
    uint32_t pl = 2, pd = 0;
    if (tag == TAG_C128) {
        pl = mrec_l128(rpm1);
        pd = mrec_d128(rpm1);
    } else if (tag == TAG_C32) {
        pl = mrec_l32(rpm1);
        pd = mrec_d32(rpm1);
    }
    const bool avail = tag != TAG_A;
    uint32_t ml = 2;
    int ktag = TAG_C128;
    if (p + MIN_MATCH <= n && pl < (uint32_t)MAX_LAZY && mrec_l128(rp) != 0 &&
        !(mrec_flag(rp) && tail_slide_nil(p, n))) {
        const bool short_chain = pl >= (uint32_t)GOOD_LENGTH;
        ktag = short_chain ? TAG_C32 : TAG_C128;
        const uint32_t M = short_chain ? mrec_l32(rp) : mrec_l128(rp);
        const uint32_t D = short_chain ? mrec_d32(rp) : mrec_d128(rp);
        if (M > pl) {
            ml = M;
            if (ml == MIN_MATCH && D > (uint32_t)TOO_FAR) ml = 2;
        } else {
            ml = pl;  // min(pl, lookahead): only used for the emit test below
        }
    }
    if (pl >= MIN_MATCH && ml <= pl) {
        s.emit = 2;
        s.len = pl;
        s.dist = pd;
        s.next_p = p - 1 + pl;
        s.next_tag = TAG_A;
        return s;
    }
    s.next_p = p + 1;
    s.next_tag = ml >= MIN_MATCH ? ktag : TAG_B;
    if (avail) {
        s.emit = 1;
        s.len = bytes(p - 1);
        s.dist = 0;
    } else {
        s.emit = 0;
        s.len = s.dist = 0;
    }
    return s;
}

// symbol encoding in the symbol stream: literal = byte; match = 1<<31 | (len-3)<<16 | (dist-1)
HD uint32_t sym_literal(uint32_t c) { return c; }
HD uint32_t sym_match(uint32_t len, uint32_t dist) { return 0x80000000u | ((len - 3) << 16) | (dist - 1); }
HD bool sym_is_match(uint32_t s) { return (s & 0x80000000u) != 0; }
HD uint32_t sym_lc(uint32_t s) { return (s >> 16) & 0xff; }     // len - 3
HD uint32_t sym_dist1(uint32_t s) { return s & 0xffff; }        // dist - 1
HD uint32_t sym_bytes(uint32_t s) { return sym_is_match(s) ? sym_lc(s) + 3 : 1; }

// ------------------------------------------------------- on-demand lazy parse
// The lazy parse (deflate_slow) needs longest_match only at the loop tops it visits, and only
// with one chain limit: 128, or 32 once prev_length >= good_length (zlib's chain_length >>= 2).
// A Walker runs the parse from any state, searching on demand; a state is (loop top p, tag) --
// the pending match of a C tag is the search result at p-1 with that tag's chain, so two walkers
// in the same (p, tag) continue identically.  The GPU runs one walker per chunk from (chunk
// start, A) and joins each chunk's walk onto the previous one's where the latter reaches a state
// the former visited (deflate.cu: k_od_walk / k_od_sync / k_od_chain / k_od_place).
struct Match {
    uint32_t len, dist, flag;
};

template <class Words, class Prev>
HD Match match_on_demand(uint32_t p, uint32_t n, const Words &w, const Prev &prevd, int chain) {
    Walk32 s;
    uint64_t rec;
    if (!walk32_start(p, n, w, prevd, s, rec, chain)) walk32_run<false>(n, w, prevd, s, 0, rec, chain);
    return chain == 32 ? Match{mrec_l32(rec), mrec_d32(rec), mrec_flag(rec)}
                       : Match{mrec_l128(rec), mrec_d128(rec), mrec_flag(rec)};
}

constexpr uint32_t NOSYM = 0xFFFFFFFFu;

struct Walker {
    uint32_t p, tag, pl, pd;  // loop top, tag, pending match (tags C128 / C32)
};

// one iteration of deflate_slow's loop from state s (the decisions of parse_step, the match at
// p searched here); returns the symbol it emits or NOSYM
template <class Words, class Prev>
HD uint32_t walker_step(Walker &s, uint32_t n, const Words &w, const Prev &prevd) {
    const uint32_t p = s.p;
    const bool pending = s.tag == TAG_C128 || s.tag == TAG_C32;
    const uint32_t pl = pending ? s.pl : 2u;
    uint32_t ml = 2, md = 0;
    uint32_t ktag = TAG_C128;
    if (p + MIN_MATCH <= n && pl < (uint32_t)MAX_LAZY) {
        const int chain = pl >= (uint32_t)GOOD_LENGTH ? 32 : MAX_CHAIN;
        const Match m = match_on_demand(p, n, w, prevd, chain);
        if (m.len != 0 && !(m.flag && tail_slide_nil((int64_t)p, (int64_t)n))) {
            ktag = chain == 32 ? TAG_C32 : TAG_C128;
            if (m.len > pl) {
                ml = m.len, md = m.dist;
                if (ml == (uint32_t)MIN_MATCH && md > (uint32_t)TOO_FAR) ml = 2;
            } else {
                ml = pl;
            }
        }
    }
    if (pl >= (uint32_t)MIN_MATCH && ml <= pl) {
        const uint32_t sym = sym_match(pl, s.pd);
        s.p = p - 1 + pl;
        s.tag = TAG_A;
        return sym;
    }
    const uint32_t sym = s.tag != TAG_A ? sym_literal(w.byte(p - 1)) : NOSYM;
    s.p = p + 1;
    s.tag = ml >= (uint32_t)MIN_MATCH ? ktag : (uint32_t)TAG_B;
    s.pl = ml, s.pd = md;
    return sym;
}

// visit word of a chunk walk at position p: bit 15 visited, bits 13-14 tag, bits 0-12 the number
// of symbols the walk emitted before that state (chunks of at most 8192 positions)
HD uint16_t vis_pack(uint32_t tag, uint32_t symidx) { return (uint16_t)(0x8000u | (tag << 13) | symidx); }
HD bool vis_match(uint16_t v, uint32_t tag) { return (v >> 13) == (0x4u | tag); }
HD uint32_t vis_symidx(uint16_t v) { return v & 0x1fffu; }

// ------------------------------------------------------------ static tables
HD int ilog2(uint32_t v) {  // v >= 1
#if defined(__CUDA_ARCH__)
    return 31 - __clz((int)v);
#else
    int r = 0;
    while (v >>= 1) ++r;
    return r;
#endif
}
HD uint32_t length_code(uint32_t lc) {  // _length_code[len-3]
    if (lc < 8) return lc;
    if (lc == 255) return 28;
    const int e = ilog2(lc) - 2;
    return 4u * (uint32_t)e + 4u + ((lc >> e) & 3u);
}
HD int extra_lbits(uint32_t code) { return (code < 8 || code == 28) ? 0 : (int)(code - 4) / 4; }
HD uint32_t base_length(uint32_t code) {
    if (code < 8) return code;
    if (code == 28) return 0;
    const int e = (int)(code - 4) / 4;
    return (4u + (code & 3u)) << e;
}
HD uint32_t dist_code(uint32_t d) {  // d = dist - 1
    if (d < 4) return d;
    const int e = ilog2(d) - 1;
    return 2u * (uint32_t)e + 2u + ((d >> e) & 1u);
}
HD int extra_dbits(uint32_t code) { return code < 4 ? 0 : (int)code / 2 - 1; }
HD uint32_t base_dist(uint32_t code) {
    if (code < 4) return code;
    const int e = (int)code / 2 - 1;
    return (2u + (code & 1u)) << e;
}
HD int extra_blbits(int code) { return code == 16 ? 2 : code == 17 ? 3 : code == 18 ? 7 : 0; }
HD int bl_order(int i) {
    const int8_t t[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    return t[i];
}
HD uint32_t bi_reverse(uint32_t code, int len) {  // len in 1..15
#if defined(__CUDA_ARCH__)
    return __brev(code) >> (32 - len);
#else
    uint32_t r = 0;
    for (int i = 0; i < len; ++i) {
        r = (r << 1) | (code & 1u);
        code >>= 1;
    }
    return r;
#endif
}
HD int static_llen(int n) { return n < 144 ? 8 : n < 256 ? 9 : n < 280 ? 7 : 8; }
HD uint32_t static_lcode(int n) {
    if (n < 144) return bi_reverse(48u + (uint32_t)n, 8);
    if (n < 256) return bi_reverse(400u + (uint32_t)(n - 144), 9);
    if (n < 280) return bi_reverse((uint32_t)(n - 256), 7);
    return bi_reverse(192u + (uint32_t)(n - 280), 8);
}
HD uint32_t static_dcode(int n) { return bi_reverse((uint32_t)n, 5); }

// ------------------------------------------------------------- Huffman trees
struct BlockTrees {
    uint16_t lcode[L_CODES + 2];
    uint8_t llen[L_CODES + 2];
    uint16_t dcode[D_CODES + 2];
    uint8_t dlen[D_CODES + 2];
    uint16_t blcode[BL_CODES];
    uint8_t bllen[BL_CODES];
    int16_t lmax, dmax, max_blindex;
    uint8_t type;      // 0 stored, 1 static, 2 dynamic
    uint8_t last;
    uint64_t opt_len, static_len;
    uint64_t body_bits;  // bits after the 3-bit header (stored: 32 + 8*len, alignment not included)
};

// zlib's heap orders nodes by smaller(n, m) = freq[n] < freq[m] || (freq[n] == freq[m] &&
// depth[n] <= depth[m]), i.e. (freq, depth) compared lexicographically with ties counting as
// "smaller".  Heap entries pack freq << 17 | depth << 10 | node into 32 bits so one load gives
// the whole key: a block's frequencies sum to at most 16384 (16383 symbols + END_BLOCK), and a
// Huffman tree over a total weight <= 16384 is at most ~21 levels deep, so zlib's uch depth never
// reaches the 7 bits kept here.  heap[heap_max..] then holds the nodes in zlib's order for
// gen_bitlen.
struct TreeScratch {
    alignas(16) uint32_t heap[HEAP_SIZE + 4];  // 16-byte aligned, spare entries: pqdownheap reads child pairs and grandchild quads
    uint16_t freq[HEAP_SIZE];     // leaf frequencies (input; forced leaves set to 1)
    uint16_t dad_len[HEAP_SIZE];  // zlib's dl union: Dad during build, Len after gen_bitlen
    uint16_t bl_count[MAX_BITS + 1];
    int heap_len, heap_max;
};

HD uint32_t hmake(uint32_t freq, uint32_t depth, int node) {
    return (freq << 17) | ((depth & 0x7f) << 10) | (uint32_t)node;
}
HD uint32_t hkey(uint32_t e) { return e >> 10; }
HD int hnode(uint32_t e) { return (int)(e & 1023); }

// (the two children heap[j], heap[j+1] -- j even -- come in one 8-byte load; keys compare as
// e | 1023, the node bits set, which orders like e >> 10; heap_len stays in a register.  The
// k_plan tree builds are issue-bound and this loop was over half of their instructions.)
struct alignas(8) HeapPair {
    uint32_t x, y;
};
struct alignas(16) HeapQuad {
    uint32_t x, y, z, w;
};
// The two children heap[j], heap[j+1] (j even) come in one 8-byte load, and the four
// grandchildren heap[2j .. 2j+3] are loaded (one 16-byte load) while this level compares, so the
// chain of dependent shared-memory loads is one per two levels; keys compare as e | 1023 (the
// node bits set), which orders like e >> 10; heap_len stays in a register.  The k_plan tree
// builds are latency/issue-bound and this loop was over half of their instructions.
HD void pqdownheap(TreeScratch &t, int k) {
    const uint32_t v = t.heap[k];
    const uint32_t vk = v | 1023u;
    const int len = t.heap_len;
    int j = k << 1;
    if (j <= len) {
        const HeapPair c0 = *reinterpret_cast<const HeapPair *>(&t.heap[j]);  // heap[j + 1] unused when j == len
        uint32_t cx = c0.x, cy = c0.y;
        for (;;) {
            const int g = j << 1;  // grandchildren: heap[g .. g+3] (children of j and j+1)
            HeapQuad q{0u, 0u, 0u, 0u};
            if (g <= len) q = *reinterpret_cast<const HeapQuad *>(&t.heap[g]);
            uint32_t hj = cx;
            int jj = j;
            if (j < len && (cy | 1023u) <= (cx | 1023u)) jj = j + 1, hj = cy;
            if (vk <= (hj | 1023u)) break;
            t.heap[k] = hj;
            k = jj;
            j = k << 1;
            if (j > len) break;
            if (jj == (g >> 1)) cx = q.x, cy = q.y;
            else cx = q.z, cy = q.w;
        }
    }
    t.heap[k] = v;
}

// build_tree + gen_bitlen + gen_codes (trees.c).  kind: 0 lit/len, 1 dist, 2 bit-length.
// freq[] of the `elems` leaves must be loaded into t.freq; returns max_code, writes
// lengths/codes; accumulates opt_len/static_len exactly as zlib does.
HD int build_tree(TreeScratch &t, int kind, int elems, uint8_t *len_out, uint16_t *code_out, uint64_t &opt_len,
                  uint64_t &static_len) {
    const int max_length = kind == 2 ? MAX_BL_BITS : MAX_BITS;
    int max_code = -1;
    t.heap_len = 0;
    t.heap_max = HEAP_SIZE;
    for (int n = 0; n < elems; n++) {
        if (t.freq[n] != 0) {
            t.heap[++t.heap_len] = hmake(t.freq[n], 0, max_code = n);
        } else {
            t.dad_len[n] = 0;
        }
    }
    while (t.heap_len < 2) {
        const int node = max_code < 2 ? ++max_code : 0;
        t.heap[++t.heap_len] = hmake(1, 0, node);
        t.freq[node] = 1;
        opt_len--;
        if (kind == 0) static_len -= (uint64_t)static_llen(node);
        else if (kind == 1) static_len -= 5;
    }
    for (int n = t.heap_len / 2; n >= 1; n--) pqdownheap(t, n);
    int node = elems;
    do {
        const uint32_t en = t.heap[1];  // pqremove
        t.heap[1] = t.heap[t.heap_len--];
        pqdownheap(t, 1);
        const uint32_t em = t.heap[1];
        t.heap[--t.heap_max] = en;
        t.heap[--t.heap_max] = em;
        const uint32_t dn = (en >> 10) & 0x7f, dm = (em >> 10) & 0x7f;
        t.dad_len[hnode(en)] = t.dad_len[hnode(em)] = (uint16_t)node;
        t.heap[1] = hmake((en >> 17) + (em >> 17), (dn >= dm ? dn : dm) + 1, node++);
        pqdownheap(t, 1);
    } while (t.heap_len >= 2);
    t.heap[--t.heap_max] = t.heap[1];

    // gen_bitlen
    for (int b = 0; b <= MAX_BITS; b++) t.bl_count[b] = 0;
    t.dad_len[hnode(t.heap[t.heap_max])] = 0;
    int overflow = 0;
    int h;
    for (h = t.heap_max + 1; h < HEAP_SIZE; h++) {
        const int n = hnode(t.heap[h]);
        int bits = t.dad_len[t.dad_len[n]] + 1;
        if (bits > max_length) bits = max_length, overflow++;
        t.dad_len[n] = (uint16_t)bits;
        if (n > max_code) continue;
        t.bl_count[bits]++;
        int xbits = 0;
        if (kind == 0 && n >= 257) xbits = extra_lbits((uint32_t)(n - 257));
        else if (kind == 1) xbits = extra_dbits((uint32_t)n);
        else if (kind == 2) xbits = extra_blbits(n);
        const uint64_t f = t.freq[n];
        opt_len += f * (uint64_t)(bits + xbits);
        if (kind == 0) static_len += f * (uint64_t)(static_llen(n) + xbits);
        else if (kind == 1) static_len += f * (uint64_t)(5 + xbits);
    }
    if (overflow != 0) {
        do {
            int bits = max_length - 1;
            while (t.bl_count[bits] == 0) bits--;
            t.bl_count[bits]--;
            t.bl_count[bits + 1] += 2;
            t.bl_count[max_length]--;
            overflow -= 2;
        } while (overflow > 0);
        h = HEAP_SIZE;
        for (int bits = max_length; bits != 0; bits--) {
            int n = t.bl_count[bits];
            while (n != 0) {
                const int m = hnode(t.heap[--h]);
                if (m > max_code) continue;
                if ((unsigned)t.dad_len[m] != (unsigned)bits) {
                    opt_len += ((uint64_t)bits - (uint64_t)t.dad_len[m]) * (uint64_t)t.freq[m];
                    t.dad_len[m] = (uint16_t)bits;
                }
                n--;
            }
        }
    }
    // gen_codes
    uint16_t next_code[MAX_BITS + 1];
    uint32_t code = 0;
    for (int bits = 1; bits <= MAX_BITS; bits++) {
        code = (code + t.bl_count[bits - 1]) << 1;
        next_code[bits] = (uint16_t)code;
    }
    for (int n = 0; n < elems; n++) {
        const int len = n <= max_code ? t.dad_len[n] : 0;
        len_out[n] = (uint8_t)len;
        code_out[n] = len ? (uint16_t)bi_reverse(next_code[len]++, len) : 0;
    }
    return max_code;
}

// scan_tree (counting) / send_tree (emitting) share this run-length walk.
template <class Visit>
HD void walk_tree_lengths(const uint8_t *len, int max_code, Visit &&visit) {
    int prevlen = -1, curlen, nextlen = len[0];
    int count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    for (int n = 0; n <= max_code; n++) {
        curlen = nextlen;
        nextlen = n + 1 <= max_code ? len[n + 1] : 0xffff;  // guard tree[max_code+1].Len = 0xffff
        if (++count < max_count && curlen == nextlen) {
            continue;
        } else if (count < min_count) {
            for (int c = 0; c < count; ++c) visit(curlen, 0);
        } else if (curlen != 0) {
            if (curlen != prevlen) {
                visit(curlen, 0);
                count--;
            }
            visit(16, count - 3);
        } else if (count <= 10) {
            visit(17, count - 3);
        } else {
            visit(18, count - 11);
        }
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) {
            max_count = 138, min_count = 3;
        } else if (curlen == nextlen) {
            max_count = 6, min_count = 3;
        } else {
            max_count = 7, min_count = 4;
        }
    }
}
// NOTE: scan_tree increments bl_tree[curlen].Freq += count in the count<min_count case,
// which the per-call visit above reproduces one at a time.

// Build the trees of one block from its symbol histogram (lfreq[286] incl. END_BLOCK=1,
// dfreq[30]) and choose stored / static / dynamic as _tr_flush_block does.
HD void plan_block(const uint32_t *lfreq, const uint32_t *dfreq, uint64_t stored_len, bool stored_ok, bool last,
                   TreeScratch &t, BlockTrees &bt) {
    uint64_t opt_len = 0, static_len = 0;
    for (int i = 0; i < HEAP_SIZE; ++i) t.freq[i] = 0;
    for (int i = 0; i < L_CODES; ++i) t.freq[i] = (uint16_t)lfreq[i];
    bt.lmax = (int16_t)build_tree(t, 0, L_CODES, bt.llen, bt.lcode, opt_len, static_len);
    for (int i = 0; i < HEAP_SIZE; ++i) t.freq[i] = 0;
    for (int i = 0; i < D_CODES; ++i) t.freq[i] = (uint16_t)dfreq[i];
    bt.dmax = (int16_t)build_tree(t, 1, D_CODES, bt.dlen, bt.dcode, opt_len, static_len);
    // build_bl_tree
    uint32_t blf[BL_CODES];
    for (int i = 0; i < BL_CODES; ++i) blf[i] = 0;
    auto count_visit = [&](int sym, int) { blf[sym]++; };
    walk_tree_lengths(bt.llen, bt.lmax, count_visit);
    walk_tree_lengths(bt.dlen, bt.dmax, count_visit);
    for (int i = 0; i < HEAP_SIZE; ++i) t.freq[i] = 0;
    for (int i = 0; i < BL_CODES; ++i) t.freq[i] = (uint16_t)blf[i];
    build_tree(t, 2, BL_CODES, bt.bllen, bt.blcode, opt_len, static_len);
    int max_blindex;
    for (max_blindex = BL_CODES - 1; max_blindex >= 3; max_blindex--)
        if (bt.bllen[bl_order(max_blindex)] != 0) break;
    opt_len += 3 * ((uint64_t)max_blindex + 1) + 5 + 5 + 4;
    bt.max_blindex = (int16_t)max_blindex;
    bt.opt_len = opt_len;
    bt.static_len = static_len;
    bt.last = last ? 1 : 0;
    uint64_t opt_lenb = (opt_len + 3 + 7) >> 3;
    const uint64_t static_lenb = (static_len + 3 + 7) >> 3;
    if (static_lenb <= opt_lenb) opt_lenb = static_lenb;
    if (stored_len + 4 <= opt_lenb && stored_ok) {
        bt.type = 0;
        bt.body_bits = 32 + 8 * stored_len;
    } else if (static_lenb == opt_lenb) {
        bt.type = 1;
        bt.body_bits = static_len;
    } else {
        bt.type = 2;
        // exact emitted bits: counts + bl lengths + tree runs + data (opt_len accounts the same)
        uint64_t bits = 5 + 5 + 4 + 3 * (uint64_t)(max_blindex + 1);
        auto size_visit = [&](int sym, int) { bits += bt.bllen[sym] + extra_blbits(sym); };
        walk_tree_lengths(bt.llen, bt.lmax, size_visit);
        walk_tree_lengths(bt.dlen, bt.dmax, size_visit);
        for (int i = 0; i < L_CODES; ++i) {
            if (!lfreq[i]) continue;
            const int xb = i >= 257 ? extra_lbits((uint32_t)(i - 257)) : 0;
            bits += (uint64_t)lfreq[i] * (uint64_t)(bt.llen[i] + xb);
        }
        for (int i = 0; i < D_CODES; ++i) {
            if (!dfreq[i]) continue;
            bits += (uint64_t)dfreq[i] * (uint64_t)(bt.dlen[i] + extra_dbits((uint32_t)i));
        }
        bt.body_bits = bits;
    }
}

// bits one symbol costs under the block's chosen (static or dynamic) trees
HD uint32_t symbol_bits(uint32_t s, const BlockTrees &bt) {
    if (!sym_is_match(s)) return bt.type == 1 ? (uint32_t)static_llen((int)s) : bt.llen[s];
    const uint32_t lc = sym_lc(s), code = length_code(lc), d = sym_dist1(s), dc = dist_code(d);
    const uint32_t ll = bt.type == 1 ? (uint32_t)static_llen((int)(code + 257)) : bt.llen[code + 257];
    const uint32_t dl = bt.type == 1 ? 5u : bt.dlen[dc];
    return ll + (uint32_t)extra_lbits(code) + dl + (uint32_t)extra_dbits(dc);
}

// the (up to 48) bits of one symbol, LSB-first, and their count
HD uint64_t symbol_code(uint32_t s, const BlockTrees &bt, uint32_t &nbits) {
    const bool st = bt.type == 1;
    if (!sym_is_match(s)) {
        nbits = st ? (uint32_t)static_llen((int)s) : bt.llen[s];
        return st ? static_lcode((int)s) : bt.lcode[s];
    }
    const uint32_t lc = sym_lc(s), code = length_code(lc), d = sym_dist1(s), dc = dist_code(d);
    uint64_t v = 0;
    uint32_t pos = 0;
    const int lsym = (int)code + 257;
    const uint32_t ll = st ? (uint32_t)static_llen(lsym) : bt.llen[lsym];
    v |= (uint64_t)(st ? static_lcode(lsym) : bt.lcode[lsym]) << pos;
    pos += ll;
    const int xl = extra_lbits(code);
    if (xl) {
        v |= (uint64_t)(lc - base_length(code)) << pos;
        pos += (uint32_t)xl;
    }
    const uint32_t dl = st ? 5u : bt.dlen[dc];
    v |= (uint64_t)(st ? static_dcode((int)dc) : bt.dcode[dc]) << pos;
    pos += dl;
    const int xd = extra_dbits(dc);
    if (xd) {
        v |= (uint64_t)(d - base_dist(dc)) << pos;
        pos += (uint32_t)xd;
    }
    nbits = pos;
    return v;
}

// ------------------------------------------------------------------ checksums
HD uint32_t crc_multmodp(uint32_t a, uint32_t b) {  // crc32.c multmodp
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = b & 1 ? (b >> 1) ^ 0xedb88320u : b >> 1;
    }
    return p;
}
// x^(8*len) mod P, by square-and-multiply on x^(2^k)
HD uint32_t crc_x8n(uint64_t len) {
    uint32_t p = 1u << 31;     // x^0
    uint32_t sq = 1u << 23;    // x^8 (reflected: x^k is 1 << (31-k))
    while (len) {
        if (len & 1) p = crc_multmodp(sq, p);
        sq = crc_multmodp(sq, sq);
        len >>= 1;
    }
    return p;
}
HD uint32_t crc_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) { return crc_multmodp(crc_x8n(len2), crc1) ^ crc2; }

}  // namespace ipz
