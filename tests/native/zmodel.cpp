// zmodel.cpp -- TEST HARNESS: runs the position-parallel deflate decomposition of
// paper_2502_04093_b200/csrc/deflate_core.cuh sequentially on the CPU (same device
// functions, kernel grids emulated by loops) so the semantics can be diffed against
// the system libz's compress2(level 6) without a GPU.  Not part of the product.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../paper_2502_04093_b200/csrc/deflate_core.cuh"

using namespace ipz;

namespace {

struct BitWriter {
    std::vector<uint8_t> &buf;
    uint64_t pos = 0;  // bit position
    explicit BitWriter(std::vector<uint8_t> &b) : buf(b) {}
    void put(uint64_t v, uint32_t n) {
        for (uint32_t i = 0; i < n; ++i, ++pos) {
            if ((pos >> 3) >= buf.size()) buf.resize((pos >> 3) + 1024, 0);
            if ((v >> i) & 1) buf[pos >> 3] |= (uint8_t)(1u << (pos & 7));
        }
    }
    void align() { pos = (pos + 7) & ~uint64_t(7); }
};

// 4-byte little-endian words; bytes past n read as 0 (the GPU reads padding there, which
// match_len32 masks off)
struct HostWords {
    const uint8_t *in;
    uint64_t n;
    uint32_t word(uint32_t k) const {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b)
            if (4ull * k + b < n) v |= (uint32_t)in[4ull * k + b] << (8 * b);
        return v;
    }
    uint32_t byte(uint32_t i) const { return in[i]; }
    const uint8_t *at(uint32_t off) const { return in + off; }
};

struct Stats {
    uint64_t chunks, blocks, stored, fixed, dynamic, symbols;
};

}  // namespace

// blocks of 16383 symbols, Huffman plans, bits, Adler-32 (shared by both parse models)
static int emit_stream(const uint8_t *in, uint64_t n, std::vector<uint32_t> &syms, std::vector<int64_t> &tops,
                       int final_tag, int64_t nchunks, uint8_t *out, uint64_t cap, uint64_t *out_len,
                       uint64_t *stats) {
    const uint64_t S_loop = syms.size();
    const bool final_lit = final_tag != TAG_A && n > 0;
    if (final_lit) {
        syms.push_back(sym_literal(in[n - 1]));
        tops[syms.size() - 1] = (int64_t)n;
    }
    const uint64_t S = syms.size();
    // 7. blocks: every in-loop tally that fills 16383 symbols flushes; then a final block
    const uint64_t nfull = S_loop / BLOCK_SYMS;
    const uint64_t nblocks = nfull + 1;
    std::vector<uint8_t> buf(16, 0);
    BitWriter bw(buf);
    bw.put(0x78, 8);
    bw.put(0x9c, 8);
    TreeScratch ts;
    BlockTrees bt;
    uint64_t sym_start = 0, byte_start = 0;
    Stats st{};
    st.chunks = (uint64_t)nchunks;
    st.blocks = nblocks;
    st.symbols = S;
    for (uint64_t b = 0; b < nblocks; ++b) {
        const bool last = b + 1 == nblocks;
        const uint64_t sym_end = last ? S : (b + 1) * BLOCK_SYMS;
        uint32_t lf[L_CODES] = {0}, df[D_CODES] = {0};
        uint64_t blen = 0;
        for (uint64_t i = sym_start; i < sym_end; ++i) {
            const uint32_t s = syms[i];
            blen += sym_bytes(s);
            if (sym_is_match(s)) {
                lf[length_code(sym_lc(s)) + 257]++;
                df[dist_code(sym_dist1(s))]++;
            } else {
                lf[s]++;
            }
        }
        lf[END_BLOCK] = 1;
        // flush loop top: last block flushes at p = n; others at the tallying iteration
        int64_t pf;
        if (last) {
            pf = (int64_t)n;
        } else {
            pf = tops[sym_end - 1];
        }
        const int64_t offset = 32768 * slides_before(pf, (int64_t)n);
        const bool stored_ok = (int64_t)byte_start >= offset;
        plan_block(lf, df, blen, stored_ok, last, ts, bt);
        bw.put((uint64_t)(bt.type == 0 ? 0 : bt.type == 1 ? 1 : 2) * 2 + (last ? 1 : 0), 3);
        if (bt.type == 0) {
            ++st.stored;
            bw.align();
            bw.put(blen & 0xffff, 16);
            bw.put(~blen & 0xffff, 16);
            for (uint64_t i = 0; i < blen; ++i) bw.put(in[byte_start + i], 8);
        } else {
            if (bt.type == 2) {
                ++st.dynamic;
                const int lcodes = bt.lmax + 1, dcodes = bt.dmax + 1, blcodes = bt.max_blindex + 1;
                bw.put((uint64_t)(lcodes - 257), 5);
                bw.put((uint64_t)(dcodes - 1), 5);
                bw.put((uint64_t)(blcodes - 4), 4);
                for (int r = 0; r < blcodes; ++r) bw.put(bt.bllen[bl_order(r)], 3);
                auto send = [&](int sym, int extra) {
                    bw.put(bt.blcode[sym], bt.bllen[sym]);
                    if (sym == 16) bw.put((uint64_t)extra, 2);
                    else if (sym == 17) bw.put((uint64_t)extra, 3);
                    else if (sym == 18) bw.put((uint64_t)extra, 7);
                };
                walk_tree_lengths(bt.llen, bt.lmax, send);
                walk_tree_lengths(bt.dlen, bt.dmax, send);
            } else {
                ++st.fixed;
            }
            for (uint64_t i = sym_start; i < sym_end; ++i) {
                uint32_t nb;
                const uint64_t v = symbol_code(syms[i], bt, nb);
                bw.put(v, nb);
            }
            if (bt.type == 1) bw.put(static_lcode(END_BLOCK), 7);
            else bw.put(bt.lcode[END_BLOCK], bt.llen[END_BLOCK]);
        }
        sym_start = sym_end;
        byte_start += blen;
    }
    bw.align();
    // adler32 trailer, big-endian
    uint32_t a = 1, bsum = 0;
    for (uint64_t i = 0; i < n; ++i) {
        a = (a + in[i]) % 65521u;
        bsum = (bsum + a) % 65521u;
    }
    const uint32_t adler = (bsum << 16) | a;
    for (int i = 3; i >= 0; --i) bw.put((adler >> (8 * i)) & 0xff, 8);
    const uint64_t len = bw.pos >> 3;
    if (len > cap) return -2;
    std::memcpy(out, buf.data(), len);
    *out_len = len;
    if (stats) {
        stats[0] = st.chunks;
        stats[1] = st.blocks;
        stats[2] = st.stored;
        stats[3] = st.fixed;
        stats[4] = st.dynamic;
        stats[5] = st.symbols;
    }
    return 0;
}

extern "C" int zmodel_compress(const uint8_t *in, uint64_t n, int chunk, uint8_t *out, uint64_t cap,
                               uint64_t *out_len, uint64_t *stats) {
    struct HostBytes {
        const uint8_t *in;
        uint32_t operator()(int64_t i) const { return in[i]; }
        int64_t match_len(int64_t a, int64_t b, int64_t maxlen) const {
            int64_t len = 0;
            while (len < maxlen && in[a + len] == in[b + len]) ++len;
            return len;
        }
    } bytes{in};
    // 1. hash-chain links
    std::vector<uint16_t> prevd(n + 1, 0);
    {
        std::vector<int64_t> head(1 << 15, -1);
        for (int64_t p = 0; p + MIN_MATCH <= (int64_t)n; ++p) {
            const uint32_t h = hash3(in[p], in[p + 1], in[p + 2]);
            const int64_t q = head[h];
            prevd[p] = (q >= 0 && p - q < WSIZE) ? (uint16_t)(p - q) : 0;
            head[h] = p;
        }
    }
    auto prevfn = [&](int64_t i) -> uint32_t { return prevd[i]; };
    // 2. match records (the GPU's fast form; zmodel_match_check pins it to match_search)
    std::vector<uint64_t> rec(n + 1, 0);
    const HostWords words{in, n};
    for (int64_t p = 0; p < (int64_t)n; ++p) rec[p] = match_search32((uint32_t)p, (uint32_t)n, words, prevfn);
    // 3. anchors: no match found at q < p can reach past p
    std::vector<uint8_t> anchor(n + 1, 0);
    {
        int64_t reach = 0;
        for (int64_t p = 0; p <= (int64_t)n; ++p) {
            anchor[p] = reach <= p;
            if (p < (int64_t)n) {
                const int64_t r = p + (int64_t)(mrec_l128(rec[p]) ? mrec_l128(rec[p]) : 1);
                if (r > reach) reach = r;
            }
        }
    }
    const int64_t CH = chunk > 0 ? chunk : 4096;
    const int64_t nchunks = ((int64_t)n + CH - 1) / CH;
    std::vector<int64_t> bnd(nchunks + 1);
    bnd[nchunks] = (int64_t)n;
    for (int64_t k = nchunks - 1; k >= 0; --k) {  // first anchor >= k*CH (suffix-min)
        int64_t b = bnd[k + 1];
        for (int64_t p = k * CH; p < (k + 1) * CH && p < (int64_t)n; ++p)
            if (anchor[p]) {
                b = p;
                break;
            }
        bnd[k] = b;
    }
    bnd[0] = 0;
    // 4. per chunk, the exit tag for each entry tag
    auto run_chunk = [&](int64_t b0, int64_t b1, int tag, std::vector<uint32_t> *syms, int64_t *loop_tops) {
        int64_t p = b0;
        uint64_t count = 0;
        while (p < b1) {
            const Step s = parse_step(p, tag, (int64_t)n, rec[p], p > 0 ? rec[p - 1] : 0, bytes);
            if (s.emit) {
                const uint32_t sym = s.emit == 2 ? sym_match(s.len, s.dist) : sym_literal(s.len);
                if (syms) syms->push_back(sym);
                if (loop_tops) loop_tops[syms->size() - 1] = p;
                ++count;
            }
            p = s.next_p;
            tag = s.next_tag;
        }
        if (p != b1) return -1;  // anchors guarantee exact exit
        return tag;
    };
    std::vector<uint8_t> exits(nchunks * 4, 0);
    for (int64_t k = 0; k < nchunks; ++k) {
        if (bnd[k] >= bnd[k + 1]) {
            for (int t = 0; t < 4; ++t) exits[k * 4 + t] = (uint8_t)t;  // empty chunk: identity
            continue;
        }
        for (int t = 0; t < 4; ++t) {
            const int e = run_chunk(bnd[k], bnd[k + 1], t, nullptr, nullptr);
            if (e < 0) return -10;
            exits[k * 4 + t] = (uint8_t)e;
        }
    }
    // 5. resolve entry tags (a scan of 4->4 maps)
    std::vector<int> entry(nchunks + 1);
    entry[0] = TAG_A;
    for (int64_t k = 0; k < nchunks; ++k) entry[k + 1] = exits[k * 4 + entry[k]];
    // 6. emit symbols from the true entries; remember each symbol's loop top
    std::vector<uint32_t> syms;
    std::vector<int64_t> tops(n + 2);
    for (int64_t k = 0; k < nchunks; ++k)
        if (bnd[k] < bnd[k + 1]) run_chunk(bnd[k], bnd[k + 1], entry[k], &syms, tops.data());
    return emit_stream(in, n, syms, tops, entry[nchunks], nchunks, out, cap, out_len, stats);
}

extern "C" uint32_t zmodel_crc_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) { return crc_combine(crc1, crc2, len2); }

// match_search32 (the GPU's form) against the reference-shaped match_search at every
// position; returns the number of positions whose records differ.
extern "C" uint64_t zmodel_match_check(const uint8_t *in, uint64_t n) {
    struct HB {
        const uint8_t *in;
        uint32_t operator()(int64_t i) const { return in[i]; }
        int64_t match_len(int64_t a, int64_t b, int64_t maxlen) const {
            int64_t len = 0;
            while (len < maxlen && in[a + len] == in[b + len]) ++len;
            return len;
        }
    } bytes{in};
    std::vector<uint16_t> prevd(n + 1, 0);
    std::vector<int64_t> head(1 << 15, -1);
    for (int64_t p = 0; p + MIN_MATCH <= (int64_t)n; ++p) {
        const uint32_t h = hash3(in[p], in[p + 1], in[p + 2]);
        const int64_t q = head[h];
        prevd[p] = (q >= 0 && p - q < WSIZE) ? (uint16_t)(p - q) : 0;
        head[h] = p;
    }
    auto prevfn = [&](int64_t i) -> uint32_t { return prevd[i]; };
    const HostWords words{in, n};
    uint64_t bad = 0;
    for (int64_t p = 0; p < (int64_t)n; ++p) {
        const uint64_t ref = match_search(p, (int64_t)n, bytes, prevfn);
        bad += ref != match_search32((uint32_t)p, (uint32_t)n, words, prevfn);
        // the resumable walk (k_match's budgeted first pass + queued second pass), stopped
        // and resumed every `budget` candidates
        for (int budget : {1, 2, 5, 31}) {
            Walk32 s;
            uint64_t rec;
            if (!walk32_start((uint32_t)p, (uint32_t)n, words, prevfn, s, rec))
                while (!walk32_run((uint32_t)n, words, prevfn, s, budget, rec)) {
                    Walk32 t = s;  // the state round-trips through memory
                    s = t;
                }
            bad += rec != ref;
        }
    }
    return bad;
}

// dev statistics: parse steps (positions whose match record the lazy parse reads) and the
// match_step work spent on them vs on all positions
extern "C" void zmodel_parse_visits(const uint8_t *in, uint64_t n, uint64_t *out3) {
    struct HB {
        const uint8_t *in;
        uint32_t operator()(int64_t i) const { return in[i]; }
        int64_t match_len(int64_t a, int64_t b, int64_t maxlen) const {
            int64_t len = 0;
            while (len < maxlen && in[a + len] == in[b + len]) ++len;
            return len;
        }
    } bytes{in};
    std::vector<uint16_t> prevd(n + 1, 0);
    std::vector<int64_t> head(1 << 15, -1);
    for (int64_t p = 0; p + MIN_MATCH <= (int64_t)n; ++p) {
        const uint32_t h = hash3(in[p], in[p + 1], in[p + 2]);
        const int64_t q = head[h];
        prevd[p] = (q >= 0 && p - q < WSIZE) ? (uint16_t)(p - q) : 0;
        head[h] = p;
    }
    auto prevfn = [&](int64_t i) -> uint32_t { return prevd[i]; };
    std::vector<uint64_t> rec(n + 1, 0), steps(n + 1, 0);
    for (int64_t p = 0; p < (int64_t)n; ++p) {
        MatchState s;
        match_init(s, p, (int64_t)n, bytes, prevfn);
        uint64_t k = 0;
        while (!s.done) match_step(s, bytes, prevfn), ++k;
        steps[p] = k;
        rec[p] = match_result(s);
    }
    uint64_t visits = 0, vsteps = 0, allsteps = 0;
    for (int64_t p = 0; p < (int64_t)n; ++p) allsteps += steps[p];
    int64_t p = 0;
    int tag = TAG_A;
    while (p < (int64_t)n) {
        ++visits;
        vsteps += steps[p];
        const Step s = parse_step(p, tag, (int64_t)n, rec[p], p > 0 ? rec[p - 1] : 0, bytes);
        p = s.next_p;
        tag = s.next_tag;
    }
    out3[0] = visits;
    out3[1] = vsteps;
    out3[2] = allsteps;
}

// The on-demand chunked parse, run sequentially exactly as the GPU's k_od_* kernels run it in
// parallel: (1) one walker per chunk from (chunk start, A), recording each visited state and
// the symbols it emits; (2) from each chunk walk's exit state, a continuation walk until it
// reaches a state the walk of the chunk it is in visited (sync); (3) from chunk 0, follow the
// syncs: the true parse is chunk 0's walk, its continuation, the synced chunk's walk from the
// sync state, ...; (4) place the adopted symbols (re-walking the continuations).
extern "C" int zmodel_compress_od(const uint8_t *in, uint64_t n, int chunk, uint8_t *out, uint64_t cap,
                                  uint64_t *out_len, uint64_t *stats) {
    std::vector<uint16_t> prevd(n + 1, 0);
    {
        std::vector<int64_t> head(1 << 15, -1);
        for (int64_t p = 0; p + MIN_MATCH <= (int64_t)n; ++p) {
            const uint32_t h = hash3(in[p], in[p + 1], in[p + 2]);
            const int64_t q = head[h];
            prevd[p] = (q >= 0 && p - q < WSIZE) ? (uint16_t)(p - q) : 0;
            head[h] = p;
        }
    }
    auto prevfn = [&](uint32_t i) -> uint32_t { return prevd[i]; };
    const HostWords words{in, n};
    const uint64_t C = chunk > 0 ? (uint64_t)chunk : 1024;
    if (C > 8192) return -20;
    const uint64_t nch = (n + C - 1) / C;
    auto b = [&](uint64_t k) { return std::min<uint64_t>(k * C, n); };
    // 1. chunk walks
    std::vector<uint16_t> vis(n + 1, 0), spos(n + 1, 0);
    std::vector<uint32_t> ssym(n + 1, 0), nsym(nch, 0);
    std::vector<Walker> ex(nch);
    for (uint64_t k = 0; k < nch; ++k) {
        Walker w{(uint32_t)b(k), TAG_A, 0, 0};
        uint32_t cnt = 0;
        while (w.p < b(k + 1)) {
            const uint32_t p = w.p;
            vis[p] = vis_pack(w.tag, cnt);
            const uint32_t sym = walker_step(w, (uint32_t)n, words, prevfn);
            if (sym != NOSYM) {
                ssym[b(k) + cnt] = sym;
                spos[b(k) + cnt] = (uint16_t)(p - b(k));
                ++cnt;
            }
        }
        nsym[k] = cnt;
        ex[k] = w;
    }
    // 2. continuations until they meet a visited state
    std::vector<uint64_t> nxt(nch), nidx(nch, 0), ncont(nch, 0);
    std::vector<int> fin(nch, TAG_A);
    auto follow = [&](Walker w, uint64_t &c, uint32_t &idx, std::vector<uint32_t> *syms, std::vector<int64_t> *tops) {
        uint64_t cnt = 0;
        for (;;) {
            if (w.p >= n) {
                c = nch;
                idx = w.tag;  // the final tag
                return cnt;
            }
            c = w.p / C;
            const uint16_t v = vis[w.p];
            if (vis_match(v, w.tag)) {
                idx = vis_symidx(v);
                return cnt;
            }
            const uint32_t p = w.p;
            // the GPU's run jump (deflate.cu od_follow): floor(R / 258) periodic match(258, 1) cycles
            if (w.tag == TAG_A && p >= 1 && p + 516 <= n && in[p - 1] == in[p] && in[p + 257] == in[p] &&
                in[p + 515] == in[p]) {
                uint64_t e = p + 1;
                while (e < n && in[e] == in[e - 1]) ++e;
                const uint64_t m = (e - p) / MAX_MATCH;
                if (m >= 2) {
                    for (uint64_t i = 0; i < m; ++i)
                        if (syms) syms->push_back(sym_match(MAX_MATCH, 1)), tops->push_back((int64_t)(p + 1 + MAX_MATCH * i));
                    cnt += m;
                    w.p = (uint32_t)(p + MAX_MATCH * m);
                    continue;
                }
            }
            const uint32_t sym = walker_step(w, (uint32_t)n, words, prevfn);
            if (sym != NOSYM) {
                if (syms) syms->push_back(sym), tops->push_back(p);
                ++cnt;
            }
        }
    };
    uint64_t cont_steps = 0;
    for (uint64_t k = 0; k < nch; ++k) {
        uint64_t c;
        uint32_t idx;
        ncont[k] = follow(ex[k], c, idx, nullptr, nullptr);
        nxt[k] = c;
        if (c == nch) fin[k] = (int)idx;
        else nidx[k] = idx;
        cont_steps += ncont[k];
    }
    // 3. the adopted chain; 4. placement
    std::vector<uint32_t> syms;
    std::vector<int64_t> tops;
    int final_tag = TAG_A;
    uint64_t a = 0, idx = 0, adopted = 0;
    while (a < nch) {
        ++adopted;
        for (uint64_t i = idx; i < nsym[a]; ++i) syms.push_back(ssym[b(a) + i]), tops.push_back((int64_t)(b(a) + spos[b(a) + i]));
        uint64_t c;
        uint32_t id;
        follow(ex[a], c, id, &syms, &tops);
        if (c == nch) final_tag = (int)id;
        else idx = id;
        a = c;
    }
    tops.resize(syms.size() + 2);
    const int rc = emit_stream(in, n, syms, tops, final_tag, (int64_t)nch, out, cap, out_len, stats);
    if (stats) stats[0] = adopted, stats[1] = cont_steps;
    return rc;
}
