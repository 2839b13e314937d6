// watermark.cpp -- TEST PROGRAM (after proj/tests/test_archive.cpp:139-150): an istream whose
// buffer counts every byte it serves and the furthest offset read.  Checks, through the
// source-compatible API (include/ipcomp/), that opening + planning reads exactly the index,
// and that a partial retrieval then reads exactly index_bytes + plan_payload_bytes, each byte
// once -- the partial-bitplane fetch at the I/O level.
//   watermark <n> <seed>   (prints "index <b> after_plan <b> plan <b> after_retrieve <b> watermark <b>")
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <streambuf>

#include "ipcomp/pipeline.hpp"

using namespace ipcomp;

class CountingBuf : public std::streambuf {
   public:
    explicit CountingBuf(const std::string &s) : s_(s) {}
    std::uint64_t served = 0, watermark = 0;

   protected:
    std::streamsize xsgetn(char *dst, std::streamsize n) override {
        const std::streamsize got = std::min<std::streamsize>(n, (std::streamsize)(s_.size() - pos_));
        if (got <= 0) return 0;
        std::copy(s_.data() + pos_, s_.data() + pos_ + got, dst);
        pos_ += (std::size_t)got;
        served += (std::uint64_t)got;
        watermark = std::max<std::uint64_t>(watermark, pos_);
        setg(nullptr, nullptr, nullptr);
        return got;
    }
    int_type underflow() override {
        if (pos_ >= s_.size()) return traits_type::eof();
        one_ = s_[pos_];
        ++pos_;
        ++served;
        watermark = std::max<std::uint64_t>(watermark, pos_);
        setg(&one_, &one_, &one_ + 1);
        return traits_type::to_int_type(one_);
    }
    pos_type seekoff(off_type off, std::ios_base::seekdir dir, std::ios_base::openmode) override {
        const off_type base = dir == std::ios_base::beg ? 0 : dir == std::ios_base::end ? (off_type)s_.size() : (off_type)pos_;
        return seekpos(pos_type(base + off), std::ios_base::in);
    }
    pos_type seekpos(pos_type p, std::ios_base::openmode) override {
        if (p < 0 || (std::size_t)p > s_.size()) return pos_type(off_type(-1));
        pos_ = (std::size_t)p;
        setg(nullptr, nullptr, nullptr);
        return p;
    }

   private:
    const std::string &s_;
    std::size_t pos_ = 0;
    char one_ = 0;
};

int main(int argc, char **argv) {
    const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 40;
    const unsigned seed = argc > 2 ? (unsigned)std::atoi(argv[2]) : 1;
    const Dims dims{n, n + 3, n - 5};
    std::vector<double> f(element_count(dims));
    for (std::size_t i = 0; i < f.size(); ++i)
        f[i] = std::sin(0.07 * (double)(i % 997) + seed) + 0.3 * std::cos(0.011 * (double)i);
    const ArchiveData a = compress_field<double>(f, dims, {.eb = 1e-6});
    std::ostringstream os(std::ios::binary);
    write_archive(os, a);
    const std::string bytes = os.str();

    CountingBuf buf(bytes);
    std::istream in(&buf);
    ArchiveReader reader(in);
    const ErrorModel model = build_error_model(reader.header(), reader.records());
    const std::uint64_t after_open = buf.served, mark_open = buf.watermark;
    const RetrievalPlan plan = plan_for_error(model, 1e-3);
    (void)plan_for_size(model, total_payload_bytes(model));
    const std::uint64_t after_plan = buf.served;
    const Retrieved<double> r = reconstruct_field<double>(reader, plan);
    double worst = 0.0;
    for (std::size_t i = 0; i < f.size(); ++i) worst = std::max(worst, std::fabs(f[i] - r.values[i]));
    std::printf("index %llu open_served %llu open_watermark %llu after_plan %llu plan %llu after_retrieve %llu "
                "watermark %llu loaded %llu archive %llu err_ok %d\n",
                (unsigned long long)reader.index_bytes(), (unsigned long long)after_open, (unsigned long long)mark_open,
                (unsigned long long)after_plan, (unsigned long long)plan_payload_bytes(model, plan),
                (unsigned long long)buf.served, (unsigned long long)buf.watermark,
                (unsigned long long)r.stats.payload_bytes_loaded, (unsigned long long)bytes.size(), worst <= 1e-3);
    return 0;
}
