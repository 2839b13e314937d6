// cxx_api.cpp -- TEST PROGRAM: drives include/ipcomp_b200.hpp the way a reference user
// drives <ipcomp/pipeline.hpp> (compress -> write -> read back from an istream ->
// plan_for_error -> reconstruct -> refine to the full plan -> session file round trip ->
// compute_metrics) and writes the archive and
// both reconstructions to files so tests/test_cxx_api.py can diff them with the oracle.
//   cxx_api <field.f32> <nx> <ny> <nz> <eb> <max_error> <out_prefix>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "ipcomp_b200.hpp"

namespace ib = ipcomp_b200;

static void dump(const std::string &path, const void *p, size_t n) {
    std::ofstream f(path, std::ios::binary);
    f.write(static_cast<const char *>(p), (std::streamsize)n);
}

int main(int argc, char **argv) {
    if (argc != 8) {
        std::fprintf(stderr, "usage: cxx_api field nx ny nz eb max_error out_prefix\n");
        return 2;
    }
    try {
        const ib::Dims dims{std::strtoul(argv[2], nullptr, 10), std::strtoul(argv[3], nullptr, 10),
                            std::strtoul(argv[4], nullptr, 10)};
        std::vector<float> field(dims[0] * dims[1] * dims[2]);
        std::ifstream in(argv[1], std::ios::binary);
        in.read(reinterpret_cast<char *>(field.data()), (std::streamsize)(field.size() * sizeof(float)));
        ib::CompressOptions opt;
        opt.eb = std::atof(argv[5]);
        opt.interp = ib::InterpKind::cubic;
        ib::ArchiveReader compressed = ib::compress_field<float>(field, dims, opt);
        std::stringstream ss;
        ib::write_archive(ss, compressed);
        const std::string bytes = ss.str();
        const std::string pre = argv[7];
        dump(pre + ".archive", bytes.data(), bytes.size());

        ib::ArchiveReader reader(ss);  // the reference's ArchiveReader(std::istream&)
        const ib::RetrievalPlan plan = ib::plan_for_error(reader, std::atof(argv[6]));
        ib::Retrieved<float> r1 = ib::reconstruct_field<float>(reader, plan);
        dump(pre + ".recon", r1.values.data(), r1.values.size() * sizeof(float));
        ib::Retrieved<float> r2 = ib::refine_field<float>(reader, r1.session, r1.values, ib::full_plan(reader));
        dump(pre + ".refine", r2.values.data(), r2.values.size() * sizeof(float));
        // session file round trip (write_session / read_session), then refine from it
        std::stringstream sess;
        ib::write_session(sess, r1.session);
        const std::string sbytes = sess.str();
        dump(pre + ".session", sbytes.data(), sbytes.size());
        const ib::RetrievalSession back = ib::read_session(sess, reader);
        ib::Retrieved<float> r3 = ib::refine_field<float>(reader, back, r1.values, ib::full_plan(reader));
        dump(pre + ".refine2", r3.values.data(), r3.values.size() * sizeof(float));
        const ib::FieldMetrics m = ib::compute_metrics<float>(field, r3.values);
        std::printf("max_error %.17g mse %.17g psnr %.17g\n", m.max_error, m.mse, m.psnr);
        std::printf("levels %d plan", reader.header().levels);
        for (int k : plan.k) std::printf(" %d", k);
        std::printf(" bytes_read %llu\n", (unsigned long long)reader.payload_bytes_read());
        // error behaviour: a plan of the wrong length is std::invalid_argument
        try {
            ib::reconstruct_field<float>(reader, ib::RetrievalPlan{{1}});
            return 3;
        } catch (const std::invalid_argument &) {
        }
        try {
            ib::plan_for_error(reader, opt.eb * 0.5);
            return 4;
        } catch (const ib::InfeasibleRequest &) {
        }
    } catch (const ib::CudaError &e) {
        std::fprintf(stderr, "cuda: %s\n", e.what());
        return 10;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
