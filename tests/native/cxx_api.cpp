// cxx_api.cpp -- TEST PROGRAM: a reference user's program, written against the reference's
// public headers (<ipcomp/pipeline.hpp>, namespace ipcomp) and built against this repo's
// source-compatible include/ipcomp/ + libipcomp_b200.so: compress -> write_archive ->
// ArchiveReader(std::istream&) -> build_error_model -> plan_for_error -> reconstruct ->
// refine to the full plan -> session file round trip -> compute_metrics.  Writes the archive
// and the reconstructions so tests/test_cxx_api.py can diff them with the oracle.
//   cxx_api <field.f32> <nx> <ny> <nz> <eb> <max_error> <out_prefix>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "ipcomp/pipeline.hpp"

using namespace ipcomp;

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
        const Dims dims{std::strtoul(argv[2], nullptr, 10), std::strtoul(argv[3], nullptr, 10),
                        std::strtoul(argv[4], nullptr, 10)};
        std::vector<float> field(dims[0] * dims[1] * dims[2]);
        std::ifstream in(argv[1], std::ios::binary);
        in.read(reinterpret_cast<char *>(field.data()), (std::streamsize)(field.size() * sizeof(float)));
        const ArchiveData archive = compress_field<float>(field, dims, {.eb = std::atof(argv[5]), .interp = InterpKind::cubic});
        std::stringstream ss;
        write_archive(ss, archive);
        const std::string bytes = ss.str();
        const std::string pre = argv[7];
        dump(pre + ".archive", bytes.data(), bytes.size());

        ArchiveReader reader(ss);
        const ErrorModel model = build_error_model(reader.header(), reader.records());
        const RetrievalPlan plan = plan_for_error(model, std::atof(argv[6]));
        const Retrieved<float> r1 = reconstruct_field<float>(reader, plan);
        dump(pre + ".recon", r1.values.data(), r1.values.size() * sizeof(float));
        const Retrieved<float> r2 = refine_field<float>(reader, r1.session, r1.values, full_plan(model));
        dump(pre + ".refine", r2.values.data(), r2.values.size() * sizeof(float));
        std::stringstream sess;
        write_session(sess, r1.session);
        const std::string sbytes = sess.str();
        dump(pre + ".session", sbytes.data(), sbytes.size());
        const RetrievalSession back = read_session(sess, reader);
        const Retrieved<float> r3 = refine_field<float>(reader, back, r1.values, full_plan(model));
        dump(pre + ".refine2", r3.values.data(), r3.values.size() * sizeof(float));
        const FieldMetrics m = compute_metrics<float>(field, r3.values);
        std::printf("max_error %.17g mse %.17g psnr %.17g\n", m.max_error, m.mse, m.psnr);
        std::printf("levels %d plan", reader.header().levels);
        for (int k : plan.k) std::printf(" %d", k);
        std::printf(" bytes_read %llu\n", (unsigned long long)reader.payload_bytes_read());
        try {
            reconstruct_field<float>(reader, RetrievalPlan{{1}});
            return 3;
        } catch (const std::invalid_argument &) {
        }
        try {
            plan_for_error(model, archive.header.eb * 0.5);
            return 4;
        } catch (const InfeasibleRequest &) {
        }
    } catch (const b200::CudaError &e) {
        std::fprintf(stderr, "cuda: %s\n", e.what());
        return 10;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
