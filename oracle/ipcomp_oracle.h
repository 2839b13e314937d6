/*
 * ipcomp_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference IPComp hot path
 * (/root/reference/proj, arXiv 2502.04093), used ONLY as the parity checker
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  The
 * product path (paper_2502_04093_b200/, include/) never links or calls it.
 *
 * Pinning: the restatement is validated against the reference itself,
 * compiled from its own sources into oracle/_ref/ (oracle/Makefile, target
 * `ref`), and against the golden archives under tests/golden/ that
 * tests/golden/make_golden.py generated from that build.
 *
 * Third-party arithmetic: the reference's lossless stage is zlib
 * (compress2 level 6 / uncompress / crc32, proj/src/backend.cpp:10,18,27).
 * zlib is not vendored in the reference; its version is not pinned by the
 * reference (proj/CMakeLists.txt:13 `find_package(ZLIB)`).  This oracle links
 * the same system libz the reference links in this image (zlib 1.3,
 * ZLIB_VERNUM 0x1300) and makes the same calls.
 *
 * Error codes (mirroring the reference's exception types):
 *   0 ok, 1 std::invalid_argument, 2 std::runtime_error,
 *   3 std::domain_error, 4 ipcomp::InfeasibleRequest.
 */
#ifndef IPCOMP_ORACLE_H
#define IPCOMP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LEVELS 16

typedef struct {
    int levels;
    uint64_t count[ORC_MAX_LEVELS];           /* [l-1] points of level l          */
    int32_t *codes[ORC_MAX_LEVELS];           /* quantization codes, ordinal order */
    uint32_t *negabinary[ORC_MAX_LEVELS];     /* codewords                         */
    uint64_t n_outliers[ORC_MAX_LEVELS];
    uint64_t *outlier_ordinal[ORC_MAX_LEVELS];
    uint8_t *outlier_bytes[ORC_MAX_LEVELS];   /* raw outlier block bytes           */
    uint8_t *xor_planes[ORC_MAX_LEVELS];      /* 32 planes * plane_bytes, post-XOR */
    double delta[ORC_MAX_LEVELS][33];
} orc_trace;

typedef struct {
    int scalar, interp, ndims, levels, progressive_levels, anchor_cap;
    uint64_t dims[4];
    double eb, range;
    uint64_t index_bytes, payload_bytes;
    uint32_t identity;
    uint64_t count[ORC_MAX_LEVELS];
    double delta[ORC_MAX_LEVELS][33];
    uint64_t outlier_offset[ORC_MAX_LEVELS], outlier_length[ORC_MAX_LEVELS], outlier_count[ORC_MAX_LEVELS];
    uint64_t plane_offset[ORC_MAX_LEVELS][32], plane_length[ORC_MAX_LEVELS][32];
} orc_info;

/* compress_field<T> + write_archive: archive file bytes (malloc'd, orc_free) */
int orc_compress(int scalar, const void *values, const uint64_t *dims, int nd, double eb, int interp,
                 int progressive_levels, uint64_t anchor_cap, uint8_t **out, uint64_t *out_size,
                 orc_trace *trace /* may be NULL */, char *err, int errlen);
void orc_trace_free(orc_trace *t);
void orc_free(void *p);

int orc_archive_info(const uint8_t *archive, uint64_t size, orc_info *info, char *err, int errlen);

/* reconstruct_field<T>; merged[l-1] malloc'd for progressive levels (NULL otherwise) */
int orc_reconstruct(const uint8_t *archive, uint64_t size, int scalar, const int *k, void *out_values,
                    uint32_t **merged, uint64_t *payload_bytes_loaded, char *err, int errlen);

/* refine_field<T> */
int orc_refine(const uint8_t *archive, uint64_t size, int scalar, const int *session_k,
               uint32_t *const *session_merged, const void *previous, const int *target_k, void *out_values,
               uint32_t **merged_out, uint64_t *payload_bytes_loaded, char *err, int errlen);

/* planner (proj/src/planner.cpp) over the archive index */
int orc_plan_for_error(const uint8_t *archive, uint64_t size, double max_error, int *k_out, char *err, int errlen);
int orc_plan_for_size(const uint8_t *archive, uint64_t size, uint64_t budget, int *k_out, char *err, int errlen);
double orc_bound_for_plan(const uint8_t *archive, uint64_t size, const int *k);
uint64_t orc_plan_payload_bytes(const uint8_t *archive, uint64_t size, const int *k);

/* the lossless stage alone (backend_encode / crc32_bytes) */
int orc_backend_encode(const uint8_t *raw, uint64_t n, int preferred, uint8_t **payload, uint64_t *payload_len,
                       int *backend, uint32_t *crc);
uint32_t orc_crc32(const uint8_t *p, uint64_t n);

/* session file (session.cpp) */
int orc_write_session(uint32_t archive_crc, int levels, const int *k, uint32_t *const *merged,
                      const uint64_t *counts, uint8_t **out, uint64_t *out_size);
/* compute_metrics (pipeline.hpp:354-372): out = {max_error, mse, psnr} */
int orc_compute_metrics(int scalar, const void *original, const void *decoded, uint64_t n, double *out);
int orc_read_session(const uint8_t *archive, uint64_t size, const uint8_t *bytes, uint64_t n, int *k_out,
                     uint32_t **merged_out, char *err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
