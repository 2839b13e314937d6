/*
 * ipcomp_b200.h -- the C-ABI drop-in boundary of the B200-native IPComp hot path.
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.  Every
 * call returns an IPCG_* status; the message of the last failure is available from
 * ipcg_last_error().  The status codes map one-to-one onto the exception types the
 * reference throws (std::invalid_argument, std::runtime_error, std::domain_error,
 * ipcomp::InfeasibleRequest), so the C++ host layer (include/ipcomp/pipeline.hpp)
 * rethrows exactly what the reference would.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 */
#ifndef IPCOMP_B200_H
#define IPCOMP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPCG_OK 0
#define IPCG_EINVAL 1      /* std::invalid_argument */
#define IPCG_ERUNTIME 2    /* std::runtime_error    */
#define IPCG_EDOMAIN 3     /* std::domain_error     */
#define IPCG_EINFEASIBLE 4 /* ipcomp::InfeasibleRequest (common.hpp:23-25) */
#define IPCG_ECUDA 5       /* device failure (no reference counterpart) */

#define IPCG_MAX_LEVELS 16

typedef struct ipcg_ctx ipcg_ctx;         /* one CUDA device + stream + workspace  */
typedef struct ipcg_archive ipcg_archive; /* parsed index + payload (host or device) */
typedef struct ipcg_session ipcg_session; /* device-resident RetrievalSession        */

/* ArchiveHeader + LevelRecord (include/ipcomp/archive.hpp:19-46), records[l-1] = level l */
typedef struct {
    uint64_t count;
    double delta[33];
    uint64_t outlier_offset, outlier_length, outlier_count;
    uint64_t plane_offset[32], plane_length[32];
} ipcg_level_record;

typedef struct {
    uint16_t version;
    uint8_t scalar; /* 0 f32, 1 f64 (common.hpp:14) */
    uint8_t interp; /* 0 linear, 1 cubic */
    uint8_t ndims, levels, progressive_levels, anchor_cap;
    uint64_t dims[4];
    double eb, range;
    uint64_t payload_bytes, index_bytes;
    uint32_t identity; /* crc32 of the index bytes (archive.cpp:161-162) */
    ipcg_level_record records[IPCG_MAX_LEVELS];
} ipcg_index;

/* context ---------------------------------------------------------------- */
/* A context is used by one host thread at a time.  Its device scratch, archive payloads
 * and session codewords come from a grow-only pool it owns: destroy archives and sessions
 * before their context. */
int ipcg_ctx_create(int device, ipcg_ctx **out);
void ipcg_ctx_destroy(ipcg_ctx *ctx);
const char *ipcg_last_error(const ipcg_ctx *ctx);
/* CUDA stream all work of this context is ordered on (cudaStream_t; NULL restores the
 * context's own stream).  Device buffers of archives and sessions are allocated and freed
 * stream-ordered on the stream current when they were created, which must outlive them. */
int ipcg_set_stream(ipcg_ctx *ctx, void *cuda_stream);
int ipcg_synchronize(ipcg_ctx *ctx);
/* Host-async mode (off by default; no reference counterpart -- the reference's calls are
 * synchronous).  When on, ipcg_reconstruct / ipcg_refine with a HOST `out` return once the
 * values are final on the device; the device->host copy into `out` runs on a context-owned
 * copy stream and has landed when ipcg_synchronize returns (or the next ipcg_set_* call).
 * Later calls overlap it; a refine whose `previous` is host memory waits for pending copies
 * before reading it.  `out` should be page-locked for the copy to be asynchronous. */
int ipcg_set_host_async(ipcg_ctx *ctx, int enable);
/* Upload a HOST field ahead of its ipcg_compress (no reference counterpart: the reference has no
 * device).  Returns at once; the copy of `bytes` bytes runs on a context-owned stream under the
 * calls that follow.  The next ipcg_compress of this context given the same host pointer (and a
 * shape of `bytes` bytes) compresses the staged device copy instead of uploading again; any other
 * compress ignores it.  The copy is enqueued in shares by the retrieval calls that follow (behind
 * their own block uploads, so it does not delay them) and the rest by that compress.  One field
 * is staged at a time; the host field must stay unmodified and valid until the compress that
 * takes it returns (or, if none does, until ipcg_synchronize).  `host_values` should be
 * page-locked for the copy to be asynchronous. */
int ipcg_stage_field(ipcg_ctx *ctx, const void *host_values, uint64_t bytes);

/* compress_field<T> (include/ipcomp/pipeline.hpp:140-223).  `values` is a host or
 * device pointer (values_on_device); the archive is produced device-resident. */
int ipcg_compress(ipcg_ctx *ctx, int scalar, const void *values, int values_on_device, const uint64_t *dims,
                  int ndims, double eb, int interp, int progressive_levels, uint64_t anchor_cap, ipcg_archive **out);

/* ArchiveReader(std::istream&) (src/archive.cpp:117-170): parse the index of an
 * archive held in caller memory (host or device).  The bytes are borrowed, like
 * the reference's istream, and must outlive the handle. */
int ipcg_archive_open(ipcg_ctx *ctx, const void *bytes, uint64_t size, int on_device, ipcg_archive **out);
/* ArchiveReader(std::istream&) over a seekable source, as the reference reads its stream
 * (archive.cpp:117-181): `read` copies `len` bytes at absolute offset `offset` into host
 * memory `dst` and returns the number of bytes it delivered (fewer = end of source, < 0 =
 * failure).  Opening reads exactly the index (the header, then each level record in
 * turn); a retrieval then reads only the blocks its plan names, each once, at
 * index_bytes + block offset -- the reference's read_range.  `user` and the source must
 * outlive the handle.  Index errors carry the reference's messages ("truncated archive
 * index", "not an archive: bad magic", ...); a short block read raises "truncated archive
 * payload". */
typedef int64_t (*ipcg_read_fn)(void *user, uint64_t offset, void *dst, uint64_t len);
int ipcg_archive_open_source(ipcg_ctx *ctx, ipcg_read_fn read, void *user, ipcg_archive **out);
/* ArchiveReader::read_range (archive.cpp:172-181): `length` payload bytes at payload offset
 * `offset` into host memory, accounted in payload_bytes_read ("block offset outside
 * payload" / "truncated archive payload" as the reference). */
int ipcg_archive_read_range(ipcg_ctx *ctx, ipcg_archive *a, uint64_t offset, uint64_t length, void *dst);
int ipcg_archive_index(const ipcg_archive *a, ipcg_index *out);
/* write_archive (src/archive.cpp:72-81): serialized size and copy-out */
uint64_t ipcg_archive_size(const ipcg_archive *a);
int ipcg_archive_write(ipcg_ctx *ctx, const ipcg_archive *a, void *dst, int dst_on_device, uint64_t capacity);
/* bytes [offset, offset + length) of the serialized archive (e.g. the payload alone, for
 * ArchiveData::payload) into host or device memory; archives opened from a source read them
 * through it (not accounted as block reads) */
int ipcg_archive_copy(ipcg_ctx *ctx, const ipcg_archive *a, uint64_t offset, uint64_t length, void *dst,
                      int dst_on_device);
/* ArchiveReader::payload_bytes_read (archive.hpp:81) */
uint64_t ipcg_archive_payload_bytes_read(const ipcg_archive *a);
void ipcg_archive_free(ipcg_archive *a);
/* serialize_index (archive.cpp:31-65) of header + records (payload_bytes, index_bytes and
 * identity are derived, not read); *size_out receives the index size, also when capacity is too
 * small (IPCG_EINVAL).  Context-free (errors via ipcg_last_error(NULL)). */
int ipcg_index_serialize(const ipcg_index *ix, uint8_t *dst, uint64_t capacity, uint64_t *size_out);
/* parse an index held in host memory (the archive's first `size` bytes, payload optional) */
int ipcg_index_parse(const uint8_t *bytes, uint64_t size, ipcg_index *out);
/* crc32_bytes (backend.cpp:9-11): zlib's CRC-32, host (archive identity, small blocks) */
uint32_t ipcg_crc32(const void *bytes, uint64_t len);

/* ReconstructStats (pipeline.hpp:37-40) */
typedef struct {
    uint64_t payload_bytes_loaded;
    int level_visits[IPCG_MAX_LEVELS]; /* [l-1]: times level l was reconstructed */
} ipcg_retrieve_stats;

/* reconstruct_field<T> (pipeline.hpp:260-287): plan k[levels] (RetrievalPlan,
 * archive.hpp:59-61); out is host or device and holds out_count elements (must equal the
 * grid's point count: IPCG_EINVAL otherwise); *session_out and stats may be NULL. */
int ipcg_reconstruct(ipcg_ctx *ctx, ipcg_archive *a, int scalar, const int *k, void *out, int out_on_device,
                     uint64_t out_count, ipcg_session **session_out, ipcg_retrieve_stats *stats);

/* refine_field<T> (pipeline.hpp:294-352); previous_count / out_count elements, each must
 * equal the grid's point count ("previous reconstruction has wrong size", pipeline.hpp:303) */
int ipcg_refine(ipcg_ctx *ctx, ipcg_archive *a, int scalar, const ipcg_session *session, const void *previous,
                int previous_on_device, uint64_t previous_count, const int *k, void *out, int out_on_device,
                uint64_t out_count, ipcg_session **session_out, ipcg_retrieve_stats *stats);

/* RetrievalSession (session.hpp:19-34): planes_loaded[levels] (0..32, 32 for levels above
 * the progressive bound) and merged[l] = host codewords of progressive level l+1 (count of
 * that level; required when planes_loaded > 0, may be NULL when it is 0) */
int ipcg_session_create(ipcg_ctx *ctx, const ipcg_archive *a, const int *planes_loaded,
                        const uint32_t *const *merged /* [levels], host, NULL for non-progressive */,
                        ipcg_session **out);
int ipcg_session_levels(const ipcg_session *s);
uint32_t ipcg_session_archive_crc(const ipcg_session *s);
int ipcg_session_planes_loaded(const ipcg_session *s, int *k_out);
uint64_t ipcg_session_count(const ipcg_session *s, int level);
int ipcg_session_merged(ipcg_ctx *ctx, const ipcg_session *s, int level, uint32_t *dst, int dst_on_device);
void ipcg_session_free(ipcg_session *s);
/* write_session (src/session.cpp:8-24): the session file, each progressive level's merged
 * codewords deflated on the device.  dst is host or device memory of `capacity` bytes;
 * *size_out receives the file size (also when the call fails with IPCG_EINVAL because
 * capacity is too small or dst is NULL -- a size query).  ipcg_session_write_bound gives a
 * capacity that always suffices. */
uint64_t ipcg_session_write_bound(const ipcg_session *s);
int ipcg_session_write(ipcg_ctx *ctx, const ipcg_session *s, void *dst, int dst_on_device, uint64_t capacity,
                       uint64_t *size_out);
/* read_session (src/session.cpp:26-61): parse + CRC-check + inflate on the device into a
 * device-resident session bound to `a`; errors carry the reference's messages. */
int ipcg_session_read(ipcg_ctx *ctx, const ipcg_archive *a, const void *bytes, uint64_t size, int on_device,
                      ipcg_session **out);

/* compute_metrics<T> (pipeline.hpp:354-372): max pointwise error, MSE and PSNR of `decoded`
 * against `original` (n elements of f32/f64 each, host or device), one device pass.  max_error
 * is exact; mse/psnr differ from the reference's left-to-right double sum only by summation
 * order.  Sizes differing -> IPCG_EINVAL "metrics inputs differ in size". */
int ipcg_compute_metrics(ipcg_ctx *ctx, int scalar, const void *original, int original_on_device, uint64_t n_original,
                         const void *decoded, int decoded_on_device, uint64_t n_decoded, double *max_error,
                         double *mse, double *psnr);

/* planner (src/planner.cpp:30-290) over the index */
int ipcg_plan_for_error(ipcg_ctx *ctx, const ipcg_archive *a, double max_error, int *k_out);
int ipcg_plan_for_size(ipcg_ctx *ctx, const ipcg_archive *a, uint64_t byte_budget, int *k_out);
double ipcg_bound_for_plan(const ipcg_archive *a, const int *k);
uint64_t ipcg_plan_payload_bytes(const ipcg_archive *a, const int *k);

/* ErrorModel / LevelCosts (planner.hpp:13-32): a plain model callers may also build by hand;
 * the planner below works on it alone (planner.cpp:30-290).  Context-free calls; errors
 * (IPCG_EINFEASIBLE, IPCG_EINVAL for a malformed model) via ipcg_last_error(NULL). */
typedef struct {
    double delta[33];
    uint64_t plane_bytes[32];
    uint64_t outlier_bytes;
    int progressive;
} ipcg_level_costs;
typedef struct {
    int levels, progressive_levels;
    double eb, amplification;
    ipcg_level_costs level[IPCG_MAX_LEVELS]; /* [l-1] */
} ipcg_error_model;
int ipcg_build_error_model(const ipcg_index *ix, ipcg_error_model *out);
int ipcg_model_plan_for_error(const ipcg_error_model *m, double max_error, int *k_out);
int ipcg_model_plan_for_size(const ipcg_error_model *m, uint64_t byte_budget, int *k_out);
/* The same planners (planner.cpp:125-290) as one GPU launch on the context's stream: by_size = 0
 * plans for `max_error` (plan_for_error), 1 for `byte_budget` (plan_for_size).  Plans, error
 * kinds and messages are the host planner's; the host calls above stay the default. */
int ipcg_model_plan_device(ipcg_ctx *ctx, const ipcg_error_model *m, int by_size, double max_error,
                           uint64_t byte_budget, int *k_out);
double ipcg_model_bound_for_plan(const ipcg_error_model *m, const int *k);
uint64_t ipcg_model_plan_payload_bytes(const ipcg_error_model *m, const int *k);
uint64_t ipcg_model_mandatory_payload_bytes(const ipcg_error_model *m);
uint64_t ipcg_model_total_payload_bytes(const ipcg_error_model *m);

/* bitplane.cpp:7-68 on the device, for host arrays: 32 plane rows planes[p] of
 * ceil(count/8) bytes each (bit i of plane p = digit 31-p of codeword i, LSB-first).
 *   split (+ xor_encode when xor_encode != 0)                    bitplane.cpp:7-22,44-49
 *   xor_encode (decode = 0) / xor_decode of the first `nplanes` planes (decode = 1), in place
 *   merge of the first planes_loaded raw planes                  bitplane.cpp:24-38 */
int ipcg_split(ipcg_ctx *ctx, const uint32_t *codewords, uint64_t count, int xor_encode, uint8_t *const *planes);
int ipcg_plane_xor(ipcg_ctx *ctx, uint8_t *const *planes, uint64_t count, int nplanes, int decode);
int ipcg_merge(ipcg_ctx *ctx, const uint8_t *const *planes, uint64_t count, int planes_loaded, uint32_t *codewords);

/* backend_encode (src/backend.cpp:34-53) for `count` equal-length raw planes laid out
 * at raw + i*raw_stride (host or device).  Payloads are written to out_payload
 * (host, capacity count*plane_bytes), with per-plane backend id / length / crc32. */
int ipcg_backend_encode(ipcg_ctx *ctx, const uint8_t *raw, int raw_on_device, uint64_t plane_bytes,
                        uint64_t raw_stride, int count, uint8_t *backend, uint64_t *length, uint32_t *crc,
                        uint8_t *out_payload, uint64_t out_capacity);

/* backend_decode (src/backend.cpp:55-65) for `count` blocks whose payloads are concatenated
 * in host memory; outputs are concatenated (raw_bytes[i] each) into out.  status[i]:
 * 0 ok, 1 "block checksum mismatch", 2 "deflate backend failed to decompress block",
 * 3 "identity block has wrong length". */
int ipcg_backend_decode(ipcg_ctx *ctx, const uint8_t *payloads, const uint64_t *payload_len, const uint8_t *backend,
                        const uint32_t *crc, const uint64_t *raw_bytes, int count, uint8_t *out, int *status);

/* number of kernels this context launched so far (evidence for bench.py) */
uint64_t ipcg_kernel_launches(const ipcg_ctx *ctx);
/* per-kernel-family CUDA-event timing on the launching stream (bench.py roofline) */
int ipcg_profile_enable(ipcg_ctx *ctx, int enable);
int ipcg_profile_read(ipcg_ctx *ctx, char *json, uint64_t capacity);

#ifdef __cplusplus
}
#endif
#endif
