// host.h -- host-side C++ of the drop-in: archive index format (src/archive.cpp),
// retrieval planner (src/planner.cpp) and CRC-32 for the index identity.  This is
// the reference's host layer restated; it never touches payload bytes.
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/ipcomp_b200.h"

namespace ipcg {

uint32_t crc32_host(const uint8_t *p, size_t n, uint32_t crc = 0);

// serialize_index (archive.cpp:31-65) incl. check_header / check_record
std::vector<uint8_t> serialize_index(const ipcg_index &ix);
// bytes needed to hold any index (header + 16 records)
constexpr uint64_t kMaxIndexBytes = 12 + 32 + 20 + IPCG_MAX_LEVELS * 808;
// ArchiveReader constructor (archive.cpp:117-170): parses `avail` bytes, fills ix
// (including index_bytes, identity, derived payload_bytes)
void parse_index(const uint8_t *bytes, uint64_t avail, ipcg_index &ix);
// the same over a seekable source, reading the index field by field (never past its end)
struct IndexSource {
    ipcg_read_fn read;
    void *user;
};
void parse_index(const IndexSource &src, ipcg_index &ix);

void validate_plan(const ipcg_index &ix, const int *k);  // archive.cpp:202-211

// planner.cpp:30-290 on the plain model (planner.hpp:13-32)
void check_model(const ipcg_error_model &m);
void build_error_model(const ipcg_index &ix, ipcg_error_model &m);
double bound_for_plan(const ipcg_error_model &m, const int *k);
uint64_t plan_payload_bytes(const ipcg_error_model &m, const int *k);
uint64_t mandatory_payload_bytes(const ipcg_error_model &m);
uint64_t total_payload_bytes(const ipcg_error_model &m);
void plan_for_error(const ipcg_error_model &m, double max_error, int *k);
void plan_for_size(const ipcg_error_model &m, uint64_t budget, int *k);
// the same two planners as one single-CTA launch (planner.cu); identical plans and errors.
// (cuda_runtime's cudaStream_t: declared as the opaque pointer it is to keep this header host-only)
void plan_on_device(const ipcg_error_model &m, int mode, double max_error, uint64_t budget, int *k,
                    struct CUstream_st *stream);
// the same from an index (build_error_model first)
double bound_for_plan(const ipcg_index &ix, const int *k);
uint64_t plan_payload_bytes(const ipcg_index &ix, const int *k);
uint64_t mandatory_payload_bytes(const ipcg_index &ix);
void plan_for_error(const ipcg_index &ix, double max_error, int *k);
void plan_for_size(const ipcg_index &ix, uint64_t budget, int *k);

}  // namespace ipcg
