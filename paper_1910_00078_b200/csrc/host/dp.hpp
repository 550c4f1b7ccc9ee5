// Data-parallel weight-gradient all-reduce (dp.cpp): NCCL buckets in
// backward order on a comm stream, overlapped with the remaining backward.
#pragma once

#include <cstddef>
#include <cstdint>

#include "core.hpp"

namespace primkit {

class Handle;
class DataParallel;

void dp_unique_id(unsigned char out[128]);
DataParallel* dp_create(Handle& h, const unsigned char id[128], int nranks, int rank, bool average);
void dp_destroy(DataParallel* dp);
void dp_set_bucket_bytes(DataParallel& dp, std::size_t bytes);
int dp_add(DataParallel& dp, void* grad, std::uint64_t elems, ElementType et);
void dp_ready(DataParallel& dp, int index);
void dp_finish(DataParallel& dp);
void dp_check(DataParallel& dp);
int dp_bucket_count(DataParallel& dp);
int dp_bucket_of(DataParallel& dp, int index);

}  // namespace primkit
