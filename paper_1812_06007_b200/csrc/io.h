// Streaming file <-> device transfer of column-major float64 payloads (io.cu).
#pragma once

#include "common.cuh"

namespace urv {

void read_file_to_device(const char* path, long long offset, long long rows, long long cols, double* dst,
                         long long ldd, cudaStream_t st);
void write_device_to_file(const char* path, long long offset, const double* src, long long rows, long long cols,
                          long long lds, cudaStream_t st);

}  // namespace urv
