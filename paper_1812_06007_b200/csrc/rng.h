// Internal interface of the device Gaussian generator (rng.cu).
#pragma once
#include "common.cuh"

namespace urv {

void rng_set_tables(const double* wi, const double* fi, const unsigned long long* ki, double r, double inv_r);
bool rng_tables_ready();
// rows x cols column-major N(0,1) draw into device memory, bit-identical to NumPy's
// Generator(Philox(key=[seed, stream])).standard_normal; false if unresolvable.
bool gaussian_device(unsigned long long seed, unsigned long long stream, long long rows, long long cols, double* out,
                     long long ld, cudaStream_t st);

}  // namespace urv
