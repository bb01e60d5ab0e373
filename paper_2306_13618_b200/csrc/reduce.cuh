// Launchers of reduce.cu.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace uotk {

void uot_terms(const double* pot, const double* mass, const double* t, int64_t n, double lam, double eta,
               double* cols, cudaStream_t s);
void uot_transport(const double* pot, const double* mass, const double* tp, int64_t n, double lam, double* out,
                   cudaStream_t s);
void check_mass(const double* a, int64_t n, int* flag, cudaStream_t s);
// flag |= bit if any of the n values is not finite
void check_finite(const double* a, int64_t n, int* flag, int bit, cudaStream_t s);
// the 4 low bits of *flag as 4 words (0/1) and back (for an or-all-reduce as a max)
void split_bits(const int* flag, int32_t* bits, cudaStream_t s);
void join_bits(const int32_t* bits, int* flag, cudaStream_t s);
void scaled_mass(const double* mass, const double* pot, int64_t n, double lam, double* w, cudaStream_t s);
// cols (n x (2 + d), column-major): a, a ||x - c||^2, a (x - c)  (c: d device values or NULL)
void moment_cols(const double* x, const double* a, int64_t n, int d, const double* c, double* cols, cudaStream_t s);
// prod[i] = a[i] * b[i]
void multiply(const double* a, const double* b, int64_t n, double* prod, cudaStream_t s);
void permute_signed(double* ws, const double* a, int64_t n, const double* b, const int32_t* perm, int64_t nz,
                    cudaStream_t s);
void signed_concat(const double* a, int64_t n, const double* b, int64_t m, double* w, cudaStream_t s);

}  // namespace uotk
