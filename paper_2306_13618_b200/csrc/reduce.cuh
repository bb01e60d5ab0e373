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
void scaled_mass(const double* mass, const double* pot, int64_t n, double lam, double* w, cudaStream_t s);
// cols (n x (2 + d), column-major): a, a ||x - c||^2, a (x - c)  (c: d device values or NULL)
void moment_cols(const double* x, const double* a, int64_t n, int d, const double* c, double* cols, cudaStream_t s);
void signed_concat(const double* a, int64_t n, const double* b, int64_t m, double* w, cudaStream_t s);

}  // namespace uotk
