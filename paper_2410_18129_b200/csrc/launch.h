// launch.h -- host-side launchers of the templated kernels, one explicit instantiation per
// compiled shape (C limbs per block, NB blocks; L = C*NB).  No CUDA types beyond cudaStream_t.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace mpb {

template <int C, int NB>
struct Launch {
    static void mp_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, bool sqr, cudaStream_t s);
    static void mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, bool trunc, bool sqr, uint32_t* ws, cudaStream_t s);
    static void mont_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count, bool trunc,
                          uint32_t* ws, cudaStream_t s);
    static void modexp(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc, uint32_t* ws,
                       cudaStream_t s);
};

#define MPB_SHAPES(X) X(16, 1) X(16, 2) X(16, 4) X(16, 6) X(16, 8) X(12, 11) X(8, 8)
#define MPB_EXTERN(C, NB) extern template struct Launch<C, NB>;
MPB_SHAPES(MPB_EXTERN)
#undef MPB_EXTERN

}  // namespace mpb
