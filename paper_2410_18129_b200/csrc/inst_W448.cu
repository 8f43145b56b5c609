// inst_W448.cu -- one-wave exponentiation instances: k_modexp<C, RM, NB, schoolbook> (C = 16, NB = 8; C = 12, NB = 11)
// compiled for CTAs of up to 448 threads (stage stride 448 x 16 bytes, 128 registers, a few spill bytes), one CTA per SM
// (DESIGN.md 5.3c).  The whole kernel family is compiled in its own namespace (mpb_w448) so its
// templates, which read the block size as a compile-time constant, do not collide with the
// 128-thread instances of inst_C16.cu; only mpb_modexp_w448 (launch.h) is exported.
#define MPB_THREADS 448
#define MPB_MINB 1
#define mpb mpb_w448
#include "kernels.cuh"
#undef mpb

namespace {
template <int C, int RM, int NBT>
void go_w(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base, const uint32_t* exp,
          uint32_t* out, size_t count, size_t k0, size_t n, int bits, int window, uint32_t* ws, unsigned grid,
          unsigned threads, cudaStream_t s) {
    using namespace mpb_w448;
    const size_t sm = stage_bytes<C>();
    smem_optin(k_modexp<C, RM, NBT, 0>, sm);
    k_modexp<C, RM, NBT, 0><<<grid, threads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, NBT, bits, window,
                                                        ws);
}
}  // namespace

bool mpb_modexp_w448(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                     const uint32_t* exp, uint32_t* out, size_t count, size_t k0, size_t n, int C, int nb,
                     int bits, int window, int redc, uint32_t* ws, unsigned grid, unsigned threads, cudaStream_t s) {
    if (threads == 0 || threads > 448 || threads % 32 != 0 || grid == 0) return false;
#define MPB_W_CASE(CV, NBV)                                                                                    \
    if (C == CV && nb == NBV) {                                                                                       \
        if (redc == 1) go_w<CV, 1, NBV>(N, NP, R2, base, exp, out, count, k0, n, bits, window, ws, grid, threads, s); \
        else if (redc == 0) go_w<CV, 0, NBV>(N, NP, R2, base, exp, out, count, k0, n, bits, window, ws, grid, threads, s); \
        else return false;                                                                                         \
        return true;                                                                                       \
    }
    MPB_W_CASE(16, 8)
    MPB_W_CASE(12, 11)
#undef MPB_W_CASE
    return false;
}
