// corr_count.cu -- TEST ARTEFACT (libmpb_corr.so), never part of the product path.
//
// The same k_modexp<C = 16, truncated REDC, NB = 4, schoolbook> instantiation that
// mont_batch_modexp_ct runs for 2048-bit operands (kernels.cuh, warp-tiled workspace), compiled
// with MPB_CORR_COUNT so the engine counts every time Theorem 2's exact carry correction
// [S mod 2^32 > K] evaluates to 1.  tests/test_gpu_parity.py
// feeds it crafted inputs (a gamma-family T as the "R^2" operand, whose REDC is the first operation
// of the exponentiation) and checks that the correction fired inside this kernel, and that the
// release library's result for the same inputs equals the exact schedule.
#define MPB_CORR_COUNT 1
#include "../kernels.cuh"

extern "C" {

// Arguments as mont_batch_modexp_ct at bits = 2048, redc = truncated, schoolbook (word-sliced
// device arrays; ws: mont_batch_modexp_ct_workspace(count, 2048, window, AUTO) bytes).
int mpb_corr_modexp_2048(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                         const uint32_t* exp, uint32_t* out, size_t count, int window, void* ws, void* stream) {
    using namespace mpb;
    if (count == 0) return 0;
    k_modexp<16, 1, 4, 0><<<(unsigned)((count + kThreads - 1) / kThreads), kThreads, stage_bytes<16>(),
                            (cudaStream_t)stream>>>(N, NP, R2, base, exp, out, count, 0, count, 4, 2048, window,
                                                   (uint32_t*)ws);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// The counter's value; reset to 0 afterwards.  Synchronises the device.
unsigned long long mpb_corr_count_take(void) {
    unsigned long long v = 0, z = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&v, mpb::g_corr_count, sizeof v);
    cudaMemcpyToSymbol(mpb::g_corr_count, &z, sizeof z);
    return v;
}

}  // extern "C"
