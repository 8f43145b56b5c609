// DIAGNOSTIC (tools only): the 2048-bit headline instantiation k_modexp<16, 1, 4, 0> with per-CTA
// %globaltimer start / end and %smid, to see how CTA durations differ between the first and the
// later waves of a launch.  Build: nvcc ... -DMPB_CTA_TIMES -shared tools/cta_times.cu
#define MPB_CTA_TIMES 1
#include "../paper_2410_18129_b200/csrc/kernels.cuh"

extern "C" {
int cta_modexp_2048(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                    const uint32_t* exp, uint32_t* out, size_t count, int window, void* ws) {
    using namespace mpb;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    if (g > (1u << 14)) return -1;
    static unsigned long long z[1 << 14];
    cudaMemcpyToSymbol(g_cta_t1, z, sizeof z);
    smem_optin(k_modexp<16, 1, 4, 0>, stage_bytes<16>());
    k_modexp<16, 1, 4, 0><<<g, kThreads, stage_bytes<16>()>>>(N, NP, R2, base, exp, out, count, 0, count, 4, 2048,
                                                               window, (uint32_t*)ws);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}
void cta_times_take(unsigned long long* t0, unsigned long long* t1, uint32_t* sm, int n) {
    using namespace mpb;
    cudaMemcpyFromSymbol(t0, g_cta_t0, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(t1, g_cta_t1, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(sm, g_cta_sm, sizeof(uint32_t) * n);
}
}
