// mpb.cu -- kernels and the C ABI (include/mpb.h) of libmpb.so, sm_100a.
//
// One thread per operand (the warp is the paper's "batch of 8" widened to 32 lanes,
// PAPER.md L66-98); operands are word-sliced in HBM so each uint4 access of a warp
// is 512 contiguous bytes.  See DESIGN.md for the data layout, the per-kernel
// roofline and the readings of the paper.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/mpb.h"
#include "launch.h"

#define MPB_DEVI __device__ __forceinline__

using mpb::Launch;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#ifdef MPB_THREADS
constexpr int kThreads = MPB_THREADS;
#else
constexpr int kThreads = 128;
#endif

MPB_DEVI size_t tid_global() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }

// word-sliced accessor for operand k of an array with `count` operands
// word i of operand k (32-bit access)
MPB_DEVI uint32_t word_at(const uint32_t* base, size_t count, size_t k, int i) {
    return __ldg(base + ((size_t)(i >> 2) * count + k) * 4 + (i & 3));
}

// ------------------------------------------------------------- layout kernels
__global__ void k_expand(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t count, int chunks) {
    const size_t t = tid_global();
    if (t >= count * (size_t)chunks) return;
    const size_t q = t / count, k = t % count;
    dst[q * count + k] = src[k * chunks + q];
}
__global__ void k_contract(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t count, int chunks) {
    const size_t t = tid_global();
    if (t >= count * (size_t)chunks) return;
    const size_t q = t / count, k = t % count;
    dst[k * chunks + q] = src[q * count + k];
}

// ------------------------------------------------------------- dispatch
// Kernels are instantiated per block size C in {16, 12, 8, 4}; nb = L / C is a runtime
// argument.  Block size for a limb count: the largest C dividing L (mpb::block_for), unless
// the environment variable MPB_BLOCK forces one (tuning only).
int block_of(int L) {
    static int forced = [] {
        const char* e = getenv("MPB_BLOCK");
        return e ? atoi(e) : 0;
    }();
    if ((forced == 16 || forced == 12 || forced == 8 || forced == 4) && L % forced == 0) return forced;
    return mpb::block_for(L);
}
template <typename F>
int dispatch_L(int L, F&& f) {
    switch (block_of(L)) {
        case 16: return f(std::integral_constant<int, 16>{}, L / 16);
        case 12: return f(std::integral_constant<int, 12>{}, L / 12);
        case 8: return f(std::integral_constant<int, 8>{}, L / 8);
        default: return f(std::integral_constant<int, 4>{}, L / 4);
    }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int check_ptrs(std::initializer_list<const void*> ps) {
    for (const void* p : ps) {
        if (!p) return fail(MPB_EINVAL, "null pointer");
        if (!aligned16(p)) return fail(MPB_EINVAL, "pointer not 16-byte aligned");
    }
    return MPB_OK;
}

int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MPB_ECUDA, std::string("CUDA launch failed: ") + cudaGetErrorString(e));
    return MPB_OK;
}

unsigned grid_for(size_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

// MPB_REG=0 routes 1024-bit CIOS exponentiations to the block engine instead of the register-resident
// kernel (tests and A/B only)
int reg_policy() {
    static int v = [] {
        const char* e = getenv("MPB_REG");
        return e ? atoi(e) : 1;
    }();
    return v;
}

// MPB_REG_TRUNC=1 runs stand-alone 1024-bit truncated MontMul / MontSqr on the register-resident
// truncated kernel (k_mont_mul_rtr) instead of the block engine (A/B until measured)
int reg_trunc_policy() {
    static int v = [] {
        const char* e = getenv("MPB_REG_TRUNC");
        return e ? atoi(e) : 0;
    }();
    return v;
}

// The library's own stream-ordered memory pool for the current device (mpb_modexp_host), created
// once per device with an unlimited release threshold so repeated calls reuse their allocation;
// the device's default pool (and every other cudaMallocAsync user in the process) is untouched.
cudaMemPool_t private_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = p;
    }
    return pools[dev];
}

constexpr int kMaxLimbs = 512;  // 16384-bit operands
// Word-sliced chunk strides are count * 16 bytes held in 32 bits (one mad.wide.u32 per address);
// the CRT path holds 2 * count operands.
constexpr size_t kMaxCount = (size_t)1 << 27;

int limbs_checked(int bits, int& L) {
    L = mpb_limbs(bits);
    if (L <= 0) return fail(MPB_EUNSUPPORTED, "bits must be positive");
    if (L > kMaxLimbs)
        return fail(MPB_EUNSUPPORTED, "bits=" + std::to_string(bits) + " exceeds the compiled maximum of " +
                                          std::to_string(32 * kMaxLimbs));
    return MPB_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int mpb_limbs(int bits) { return bits <= 0 ? 0 : 4 * ((bits + 127) / 128); }

int mpb_supported(int bits) {
    int L;
    const std::string keep = g_err;
    const int ok = limbs_checked(bits, L) == MPB_OK;
    g_err = keep;
    return ok;
}

const char* mpb_last_error(void) { return g_err.c_str(); }

int mpb_layout_expand(const uint32_t* src, uint32_t* dst, size_t count, int limbs, void* stream) {
    g_err.clear();
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (limbs <= 0 || limbs % 4) return fail(MPB_EINVAL, "limbs must be a positive multiple of 4");
    if (int rc = check_ptrs({src, dst})) return rc;
    if (src == dst) return fail(MPB_EINVAL, "in-place layout change not supported");
    const size_t n = count * (size_t)(limbs / 4);
    k_expand<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, count, limbs / 4);
    return check_launch();
}

int mpb_layout_contract(const uint32_t* src, uint32_t* dst, size_t count, int limbs, void* stream) {
    g_err.clear();
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (limbs <= 0 || limbs % 4) return fail(MPB_EINVAL, "limbs must be a positive multiple of 4");
    if (int rc = check_ptrs({src, dst})) return rc;
    if (src == dst) return fail(MPB_EINVAL, "in-place layout change not supported");
    const size_t n = count * (size_t)(limbs / 4);
    k_contract<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, count, limbs / 4);
    return check_launch();
}

// Karatsuba levels for an algo request.  AUTO = schoolbook: the blocked schoolbook engine beat
// every Karatsuba variant at every measured size on sm_100a, so no crossover exists.
static int kara_levels(int algo, int /*L*/) {
    switch (algo) {
        case MPB_ALGO_KARATSUBA: return 1;
        case MPB_ALGO_KARATSUBA2: return 2;
        default: return 0;  // SCHOOLBOOK, AUTO
    }
}

size_t mp_batch_workspace(size_t count, int bits, int algo) {
    const int L = mpb_limbs(bits);
    if (L <= 0) return 0;
    const int C = block_of(L);
    return count * (size_t)mpb::kara_scratch_blocks_host(L / C, kara_levels(algo, L)) * C * sizeof(uint32_t);
}

static int mp_product(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, int bits, int algo, bool sqr,
                      void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    if (algo < MPB_ALGO_AUTO || algo > MPB_ALGO_HYBRID) return fail(MPB_EINVAL, "algo out of range");
    if (algo >= MPB_ALGO_RADIX52)
        return fail(MPB_EUNSUPPORTED, "MPB_ALGO_RADIX52 / HYBRID are exponentiation paths (mont_batch_modexp_ct)");
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (int rc = check_ptrs({a, b, c})) return rc;
    if (c == a || c == b) return fail(MPB_EINVAL, "output aliases an input");
    const int levels = kara_levels(algo, L);
    const size_t need = mp_batch_workspace(count, bits, algo);
    if (need > 0) {
        if (int rc = check_ptrs({ws})) return rc;
        if (ws_bytes < need) return fail(MPB_EINVAL, "workspace too small");
    }
    return dispatch_L(L, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::mp_mul(a, b, c, count, nb, sqr, levels, (uint32_t*)ws, (cudaStream_t)stream);
        return check_launch();
    });
}

int mp_batch_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, int bits, int algo, void* ws,
                 size_t ws_bytes, void* stream) {
    return mp_product(a, b, c, count, bits, algo, false, ws, ws_bytes, stream);
}
int mp_batch_sqr(const uint32_t* a, uint32_t* c, size_t count, int bits, int algo, void* ws, size_t ws_bytes,
                 void* stream) {
    return mp_product(a, a, c, count, bits, algo, true, ws, ws_bytes, stream);
}

size_t mont_batch_workspace(size_t count, int bits) {
    // T, Q word-sliced (3L per operand), or -- mont_batch_redc at the compile-time block counts --
    // T, Q, N, N', OUT in warp tiles (6L per operand over count rounded up to 32)
    const int L = mpb_limbs(bits);
    const size_t sliced = count * (size_t)(3 * L), tiled = ((count + 31) & ~(size_t)31) * (size_t)(6 * L);
    return (sliced > tiled ? sliced : tiled) * sizeof(uint32_t);
}

static bool redc_ok(int redc) { return redc == MPB_REDC_FULL || redc == MPB_REDC_TRUNCATED || redc == MPB_REDC_CIOS; }

static int mont_op(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                   size_t count, int bits, int redc, void* ws, size_t ws_bytes, bool sqr, void* stream) {
    g_err.clear();
    if (!redc_ok(redc)) return fail(MPB_EINVAL, "redc out of range");
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (int rc = check_ptrs({a, b, N, NP, c, ws})) return rc;
    if (c == a || c == b || c == N || c == NP) return fail(MPB_EINVAL, "output aliases an input");
    if (ws_bytes < mont_batch_workspace(count, bits)) return fail(MPB_EINVAL, "workspace too small");
    if (redc == MPB_REDC_CIOS && L == 32 && reg_policy() != 0) {  // 1024 bits: register-resident CIOS
        if (!mpb::launch_mont_mul_reg(a, sqr ? a : b, N, NP, c, count, bits, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_mont_mul_reg: launch refused");
        return check_launch();
    }
    if (redc == MPB_REDC_TRUNCATED && L == 32 && reg_trunc_policy() > 0) {  // opt-in (A/B): register truncated
        if (!mpb::launch_mont_mul_rtr(a, sqr ? a : b, N, NP, c, count, bits, sqr, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_mont_mul_rtr: launch refused");
        return check_launch();
    }
    return dispatch_L(L, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::mont_mul(a, b, N, NP, c, count, nb, redc, sqr, (uint32_t*)ws, (cudaStream_t)stream);
        return check_launch();
    });
}

int mont_batch_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                   size_t count, int bits, int redc, void* ws, size_t ws_bytes, void* stream) {
    return mont_op(a, b, N, NP, c, count, bits, redc, ws, ws_bytes, false, stream);
}
int mont_batch_sqr(const uint32_t* a, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count, int bits,
                   int redc, void* ws, size_t ws_bytes, void* stream) {
    return mont_op(a, a, N, NP, c, count, bits, redc, ws, ws_bytes, true, stream);
}

int mont_batch_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count, int bits,
                    int redc, void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    if (!redc_ok(redc)) return fail(MPB_EINVAL, "redc out of range");
    if (redc == MPB_REDC_CIOS)
        return fail(MPB_EUNSUPPORTED, "CIOS interleaves the reduction with a multiplication (alg:8BlockMontRed); "
                                      "a stand-alone REDC takes MPB_REDC_FULL or MPB_REDC_TRUNCATED");
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (int rc = check_ptrs({T, N, NP, c, ws})) return rc;
    if (c == T || c == N || c == NP) return fail(MPB_EINVAL, "output aliases an input");
    if (ws_bytes < mont_batch_workspace(count, bits)) return fail(MPB_EINVAL, "workspace too small");
    return dispatch_L(L, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::mont_redc(T, N, NP, c, count, nb, redc == MPB_REDC_TRUNCATED, (uint32_t*)ws, (cudaStream_t)stream);
        return check_launch();
    });
}

size_t mont_batch_modexp_ct_workspace(size_t count, int bits, int window, int algo) {
    const int L = mpb_limbs(bits);
    if (L <= 0 || window < 1 || window > 6) return 0;
    if (algo == MPB_ALGO_RADIX52) {  // (block engine: truncated / full; register CIOS at 1024 bits)
        const size_t a = mpb::d52_workspace_bytes(count, bits, window), b = mpb::d52r_workspace_bytes(count, bits, window);
        return a > b ? a : b;
    }
    if (algo == MPB_ALGO_HYBRID) return mpb::hybrid_workspace_bytes(count, bits, window);
    const int C = block_of(L);
    const int lev = kara_levels(algo, L);
    // Karatsuba product scratch, plus the truncated-Karatsuba REDC's 6 NB blocks (mp_kara.cuh)
    const size_t kara = (size_t)mpb::kara_scratch_blocks_host(L / C, lev) * C + (lev > 0 ? (size_t)6 * L : 0);
    // word-sliced layout (Karatsuba products, TMA tiles): G | Y | T | Q | S | scratch, stride count;
    // warp-tiled layout (the default path): G | Y | T | Q | S | N | N' over count rounded up to 32
    const size_t sliced = count * ((size_t)L * (size_t)((1 << window) + 5) + kara);
    const size_t tiled = ((count + 31) & ~(size_t)31) * (size_t)L * (size_t)((1 << window) + 7);
    return (sliced > tiled ? sliced : tiled) * sizeof(uint32_t);
}

int mont_batch_modexp_ct(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                         const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, int redc, int algo,
                         void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    if (!redc_ok(redc)) return fail(MPB_EINVAL, "redc out of range");
    if (algo < MPB_ALGO_AUTO || algo > MPB_ALGO_HYBRID) return fail(MPB_EINVAL, "algo out of range");
    if (window < 1 || window > 6) return fail(MPB_EINVAL, "window must be in 1..6");
    if (redc == MPB_REDC_CIOS && (algo == MPB_ALGO_KARATSUBA || algo == MPB_ALGO_KARATSUBA2))
        return fail(MPB_EUNSUPPORTED, "CIOS (alg:8BlockMontRed) interleaves rows of a schoolbook product; "
                                      "Karatsuba needs MPB_REDC_FULL or MPB_REDC_TRUNCATED");
    if (algo == MPB_ALGO_HYBRID && redc == MPB_REDC_CIOS)
        return fail(MPB_EUNSUPPORTED, "the hybrid path has truncated and full REDC only");
    if (algo == MPB_ALGO_RADIX52 && redc == MPB_REDC_CIOS && !mpb::d52r_workspace_bytes(1, bits, window))
        return fail(MPB_EUNSUPPORTED, "radix-2^52 CIOS (register-resident) exists for 1024-bit operands only");
    if (algo == MPB_ALGO_HYBRID && !mpb::hybrid_workspace_bytes(1, bits, window))
        return fail(MPB_EUNSUPPORTED, "the hybrid path serves 1921..2048-bit operands");
    if (algo == MPB_ALGO_RADIX52 && !mpb::d52_digits(bits))
        return fail(MPB_EUNSUPPORTED, "bits=" + std::to_string(bits) + " has no radix-2^52 instance");
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (int rc = check_ptrs({N, NP, R2, base, exp, out, ws})) return rc;
    if (out == N || out == NP || out == R2 || out == base || out == exp)
        return fail(MPB_EINVAL, "output aliases an input");
    if (ws_bytes < mont_batch_modexp_ct_workspace(count, bits, window, algo))
        return fail(MPB_EINVAL, "workspace too small");
    if (redc == MPB_REDC_CIOS && L == 32 && algo <= MPB_ALGO_SCHOOLBOOK && reg_policy() != 0) {
        // 1024 bits, CIOS: the register-resident exponentiation (inst_R32.cu)
        if (!mpb::launch_modexp_reg(N, NP, R2, base, exp, out, count, bits, window, (uint32_t*)ws, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_modexp_reg: launch refused");
        return check_launch();
    }
    if (redc == MPB_REDC_TRUNCATED && L == 32 && algo <= MPB_ALGO_SCHOOLBOOK && reg_policy() == 2) {
        // 1024 bits, truncated: the register-resident truncated exponentiation (inst_R32.cu; opt-in
        // MPB_REG=2 until measured)
        if (!mpb::launch_modexp_rtr(N, NP, R2, base, exp, out, count, bits, window, (uint32_t*)ws, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_modexp_rtr: launch refused");
        return check_launch();
    }
    if (algo == MPB_ALGO_HYBRID) {
        if (!mpb::launch_modexp_hybrid(N, NP, R2, base, exp, out, count, bits, window, redc == MPB_REDC_TRUNCATED,
                                  (uint32_t*)ws, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_modexp_hybrid: launch refused");
        return check_launch();
    }
    if (algo == MPB_ALGO_RADIX52 && redc == MPB_REDC_CIOS) {
        if (!mpb::launch_modexp_d52r(N, R2, base, exp, out, count, bits, window, (uint32_t*)ws, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_modexp_d52r: launch refused");
        return check_launch();
    }
    if (algo == MPB_ALGO_RADIX52) {
        if (!mpb::launch_modexp_d52(N, NP, R2, base, exp, out, count, bits, window, redc == MPB_REDC_TRUNCATED,
                               (uint32_t*)ws, (cudaStream_t)stream))
            return fail(MPB_ECUDA, "launch_modexp_d52: launch refused");
        return check_launch();
    }
    return dispatch_L(L, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::modexp(N, NP, R2, base, exp, out, count, nb, bits, window, redc,
                          redc == MPB_REDC_CIOS ? 0 : kara_levels(algo, L), (uint32_t*)ws, (cudaStream_t)stream);
        return check_launch();
    });
}

size_t mont_batch_setup_workspace(size_t count, int bits) {
    const int L = mpb_limbs(bits);
    return count * (size_t)(6 * L) * sizeof(uint32_t);
}

static int setup_impl(const uint32_t* N, uint32_t* NP, uint32_t* R2, size_t count, int bits, int pub_bits, void* ws,
                      size_t ws_bytes, void* stream) {
    g_err.clear();
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (int rc = check_ptrs({N, NP, R2, ws})) return rc;
    if (NP == N || R2 == N || NP == R2) return fail(MPB_EINVAL, "output aliases an input");
    if (ws_bytes < mont_batch_setup_workspace(count, bits)) return fail(MPB_EINVAL, "workspace too small");
    return dispatch_L(L, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::setup(N, NP, R2, count, nb, pub_bits, (uint32_t*)ws, (cudaStream_t)stream);
        return check_launch();
    });
}

int mont_batch_setup(const uint32_t* N, uint32_t* NP, uint32_t* R2, size_t count, int bits, void* ws, size_t ws_bytes,
                     void* stream) {
    return setup_impl(N, NP, R2, count, bits, 0, ws, ws_bytes, stream);
}

// ------------------------------------------------------------------ CRT-RSA
// Layout of the CRT workspace (uint32 words; n2 = 2*count operands of Lh limbs, word-sliced):
//   PQ | NPQ | R2Q | E | B | M   (6 * n2 * Lh)  then scratch shared by the steps.
static size_t crt_scratch_words(size_t count, int bits, int window) {
    const int h = bits / 2, Lh = mpb_limbs(h);
    const size_t n2 = 2 * count;
    size_t w = mont_batch_setup_workspace(n2, h) / 4;
    const size_t me = mont_batch_modexp_ct_workspace(n2, h, window, MPB_ALGO_AUTO) / 4;
    if (me > w) w = me;
    if ((size_t)4 * Lh * n2 > w) w = (size_t)4 * Lh * n2;        // reduce: T, Q, X
    if ((size_t)7 * Lh * count > w) w = (size_t)7 * Lh * count;  // recombine: T, Q, X, H, PR
    return w;
}

size_t rsa_batch_crt_workspace(size_t count, int bits, int window) {
    if (bits < 128 || (bits & 1) || window < 1 || window > 6) return 0;
    const int Lh = mpb_limbs(bits / 2);
    return (6 * (2 * count) * (size_t)Lh + crt_scratch_words(count, bits, window)) * sizeof(uint32_t);
}

int rsa_batch_crt_ct(const uint32_t* c, const uint32_t* p, const uint32_t* q, const uint32_t* dp, const uint32_t* dq,
                     const uint32_t* qinv, uint32_t* m, size_t count, int bits, int window, int redc, void* ws,
                     size_t ws_bytes, void* stream) {
    g_err.clear();
    if (!redc_ok(redc)) return fail(MPB_EINVAL, "redc out of range");
    if (window < 1 || window > 6) return fail(MPB_EINVAL, "window must be in 1..6");
    if (bits < 128 || (bits & 1)) return fail(MPB_EUNSUPPORTED, "bits must be even and >= 128");
    int L, Lh;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (int rc = limbs_checked(bits / 2, Lh)) return rc;
    if (count == 0) return MPB_OK;
    if (count > kMaxCount / 2)  // the half-size modexp runs 2 * count operands in one call
        return fail(MPB_EUNSUPPORTED, "count exceeds 2^26 RSA operations per call");
    if (int rc = check_ptrs({c, p, q, dp, dq, qinv, m, ws})) return rc;
    for (const void* in : {(const void*)c, (const void*)p, (const void*)q, (const void*)dp, (const void*)dq,
                           (const void*)qinv})
        if (in == m) return fail(MPB_EINVAL, "output aliases an input");
    if (ws_bytes < rsa_batch_crt_workspace(count, bits, window)) return fail(MPB_EINVAL, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const int h = bits / 2;
    const size_t n2 = 2 * count, arr_w = n2 * (size_t)Lh;
    uint32_t* base = (uint32_t*)ws;
    uint32_t *PQ = base, *NPQ = base + arr_w, *R2Q = base + 2 * arr_w, *E = base + 3 * arr_w, *B = base + 4 * arr_w,
             *M = base + 5 * arr_w, *scr = base + 6 * arr_w;
    const size_t scr_bytes = crt_scratch_words(count, bits, window) * sizeof(uint32_t);
    // [p; q] and [dp; dq] as 2*count-operand word-sliced arrays: per 16-byte chunk row, count
    // operands from each source (a pitched copy; no arithmetic)
    auto concat = [&](const uint32_t* a, const uint32_t* b, uint32_t* dst) -> bool {
        const size_t row = count * 16, drow = n2 * 16;
        return cudaMemcpy2DAsync(dst, drow, a, row, row, Lh / 4, cudaMemcpyDeviceToDevice, s) == cudaSuccess &&
               cudaMemcpy2DAsync((char*)dst + row, drow, b, row, row, Lh / 4, cudaMemcpyDeviceToDevice, s) ==
                   cudaSuccess;
    };
    if (!concat(p, q, PQ) || !concat(dp, dq, E)) return fail(MPB_ECUDA, "device copy failed");
    // the primes' bit length is the public bits/2 (precondition), never derived from p or q
    if (int rc = setup_impl(PQ, NPQ, R2Q, n2, h, h, scr, scr_bytes, stream)) return rc;
    int rc = dispatch_L(Lh, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::crt_reduce(c, L, PQ, NPQ, R2Q, B, count, nb, scr, s);
        return check_launch();
    });
    if (rc) return rc;
    if ((rc = mont_batch_modexp_ct(PQ, NPQ, R2Q, B, E, M, n2, h, window, redc, MPB_ALGO_AUTO, scr, scr_bytes, stream)))
        return rc;
    return dispatch_L(Lh, [&](auto Ci, int nb) {
        constexpr int C = decltype(Ci)::value;
        Launch<C>::crt_recombine(M, PQ, NPQ, R2Q, qinv, m, L, count, nb, scr, s);
        return check_launch();
    });
}

int mpb_modexp_host(const uint32_t* N, const uint32_t* base, const uint32_t* exp, uint32_t* out, size_t count,
                    int bits, int window, int redc, void* stream) {
    g_err.clear();
    int L;
    if (int rc = limbs_checked(bits, L)) return rc;
    if (!redc_ok(redc)) return fail(MPB_EINVAL, "redc out of range");
    if (count == 0) return MPB_OK;
    if (count > kMaxCount) return fail(MPB_EUNSUPPORTED, "count exceeds 2^27 operands per call");
    if (!N || !base || !exp || !out) return fail(MPB_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nb = count * (size_t)L * sizeof(uint32_t);
    const size_t ws_bytes = mont_batch_modexp_ct_workspace(count, bits, window, 0);
    const size_t setup_bytes = mont_batch_setup_workspace(count, bits);
    uint8_t* dev = nullptr;
    cudaMemPool_t pool = private_pool();
    if (!pool) return fail(MPB_ECUDA, "could not create the library's memory pool");
    // 7 arrays of L limbs (N, N', R2, base, exp, out, staging) + workspace
    const size_t total = 7 * nb + (ws_bytes > setup_bytes ? ws_bytes : setup_bytes) + 256;
    if (cudaMallocFromPoolAsync((void**)&dev, total, pool, s) != cudaSuccess)
        return fail(MPB_ECUDA, "cudaMallocFromPoolAsync failed");
    uint32_t* d[7];
    for (int i = 0; i < 7; i++) d[i] = (uint32_t*)(dev + i * nb);
    void* ws = dev + 7 * nb;
    const size_t wsz = total - 7 * nb;
    int rc = MPB_OK;
    auto h2d = [&](const uint32_t* h, uint32_t* dst) {
        if (rc) return;
        if (cudaMemcpyAsync(d[6], h, nb, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            rc = fail(MPB_ECUDA, "H2D copy failed");
            return;
        }
        rc = mpb_layout_expand(d[6], dst, count, L, stream);
    };
    h2d(N, d[0]);
    h2d(base, d[3]);
    h2d(exp, d[4]);
    if (!rc) rc = mont_batch_setup(d[0], d[1], d[2], count, bits, ws, wsz, stream);
    if (!rc) rc = mont_batch_modexp_ct(d[0], d[1], d[2], d[3], d[4], d[5], count, bits, window, redc, 0, ws, wsz, stream);
    if (!rc) rc = mpb_layout_contract(d[5], d[6], count, L, stream);
    if (!rc && cudaMemcpyAsync(out, d[6], nb, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        rc = fail(MPB_ECUDA, "D2H copy failed");
    cudaFreeAsync(dev, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && !rc) rc = fail(MPB_ECUDA, "stream sync failed");
    return rc;
}

}  // extern "C"
