// Leaf product on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64):
//   C <- alpha*A*B + beta*C                     (classical_mul, ring.hpp:315-384)
// For Z/pZ with p < 2^16 the float64 dot product is exact while
// k*(p-1)^2 < 2^53 (k < 2^21), so one exact floor-based reduction per output
// replaces the reference's lazy u64 accumulation (ring.hpp:327-357); alpha and
// beta are applied in residue arithmetic (products < 2^32, exact).  For the
// REAL64 field the same kernel is a plain float64 GEMM.
//
// Tiling: 64x64 output tile per 128-thread CTA (2x2 warps of 32x32, i.e. 4x4
// m8n8 tiles and 32 accumulator registers per thread), K stepped by 16 with a
// two-stage cp.async (zero-fill) pipeline, so any m, k, n and any leading
// dimension are handled.
#include <cstdint>

#include "wm_launch.h"
#include "wm_device.h"

namespace wm {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int APAD = 4, BPAD = 4;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double reduce_modp(double v, double p, double pinv) {
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

template <bool REAL>
__global__ void __launch_bounds__(128) k_leaf_dmma(const MulParams P) {
    __shared__ double As[2][BM][BK + APAD];
    __shared__ double Bs[2][BK][BN + BPAD];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t4 = lane & 3;
    const std::uint64_t row0 = static_cast<std::uint64_t>(blockIdx.y) * BM;
    const std::uint64_t col0 = static_cast<std::uint64_t>(blockIdx.x) * BN;
    const std::uint32_t M = P.m, N = P.n, K = P.k;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_C();

    auto load_tile = [&](int buf, std::uint32_t k0) {
#pragma unroll
        for (int e = 0; e < (BM * BK) / 128; ++e) {
            const int idx = e * 128 + tid;
            const int r = idx / BK, c = idx % BK;
            const std::uint64_t gr = row0 + r, gc = k0 + c;
            const bool ok = gr < M && gc < K;
            cp_async8(&As[buf][r][c], ok ? P.A + gr * P.lda + gc : P.A, ok);
        }
#pragma unroll
        for (int e = 0; e < (BK * BN) / 128; ++e) {
            const int idx = e * 128 + tid;
            const int r = idx / BN, c = idx % BN;
            const std::uint64_t gr = k0 + r, gc = col0 + c;
            const bool ok = gr < K && gc < N;
            cp_async8(&Bs[buf][r][c], ok ? P.B + gr * P.ldb + gc : P.B, ok);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const std::uint32_t ktiles = (K + BK - 1) / BK;
    load_tile(0, 0);
    cp_async_commit();
    for (std::uint32_t kt = 0; kt < ktiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) load_tile(buf ^ 1, (kt + 1) * BK);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[buf][wm * 32 + i * 8 + g][kk + t4];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + t4][wn * 32 + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
        __syncthreads();
    }
    WM_PDL_LATE_C();

    const double p = P.pd, pinv = P.pinv;
    const double al = REAL ? P.alphad : static_cast<double>(P.alpha);
    const double be = REAL ? P.betad : static_cast<double>(P.beta);
    const bool use_c = REAL ? (P.betad != 0.0) : (P.beta != 0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const std::uint64_t r = row0 + wm * 32 + i * 8 + g;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const std::uint64_t c = col0 + wn * 32 + j * 8 + t4 * 2 + e;
                if (c >= N) continue;
                double* cp = P.C + r * P.ldc + c;
                double v = acc[i][j][e];
                if (REAL) {
                    v = al * v;
                    if (use_c) v = fma(be, *cp, v);
                } else {
                    v = reduce_modp(v, p, pinv);
                    v = v * al;  // < 2^32
                    if (use_c) v = fma(be, *cp, v);  // < 2^33
                    v = reduce_modp(v, p, pinv);
                }
                *cp = v;
            }
        }
    }
}

}  // namespace

cudaError_t launch_leaf_dmma(const MulParams& P, bool real, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((P.n + BN - 1) / BN, (P.m + BM - 1) / BM);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (real) return cudaLaunchKernelEx(&cfg, k_leaf_dmma<true>, P);
    return cudaLaunchKernelEx(&cfg, k_leaf_dmma<false>, P);
}

}  // namespace wm
