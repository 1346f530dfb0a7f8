// Leaf product on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64):
//   C <- alpha*A*B + beta*C                     (classical_mul, ring.hpp:315-384)
// For Z/pZ with p < 2^16 the float64 dot product is exact while
// k*(p-1)^2 < 2^53 (k < 2^21), so one exact floor-based reduction per output
// replaces the reference's lazy u64 accumulation (ring.hpp:327-357); alpha and
// beta are applied in residue arithmetic (products < 2^32, exact).  For the
// REAL64 field the same kernel is a plain float64 GEMM.
//
// Tiling: a BM x BN output tile per CTA of WM x WN warps (each warp a grid of
// m8n8 tiles held in registers), K stepped by 16 through an NST-stage cp.async
// (zero-fill) ring, so any m, k, n and any leading dimension are handled;
// 16-byte copies when the operands allow them (even leading dimensions and
// extents, 16-byte aligned bases), 8-byte copies otherwise.
#include <cstdint>

#include "wm_launch.h"
#include "wm_device.h"

namespace wm {
namespace {

constexpr int BK = 16;
constexpr int APAD = 4, BPAD = 4;

template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = pred ? BYTES : 0;
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
    else
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

template <bool REAL, int BM, int BN, int WM, int WN, int NST, bool VEC>
__global__ void __launch_bounds__(32 * WM * WN) k_leaf_dmma(const MulParams P) {
    constexpr int NT = 32 * WM * WN;
    constexpr int MI = BM / WM / 8, NJ = BN / WN / 8;  // m8n8 tiles per warp
    constexpr int LDA = BK + APAD, LDB = BN + BPAD;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                        // [NST][BM][LDA]
    double* Bs = smem + NST * BM * LDA;       // [NST][BK][LDB]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, t4 = lane & 3;
    const std::uint64_t row0 = static_cast<std::uint64_t>(blockIdx.y) * BM;
    const std::uint64_t col0 = static_cast<std::uint64_t>(blockIdx.x) * BN;
    const std::uint32_t M = P.m, N = P.n, K = P.k;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_C();

    auto load_tile = [&](int buf, std::uint32_t k0) {
        constexpr int W = VEC ? 2 : 1;  // doubles per copy
        double* a = As + buf * BM * LDA;
        double* b = Bs + buf * BK * LDB;
#pragma unroll
        for (int e = 0; e < (BM * BK / W + NT - 1) / NT; ++e) {
            const int idx = e * NT + tid;
            if ((BM * BK / W) % NT != 0 && idx >= BM * BK / W) break;
            const int r = idx / (BK / W), c = (idx % (BK / W)) * W;
            const std::uint64_t gr = row0 + r, gc = k0 + c;
            const bool ok = gr < M && gc < K;
            cp_async_zfill<8 * W>(a + r * LDA + c, ok ? P.A + gr * P.lda + gc : P.A, ok);
        }
#pragma unroll
        for (int e = 0; e < (BK * BN / W + NT - 1) / NT; ++e) {
            const int idx = e * NT + tid;
            if ((BK * BN / W) % NT != 0 && idx >= BK * BN / W) break;
            const int r = idx / (BN / W), c = (idx % (BN / W)) * W;
            const std::uint64_t gr = k0 + r, gc = col0 + c;
            const bool ok = gr < K && gc < N;
            cp_async_zfill<8 * W>(b + r * LDB + c, ok ? P.B + gr * P.ldb + gc : P.B, ok);
        }
    };

    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const std::uint32_t ktiles = (K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        if (static_cast<std::uint32_t>(s) < ktiles) load_tile(s, s * BK);
        cp_async_commit();
    }
    for (std::uint32_t kt = 0; kt < ktiles; ++kt) {
        const int buf = kt % NST;
        cp_async_wait<NST - 2>();  // tile kt has landed
        __syncthreads();           // ... for every thread, and tile kt - 1's buffer is free
        if (kt + NST - 1 < ktiles) load_tile((kt + NST - 1) % NST, (kt + NST - 1) * BK);
        cp_async_commit();
        const double* a = As + buf * BM * LDA + (wm * MI * 8 + g) * LDA + t4;
        const double* b = Bs + buf * BK * LDB + t4 * LDB + wn * NJ * 8 + g;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[MI], bf[NJ];
#pragma unroll
            for (int i = 0; i < MI; ++i) af[i] = a[i * 8 * LDA + kk];
#pragma unroll
            for (int j = 0; j < NJ; ++j) bf[j] = b[kk * LDB + j * 8];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
    }
    WM_PDL_LATE_C();

    const double p = P.pd, pinv = P.pinv;
    const double al = REAL ? P.alphad : static_cast<double>(P.alpha);
    const double be = REAL ? P.betad : static_cast<double>(P.beta);
    const bool use_c = REAL ? (P.betad != 0.0) : (P.beta != 0);
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const std::uint64_t r = row0 + wm * MI * 8 + i * 8 + g;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const std::uint64_t c = col0 + wn * NJ * 8 + j * 8 + t4 * 2 + e;
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

template <bool REAL, int BM, int BN, int WM, int WN, int NST, bool VEC>
cudaError_t launch_cfg(const MulParams& P, cudaStream_t s) {
    constexpr std::size_t smem = sizeof(double) * NST * (BM * (BK + APAD) + BK * (BN + BPAD));
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_leaf_dmma<REAL, BM, BN, WM, WN, NST, VEC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((P.n + BN - 1) / BN, (P.m + BM - 1) / BM);
    cfg.blockDim = dim3(32 * WM * WN);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_leaf_dmma<REAL, BM, BN, WM, WN, NST, VEC>, P);
}

// One shape: 64 x 64 tiles, four warps, two-stage ring.  It saturates the SMs once
// the grid is several waves deep (31.7 TFLOP/s at 2048^3 in isolation); a 1024^3
// leaf is only 256 tiles on 148 SMs (20 TFLOP/s alone), but inside a
// multiplication the lanes overlap neighbouring leaves and this shape wins.
// Measured inside config 5, whose 2-temporary schedule runs its 16,807 leaves
// strictly one after another (profiles/r2/dmma_c5_bench.txt; this shape 1570 ms):
// 64 x 32 tiles 1616, 32 x 64 1650, 128 x 64 1680, 64 x 128 1712, 32 x 32 2365,
// 128 x 128 2942-3044, a three-stage ring 1567 (no difference), two warp groups
// splitting the k steps of a tile 1650 (faster on a lone leaf in a replay loop,
// profiles/r2/dmma_sweep.log, slower in the real chain).
template <bool REAL, bool VEC>
cudaError_t launch_shape(const MulParams& P, cudaStream_t s) {
    return launch_cfg<REAL, 64, 64, 2, 2, 2, VEC>(P, s);
}

}  // namespace

cudaError_t launch_leaf_dmma(const MulParams& P, bool real, cudaStream_t s) {
    const bool vec = P.lda % 2 == 0 && P.ldb % 2 == 0 && P.k % 2 == 0 && P.n % 2 == 0 &&
                     (reinterpret_cast<std::uintptr_t>(P.A) & 15u) == 0 &&
                     (reinterpret_cast<std::uintptr_t>(P.B) & 15u) == 0;
    if (real) return vec ? launch_shape<true, true>(P, s) : launch_shape<true, false>(P, s);
    return vec ? launch_shape<false, true>(P, s) : launch_shape<false, false>(P, s);
}

}  // namespace wm
