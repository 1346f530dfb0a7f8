// Micro-plan executor: one CTA runs a whole plan of tiny operations.
//
// The reference's own correctness shapes (acceptance.cpp:55-84, test_executor.cpp)
// recurse down to cutoff 1..4 on problems of at most 64^3: std2 at 64^3 and
// cutoff 1 is 117,649 one-word leaf products and ~2.5 x 10^5 block additions of
// a few words.  Issued as launches that is ~10^5 dependent launches (hundreds of
// ms per multiplication, and seconds to capture and instantiate as a graph);
// here the host planner's operation list is uploaded once and ONE CTA walks it
// in program order:
//   * the whole working set (A, B, C and the schedule's temporaries) is staged
//     in shared memory when it fits, so every operation touches on-chip data
//     (~30-cycle accesses instead of ~500-cycle L2 round trips); C -- and A / B
//     when the contract lets the schedule overwrite them -- go back at the end;
//   * the operation descriptors stream through shared memory in chunks loaded
//     cooperatively, so no operation waits on its own descriptor fetch;
//   * the threads share each operation's elements and a barrier separates
//     consecutive operations (it also orders the memory accesses); when every
//     operation is small one warp walks the plan with warp barriers.
// Same arithmetic as the production kernels: residues exact in float64, one
// floor-based reduction per result; leaf dot products stay exact while
// k (p-1)^2 < 2^53.
#include <cstdint>

#include "wm_apply.cuh"
#include "wm_micro.h"

namespace wm {
namespace {

constexpr int kChunk = 64;  // operation descriptors staged per chunk (4 KB)

__device__ __forceinline__ double reduce(double v, double p, double pinv) {
    double r = fma(-floor(v * pinv), p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

// SMEM: operand "addresses" are byte offsets into the shared working-set image
template <bool SMEM>
__device__ __forceinline__ double* at(double* img, const double* ptr) {
    return SMEM ? img + (reinterpret_cast<std::uintptr_t>(ptr) >> 3) : const_cast<double*>(ptr);
}

// NT == 32: one warp walks the plan (every operation is small), warp barriers
template <int NT>
__device__ __forceinline__ void step_sync() {
    if (NT == 32) __syncwarp();
    else __syncthreads();
}

template <bool SMEM, int NT>
__device__ __forceinline__ void run_op(const MicroOp& o, double* img, double p, double pinv) {
    const std::uint32_t total = o.rows * o.cols;
    double* d = at<SMEM>(img, o.d);
    const double* a = at<SMEM>(img, o.a);
    const double* b = at<SMEM>(img, o.b);
    // power-of-two widths (every recursion of a power-of-two problem) index
    // without an integer division
    const bool pow2 = o.csh != 0xFFu;
    if (o.kind == MicroOp::ADD) {
        const double sa = static_cast<double>(o.sa), sb = static_cast<double>(o.sb);
        const bool two = o.mode <= M_GEN;
        for (std::uint32_t e = threadIdx.x; e < total; e += NT) {
            const std::uint32_t r = pow2 ? e >> o.csh : e / o.cols, c = e - r * o.cols;
            const double x = a[r * o.lda + c];
            const double y = two ? b[r * o.ldb + c] : 0.0;
            d[r * o.ldd + c] = apply<false>(x, y, o.mode, sa, sb, p, pinv);
        }
    } else {  // C <- alpha*A*B + beta*C
        const double al = static_cast<double>(o.sa), be = static_cast<double>(o.sb);
        for (std::uint32_t e = threadIdx.x; e < total; e += NT) {
            const std::uint32_t r = pow2 ? e >> o.csh : e / o.cols, c = e - r * o.cols;
            double s = 0.0;
            for (std::uint32_t l = 0; l < o.k; ++l) s = fma(a[r * o.lda + l], b[l * o.ldb + c], s);
            double v = al * reduce(s, p, pinv);
            if (o.sb) v = fma(be, d[r * o.ldd + c], v);
            d[r * o.ldd + c] = reduce(v, p, pinv);
        }
    }
}

template <bool SMEM, int NT>
__global__ void __launch_bounds__(NT) k_micro(const MicroOp* __restrict__ ops, std::uint32_t n,
                                              const MicroImage img_desc, double p, double pinv) {
    extern __shared__ double smem[];
    MicroOp* chunk = reinterpret_cast<MicroOp*>(smem);
    double* img = smem + kChunk * sizeof(MicroOp) / sizeof(double);
    if (SMEM)
        for (int r = 0; r < img_desc.nregions; ++r) {
            const MicroRegion& R = img_desc.region[r];
            if (!R.load) continue;
            for (std::uint64_t e = threadIdx.x; e < R.rows * R.cols; e += NT) {
                const std::uint64_t i = e / R.cols, j = e - i * R.cols;
                img[R.offset + i * R.ld + j] = R.global[i * R.ld + j];
            }
        }
    for (std::uint32_t base = 0; base < n; base += kChunk) {
        const std::uint32_t m = n - base < kChunk ? n - base : kChunk;
        __syncthreads();  // the previous chunk (and the image load) is complete
        const std::uint32_t words = m * static_cast<std::uint32_t>(sizeof(MicroOp) / 8);
        const std::uint64_t* src = reinterpret_cast<const std::uint64_t*>(ops + base);
        for (std::uint32_t w = threadIdx.x; w < words; w += NT)
            reinterpret_cast<std::uint64_t*>(chunk)[w] = src[w];
        __syncthreads();
        for (std::uint32_t i = 0; i < m; ++i) {
            run_op<SMEM, NT>(chunk[i], img, p, pinv);
            step_sync<NT>();
        }
    }
    __syncthreads();
    if (SMEM)
        for (int r = 0; r < img_desc.nregions; ++r) {
            const MicroRegion& R = img_desc.region[r];
            if (!R.store) continue;
            for (std::uint64_t e = threadIdx.x; e < R.rows * R.cols; e += NT) {
                const std::uint64_t i = e / R.cols, j = e - i * R.cols;
                R.global[i * R.ld + j] = img[R.offset + i * R.ld + j];
            }
        }
}

template <bool SMEM, int NT>
cudaError_t micro_launch(const MicroOp* ops, std::uint32_t n, const MicroImage& img, double pd,
                         std::size_t bytes, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_micro<SMEM, NT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_micro<SMEM, NT><<<1, NT, bytes, s>>>(ops, n, img, pd, 1.0 / pd);
    return cudaGetLastError();
}

}  // namespace

std::size_t micro_smem_limit() { return 200 * 1024 - kChunk * sizeof(MicroOp); }

cudaError_t launch_micro(const MicroOp* ops, std::uint32_t n, const MicroImage& img, bool small,
                         std::uint32_t p, cudaStream_t s) {
    const double pd = static_cast<double>(p);
    std::size_t bytes = kChunk * sizeof(MicroOp);
    if (img.nregions) {
        bytes += img.words * sizeof(double);
        return small ? micro_launch<true, 32>(ops, n, img, pd, bytes, s)
                     : micro_launch<true, 256>(ops, n, img, pd, bytes, s);
    }
    return small ? micro_launch<false, 32>(ops, n, img, pd, bytes, s)
                 : micro_launch<false, 256>(ops, n, img, pd, bytes, s);
}

}  // namespace wm
