// Elementwise kernels: batched block additions over Z/pZ held in float64
// (block_addsub / block_scale_copy, ring.hpp:241-310), boundary conversions and
// the seeded generator.
//
// The additions are HBM-bound (3 x 8 B per element for a two-term addition).
// One launch carries up to kMaxAddBatch independent items (e.g. a schedule's
// S_i / T_i pair), each split into 256-thread blocks that stream 4 x 16 B per
// thread with all loads issued before the stores.  Residue arithmetic is exact
// in float64: operands are canonical (< 2^16), so a +/- b needs one conditional
// correction and the general sa*a + sb*b (< 2^33) one floor-based reduction.
#include <cstdint>

#include "wm_launch.h"
#include "wm_device.h"
#include "wm_fused.h"
#include "wm_apply.cuh"

namespace wm {

bool g_pdl = true;
namespace {

// d = ca*a + cb*b over canonical operands, reduced once (MODP: residue
// scalars, |v| < 2^33, exact): one FMA path for every addition mode
template <bool REAL>
__device__ __forceinline__ double lin_item(double a, double b, double ca, double cb, double p,
                                           double pinv) {
    const double v = fma(ca, a, cb * b);
    if (REAL) return v;
    double r = fma(-floor(v * pinv), p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

template <bool REAL, int ILP>
__global__ void __launch_bounds__(kAddThreads) k_addsub(const AddBatch B) {
    // programmatic dependent launch: wait for the producer grid, then let the
    // next kernel in the chain start its launch
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    WM_TL_BEGIN(B.tl);
    int i = 0;
#pragma unroll 1
    while (i + 1 < B.n && blockIdx.x >= B.it[i + 1].blk0) ++i;
    const AddItem& t = B.it[i];
    const std::uint32_t mode = t.mode;
    const double p = B.pd, pinv = B.pinv;
    const bool two = mode <= M_GEN;
    const std::uint64_t blk = blockIdx.x - t.blk0;
    if (t.vec == 2) {
        const std::uint32_t cv = t.cols >> 1;
        const std::uint64_t total = static_cast<std::uint64_t>(t.rows) * cv;
        const std::uint64_t start = blk * (kAddThreads * ILP) + threadIdx.x;
        double2 av[ILP], bv[ILP];
        std::uint64_t r[ILP], c[ILP];
        bool ok[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const std::uint64_t idx = start + static_cast<std::uint64_t>(u) * kAddThreads;
            ok[u] = idx < total;
            r[u] = idx / cv;
            c[u] = (idx - r[u] * cv) * 2;
            if (ok[u]) {
                av[u] = __ldg(reinterpret_cast<const double2*>(t.a + r[u] * t.lda + c[u]));
                if (two) bv[u] = __ldg(reinterpret_cast<const double2*>(t.b + r[u] * t.ldb + c[u]));
            }
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            if (!ok[u]) continue;
            double2 o;
            o.x = lin_item<REAL>(av[u].x, two ? bv[u].x : 0.0, t.ca, t.cb, p, pinv);
            o.y = lin_item<REAL>(av[u].y, two ? bv[u].y : 0.0, t.ca, t.cb, p, pinv);
            *reinterpret_cast<double2*>(t.d + r[u] * t.ldd + c[u]) = o;
        }
    } else {
        const std::uint64_t total = static_cast<std::uint64_t>(t.rows) * t.cols;
        const std::uint64_t start = blk * (kAddThreads * ILP) + threadIdx.x;
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const std::uint64_t idx = start + static_cast<std::uint64_t>(u) * kAddThreads;
            if (idx >= total) break;
            const std::uint64_t rr = idx / t.cols, cc = idx - rr * t.cols;
            const double a = t.a[rr * t.lda + cc];
            const double b = two ? t.b[rr * t.ldb + cc] : 0.0;
            t.d[rr * t.ldd + cc] = lin_item<REAL>(a, b, t.ca, t.cb, p, pinv);
        }
    }
    WM_TL_END(B.tl);
    WM_PDL_LATE_M();
}

}  // namespace



namespace {

// One fused run of a schedule's block additions: every thread owns one 16-B
// position of the (identically shaped, pairwise disjoint) slot views and
// executes the run's dataflow on registers -- each slot read once, written once.
// One kernel per run (GID): each launch carries only its own body.
template <bool REAL, int GID>
__global__ void __launch_bounds__(256) k_group(const fused::GroupParams G, unsigned long long* tl) {
    // the position is worked out ahead of the wait (nothing here touches memory)
    const std::uint32_t cv = G.cols >> 1;
    const std::uint64_t total = static_cast<std::uint64_t>(G.rows) * cv;
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    const std::uint64_t r = idx / cv, c = (idx - r * cv) * 2;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    WM_TL_BEGIN(tl);
    if (idx < total) fused::GroupBody<REAL, GID>::run(G, r, c);
    WM_TL_END(tl);
    WM_PDL_LATE_M();
}

using GroupKernel = void (*)(const fused::GroupParams, unsigned long long*);
#define WM_GK_MODP(i) k_group<false, i>,
#define WM_GK_REAL(i) k_group<true, i>,
const GroupKernel kGroupModp[] = {WM_FUSED_GROUP_IDS(WM_GK_MODP)};
const GroupKernel kGroupReal[] = {WM_FUSED_GROUP_IDS(WM_GK_REAL)};
#undef WM_GK_MODP
#undef WM_GK_REAL
static_assert(sizeof(kGroupModp) / sizeof(kGroupModp[0]) == fused::kNumGroups, "one kernel per run");

__global__ void k_u32_to_f64(double* __restrict__ dst, std::uint64_t ldd,
                             const std::uint32_t* __restrict__ src, std::uint64_t lds,
                             std::uint64_t rows, std::uint64_t cols, unsigned long long* tl) {
    WM_TL_BEGIN(tl);
    const std::uint64_t total = rows * cols;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
         i < total; i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t r = i / cols, c = i - r * cols;
        dst[r * ldd + c] = static_cast<double>(src[r * lds + c]);
    }
    WM_TL_END(tl);
}

// canonicalise (values are exact integers; reduce any representative into [0, p))
__global__ void k_f64_to_u32(std::uint32_t* __restrict__ dst, std::uint64_t ldd,
                             const double* __restrict__ src, std::uint64_t lds,
                             std::uint64_t rows, std::uint64_t cols, double p,
                             unsigned long long* tl) {
    WM_TL_BEGIN(tl);
    const std::uint64_t total = rows * cols;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
         i < total; i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t r = i / cols, c = i - r * cols;
        double v = src[r * lds + c];
        v = v - floor(v / p) * p;
        if (v >= p) v -= p;
        if (v < 0) v += p;
        dst[r * ldd + c] = static_cast<std::uint32_t>(v);
    }
    WM_TL_END(tl);
}

__device__ __forceinline__ std::uint64_t sm64_mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// SplitMix64 stream of Matrix::fill_random (ring.hpp:93-105,202-205): element i of
// the row-major fill is mix(seed + (i+1)*gamma) % p -- index-addressable.
__global__ void k_fill_splitmix(double* __restrict__ dst, std::uint64_t ld, std::uint64_t rows,
                                std::uint64_t cols, std::uint64_t seed, std::uint32_t p,
                                int real) {
    const std::uint64_t total = rows * cols;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
         i < total; i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t z = sm64_mix(seed + (i + 1) * 0x9e3779b97f4a7c15ull);
        const std::uint64_t r = i / cols, c = i - r * cols;
        double v;
        if (real) v = 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
        else v = static_cast<double>(z % p);
        dst[r * ld + c] = v;
    }
}

// dst = sum_i coef_i * src_i over up to kMaxLincomb equally shaped blocks in one
// HBM pass (the S_i / T_i operand of a distributed product is a combination of
// up to four quadrants; the gathered P_i folds into C with alpha * coef).
// Canonical residues times coefficients < 2^16 sum to < 2^34: exact in float64.
template <bool REAL, bool VEC>
__global__ void __launch_bounds__(256) k_lincomb(const LincombParams L) {
    const std::uint64_t cols = VEC ? L.cols / 2 : L.cols;
    const std::uint64_t total = L.rows * cols;
    const double p = L.p, pinv = 1.0 / L.p;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
         i < total; i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t r = i / cols, c = (i - r * cols) * (VEC ? 2 : 1);
        double v0 = 0.0, v1 = 0.0;
#pragma unroll
        for (int t = 0; t < kMaxLincomb; ++t) {
            if (t >= L.n) break;
            const double* src = L.src[t] + r * L.lds[t] + c;
            if (VEC) {
                const double2 x = __ldg(reinterpret_cast<const double2*>(src));
                v0 = fma(L.coef[t], x.x, v0);
                v1 = fma(L.coef[t], x.y, v1);
            } else {
                v0 = fma(L.coef[t], __ldg(src), v0);
            }
        }
        if (!REAL) {  // v is an exact integer, |v| < 2^36
            v0 = fma(-floor(v0 * pinv), p, v0);
            v0 = v0 < 0.0 ? v0 + p : (v0 >= p ? v0 - p : v0);
            v1 = fma(-floor(v1 * pinv), p, v1);
            v1 = v1 < 0.0 ? v1 + p : (v1 >= p ? v1 - p : v1);
        }
        double* dst = L.dst + r * L.ldd + c;
        if (VEC) *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
        else *dst = v0;
    }
}

unsigned grid_for(std::uint64_t total) {
    std::uint64_t b = (total + 255) / 256;
    if (b > 148ull * 32) b = 148ull * 32;
    return static_cast<unsigned>(b ? b : 1);
}

}  // namespace

cudaError_t launch_addsub(const AddBatch& b, bool real, unsigned blocks, cudaStream_t s) {
    // blocks were counted at kAddIlp units per thread; small launches spread the
    // same work over more CTAs (fewer units per thread) to fill the 148 SMs
    int ilp = kAddIlp;
    if (blocks * 4 <= 2 * 148) ilp = 1;
    else if (blocks * 2 <= 2 * 148) ilp = 2;
    AddBatch bb = b;
    if (ilp != kAddIlp)
        for (int i = 0; i < bb.n; ++i) bb.it[i].blk0 *= kAddIlp / ilp;
    blocks *= kAddIlp / ilp;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kAddThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define WM_ADD_LAUNCH(I)                                                       \
    if (ilp == I)                                                              \
        return real ? cudaLaunchKernelEx(&cfg, k_addsub<true, I>, bb)          \
                    : cudaLaunchKernelEx(&cfg, k_addsub<false, I>, bb);
    WM_ADD_LAUNCH(1)
    WM_ADD_LAUNCH(2)
    WM_ADD_LAUNCH(4)
#undef WM_ADD_LAUNCH
    return cudaErrorInvalidValue;
}

cudaError_t launch_group(int gid, const fused::GroupParams& G, bool real, cudaStream_t s,
                         unsigned long long* tl) {
    const std::uint64_t total = static_cast<std::uint64_t>(G.rows) * (G.cols / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((total + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (gid < 0 || gid >= fused::kNumGroups) return cudaErrorInvalidValue;
    return cudaLaunchKernelEx(&cfg, real ? kGroupReal[gid] : kGroupModp[gid], G, tl);
}

cudaError_t launch_lincomb(const LincombParams& L, bool real, cudaStream_t s) {
    bool vec = L.cols % 2 == 0 && L.ldd % 2 == 0 && reinterpret_cast<std::uintptr_t>(L.dst) % 16 == 0;
    for (int t = 0; t < L.n; ++t)
        vec = vec && L.lds[t] % 2 == 0 && reinterpret_cast<std::uintptr_t>(L.src[t]) % 16 == 0;
    const unsigned grid = grid_for(L.rows * (vec ? L.cols / 2 : L.cols));
    if (vec) {
        if (real) k_lincomb<true, true><<<grid, 256, 0, s>>>(L);
        else k_lincomb<false, true><<<grid, 256, 0, s>>>(L);
    } else {
        if (real) k_lincomb<true, false><<<grid, 256, 0, s>>>(L);
        else k_lincomb<false, false><<<grid, 256, 0, s>>>(L);
    }
    return cudaGetLastError();
}

cudaError_t launch_u32_to_f64(double* dst, std::uint64_t ldd, const std::uint32_t* src,
                              std::uint64_t lds, std::uint64_t rows, std::uint64_t cols,
                              cudaStream_t s, unsigned long long* tl) {
    k_u32_to_f64<<<grid_for(rows * cols), 256, 0, s>>>(dst, ldd, src, lds, rows, cols, tl);
    return cudaGetLastError();
}

cudaError_t launch_f64_to_u32(std::uint32_t* dst, std::uint64_t ldd, const double* src,
                              std::uint64_t lds, std::uint64_t rows, std::uint64_t cols,
                              std::uint32_t p, cudaStream_t s, unsigned long long* tl) {
    k_f64_to_u32<<<grid_for(rows * cols), 256, 0, s>>>(dst, ldd, src, lds, rows, cols,
                                                        static_cast<double>(p), tl);
    return cudaGetLastError();
}

cudaError_t launch_fill_splitmix(double* dst, std::uint64_t ld, std::uint64_t rows,
                                 std::uint64_t cols, std::uint64_t seed, std::uint32_t p,
                                 bool real, cudaStream_t s) {
    k_fill_splitmix<<<grid_for(rows * cols), 256, 0, s>>>(dst, ld, rows, cols, seed, p,
                                                           real ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace wm
