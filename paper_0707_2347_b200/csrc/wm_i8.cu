// Leaf product on the 5th-generation tensor cores, exact over Z/pZ (p < 2^16):
//   C <- alpha*A*B + beta*C                  (classical_mul, ring.hpp:315-384)
//
// Each canonical residue a < 2^16 (held in float64) is split into two unsigned
// 8-bit limbs a = 256*a_h + a_l.  The product needs four limb products, issued as
// tcgen05.mma kind::i8 (u8 x u8 -> s32 in TMEM) into three accumulators:
//   D_hh = A_h B_h,   D_x = A_h B_l + A_l B_h,   D_ll = A_l B_l,
// each bounded by 2*k*255^2 < 2^32 for k <= 32768 (read back as u32).  The
// epilogue recombines v = 2^16 D_hh + 2^8 D_x + D_ll < 2^49 exactly in float64,
// reduces mod p, and applies alpha / beta in residue arithmetic.
//
// Leaves are small (128^3 .. 1024^3 at the BASELINE cutoffs), so the kernel is
// built for latency and parallelism rather than peak tensor throughput -- the
// float64 operand stream, not the tensor pipe, is the bound:
//  * a 128 x BN output tile per CTA (UMMA M=128, N=BN in {32,64}), K in 32-wide
//    chunks (one MMA per limb product per chunk);
//  * the float64 chunks stream through a 4-deep cp.async ring (up to 3 chunks,
//    ~120-160 KB, in flight per SM), are converted to limbs in shared memory by
//    all 256 threads (conflict-free: 272-B padded rows, one 16-B store per
//    limb row segment) and consumed by one elected thread issuing the MMAs;
//  * for small leaves the K dimension is split across the S CTAs of a thread
//    block cluster (S in {1,2,4}); each CTA reduces its partial mod p into
//    shared memory and the cluster sums the S partials over DSMEM, so the
//    split costs no global scratch and no extra launch.
// Every kernel waits on griddepcontrol (programmatic dependent launch) before
// touching global memory, so it can be launched while its producer drains.
#include <cooperative_groups.h>

#include <cstdint>

#include "wm_device.h"
#include "wm_tc.h"

namespace cg = cooperative_groups;

namespace wm {
namespace {

constexpr int BM = 128, KC = 32, NT = 256, NF64 = 3, NLIMB = 2;
constexpr int AROW = 34;  // padded row of the float64 A stage (272 B)

template <int BN>
struct Smem {
    double a[NF64][BM * AROW];          // float64 A chunks (row-major, padded)
    double b[NF64][KC * BN];            // float64 B chunks (k rows x BN)
    std::uint8_t a_hi[NLIMB][BM * KC];  // limb tiles, canonical K-major layout
    std::uint8_t a_lo[NLIMB][BM * KC];
    std::uint8_t b_hi[NLIMB][BN * KC];
    std::uint8_t b_lo[NLIMB][BN * KC];
    std::uint64_t mbar[NLIMB];
    std::uint64_t mbar_done;
    std::uint32_t tmem_base;
};

// canonical K-major no-swizzle offset of (row r, k c) in a tile 32 bytes wide:
// 8-row x 16-byte core matrices, K halves 128 B apart (LBO), row groups 256 B (SBO)
__device__ __forceinline__ std::uint32_t koff(std::uint32_t r, std::uint32_t c) {
    return (r & 7u) * 16u + (r >> 3) * 256u + (c >> 4) * 128u + (c & 15u);
}

__device__ __forceinline__ double reduce_modp(double v, double p, double pinv) {
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BN>
__device__ __forceinline__ void issue_chunk(Smem<BN>& S, int st, const MulParams& P,
                                            std::uint64_t i0, std::uint64_t j0, std::uint32_t k0,
                                            int tid) {
    // A: 128 rows x 32 doubles = 2048 x 16 B
#pragma unroll
    for (int j = 0; j < (BM * KC / 2) / NT; ++j) {
        const int u = j * NT + tid;
        const int r = u >> 4, c = (u & 15) * 2;
        cp16(&S.a[st][r * AROW + c], P.A + (i0 + r) * P.lda + k0 + c);
    }
    // B: 32 rows x BN doubles
#pragma unroll
    for (int j = 0; j < (KC * BN / 2) / NT; ++j) {
        const int u = j * NT + tid;
        const int kk = u / (BN / 2), c = (u % (BN / 2)) * 2;
        cp16(&S.b[st][kk * BN + c], P.B + (k0 + kk) * P.ldb + j0 + c);
    }
}

template <int BN>
__device__ __forceinline__ void convert_chunk(Smem<BN>& S, int fs, int ls, int tid) {
    {  // A: thread = (row, 16-wide half)
        const int r = tid & 127, h = tid >> 7;
        const double* src = &S.a[fs][r * AROW + h * 16];
        std::uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v0 = *reinterpret_cast<const double2*>(src + q * 4);
            const double2 v1 = *reinterpret_cast<const double2*>(src + q * 4 + 2);
            const std::uint32_t x0 = __double2uint_rz(v0.x), x1 = __double2uint_rz(v0.y),
                                x2 = __double2uint_rz(v1.x), x3 = __double2uint_rz(v1.y);
            hi[q] = (x0 >> 8) | ((x1 >> 8) << 8) | ((x2 >> 8) << 16) | ((x3 >> 8) << 24);
            lo[q] = (x0 & 255u) | ((x1 & 255u) << 8) | ((x2 & 255u) << 16) | ((x3 & 255u) << 24);
        }
        const std::uint32_t o = koff(r, h * 16);
        *reinterpret_cast<uint4*>(&S.a_hi[ls][o]) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(&S.a_lo[ls][o]) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    // B: thread = (n, 4 consecutive k) -> K-major rows of the B^T tile
#pragma unroll
    for (int it = 0; it < (KC * BN) / (4 * NT); ++it) {
        const int t = it * NT + tid;
        const int n = t % BN, kg = t / BN;
        std::uint32_t hi = 0, lo = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const std::uint32_t x = __double2uint_rz(S.b[fs][(kg * 4 + e) * BN + n]);
            hi |= (x >> 8) << (8 * e);
            lo |= (x & 255u) << (8 * e);
        }
        const std::uint32_t o = koff(n, kg * 4);
        *reinterpret_cast<std::uint32_t*>(&S.b_hi[ls][o]) = hi;
        *reinterpret_cast<std::uint32_t*>(&S.b_lo[ls][o]) = lo;
    }
}

template <int BN, int SPLIT>
__global__ void __launch_bounds__(NT, 1) k_leaf_i8(const MulParams P) {
    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    Smem<BN>& S = *reinterpret_cast<Smem<BN>*>(smem_raw);
    constexpr std::uint32_t TCOLS = BN == 32 ? 128 : 256;  // D_hh | D_x | D_ll
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = SPLIT > 1 ? static_cast<int>(blockIdx.x) : 0;  // rank in the cluster
    const std::uint64_t j0 = static_cast<std::uint64_t>(blockIdx.y) * BN;
    const std::uint64_t i0 = static_cast<std::uint64_t>(blockIdx.z) * BM;
    const std::uint32_t klen = P.k / SPLIT;
    const std::uint32_t kbeg = ks * klen;
    const std::uint32_t nk = klen / KC;

    if (warp == 0) tc::tmem_alloc(&S.tmem_base, TCOLS);
    if (tid == 0) {
        for (int s = 0; s < NLIMB; ++s) tc::mbar_init(&S.mbar[s], 1);
        tc::mbar_init(&S.mbar_done, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const std::uint32_t tbase = S.tmem_base;
    constexpr std::uint32_t idesc = tc::idesc_i8(BM, BN);

    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

#pragma unroll
    for (int c = 0; c < NF64 - 1; ++c) {
        if (c < static_cast<int>(nk)) issue_chunk<BN>(S, c, P, i0, j0, kbeg + c * KC, tid);
        cp_commit();
    }
    for (std::uint32_t kc = 0; kc < nk; ++kc) {
        const std::uint32_t nxt = kc + NF64 - 1;
        if (nxt < nk) issue_chunk<BN>(S, nxt % NF64, P, i0, j0, kbeg + nxt * KC, tid);
        cp_commit();
        cp_wait<NF64 - 1>();
        const int ls = kc % NLIMB;
        if (kc >= NLIMB) tc::mbar_wait(&S.mbar[ls], ((kc / NLIMB) - 1) & 1);
        __syncthreads();  // chunk kc landed for every thread
        convert_chunk<BN>(S, kc % NF64, ls, tid);
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const std::uint64_t ah = tc::smem_desc(tc::smem_u32(S.a_hi[ls]), 128, 256);
            const std::uint64_t al = tc::smem_desc(tc::smem_u32(S.a_lo[ls]), 128, 256);
            const std::uint64_t bh = tc::smem_desc(tc::smem_u32(S.b_hi[ls]), 128, 256);
            const std::uint64_t bl = tc::smem_desc(tc::smem_u32(S.b_lo[ls]), 128, 256);
            const bool acc = kc > 0;
            tc::mma_i8(tbase + 0, ah, bh, idesc, acc);
            tc::mma_i8(tbase + BN, ah, bl, idesc, acc);
            tc::mma_i8(tbase + BN, al, bh, idesc, true);
            tc::mma_i8(tbase + 2 * BN, al, bl, idesc, acc);
            tc::commit(&S.mbar[ls]);
            if (kc + 1 == nk) tc::commit(&S.mbar_done);
        }
    }

    tc::mbar_wait(&S.mbar_done, 0);
    tc::fence_after();
    const double p = P.pd, pinv = P.pinv;
    const double al = static_cast<double>(P.alpha), be = static_cast<double>(P.beta);
    // warp w drains TMEM lanes 32*(w%4).., columns [ (w/4)*BN/2, +BN/2 )
    const int lg = warp & 3, half = warp >> 2;
    const std::uint32_t row = lg * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(lg * 32) << 16;

    if (SPLIT == 1) {
        double* crow = P.C + (i0 + row) * P.ldc + j0;
#pragma unroll
        for (int q = 0; q < BN / 32; ++q) {
            const std::uint32_t col = half * (BN / 2) + q * 16;
            std::uint32_t hh[16], xx[16], ll[16];
            tc::tmem_ld16(tbase + lane_off + col, hh);
            tc::tmem_ld16(tbase + lane_off + BN + col, xx);
            tc::tmem_ld16(tbase + lane_off + 2 * BN + col, ll);
            tc::tmem_wait_ld();
            double out[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const double v = fma(static_cast<double>(hh[e]), 65536.0,
                                     fma(static_cast<double>(xx[e]), 256.0,
                                         static_cast<double>(ll[e])));
                out[e] = reduce_modp(v, p, pinv) * al;
            }
            if (P.beta != 0) {
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                    const double2 c = *reinterpret_cast<const double2*>(crow + col + e);
                    out[e] = fma(be, c.x, out[e]);
                    out[e + 1] = fma(be, c.y, out[e + 1]);
                }
            }
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
                double2 o;
                o.x = reduce_modp(out[e], p, pinv);
                o.y = reduce_modp(out[e + 1], p, pinv);
                *reinterpret_cast<double2*>(crow + col + e) = o;
            }
        }
    } else {
        // partial (mod p) -> own shared memory (reuses the float64 A ring),
        // then the cluster sums the SPLIT partials over DSMEM.
        std::uint32_t* part = reinterpret_cast<std::uint32_t*>(&S.a[0][0]);  // [BM][BN+1]
        constexpr int PLD = BN + 1;
#pragma unroll
        for (int q = 0; q < BN / 32; ++q) {
            const std::uint32_t col = half * (BN / 2) + q * 16;
            std::uint32_t hh[16], xx[16], ll[16];
            tc::tmem_ld16(tbase + lane_off + col, hh);
            tc::tmem_ld16(tbase + lane_off + BN + col, xx);
            tc::tmem_ld16(tbase + lane_off + 2 * BN + col, ll);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const double v = fma(static_cast<double>(hh[e]), 65536.0,
                                     fma(static_cast<double>(xx[e]), 256.0,
                                         static_cast<double>(ll[e])));
                part[row * PLD + col + e] = static_cast<std::uint32_t>(reduce_modp(v, p, pinv));
            }
        }
        cg::cluster_group cluster = cg::this_cluster();
        constexpr int ROWS = BM / SPLIT;
        constexpr int ITER = ROWS * BN / NT;  // elements per thread, compile-time
        // issue the C reads (beta != 0) before the cluster barrier so their
        // latency overlaps it
        double cin[ITER];
        if (P.beta != 0) {
#pragma unroll
            for (int it = 0; it < ITER; ++it) {
                const int e = it * NT + tid;
                const int r = ks * ROWS + e / BN, c = e % BN;
                cin[it] = P.C[(i0 + r) * P.ldc + j0 + c];
            }
        }
        cluster.sync();
        const std::uint32_t* src[SPLIT];
#pragma unroll
        for (int s = 0; s < SPLIT; ++s) src[s] = cluster.map_shared_rank(part, s);
        std::uint32_t pv[ITER][SPLIT];
#pragma unroll
        for (int it = 0; it < ITER; ++it) {
            const int e = it * NT + tid;
            const int r = ks * ROWS + e / BN, c = e % BN;
#pragma unroll
            for (int s = 0; s < SPLIT; ++s) pv[it][s] = src[s][r * PLD + c];
        }
#pragma unroll
        for (int it = 0; it < ITER; ++it) {
            const int e = it * NT + tid;
            const int r = ks * ROWS + e / BN, c = e % BN;
            double v = 0.0;
#pragma unroll
            for (int s = 0; s < SPLIT; ++s) v += static_cast<double>(pv[it][s]);
            v = reduce_modp(v, p, pinv) * al;
            if (P.beta != 0) v = fma(be, cin[it], v);
            P.C[(i0 + r) * P.ldc + j0 + c] = reduce_modp(v, p, pinv);
        }
        cluster.sync();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, TCOLS);
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

template <int BN, int SPLIT>
cudaError_t set_attr() {
    return cudaFuncSetAttribute(k_leaf_i8<BN, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem<BN>)));
}

template <int BN, int SPLIT>
cudaError_t launch_cfg(const MulParams& P, cudaStream_t s) {
    auto kern = k_leaf_i8<BN, SPLIT>;
    const int smem = static_cast<int>(sizeof(Smem<BN>));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SPLIT, P.n / BN, P.m / BM);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (SPLIT > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = SPLIT;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, P);
}

}  // namespace

bool leaf_i8_supported(const MulParams& P) {
    return P.m % BM == 0 && P.n % 32 == 0 && P.k % KC == 0 && P.k <= 32768 && P.m > 0 &&
           P.n > 0 && P.k > 0 && P.lda % 2 == 0 && P.ldb % 2 == 0 && P.ldc % 2 == 0 &&
           aligned16(P.A) && aligned16(P.B) && aligned16(P.C) && P.p < 65536u;
}

// one-time function attributes (not stream-ordered, so kept out of graph capture)
cudaError_t leaf_i8_init() {
    cudaError_t e;
    if ((e = set_attr<64, 1>()) != cudaSuccess) return e;
    if ((e = set_attr<64, 2>()) != cudaSuccess) return e;
    if ((e = set_attr<64, 4>()) != cudaSuccess) return e;
    if ((e = set_attr<32, 1>()) != cudaSuccess) return e;
    if ((e = set_attr<32, 2>()) != cudaSuccess) return e;
    return set_attr<32, 4>();
}

// measurement hook: force a (BN, SPLIT) configuration
cudaError_t launch_leaf_i8_cfg(const MulParams& P, int bn, int split, cudaStream_t s) {
    if (!leaf_i8_supported(P) || P.n % bn || P.k % (split * KC)) return cudaErrorInvalidValue;
    if (bn == 64 && split == 1) return launch_cfg<64, 1>(P, s);
    if (bn == 64 && split == 2) return launch_cfg<64, 2>(P, s);
    if (bn == 64 && split == 4) return launch_cfg<64, 4>(P, s);
    if (bn == 32 && split == 1) return launch_cfg<32, 1>(P, s);
    if (bn == 32 && split == 2) return launch_cfg<32, 2>(P, s);
    if (bn == 32 && split == 4) return launch_cfg<32, 4>(P, s);
    return cudaErrorInvalidValue;
}

// Tile width and K split: aim for >= ~100 CTAs on the 148 SMs; a split needs
// every slice to be a whole number of 32-wide chunks.
cudaError_t launch_leaf_i8(const MulParams& P, cudaStream_t s) {
    if (!leaf_i8_supported(P)) return cudaErrorInvalidValue;
    const std::uint32_t tiles64 = (P.n % 64 == 0) ? (P.m / BM) * (P.n / 64) : 0;
    const std::uint32_t tiles32 = (P.m / BM) * (P.n / 32);
    const bool s2 = P.k % (2 * KC) == 0, s4 = P.k % (4 * KC) == 0;
    if (tiles64 >= 96) return launch_cfg<64, 1>(P, s);
    if (tiles64 >= 48 && s2) return launch_cfg<64, 2>(P, s);
    if (tiles64 >= 24 && s4) return launch_cfg<64, 4>(P, s);
    if (tiles32 >= 96) return launch_cfg<32, 1>(P, s);
    if (tiles32 >= 48 && s2) return launch_cfg<32, 2>(P, s);
    if (s4) return launch_cfg<32, 4>(P, s);
    if (s2) return launch_cfg<32, 2>(P, s);
    return launch_cfg<32, 1>(P, s);
}

}  // namespace wm
