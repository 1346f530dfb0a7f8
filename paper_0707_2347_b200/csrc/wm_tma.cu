// TMA-fed, warp-specialised variant of the exact int8-limb GEMM (wm_i8.cu has
// the arithmetic contract; this file changes only how operands reach shared
// memory).  Per 32-wide K chunk one elected thread issues 2-3 tensor-map TMA
// loads (cp.async.bulk.tensor.2d) into a 4-deep staging ring whose "full"
// mbarriers carry the byte count; eight converter warps turn the landed
// residues into limb tiles; one thread issues the MMAs.  Float64 A boxes use
// 128-B swizzle and uint16 A boxes 64-B swizzle so the converters' row-wise
// reads are bank-conflict-free; B boxes are read along N and need none.
// Tensor maps are encoded on the host at plan-lowering time (through
// cudaGetDriverEntryPoint, no libcuda link) and passed as __grid_constant__
// parameters, so a captured graph replays them without host work.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>

#include "wm_launch.h"
#include "wm_gemm.h"
#include "wm_tc.h"

namespace cg = cooperative_groups;

namespace wm {
namespace {

constexpr int BM = 128, KC = 32;
// Staging depth: the MMA commit -> mbarrier round trip is ~0.4 us, so the limb
// ring must be deep enough that converters never wait on it (2 stages made the
// K loop latency-bound at ~0.45 us per chunk).
template <int BN>
struct Depth {
    static constexpr int NF = BN == 64 ? 3 : 4;  // TMA staging ring
    static constexpr int NLIMB = 4;              // converted limb-tile ring
};
constexpr int NCONV = 256;
constexpr int NT = NCONV + 64;  // producer warp + MMA warp + 8 converter warps
constexpr int A_STAGE = BM * KC * 8;  // 32 KB (float64 worst case)

template <int BN>
struct Smem {
    static constexpr int NF = Depth<BN>::NF, NLIMB = Depth<BN>::NLIMB;
    std::uint8_t a[NF][A_STAGE];        // 1024-B aligned (swizzled TMA boxes)
    std::uint8_t b[NF][KC * BN * 8];
    std::uint8_t a_hi[NLIMB][BM * KC];
    std::uint8_t a_lo[NLIMB][BM * KC];
    std::uint8_t b_hi[NLIMB][BN * KC];
    std::uint8_t b_lo[NLIMB][BN * KC];
    std::uint64_t full[NF], empty[NF];
    std::uint64_t lfull[NLIMB], lempty[NLIMB];
    std::uint64_t done;
    std::uint32_t tmem_base;
};

__device__ __forceinline__ std::uint32_t koff(std::uint32_t r, std::uint32_t c) {
    return (r & 7u) * 16u + (r >> 3) * 256u + (c >> 4) * 128u + (c & 15u);
}

__device__ __forceinline__ double reduce_modp(double v, double p, double pinv) {
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

__device__ __forceinline__ void pack4(const std::uint32_t (&x)[4], std::uint32_t& hi,
                                      std::uint32_t& lo) {
    hi = (x[0] >> 8) | ((x[1] >> 8) << 8) | ((x[2] >> 8) << 16) | ((x[3] >> 8) << 24);
    lo = (x[0] & 255u) | ((x[1] & 255u) << 8) | ((x[2] & 255u) << 16) | ((x[3] & 255u) << 24);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            std::uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(tc::smem_u32(mbar))
        : "memory");
}

// A stage -> limb tiles: thread = (row r, 16-wide K half h)
__device__ __forceinline__ void convert_a(const std::uint8_t* st, std::uint8_t* hi_t,
                                          std::uint8_t* lo_t, int ct, bool u16) {
    const int r = ct & 127, h = ct >> 7;
    std::uint32_t hi[4], lo[4];
    if (!u16) {
        // two 128-B-swizzled boxes [128 rows][16 doubles]; box h holds K [16h, 16h+16)
        const std::uint8_t* row = st + h * (BM * 128) + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v0 =
                *reinterpret_cast<const double2*>(row + (((2 * q) ^ (r & 7)) << 4));
            const double2 v1 =
                *reinterpret_cast<const double2*>(row + (((2 * q + 1) ^ (r & 7)) << 4));
            const std::uint32_t x[4] = {__double2uint_rz(v0.x), __double2uint_rz(v0.y),
                                        __double2uint_rz(v1.x), __double2uint_rz(v1.y)};
            pack4(x, hi[q], lo[q]);
        }
    } else {
        // one 64-B-swizzled box [128 rows][32 uint16]
        const std::uint8_t* row = st + r * 64;
        const int sw = (r >> 1) & 3;
        const uint4 w0 = *reinterpret_cast<const uint4*>(row + (((2 * h) ^ sw) << 4));
        const uint4 w1 = *reinterpret_cast<const uint4*>(row + (((2 * h + 1) ^ sw) << 4));
        const std::uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const std::uint32_t x[4] = {wv[2 * q] & 0xFFFFu, wv[2 * q] >> 16,
                                        wv[2 * q + 1] & 0xFFFFu, wv[2 * q + 1] >> 16};
            pack4(x, hi[q], lo[q]);
        }
    }
    const std::uint32_t o = koff(r, h * 16);
    *reinterpret_cast<uint4*>(hi_t + o) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(lo_t + o) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// B stage: dense box [32 k rows][BN] -> K-major limb tiles of B^T
template <int BN>
__device__ __forceinline__ void convert_b(const std::uint8_t* st, std::uint8_t* hi_t,
                                          std::uint8_t* lo_t, int ct, bool u16) {
#pragma unroll
    for (int it = 0; it < (KC * BN) / (4 * NCONV); ++it) {
        const int t = it * NCONV + ct;
        const int n = t % BN, kg = t / BN;
        std::uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int kk = kg * 4 + e;
            x[e] = u16 ? static_cast<std::uint32_t>(
                             reinterpret_cast<const std::uint16_t*>(st)[kk * BN + n])
                       : __double2uint_rz(reinterpret_cast<const double*>(st)[kk * BN + n]);
        }
        std::uint32_t hi, lo;
        pack4(x, hi, lo);
        const std::uint32_t o = koff(n, kg * 4);
        *reinterpret_cast<std::uint32_t*>(hi_t + o) = hi;
        *reinterpret_cast<std::uint32_t*>(lo_t + o) = lo;
    }
}

template <int BN>
__device__ __forceinline__ void tmem_rows16(std::uint32_t taddr, double (&v)[16], double p,
                                            double pinv) {
    std::uint32_t hh[16], xx[16], ll[16];
    tc::tmem_ld16(taddr, hh);
    tc::tmem_ld16(taddr + BN, xx);
    tc::tmem_ld16(taddr + 2 * BN, ll);
    tc::tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const double x = fma(static_cast<double>(hh[e]), 65536.0,
                             fma(static_cast<double>(xx[e]), 256.0, static_cast<double>(ll[e])));
        v[e] = reduce_modp(x, p, pinv);
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// diagnostics: phase timestamps of one thread per CTA
#define WM_STAMP(slot)                                                                   \
    do {                                                                                 \
        if (P.trace)                                                                     \
            P.trace[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 16 + \
                    (slot)] = gtimer();                                                  \
    } while (0)

template <int BN, int SPLIT>
__global__ void __launch_bounds__(NT, 1)
    k_gemm_tma(const __grid_constant__ GemmParams P, const __grid_constant__ TmaMaps M) {
    extern __shared__ std::uint8_t smem_raw[];
    // 1024-B alignment for the swizzled boxes
    const std::uint32_t base = tc::smem_u32(smem_raw);
    Smem<BN>& S = *reinterpret_cast<Smem<BN>*>(smem_raw + ((1024 - (base & 1023)) & 1023));
    constexpr std::uint32_t TCOLS = BN == 32 ? 128 : 256;
    constexpr int NF = Depth<BN>::NF, NLIMB = Depth<BN>::NLIMB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = SPLIT > 1 ? static_cast<int>(blockIdx.x) : 0;
    const int prod = static_cast<int>(blockIdx.z / P.tiles_m);
    const std::uint32_t i0 = (blockIdx.z % P.tiles_m) * BM;
    const std::uint32_t j0 = blockIdx.y * BN;
    const std::uint32_t klen = P.k / SPLIT;
    const std::uint32_t kbeg = ks * klen;
    const std::uint32_t nk = klen / KC;
    const bool a16 = P.a[prod].fmt == 1, b16 = P.b[prod].fmt == 1;
    const GemmSrc Cd = P.c[prod];
    const bool out16 = Cd.fmt == 1;

    if (tid == 64) WM_STAMP(0);
    if (warp == 0) tc::tmem_alloc(&S.tmem_base, TCOLS);
    if (tid == 32) {
        for (int s = 0; s < NF; ++s) {
            tc::mbar_init(&S.full[s], 1);
            tc::mbar_init(&S.empty[s], NCONV / 32);
        }
        for (int s = 0; s < NLIMB; ++s) {
            tc::mbar_init(&S.lfull[s], NCONV / 32);
            tc::mbar_init(&S.lempty[s], 1);
        }
        tc::mbar_init(&S.done, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const std::uint32_t tbase = S.tmem_base;
    if (tid == 64) WM_STAMP(1);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_C();
    if (tid == 64) WM_STAMP(2);

    if (warp == 0) {
        if (lane == 0) {
            const CUtensorMap* ma = &M.a[prod];
            const CUtensorMap* mb = &M.b[prod];
            const std::uint32_t bytes = BM * KC * (a16 ? 2 : 8) + KC * BN * (b16 ? 2 : 8);
            for (std::uint32_t kc = 0; kc < nk; ++kc) {
                const int st = kc % NF;
                if (kc >= static_cast<std::uint32_t>(NF))
                    tc::mbar_wait(&S.empty[st], ((kc / NF) - 1) & 1);
                tc::mbar_arrive_expect_tx(&S.full[st], bytes);
                const int k0 = static_cast<int>(kbeg + kc * KC);
                if (a16) {
                    tma_load_2d(S.a[st], ma, k0, static_cast<int>(i0), &S.full[st]);
                } else {
                    tma_load_2d(S.a[st], ma, k0, static_cast<int>(i0), &S.full[st]);
                    tma_load_2d(S.a[st] + BM * 128, ma, k0 + 16, static_cast<int>(i0), &S.full[st]);
                }
                tma_load_2d(S.b[st], mb, static_cast<int>(j0), k0, &S.full[st]);
            }
        }
    } else if (warp == 1) {
        constexpr std::uint32_t idesc = tc::idesc_i8(BM, BN);
        for (std::uint32_t kc = 0; kc < nk; ++kc) {
            const int ls = kc % NLIMB;
            tc::mbar_wait(&S.lfull[ls], (kc / NLIMB) & 1);
            tc::fence_after();
            if (lane == 0 && kc == 4) WM_STAMP(15);
            if (lane == 0) {
                const std::uint64_t ah = tc::smem_desc(tc::smem_u32(S.a_hi[ls]), 128, 256);
                const std::uint64_t al = tc::smem_desc(tc::smem_u32(S.a_lo[ls]), 128, 256);
                const std::uint64_t bh = tc::smem_desc(tc::smem_u32(S.b_hi[ls]), 128, 256);
                const std::uint64_t bl = tc::smem_desc(tc::smem_u32(S.b_lo[ls]), 128, 256);
                const bool acc = kc > 0;
                tc::mma_i8(tbase + 0, ah, bh, idesc, acc);
                tc::mma_i8(tbase + BN, ah, bl, idesc, acc);
                tc::mma_i8(tbase + BN, al, bh, idesc, true);
                tc::mma_i8(tbase + 2 * BN, al, bl, idesc, acc);
                tc::commit(&S.lempty[ls]);
                if (kc + 1 == nk) tc::commit(&S.done);
            }
            __syncwarp();
        }
    } else {
        const int ct = tid - 64;
        for (std::uint32_t kc = 0; kc < nk; ++kc) {
            const int st = kc % NF, ls = kc % NLIMB;
            tc::mbar_wait(&S.full[st], (kc / NF) & 1);
            if (ct == 0 && kc == 0) WM_STAMP(3);
            if (ct == 0 && kc == 2) WM_STAMP(11);
            if (ct == 0 && kc == 5) WM_STAMP(13);
            if (kc >= static_cast<std::uint32_t>(NLIMB))
                tc::mbar_wait(&S.lempty[ls], ((kc / NLIMB) - 1) & 1);
            if (ct == 0 && kc == 2) WM_STAMP(12);
            if (ct == 0 && kc == 5) WM_STAMP(14);
            convert_a(S.a[st], S.a_hi[ls], S.a_lo[ls], ct, a16);
            convert_b<BN>(S.b[st], S.b_hi[ls], S.b_lo[ls], ct, b16);
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&S.lfull[ls]);
                tc::mbar_arrive(&S.empty[st]);
            }
        }
    }

    WM_PDL_LATE_C();
    const double p = P.pd, pinv = P.pinv;
    const double al = static_cast<double>(P.alpha), be = static_cast<double>(P.beta);
    if (tid == 64) WM_STAMP(4);
    if (warp >= 2) {
        tc::mbar_wait(&S.done, 0);
        tc::fence_after();
    }
    if (tid == 64) WM_STAMP(5);
    const int lg = warp & 3, half = (warp - 2) >> 2;
    const std::uint32_t row = lg * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(lg * 32) << 16;

    if (SPLIT == 1) {
        if (warp >= 2) {
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) {
                const std::uint32_t col = half * (BN / 2) + q * 16;
                double out[16];
                tmem_rows16<BN>(tbase + lane_off + col, out, p, pinv);
                if (out16) {
                    std::uint16_t* crow = static_cast<std::uint16_t*>(const_cast<void*>(Cd.p)) +
                                          static_cast<std::uint64_t>(i0 + row) * Cd.ld + j0 + col;
                    std::uint32_t w[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        w[e] = static_cast<std::uint32_t>(out[2 * e]) |
                               (static_cast<std::uint32_t>(out[2 * e + 1]) << 16);
                    reinterpret_cast<uint4*>(crow)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    reinterpret_cast<uint4*>(crow)[1] = make_uint4(w[4], w[5], w[6], w[7]);
                } else {
                    double* crow = static_cast<double*>(const_cast<void*>(Cd.p)) +
                                   static_cast<std::uint64_t>(i0 + row) * Cd.ld + j0 + col;
#pragma unroll
                    for (int e = 0; e < 16; ++e) out[e] *= al;
                    if (P.beta != 0) {
#pragma unroll
                        for (int e = 0; e < 16; e += 2) {
                            const double2 c = *reinterpret_cast<const double2*>(crow + e);
                            out[e] = fma(be, c.x, out[e]);
                            out[e + 1] = fma(be, c.y, out[e + 1]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 16; e += 2)
                        *reinterpret_cast<double2*>(crow + e) =
                            make_double2(reduce_modp(out[e], p, pinv),
                                         reduce_modp(out[e + 1], p, pinv));
                }
            }
        }
    } else {
        std::uint32_t* part = reinterpret_cast<std::uint32_t*>(S.a[0]);  // [BM][BN+1]
        constexpr int PLD = BN + 1;
        if (warp >= 2) {
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) {
                const std::uint32_t col = half * (BN / 2) + q * 16;
                double v[16];
                tmem_rows16<BN>(tbase + lane_off + col, v, p, pinv);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    part[row * PLD + col + e] = static_cast<std::uint32_t>(v[e]);
            }
        }
        cg::cluster_group cluster = cg::this_cluster();
        constexpr int ROWS = BM / SPLIT;
        constexpr int ITER = ROWS * BN / NCONV;
        const int ct = tid - 64;
        double cin[ITER];
        if (warp >= 2 && !out16 && P.beta != 0) {
#pragma unroll
            for (int it = 0; it < ITER; ++it) {
                const int e = it * NCONV + ct;
                const int r = ks * ROWS + e / BN, c = e % BN;
                cin[it] = static_cast<const double*>(Cd.p)[static_cast<std::uint64_t>(i0 + r) * Cd.ld +
                                                           j0 + c];
            }
        }
        if (tid == 64) WM_STAMP(6);
        cluster.sync();
        if (tid == 64) WM_STAMP(7);
        if (warp >= 2) {
            const std::uint32_t* src[SPLIT];
#pragma unroll
            for (int s = 0; s < SPLIT; ++s) src[s] = cluster.map_shared_rank(part, s);
            std::uint32_t pv[ITER][SPLIT];
#pragma unroll
            for (int it = 0; it < ITER; ++it) {
                const int e = it * NCONV + ct;
                const int r = ks * ROWS + e / BN, c = e % BN;
#pragma unroll
                for (int s = 0; s < SPLIT; ++s) pv[it][s] = src[s][r * PLD + c];
            }
#pragma unroll
            for (int it = 0; it < ITER; ++it) {
                const int e = it * NCONV + ct;
                const int r = ks * ROWS + e / BN, c = e % BN;
                double v = 0.0;
#pragma unroll
                for (int s = 0; s < SPLIT; ++s) v += static_cast<double>(pv[it][s]);
                v = reduce_modp(v, p, pinv);
                const std::uint64_t off = static_cast<std::uint64_t>(i0 + r) * Cd.ld + j0 + c;
                if (out16) {
                    static_cast<std::uint16_t*>(const_cast<void*>(Cd.p))[off] =
                        static_cast<std::uint16_t>(v);
                } else {
                    v *= al;
                    if (P.beta != 0) v = fma(be, cin[it], v);
                    static_cast<double*>(const_cast<void*>(Cd.p))[off] = reduce_modp(v, p, pinv);
                }
            }
        }
        if (tid == 64) WM_STAMP(8);
        cluster.sync();
    }
    if (tid == 64) WM_STAMP(9);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, TCOLS);
    if (tid == 64) WM_STAMP(10);
}

template <int BN>
constexpr std::size_t smem_bytes() {
    return sizeof(Smem<BN>) + 1024;
}

template <int BN, int SPLIT>
cudaError_t set_attr() {
    return cudaFuncSetAttribute(k_gemm_tma<BN, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem_bytes<BN>()));
}

template <int BN, int SPLIT>
cudaError_t launch_cfg(const GemmParams& P, const TmaMaps& M, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SPLIT, P.n / BN, P.tiles_m * P.nprod);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem_bytes<BN>();
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
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
    return cudaLaunchKernelEx(&cfg, k_gemm_tma<BN, SPLIT>, P, M);
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool encode(CUtensorMap* map, const GemmSrc& src, std::uint64_t cols, std::uint64_t rows,
            std::uint32_t box_c, std::uint32_t box_r, CUtensorMapSwizzle sw) {
    const CUtensorMapDataType dt =
        src.fmt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    const std::uint64_t esz = src.fmt == 1 ? 2 : 8;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {src.ld * esz};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    return g_encode(map, dt, 2, const_cast<void*>(src.p), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t gemm_tma_init() {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return e != cudaSuccess ? e : cudaErrorNotSupported;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cudaError_t e;
    if ((e = set_attr<64, 1>()) != cudaSuccess) return e;
    if ((e = set_attr<64, 2>()) != cudaSuccess) return e;
    if ((e = set_attr<64, 4>()) != cudaSuccess) return e;
    if ((e = set_attr<32, 1>()) != cudaSuccess) return e;
    if ((e = set_attr<32, 2>()) != cudaSuccess) return e;
    return set_attr<32, 4>();
}

// Encode the per-product operand maps (A: box 16 doubles / 32 uint16 x 128 rows,
// 128-B / 64-B swizzle; B: box BN x 32 rows, no swizzle).
bool gemm_tma_encode(const GemmParams& P, int bn, TmaMaps& M) {
    if (!g_encode) return false;
    std::memset(&M, 0, sizeof(M));
    for (std::uint32_t i = 0; i < P.nprod; ++i) {
        const bool a16 = P.a[i].fmt == 1;
        if (!encode(&M.a[i], P.a[i], P.k, P.m, a16 ? 32 : 16, BM,
                    a16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
            return false;
        if (!encode(&M.b[i], P.b[i], P.n, P.k, static_cast<std::uint32_t>(bn), KC,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
            return false;
    }
    return true;
}

cudaError_t launch_gemm_tma(const GemmParams& P, const TmaMaps& M, int bn, int split,
                            cudaStream_t s) {
    if (bn == 64 && split == 1) return launch_cfg<64, 1>(P, M, s);
    if (bn == 64 && split == 2) return launch_cfg<64, 2>(P, M, s);
    if (bn == 64 && split == 4) return launch_cfg<64, 4>(P, M, s);
    if (bn == 32 && split == 1) return launch_cfg<32, 1>(P, M, s);
    if (bn == 32 && split == 2) return launch_cfg<32, 2>(P, M, s);
    if (bn == 32 && split == 4) return launch_cfg<32, 4>(P, M, s);
    return cudaErrorInvalidValue;
}

}  // namespace wm
