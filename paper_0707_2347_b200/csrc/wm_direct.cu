// Direct-limb product kernel of the fused leaf frames.
//
// The frame prep kernel (wm_frame.cu) writes every GEMM operand as a pair of
// byte planes -- the high and low 8-bit limbs of the residues, a = 256 a_h + a_l
// -- side by side in one row of its host block (hi bytes [0, c), lo bytes
// [c, 2c)).  That is exactly the form the tensor cores consume, so this kernel
// has no conversion stage at all:
//
//   * one elected thread streams 128-deep K stages with TWO tensor-map TMA loads
//     per stage: A as a 3-D box {128 K bytes, 128 rows, 2 limbs} in 128-B swizzle
//     (the canonical K-major SW128 UMMA layout) and B as {BN bytes, 128 K rows,
//     2 limbs} in BN-byte swizzle (the canonical MN-major layout, so B needs no
//     transpose);
//   * one thread issues the 4 K-steps x 4 limb MMAs of a stage
//     (tcgen05.mma kind::i8 into the hh / cross / ll TMEM accumulators, the
//     arithmetic contract of wm_i8.cu) and commits them to the stage's "empty"
//     barrier;
//   * four warps read the accumulators back, recombine 2^16 hh + 2^8 x + ll
//     exactly in float64, reduce mod p and store uint16 product planes.
//
// Stage size is what matters on this part: a TMA load costs ~0.3 us of latency
// per ring slot almost independently of its size (scripts/tma_probe.cu), so the
// ring carries 40-48 KB stages rather than 10 KB ones.
//
// A product whose B operand could not be given a plane (the B22 block of an
// accumulating frame with only two temporaries) is read as float64 residues by
// the four epilogue warps, which split it into the same swizzled limb layout
// while the TMA brings A.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>

#include "wm_frame.h"
#include "wm_frame_dev.cuh"
#include "wm_launch.h"
#include "wm_gemm.h"
#include "wm_tc.h"

namespace wm {
namespace {

constexpr int BM = 128, KT = 128;
// A tiles are K-major with a KT-byte swizzle span (SW64 for KT = 64)
constexpr std::uint64_t A_LAYOUT = KT == 128 ? 2 : 4;  // UMMA SWIZZLE_128B / SWIZZLE_64B
constexpr int NEPI = 256;           // eight epilogue / B-loader warps
constexpr int NT = 64 + NEPI;      // + TMA producer warp + MMA warp
constexpr int A_PART = BM * KT;  // 16 KB per limb

template <int BN>
struct DCfg {
    static constexpr int B_PART = KT * BN;
    static constexpr int STAGE = 2 * A_PART + 2 * B_PART;  // 20 KB (BN 32) / 24 KB (BN 64)
    static constexpr std::uint32_t TCOLS = BN == 32 ? 128 : BN == 64 ? 256 : 512;  // 4 BN columns
    static constexpr int NS = BN == 128 ? 3 : 4;  // stage ring depth (<= ~200 KB)
    // UMMA layout type of the MN-major B tile (swizzle span = BN bytes)
    static constexpr std::uint64_t B_LAYOUT = BN == 32 ? 6 : BN == 64 ? 4 : 2;  // SW32 / SW64 / SW128
};

template <int BN>
struct DSmem {
    std::uint8_t stage[DCfg<BN>::NS][DCfg<BN>::STAGE];  // 1024-B aligned
    std::uint64_t full[DCfg<BN>::NS], empty[DCfg<BN>::NS];
    std::uint64_t done;
    std::uint32_t tmem_base;
};

// swizzled shared-memory descriptor: start, LBO, SBO (bytes), layout type
__device__ __forceinline__ std::uint64_t sdesc(std::uint32_t saddr, std::uint32_t lbo,
                                               std::uint32_t sbo, std::uint64_t layout) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    d |= layout << 61;
    return d;
}

// kind::i8, D s32, A/B u8, A K-major, B MN-major
__host__ __device__ constexpr std::uint32_t idesc_direct(int M, int N) {
    return (2u << 4) | (1u << 16) | (static_cast<std::uint32_t>(N >> 3) << 17) |
           (static_cast<std::uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            std::uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(z),
        "r"(tc::smem_u32(mbar))
        : "memory");
}

// byte offset of B element (k, n) in a BN-byte-swizzled MN-major limb tile
template <int BN>
__device__ __forceinline__ std::uint32_t boff(std::uint32_t k, std::uint32_t n) {
    constexpr std::uint32_t mask = BN == 32 ? 1u : BN == 64 ? 3u : 7u;
    constexpr std::uint32_t sh = BN == 32 ? 2u : BN == 64 ? 1u : 0u;
    return k * BN + ((((n >> 4) ^ (k >> sh)) & mask) << 4) + (n & 15u);
}

// 16 accumulator columns of one TMEM lane: D_h = A_h [B_h | B_l] at [0, 2BN),
// D_l = A_l [B_h | B_l] at [2BN, 4BN); v = 2^16 hh + 2^8 (hl + lh) + ll < 2^48
// (each accumulator <= k 255^2 < 2^31 for k <= 32768, so hl + lh fits 32 bits).
// The residue r = v - q p uses q = rint(v / p) from a magic-constant FMA and one
// integer sign fix: four float64 operations per element and no I2F / F2I /
// FRND.  Measured (c = 512, BN = 128): TMEM read-back ~0.9 us, the float64
// reduction ~0.9 us, not overlapped within a warp.
template <int BN>
__device__ __forceinline__ void tmem_cols16(std::uint32_t taddr, std::uint32_t (&out)[16], double p,
                                            double pinv, std::uint32_t pi) {
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: rint via addition
    std::uint32_t hh[16], hl[16], lh[16], ll[16];
    tc::tmem_ld16(taddr, hh);
    tc::tmem_ld16(taddr + BN, hl);
    tc::tmem_ld16(taddr + 2 * BN, lh);
    tc::tmem_ld16(taddr + 3 * BN, ll);
    tc::tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        // v < 2^48 assembled in integer registers; its bits OR'ed under the
        // exponent of 1.5 * 2^52 give d = v + 1.5 * 2^52 exactly (no conversion)
        const std::uint64_t v = (static_cast<std::uint64_t>(hh[e]) << 16) +
                                (static_cast<std::uint64_t>(hl[e] + lh[e]) << 8) + ll[e];
        const double d = __hiloint2double(0x43380000 | static_cast<int>(v >> 32),
                                          static_cast<int>(v & 0xFFFFFFFFu));
        const double q = fma(d - kMagic, pinv, kMagic) - kMagic;  // rint(v / p) (+-1)
        // d - q p = 1.5 * 2^52 + r exactly, |r| <= p/2 + 1: the low word is r
        // in two's complement; the sign fix runs on the integer pipe
        int r = __double2loint(fma(-q, p, d));
        r += r < 0 ? static_cast<int>(pi) : 0;
        out[e] = static_cast<std::uint32_t>(r);
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// diagnostics: phase timestamps of one thread per CTA (P.trace, 16 slots per CTA)
#define WM_DSTAMP(slot)                                                                        \
    do {                                                                                       \
        if (P.trace) P.trace[(blockIdx.y + gridDim.y * blockIdx.z) * 16 + (slot)] = gtimer(); \
    } while (0)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_arrive(std::uint64_t* mbar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(tc::smem_u32(mbar))
                 : "memory");
}

// The four roles of one output tile (product `prod`, rows i0.., columns j0..):
// TMA producer (warp 0), MMA issuer (warp 1), B loaders / converters and the
// epilogue (warps 2..9).  Barriers and TMEM are set up by the caller.
template <int BN, int BSRC>
__device__ __forceinline__ void direct_tile(const GemmParams& P, const TmaMaps& M, DSmem<BN>& S,
                                            std::uint32_t tbase, int prod, std::uint32_t i0,
                                            std::uint32_t j0, bool pdl_late) {
    using C = DCfg<BN>;
    constexpr int NS = C::NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const std::uint32_t nk = P.k / KT;
    const bool bconv = P.b[prod].fmt == 0;  // float64 B: split by the epilogue warps
    const bool blsu = !bconv && BSRC == 1;
    const GemmSrc Cd = P.c[prod];
    if (warp == 0) {
        if (lane == 0) {
            const bool btma = !bconv && !blsu;
            const std::uint32_t bytes = 2 * A_PART + (btma ? 2 * C::B_PART : 0);
            for (std::uint32_t kc = 0; kc < nk; ++kc) {
                const int st = kc % NS;
                if (kc >= static_cast<std::uint32_t>(NS))
                    tc::mbar_wait(&S.empty[st], ((kc / NS) - 1) & 1);
                tc::mbar_arrive_expect_tx(&S.full[st], bytes);
                const int k0 = static_cast<int>(kc * KT);
                tma_load_3d(S.stage[st], &M.a[prod], k0, static_cast<int>(i0), 0, &S.full[st]);
                if (btma)
                    tma_load_3d(S.stage[st] + 2 * A_PART, &M.b[prod], static_cast<int>(j0), k0, 0,
                                &S.full[st]);
            }
        }
    } else if (warp == 1) {
        // N = 2 BN: the two B limb tiles are adjacent MN atoms (LBO = B_PART)
        constexpr std::uint32_t idesc = idesc_direct(BM, 2 * BN);
        for (std::uint32_t kc = 0; kc < nk; ++kc) {
            const int st = kc % NS;
            tc::mbar_wait(&S.full[st], (kc / NS) & 1);
            tc::fence_after();
            tc::fence_proxy_async();  // cp.async / st.shared limb tiles -> tensor core
            if (lane == 0 && kc == 0) WM_DSTAMP(3);
            if (lane == 0 && kc + 1 == nk) WM_DSTAMP(4);
            if (lane == 0) {
                const std::uint32_t sa = tc::smem_u32(S.stage[st]);
                const std::uint32_t sb = sa + 2 * A_PART;
#pragma unroll
                for (int s = 0; s < KT / 32; ++s) {
                    // A: K-major, KT-byte swizzle; K step = 32 bytes inside the swizzled row
                    const std::uint64_t ah = sdesc(sa + s * 32, 16, 8 * KT, A_LAYOUT);
                    const std::uint64_t al = sdesc(sa + A_PART + s * 32, 16, 8 * KT, A_LAYOUT);
                    // B: MN-major, BN-byte swizzle, K step = 32 rows
                    const std::uint64_t b = sdesc(sb + s * 32 * BN, C::B_PART, 8 * BN, C::B_LAYOUT);
                    const bool acc = kc > 0 || s > 0;
                    tc::mma_i8(tbase + 0, ah, b, idesc, acc);
                    tc::mma_i8(tbase + 2 * BN, al, b, idesc, acc);
                }
                tc::commit(&S.empty[st]);
                if (kc + 1 == nk) tc::commit(&S.done);
            }
            __syncwarp();
        }
    } else if (blsu) {
        const int ct = tid - 64;
        const std::uint8_t* bsrc = static_cast<const std::uint8_t*>(P.b[prod].p);
        const std::uint64_t pitch = P.b[prod].ld, part = P.b[prod].part;
        constexpr int CPR = BN / 16;                     // 16-B chunks per limb row
        constexpr int PER = 2 * KT * CPR / NEPI;         // chunks per thread per stage
        for (std::uint32_t kc = 0; kc < nk; ++kc) {
            const int st = kc % NS;
            if (kc >= static_cast<std::uint32_t>(NS)) tc::mbar_wait(&S.empty[st], ((kc / NS) - 1) & 1);
            std::uint8_t* bt = S.stage[st] + 2 * A_PART;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int q = e * NEPI + ct;
                const int limb = q / (KT * CPR), rem = q % (KT * CPR);
                const std::uint32_t k = rem / CPR, nc = rem % CPR;
                cp_async16(bt + limb * C::B_PART + boff<BN>(k, nc * 16),
                           bsrc + static_cast<std::uint64_t>(kc * KT + k) * pitch + limb * part + j0 + nc * 16);
            }
            cp_async_arrive(&S.full[st]);
        }
    } else if (bconv) {
        // float64 B rows [k0, k0 + 128) x [j0, j0 + BN) -> swizzled limb tiles
        const int ct = tid - 64;
        const double* bsrc = static_cast<const double*>(P.b[prod].p);
        const std::uint64_t ldb = P.b[prod].ld;
        for (std::uint32_t kc = 0; kc < nk; ++kc) {
            const int st = kc % NS;
            if (kc >= static_cast<std::uint32_t>(NS)) tc::mbar_wait(&S.empty[st], ((kc / NS) - 1) & 1);
            std::uint8_t* bh = S.stage[st] + 2 * A_PART;
            std::uint8_t* bl = bh + C::B_PART;
            constexpr int PER = KT * BN / NEPI;
            constexpr int RSTEP = NEPI / BN;
            const std::uint32_t n = ct % BN;
#pragma unroll 8
            for (int e = 0; e < PER; ++e) {
                const std::uint32_t k = ct / BN + e * RSTEP;
                const std::uint32_t v = __double2uint_rz(
                    bsrc[static_cast<std::uint64_t>(kc * KT + k) * ldb + j0 + n]);
                const std::uint32_t o = boff<BN>(k, n);
                bh[o] = static_cast<std::uint8_t>(v >> 8);
                bl[o] = static_cast<std::uint8_t>(v & 255u);
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&S.full[st]);
        }
    }

    if (pdl_late) WM_PDL_LATE_C();
    const double p = P.pd, pinv = P.pinv;
    if (warp >= 2) {
        tc::mbar_wait(&S.done, 0);
        tc::fence_after();
        if (tid == 64) WM_DSTAMP(5);
        // eight warps: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
        const int lg = warp & 3, half = (warp - 2) >> 2;
        const std::uint32_t row = lg * 32 + lane;
        const std::uint32_t lane_off = static_cast<std::uint32_t>(lg * 32) << 16;
        std::uint16_t* crow = static_cast<std::uint16_t*>(const_cast<void*>(Cd.p)) +
                              static_cast<std::uint64_t>(i0 + row) * Cd.ld + j0 + half * (BN / 2);
        const bool wide = (reinterpret_cast<std::uintptr_t>(Cd.p) & 31u) == 0 && Cd.ld % 16 == 0;
#pragma unroll
        for (int q = 0; q < BN / 32; ++q) {
            std::uint32_t out[16];
            tmem_cols16<BN>(tbase + lane_off + half * (BN / 2) + q * 16, out, p, pinv,
                            static_cast<std::uint32_t>(p));
            std::uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = out[2 * e] | (out[2 * e + 1] << 16);
            if (wide) {
                // the thread's sixteen residues are one 32-byte sector: one 256-bit store
                // (two 16-byte stores to different rows per warp instruction wrote every
                // sector twice: ncu's 50% excessive store sectors)
                asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"l"(crow + q * 16),
                             "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]),
                             "r"(w[6]), "r"(w[7])
                             : "memory");
            } else {
                reinterpret_cast<uint4*>(crow + q * 16)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                reinterpret_cast<uint4*>(crow + q * 16)[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
        }
        if (tid == 64) WM_DSTAMP(6);
    }
}

// BSRC: how B limb tiles reach shared memory when B is a plane pair --
// 0 tensor-map TMA (with A), 1 16-B cp.async by the eight epilogue warps
template <int BN, int BSRC>
__global__ void __launch_bounds__(NT, 1)
    k_gemm_direct(const __grid_constant__ GemmParams P, const __grid_constant__ TmaMaps M) {
    using C = DCfg<BN>;
    constexpr int NS = C::NS;
    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t base = tc::smem_u32(smem_raw);
    DSmem<BN>& S = *reinterpret_cast<DSmem<BN>*>(smem_raw + ((1024 - (base & 1023)) & 1023));
    const int tid = threadIdx.x, warp = tid >> 5;
    const int prod = static_cast<int>(blockIdx.z / P.tiles_m);
    const std::uint32_t i0 = (blockIdx.z % P.tiles_m) * BM;
    const std::uint32_t j0 = blockIdx.y * BN;
    const bool bconv = P.b[prod].fmt == 0;  // float64 B: split by the epilogue warps
    const bool blsu = !bconv && BSRC == 1;

    if (tid == 32) WM_DSTAMP(0);
    if (warp == 0) tc::tmem_alloc(&S.tmem_base, C::TCOLS);
    if (tid == 32) {
        for (int s = 0; s < NS; ++s) {
            tc::mbar_init(&S.full[s], bconv ? 1 + NEPI / 32 : (blsu ? 1 + NEPI : 1));
            tc::mbar_init(&S.empty[s], 1);
        }
        tc::mbar_init(&S.done, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const std::uint32_t tbase = S.tmem_base;
    if (tid == 32) WM_DSTAMP(1);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_C();
    WM_TL_BEGIN(P.tl);
    if (tid == 32) WM_DSTAMP(2);

    direct_tile<BN, BSRC>(P, M, S, tbase, prod, i0, j0, true);

    tc::fence_before();
    __syncthreads();
    WM_TL_END(P.tl);
    if (warp == 0) tc::tmem_dealloc(tbase, C::TCOLS);
    if (tid == 32) WM_DSTAMP(7);
}

template <int BN>
constexpr std::size_t dsmem_bytes() {
    static_assert(sizeof(DSmem<BN>) + 1024 <= 232448, "shared memory budget");
    return sizeof(DSmem<BN>) + 1024;
}

template <int BN, int BSRC>
cudaError_t dset_attr() {
    return cudaFuncSetAttribute(k_gemm_direct<BN, BSRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(dsmem_bytes<BN>()));
}

template <int BN, int BSRC>
cudaError_t dlaunch(const GemmParams& P, const TmaMaps& M, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, P.n / BN, P.tiles_m * P.nprod);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = dsmem_bytes<BN>();
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_gemm_direct<BN, BSRC>, P, M);
}

PFN_cuTensorMapEncodeTiled_v12000 g_denc = nullptr;

// 3-D byte map over a limb-plane pair: {cols, rows, 2 limbs}; box_l limbs per box
bool encode_planes(CUtensorMap* map, const GemmSrc& src, std::uint64_t cols, std::uint64_t rows,
                   std::uint32_t box_c, std::uint32_t box_r, CUtensorMapSwizzle sw) {
    const std::uint32_t box_l = 2;
    cuuint64_t dims[3] = {cols, rows, 2};
    cuuint64_t strides[2] = {src.ld, src.part};
    cuuint32_t box[3] = {box_c, box_r, box_l};
    cuuint32_t es[3] = {1, 1, 1};
    return g_denc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(src.p), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool g_direct_ok = false;

}  // namespace

cudaError_t gemm_direct_init() {
    if (!g_denc) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return e != cudaSuccess ? e : cudaErrorNotSupported;
        g_denc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cudaError_t e;
    if ((e = dset_attr<32, 0>()) != cudaSuccess) return e;
    if ((e = dset_attr<64, 0>()) != cudaSuccess) return e;
    if ((e = dset_attr<128, 0>()) != cudaSuccess) return e;
    if ((e = dset_attr<32, 1>()) != cudaSuccess) return e;
    if ((e = dset_attr<64, 1>()) != cudaSuccess) return e;
    g_direct_ok = true;
    return cudaSuccess;
}

bool gemm_direct_supported(const GemmParams& P, int bn) {
    const bool lsu = bn >= 1000;
    bn %= 1000;
    if (!g_direct_ok || (bn != 32 && bn != 64 && bn != 128) || (lsu && bn == 128)) return false;
    if (P.m % BM || P.n % bn || P.k % KT || P.k > 32768 || P.nprod < 1 || P.nprod > kMaxProducts)
        return false;
    for (std::uint32_t i = 0; i < P.nprod; ++i) {
        if (P.a[i].fmt != 2 || P.c[i].fmt != 1) return false;
        if (P.b[i].fmt != 2 && P.b[i].fmt != 0) return false;
    }
    return true;
}

bool gemm_direct_encode(const GemmParams& P, int bn, TmaMaps& M) {
    bn %= 1000;
    if (!g_denc) return false;
    std::memset(&M, 0, sizeof(M));
    const CUtensorMapSwizzle bsw = bn == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                   : bn == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
    for (std::uint32_t i = 0; i < P.nprod; ++i) {
        if (!encode_planes(&M.a[i], P.a[i], P.k, P.m, KT, BM,
                           KT == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
            return false;
        if (P.b[i].fmt == 2 &&
            !encode_planes(&M.b[i], P.b[i], P.n, P.k, static_cast<std::uint32_t>(bn), KT, bsw))
            return false;
    }
    return true;
}

// BN for a direct product set: the narrowest tile that still fits the grid in
// one wave of the 148 SMs (every CTA must receive its whole 128 x K A panel, so
// fewer, wider tiles win once the grid would need a second wave)
int gemm_direct_choose(const GemmParams& P) {
    const std::uint32_t mt = P.tiles_m * P.nprod;
    // a float64 B is streamed at 8 B / element: keep its panels narrow
    bool bconv = false;
    for (std::uint32_t i = 0; i < P.nprod; ++i) bconv |= P.b[i].fmt == 0;
    const int widest = bconv ? 64 : 128;
    for (int bn : {32, 64, 128})
        if (bn <= widest && P.n % bn == 0 && mt * (P.n / bn) <= 148) return bn;
    return P.n % widest == 0 ? widest : P.n % 64 == 0 ? 64 : 32;
}

// bn: 32 / 64; + 1000 selects cp.async B loads instead of TMA
cudaError_t launch_gemm_direct(const GemmParams& P, const TmaMaps& M, int bn, cudaStream_t s) {
    switch (bn) {
        case 32: return dlaunch<32, 0>(P, M, s);
        case 64: return dlaunch<64, 0>(P, M, s);
        case 128: return dlaunch<128, 0>(P, M, s);
        case 1032: return dlaunch<32, 1>(P, M, s);
        case 1064: return dlaunch<64, 1>(P, M, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace wm
