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
// Tiling: 128 x 64 output tile per CTA (UMMA M=128, N=64), K in chunks of 32
// (one MMA per limb product per chunk).  256 threads stream the float64
// operand chunk of step k+1 into registers (coalesced 16-B loads) while step k
// is converted to limbs and written to shared memory in the canonical K-major
// no-swizzle layout; one elected thread issues the four MMAs and commits them
// to the stage's mbarrier, so limb conversion overlaps the tensor pipe.  Two
// CTAs fit per SM (24 KB shared memory, 256 TMEM columns each).
#include <cstdint>

#include "wm_device.h"
#include "wm_tc.h"

namespace wm {
namespace {

constexpr int BM = 128, BN = 64, KC = 32, NT = 256, NSTAGE = 2;
constexpr int A_TILE = BM * KC;  // bytes per limb tile
constexpr int B_TILE = BN * KC;
constexpr std::uint32_t TMEM_COLS = 256;  // D_hh @0, D_x @64, D_ll @128

struct __align__(128) Stage {
    std::uint8_t a_hi[A_TILE];
    std::uint8_t a_lo[A_TILE];
    std::uint8_t b_hi[B_TILE];
    std::uint8_t b_lo[B_TILE];
};

// canonical K-major no-swizzle offset of (row r, k c) in a tile 32 bytes wide
__device__ __forceinline__ std::uint32_t koff(std::uint32_t r, std::uint32_t c) {
    return (r & 7u) * 16u + (r >> 3) * 256u + (c >> 4) * 128u + (c & 15u);
}

__device__ __forceinline__ double reduce_modp(double v, double p, double pinv) {
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

struct Regs {
    double2 a[8];  // 8 x 16 B of the A chunk
    double2 b[4];  // 4 x 16 B of the B chunk
};

__device__ __forceinline__ void load_chunk(Regs& R, const MulParams& P, std::uint64_t i0,
                                           std::uint64_t j0, std::uint32_t k0, int tid) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int u = j * NT + tid;
        const int r = u >> 4, c = (u & 15) * 2;
        R.a[j] = __ldg(reinterpret_cast<const double2*>(P.A + (i0 + r) * P.lda + k0 + c));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int u = j * NT + tid;
        const int kk = u >> 5, c = (u & 31) * 2;
        R.b[j] = __ldg(reinterpret_cast<const double2*>(P.B + (k0 + kk) * P.ldb + j0 + c));
    }
}

__device__ __forceinline__ void store_chunk(const Regs& R, Stage& S, int tid) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int u = j * NT + tid;
        const int r = u >> 4, c = (u & 15) * 2;
        const std::uint32_t x0 = __double2uint_rz(R.a[j].x), x1 = __double2uint_rz(R.a[j].y);
        const std::uint32_t o = koff(r, c);
        *reinterpret_cast<std::uint16_t*>(S.a_hi + o) =
            static_cast<std::uint16_t>((x0 >> 8) | ((x1 >> 8) << 8));
        *reinterpret_cast<std::uint16_t*>(S.a_lo + o) =
            static_cast<std::uint16_t>((x0 & 255u) | ((x1 & 255u) << 8));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int u = j * NT + tid;
        const int kk = u >> 5, n = (u & 31) * 2;
        const std::uint32_t x0 = __double2uint_rz(R.b[j].x), x1 = __double2uint_rz(R.b[j].y);
        const std::uint32_t o0 = koff(n, kk), o1 = koff(n + 1, kk);
        S.b_hi[o0] = static_cast<std::uint8_t>(x0 >> 8);
        S.b_lo[o0] = static_cast<std::uint8_t>(x0);
        S.b_hi[o1] = static_cast<std::uint8_t>(x1 >> 8);
        S.b_lo[o1] = static_cast<std::uint8_t>(x1);
    }
}

__global__ void __launch_bounds__(NT, 2) k_leaf_i8(const MulParams P) {
    __shared__ Stage st[NSTAGE];
    __shared__ __align__(8) std::uint64_t mbar[NSTAGE];
    __shared__ __align__(8) std::uint64_t mbar_done;
    __shared__ std::uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const std::uint64_t i0 = static_cast<std::uint64_t>(blockIdx.y) * BM;
    const std::uint64_t j0 = static_cast<std::uint64_t>(blockIdx.x) * BN;
    const std::uint32_t nk = P.k / KC;

    if (warp == 0) tc::tmem_alloc(&tmem_base_s, TMEM_COLS);
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) tc::mbar_init(&mbar[s], 1);
        tc::mbar_init(&mbar_done, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const std::uint32_t tbase = tmem_base_s;
    constexpr std::uint32_t idesc = tc::idesc_i8(BM, BN);

    Regs R[2];
    load_chunk(R[0], P, i0, j0, 0, tid);

    auto body = [&](Regs& cur, Regs& nxt, std::uint32_t kc) {
        if (kc + 1 < nk) load_chunk(nxt, P, i0, j0, (kc + 1) * KC, tid);
        const int s = kc % NSTAGE;
        if (kc >= NSTAGE) tc::mbar_wait(&mbar[s], ((kc / NSTAGE) - 1) & 1);
        store_chunk(cur, st[s], tid);
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const std::uint64_t ah = tc::smem_desc(tc::smem_u32(st[s].a_hi), 128, 256);
            const std::uint64_t al = tc::smem_desc(tc::smem_u32(st[s].a_lo), 128, 256);
            const std::uint64_t bh = tc::smem_desc(tc::smem_u32(st[s].b_hi), 128, 256);
            const std::uint64_t bl = tc::smem_desc(tc::smem_u32(st[s].b_lo), 128, 256);
            const bool acc = kc > 0;
            tc::mma_i8(tbase + 0, ah, bh, idesc, acc);
            tc::mma_i8(tbase + 64, ah, bl, idesc, acc);
            tc::mma_i8(tbase + 64, al, bh, idesc, true);
            tc::mma_i8(tbase + 128, al, bl, idesc, acc);
            tc::commit(&mbar[s]);
            if (kc + 1 == nk) tc::commit(&mbar_done);
        }
    };
    std::uint32_t kc = 0;
    for (; kc + 2 <= nk; kc += 2) {
        body(R[0], R[1], kc);
        body(R[1], R[0], kc + 1);
    }
    if (kc < nk) body(R[0], R[1], kc);

    // epilogue: TMEM -> registers -> exact recombination -> C
    tc::mbar_wait(&mbar_done, 0);
    tc::fence_after();
    const int lg = warp & 3, half = warp >> 2;
    const std::uint32_t row = lg * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(lg * 32) << 16;
    const double p = P.pd, pinv = P.pinv;
    const double al = static_cast<double>(P.alpha), be = static_cast<double>(P.beta);
    double* crow = P.C + (i0 + row) * P.ldc + j0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const std::uint32_t col = half * 32 + q * 16;
        std::uint32_t hh[16], xx[16], ll[16];
        tc::tmem_ld16(tbase + lane_off + 0 + col, hh);
        tc::tmem_ld16(tbase + lane_off + 64 + col, xx);
        tc::tmem_ld16(tbase + lane_off + 128 + col, ll);
        tc::tmem_wait_ld();
        double out[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            double v = fma(static_cast<double>(hh[e]), 65536.0,
                           fma(static_cast<double>(xx[e]), 256.0, static_cast<double>(ll[e])));
            v = reduce_modp(v, p, pinv) * al;
            out[e] = v;
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
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, TMEM_COLS);
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool leaf_i8_supported(const MulParams& P) {
    return P.m % BM == 0 && P.n % BN == 0 && P.k % KC == 0 && P.k <= 32768 && P.m > 0 &&
           P.n > 0 && P.k > 0 && P.lda % 2 == 0 && P.ldb % 2 == 0 && P.ldc % 2 == 0 &&
           aligned16(P.A) && aligned16(P.B) && aligned16(P.C) && P.p < 65536u;
}

cudaError_t launch_leaf_i8(const MulParams& P, cudaStream_t s) {
    if (!leaf_i8_supported(P)) return cudaErrorInvalidValue;
    dim3 grid(P.n / BN, P.m / BM);
    k_leaf_i8<<<grid, NT, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace wm
