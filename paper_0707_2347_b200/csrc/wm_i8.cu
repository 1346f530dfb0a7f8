// Leaf products on the 5th-generation tensor cores, exact over Z/pZ (p < 2^16):
//   C <- alpha*A*B + beta*C                  (classical_mul, ring.hpp:315-384)
//
// Each canonical residue a < 2^16 is split into two unsigned 8-bit limbs
// a = 256*a_h + a_l.  The product needs four limb products, issued as
// tcgen05.mma kind::i8 (u8 x u8 -> s32 in TMEM) into three accumulators:
//   D_hh = A_h B_h,   D_x = A_h B_l + A_l B_h,   D_ll = A_l B_l,
// each bounded by 2*k*255^2 < 2^32 for k <= 32768 (read back as u32).  The
// epilogue recombines v = 2^16 D_hh + 2^8 D_x + D_ll < 2^49 exactly in float64,
// reduces mod p, and applies alpha / beta in residue arithmetic.
//
// Operands are float64 residues (the caller's matrices and the schedule's
// temporaries) or uint16 residue planes (the fused frames' S_i / T_i); the
// output is a float64 block (with alpha / beta) or a uint16 plane.  One launch
// can carry several independent products of one shape (blockIdx.z selects the
// product) -- the seven products of a fused Winograd frame.
//
// Pipeline (256 threads, one CTA per SM): every thread streams its share of the
// next K chunks with 16-B cp.async into a 3-4 deep staging ring (up to ~120 KB
// in flight per SM), then all threads split the landed chunk into limb tiles in
// the canonical K-major no-swizzle UMMA layout (conflict-free: padded rows,
// one 16-B store per limb row segment); one thread issues the four MMAs per
// chunk and commits them to the limb stage's mbarrier, so limb conversion of
// chunk k+1 overlaps the tensor pipe on chunk k.  (A warp-specialised variant
// fed by per-row cp.async.bulk copies measured 2-4x slower: the bulk-copy
// engine serialises the 160 small row copies of each chunk.)  Small leaves
// split K over a 2- or 4-CTA cluster; partials (already reduced mod p) are
// summed over DSMEM -- no scratch memory, no extra launch.
// Every kernel waits on griddepcontrol (programmatic dependent launch) before
// touching global memory, so it can be launched while its producer drains.
#include <cooperative_groups.h>

#include <cstdint>

#include "wm_launch.h"
#include "wm_device.h"
#include "wm_gemm.h"
#include "wm_tc.h"

namespace cg = cooperative_groups;

namespace wm {
namespace {

constexpr int BM = 128, KC = 32, NLIMB = 2;
constexpr int NCONV = 256;  // all threads load and convert
constexpr int NT = NCONV;
constexpr int AROW = 34;        // padded float64 A row: 272 B (conflict-free reads)
constexpr int AROW16 = 40;      // padded uint16 A row: 80 B

template <int BN>
struct Cfg {
    static constexpr int NF = BN == 32 ? 4 : 3;    // staging ring depth
    static constexpr int A_BYTES = BM * AROW * 8;  // A stage (float64 worst case)
    static constexpr int B_BYTES = KC * BN * 8;    // B stage
    static constexpr int A_LIMB = BM * KC, B_LIMB = BN * KC;
    static constexpr std::uint32_t TCOLS = BN == 32 ? 128 : 256;
};

template <int BN>
struct Smem {
    std::uint8_t a[Cfg<BN>::NF][Cfg<BN>::A_BYTES];
    std::uint8_t b[Cfg<BN>::NF][Cfg<BN>::B_BYTES];
    std::uint8_t a_hi[NLIMB][Cfg<BN>::A_LIMB];
    std::uint8_t a_lo[NLIMB][Cfg<BN>::A_LIMB];
    std::uint8_t b_hi[NLIMB][Cfg<BN>::B_LIMB];
    std::uint8_t b_lo[NLIMB][Cfg<BN>::B_LIMB];
    std::uint64_t lempty[NLIMB];
    std::uint64_t done;
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

__device__ __forceinline__ void pack4(const std::uint32_t (&x)[4], std::uint32_t& hi,
                                      std::uint32_t& lo) {
    hi = (x[0] >> 8) | ((x[1] >> 8) << 8) | ((x[2] >> 8) << 16) | ((x[3] >> 8) << 24);
    lo = (x[0] & 255u) | ((x[1] & 255u) << 8) | ((x[2] & 255u) << 16) | ((x[3] & 255u) << 24);
}

// A stage -> limb tiles: thread = (row, 16-wide K half)
template <int BN>
__device__ __forceinline__ void convert_a(Smem<BN>& S, int fs, int ls, int ct, bool u16) {
    const int r = ct & 127, h = ct >> 7;
    std::uint32_t hi[4], lo[4];
    if (!u16) {
        const double* src = reinterpret_cast<const double*>(S.a[fs]) + r * AROW + h * 16;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v0 = *reinterpret_cast<const double2*>(src + q * 4);
            const double2 v1 = *reinterpret_cast<const double2*>(src + q * 4 + 2);
            const std::uint32_t x[4] = {__double2uint_rz(v0.x), __double2uint_rz(v0.y),
                                        __double2uint_rz(v1.x), __double2uint_rz(v1.y)};
            pack4(x, hi[q], lo[q]);
        }
    } else {
        const std::uint16_t* src =
            reinterpret_cast<const std::uint16_t*>(S.a[fs]) + r * AROW16 + h * 16;
        const uint4 w0 = *reinterpret_cast<const uint4*>(src);
        const uint4 w1 = *reinterpret_cast<const uint4*>(src + 8);
        const std::uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const std::uint32_t x[4] = {wv[2 * q] & 0xFFFFu, wv[2 * q] >> 16,
                                        wv[2 * q + 1] & 0xFFFFu, wv[2 * q + 1] >> 16};
            pack4(x, hi[q], lo[q]);
        }
    }
    const std::uint32_t o = koff(r, h * 16);
    *reinterpret_cast<uint4*>(&S.a_hi[ls][o]) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(&S.a_lo[ls][o]) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// B stage (k rows x BN) -> K-major limb tiles of B^T: thread = (n, 4 consecutive k)
template <int BN>
__device__ __forceinline__ void convert_b(Smem<BN>& S, int fs, int ls, int ct, bool u16) {
#pragma unroll
    for (int it = 0; it < (KC * BN) / (4 * NCONV); ++it) {
        const int t = it * NCONV + ct;
        const int n = t % BN, kg = t / BN;
        std::uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int kk = kg * 4 + e;
            x[e] = u16 ? static_cast<std::uint32_t>(
                             reinterpret_cast<const std::uint16_t*>(S.b[fs])[kk * BN + n])
                       : __double2uint_rz(reinterpret_cast<const double*>(S.b[fs])[kk * BN + n]);
        }
        std::uint32_t hi, lo;
        pack4(x, hi, lo);
        const std::uint32_t o = koff(n, kg * 4);
        *reinterpret_cast<std::uint32_t*>(&S.b_hi[ls][o]) = hi;
        *reinterpret_cast<std::uint32_t*>(&S.b_lo[ls][o]) = lo;
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

template <int BN, int SPLIT>
__global__ void __launch_bounds__(NT, 1) k_gemm_i8(const GemmParams P) {
    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    Smem<BN>& S = *reinterpret_cast<Smem<BN>*>(smem_raw);
    using CF = Cfg<BN>;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ks = SPLIT > 1 ? static_cast<int>(blockIdx.x) : 0;  // rank in the cluster
    const int prod = static_cast<int>(blockIdx.z / P.tiles_m);
    const std::uint64_t i0 = static_cast<std::uint64_t>(blockIdx.z % P.tiles_m) * BM;
    const std::uint64_t j0 = static_cast<std::uint64_t>(blockIdx.y) * BN;
    const std::uint32_t klen = P.k / SPLIT;
    const std::uint32_t kbeg = ks * klen;
    const std::uint32_t nk = klen / KC;
    const GemmSrc A = P.a[prod], B = P.b[prod], Cd = P.c[prod];
    const bool a16 = A.fmt == 1, b16 = B.fmt == 1, out16 = Cd.fmt == 1;

    if (warp == 0) tc::tmem_alloc(&S.tmem_base, CF::TCOLS);
    if (tid == 32) {
        for (int s = 0; s < NLIMB; ++s) tc::mbar_init(&S.lempty[s], 1);
        tc::mbar_init(&S.done, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const std::uint32_t tbase = S.tmem_base;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_C();

    // 16-B units per chunk: A rows of KC residues, B rows of BN residues
    const int a_upr = a16 ? KC / 8 : KC / 2;   // units per A row
    const int b_upr = b16 ? BN / 8 : BN / 2;   // units per B row
    const int astr = a16 ? AROW16 * 2 : AROW * 8;
    const int esz_a = a16 ? 2 : 8, esz_b = b16 ? 2 : 8;
    const std::uint8_t* abase = static_cast<const std::uint8_t*>(A.p);
    const std::uint8_t* bbase = static_cast<const std::uint8_t*>(B.p);
    auto issue = [&](int st, std::uint32_t k0) {
        const int na = BM * a_upr, nb = KC * b_upr;
        for (int u = tid; u < na; u += NT) {
            const int r = u / a_upr, cu = u - r * a_upr;
            cp16(S.a[st] + r * astr + cu * 16,
                 abase + ((i0 + r) * A.ld + k0) * esz_a + cu * 16);
        }
        for (int u = tid; u < nb; u += NT) {
            const int r = u / b_upr, cu = u - r * b_upr;
            cp16(S.b[st] + r * (b_upr * 16) + cu * 16,
                 bbase + ((k0 + r) * B.ld + j0) * esz_b + cu * 16);
        }
    };
    constexpr int NF = CF::NF;
#pragma unroll
    for (int c = 0; c < NF - 1; ++c) {
        if (c < static_cast<int>(nk)) issue(c, kbeg + c * KC);
        cp_commit();
    }
    constexpr std::uint32_t idesc = tc::idesc_i8(BM, BN);
    for (std::uint32_t kc = 0; kc < nk; ++kc) {
        const std::uint32_t nxt = kc + NF - 1;
        if (nxt < nk) issue(nxt % NF, kbeg + nxt * KC);
        cp_commit();
        cp_wait<NF - 1>();
        const int ls = kc % NLIMB;
        if (kc >= NLIMB) tc::mbar_wait(&S.lempty[ls], ((kc / NLIMB) - 1) & 1);
        __syncthreads();  // chunk kc landed for every thread
        convert_a<BN>(S, kc % NF, ls, tid, a16);
        convert_b<BN>(S, kc % NF, ls, tid, b16);
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
            tc::commit(&S.lempty[ls]);
            if (kc + 1 == nk) tc::commit(&S.done);
        }
    }

    // ---------------- epilogue (converter warps): TMEM -> exact recombination
    WM_PDL_LATE_C();
    const double p = P.pd, pinv = P.pinv;
    const double al = static_cast<double>(P.alpha), be = static_cast<double>(P.beta);
    tc::mbar_wait(&S.done, 0);
    tc::fence_after();
    const int lg = warp & 3, half = warp >> 2;
    const std::uint32_t row = lg * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(lg * 32) << 16;

    if (SPLIT == 1) {
        {
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) {
                const std::uint32_t col = half * (BN / 2) + q * 16;
                double out[16];
                tmem_rows16<BN>(tbase + lane_off + col, out, p, pinv);
                if (out16) {
                    std::uint16_t* crow = static_cast<std::uint16_t*>(const_cast<void*>(Cd.p)) +
                                          (i0 + row) * Cd.ld + j0 + col;
                    std::uint32_t w[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        w[e] = static_cast<std::uint32_t>(out[2 * e]) |
                               (static_cast<std::uint32_t>(out[2 * e + 1]) << 16);
                    reinterpret_cast<uint4*>(crow)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    reinterpret_cast<uint4*>(crow)[1] = make_uint4(w[4], w[5], w[6], w[7]);
                } else {
                    double* crow = static_cast<double*>(const_cast<void*>(Cd.p)) +
                                   (i0 + row) * Cd.ld + j0 + col;
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
                    for (int e = 0; e < 16; e += 2) {
                        double2 o;
                        o.x = reduce_modp(out[e], p, pinv);
                        o.y = reduce_modp(out[e + 1], p, pinv);
                        *reinterpret_cast<double2*>(crow + e) = o;
                    }
                }
            }
        }
    } else {
        // partial (mod p) -> own shared memory (reuses staging stage 0), then the
        // cluster sums the SPLIT partials over DSMEM.
        std::uint32_t* part = reinterpret_cast<std::uint32_t*>(S.a[0]);  // [BM][BN+1]
        constexpr int PLD = BN + 1;
        {
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
        const int ct = tid;
        double cin[ITER];
        if (!out16 && P.beta != 0) {
#pragma unroll
            for (int it = 0; it < ITER; ++it) {
                const int e = it * NCONV + ct;
                const int r = ks * ROWS + e / BN, c = e % BN;
                cin[it] = static_cast<const double*>(Cd.p)[(i0 + r) * Cd.ld + j0 + c];
            }
        }
        cluster.sync();
        {
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
                if (out16) {
                    static_cast<std::uint16_t*>(const_cast<void*>(Cd.p))[(i0 + r) * Cd.ld + j0 + c] =
                        static_cast<std::uint16_t>(v);
                } else {
                    v *= al;
                    if (P.beta != 0) v = fma(be, cin[it], v);
                    static_cast<double*>(const_cast<void*>(Cd.p))[(i0 + r) * Cd.ld + j0 + c] =
                        reduce_modp(v, p, pinv);
                }
            }
        }
        cluster.sync();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, CF::TCOLS);
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

template <int BN, int SPLIT>
cudaError_t set_attr() {
    return cudaFuncSetAttribute(k_gemm_i8<BN, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem<BN>)));
}

template <int BN, int SPLIT>
cudaError_t launch_cfg(const GemmParams& P, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SPLIT, P.n / BN, P.tiles_m * P.nprod);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = sizeof(Smem<BN>);
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
    return cudaLaunchKernelEx(&cfg, k_gemm_i8<BN, SPLIT>, P);
}

cudaError_t dispatch(const GemmParams& P, int bn, int split, cudaStream_t s) {
    if (bn == 64 && split == 1) return launch_cfg<64, 1>(P, s);
    if (bn == 64 && split == 2) return launch_cfg<64, 2>(P, s);
    if (bn == 64 && split == 4) return launch_cfg<64, 4>(P, s);
    if (bn == 32 && split == 1) return launch_cfg<32, 1>(P, s);
    if (bn == 32 && split == 2) return launch_cfg<32, 2>(P, s);
    if (bn == 32 && split == 4) return launch_cfg<32, 4>(P, s);
    return cudaErrorInvalidValue;
}

bool src_ok(const GemmSrc& g) {
    return g.p && aligned16(g.p) && (g.fmt == 1 ? g.ld % 8 == 0 : g.ld % 2 == 0);
}

GemmParams from_mul(const MulParams& P) {
    GemmParams G{};
    G.a[0] = {P.A, P.lda, 0};
    G.b[0] = {P.B, P.ldb, 0};
    G.c[0] = {P.C, P.ldc, 0};
    G.m = P.m;
    G.n = P.n;
    G.k = P.k;
    G.nprod = 1;
    G.tiles_m = P.m / BM;
    G.alpha = P.alpha;
    G.beta = P.beta;
    G.pd = P.pd;
    G.pinv = P.pinv;
    return G;
}

}  // namespace

bool gemm_i8_supported(const GemmParams& P) {
    if (P.m % BM || P.n % 32 || P.k % KC || P.k > 32768 || !P.m || !P.n || !P.k) return false;
    if (P.nprod < 1 || P.nprod > static_cast<std::uint32_t>(kMaxProducts)) return false;
    if (P.tiles_m != P.m / BM) return false;
    for (std::uint32_t i = 0; i < P.nprod; ++i)
        if (!src_ok(P.a[i]) || !src_ok(P.b[i]) || !src_ok(P.c[i])) return false;
    return true;
}

bool leaf_i8_supported(const MulParams& P) {
    return P.p < 65536u && gemm_i8_supported(from_mul(P));
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

// Tile width and K split: aim for >= ~100 CTAs on the 148 SMs; a split needs
// every slice to be a whole number of 32-wide chunks.
void gemm_choose(const GemmParams& P, int* bn, int* split) {
    const std::uint32_t mt = P.tiles_m * P.nprod;
    const std::uint32_t tiles64 = (P.n % 64 == 0) ? mt * (P.n / 64) : 0;
    const std::uint32_t tiles32 = mt * (P.n / 32);
    const bool s2 = P.k % (2 * KC) == 0, s4 = P.k % (4 * KC) == 0;
    *bn = 32;
    *split = 1;
    if (tiles64 >= 96) { *bn = 64; *split = 1; }
    else if (tiles64 >= 48 && s2) { *bn = 64; *split = 2; }
    else if (tiles64 >= 24 && s4) { *bn = 64; *split = 4; }
    else if (tiles32 >= 96) { *split = 1; }
    else if (tiles32 >= 48 && s2) { *split = 2; }
    else if (s4) { *split = 4; }
    else if (s2) { *split = 2; }
}

cudaError_t launch_gemm_i8(const GemmParams& P, cudaStream_t s) {
    if (!gemm_i8_supported(P)) return cudaErrorInvalidValue;
    int bn, split;
    gemm_choose(P, &bn, &split);
    return dispatch(P, bn, split, s);
}

cudaError_t launch_leaf_i8(const MulParams& P, cudaStream_t s) {
    if (!leaf_i8_supported(P)) return cudaErrorInvalidValue;
    return launch_gemm_i8(from_mul(P), s);
}

GemmParams gemm_from_mul(const MulParams& P) { return from_mul(P); }

// measurement hook: force a (BN, SPLIT) configuration
cudaError_t launch_leaf_i8_cfg(const MulParams& P, int bn, int split, cudaStream_t s) {
    if (!leaf_i8_supported(P) || P.n % bn || P.k % (split * KC)) return cudaErrorInvalidValue;
    return dispatch(from_mul(P), bn, split, s);
}

}  // namespace wm
