// Fused leaf frames.  A Winograd frame whose seven products are classical
// leaves (the bottom level of every recursion) runs as three launches instead
// of ~15-24 additions and 7 leaf products issued one after another:
//
//  prep  S1 = A21+A22, S2 = S1-A11, S3 = A11-A21, S4 = A12-S2 and
//        T1 = B12-B11, T2 = B22-T1, T3 = B22-B12, T4 = T2-B21 (Table 1) as uint16
//        residue planes; for accumulating frames beta*C_in is packed as four
//        uint16 per position into the C11 slots;
//  gemm  the seven products P1 = A11 B11, P2 = A12 B21, P3 = S4 B22,
//        P4 = A22 T4, P5 = S1 T1, P6 = S2 T2, P7 = S3 T3 in ONE int8-limb GEMM
//        launch (wm_i8.cu, blockIdx.z = product), written as uint16 planes;
//  comb  U1 = P1+P2, U2 = P1+P6, U3 = U2+P7, U4 = U2+P5, U5 = U4+P3,
//        U6 = U3-P4, U7 = U3+P5 and C_ij = alpha*U + beta*C_in, float64 out.
//
// No memory beyond the schedule's own: a "host" is a c x c float64 block whose
// rows each hold four uint16 plane rows (8c bytes).  S/T planes live in C
// blocks that are dead until the combine (C11, C12 for plain frames; C12, C21
// once beta*C_in is packed into C11), the P planes in the frame's temporaries
// or -- for ip / ovl / ovr, which have fewer -- in the A21 / B12 blocks their
// contract lets them overwrite.  Every prep / comb thread owns a fixed set of
// float64 slots (it reads them before it overwrites them), so the in-place
// packing is race-free.
#include <cstdint>
#include <type_traits>

#include "wm_launch.h"
#include "wm_frame.h"
#include "wm_frame_dev.cuh"

namespace wm {

int g_prep_rows = 1;     // rows per prep CTA ("prep_rows" option)
unsigned g_comb_block = 128;  // combine CTA size ("comb_block" option)

namespace {

using fdev::rmod;
using fdev::addm;
using fdev::subm;
using fdev::load_operand;
using fdev::store_operand;

// thread (r, q, h), q < c/4, h in {0,1}: plane columns j = 4q + 2h, +1; the
// float64 slots (r, q + k c/4), k = 0..3, of every host / C block are owned by
// the thread pair (q, 0), (q, 1) of one CTA: both read all they need (A, B and
// beta*C_in) before a barrier, then write their halves of the slots.
__global__ void __launch_bounds__(128) k_frame_prep(const FramePrepParams P) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    WM_TL_BEGIN(P.tl);
    const std::uint32_t c4 = P.c / 4;
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    const bool live = idx < static_cast<std::uint64_t>(P.c) * c4 * 2;
    const std::uint64_t pair = idx >> 1, h = idx & 1;
    const std::uint64_t r = live ? pair / c4 : 0, q = live ? pair - r * c4 : 0;
    const std::uint64_t j = 4 * q + 2 * h;
    const double p = P.pd, pinv = P.pinv;

    double av[4][2], bv[4][2];
    double(&a11)[2] = av[0], (&a12)[2] = av[1], (&a21)[2] = av[2], (&a22)[2] = av[3];
    double(&b11)[2] = bv[0], (&b12)[2] = bv[1], (&b21)[2] = bv[2], (&b22)[2] = bv[3];
    double cin[4][2];  // [k][quadrant 2h, 2h+1]
    if (live) {
        load_operand(P.A, P.fold[0], r, j, p, pinv, av);
        load_operand(P.B, P.fold[1], r, j, p, pinv, bv);
        if (P.beta != 0) {
            const double be = static_cast<double>(P.beta);
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    cin[k][e] = rmod(be * P.C.q[2 * h + e][r * P.C.ld + q + k * c4], p, pinv);
        }
    }
    __syncthreads();  // every owned slot has been read before any is overwritten
    if (!live) return;
    store_operand(P.A, P.fold[0], r, j, av);
    store_operand(P.B, P.fold[1], r, j, bv);
    double s[4][2], t[4][2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const double s1 = addm(a21[e], a22[e], p), s2 = subm(s1, a11[e], p);
        s[0][e] = s1;
        s[1][e] = s2;
        s[2][e] = subm(a11[e], a21[e], p);
        s[3][e] = subm(a12[e], s2, p);
        const double t1 = subm(b12[e], b11[e], p), t2 = subm(b22[e], t1, p);
        t[0][e] = t1;
        t[1][e] = t2;
        t[2][e] = subm(b22[e], b12[e], p);
        t[3][e] = subm(t2, b21[e], p);
    }
    // plane values (r, j..j+1) -> 4 bytes at plane + r*pld + j
    auto put = [&](int pl, const double (&v)[2]) {
        if (P.plane[pl])
            *reinterpret_cast<std::uint32_t*>(static_cast<std::uint16_t*>(P.plane[pl]) + r * P.pld[pl] + j) =
                static_cast<std::uint32_t>(v[0]) | (static_cast<std::uint32_t>(v[1]) << 16);
    };
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        put(PL_S1 + k, s[k]);
        put(PL_T1 + k, t[k]);
    }
    put(PL_A11, a11);
    put(PL_A12, a12);
    put(PL_A22, a22);
    put(PL_B11, b11);
    put(PL_B21, b21);
    put(PL_B22, b22);
    if (P.beta != 0) {
        std::uint16_t* c11 = reinterpret_cast<std::uint16_t*>(P.C.q[0]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            *reinterpret_cast<std::uint32_t*>(c11 + 4 * (r * P.C.ld + q + k * c4) + 2 * h) =
                static_cast<std::uint32_t>(cin[k][0]) | (static_cast<std::uint32_t>(cin[k][1]) << 16);
    }
    WM_TL_END(P.tl);
    WM_PDL_LATE_M();
}

// Limb-pair variant for the direct-limb GEMM (wm_direct.cu): one CTA per row r,
// thread t owns columns j = 2t, 2t+1.  A plane row holds the high bytes of its
// residues at [0, c) and the low bytes at [c, 2c); every byte a CTA writes lies
// in row r of its host, and every C_in value of row r is read before the
// CTA's barrier, so the in-place packing stays race-free.
// HOIST (CTAs of up to 256 threads, c <= 256 at one row per CTA): every load of
// the row in flight before the first use (~100 registers); otherwise the
// 64-register form, whose loads sit next to their arithmetic -- at c = 512 the
// grid is 3.5 CTAs of 256 threads per SM and occupancy wins (measured on config
// 4: 19.1 ms of prep against 22.1-24.1 ms for the hoisted form at 64-100 registers).
// EARLY: nothing this prep reads is written by a launch it directly depends on
// (FramePrepParams::early): the loads go out before griddepcontrol.wait.
template <int MAXT, bool HOIST, bool EARLY>
__global__ void __launch_bounds__(MAXT) k_frame_prep_limbs(const FramePrepParams P) {
    // blockDim = rows * c/2: each CTA owns whole rows (reads precede writes per row)
    const std::uint32_t half = P.c / 2;
    const std::uint64_t r = blockIdx.x * (blockDim.x / half) + threadIdx.x / half;
    const std::uint64_t j = 2 * (threadIdx.x % half);
    if (!EARLY) {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        WM_PDL_EARLY_M();
        WM_TL_BEGIN(P.tl);
    }
    typename std::conditional<HOIST, fdev::PrepRegs, fdev::PrepRegsF64>::type R;
    if constexpr (HOIST) {
        fdev::PrepRaw W;
        fdev::prep_limbs_fetch(P, r, j, W);
        if (EARLY) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            WM_PDL_EARLY_M();
            WM_TL_BEGIN(P.tl);
        }
        fdev::prep_limbs_finish(P, W, R);
    } else {
        fdev::prep_limbs_load(P, r, j, R);
        if (EARLY) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            WM_PDL_EARLY_M();
            WM_TL_BEGIN(P.tl);
        }
    }
    __syncthreads();  // row r of every host has been read before any of it is overwritten
    fdev::prep_limbs_store(P, r, j, R);
    WM_TL_END(P.tl);
    WM_PDL_LATE_M();
}

// thread (r, 2 consecutive columns j, j+1) of the quadrant
// EARLY: C_in is not written by a launch this one directly depends on
// (FrameCombParams::early): it is read before griddepcontrol.wait.
template <bool EARLY>
__global__ void __launch_bounds__(256) k_frame_comb(const FrameCombParams P) {
    // the position is worked out ahead of the wait in both variants
    const std::uint32_t c2 = P.c / 2;
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    const bool live = idx < static_cast<std::uint64_t>(P.c) * c2;
    const std::uint64_t r = live ? idx / c2 : 0, j = live ? 2 * (idx - r * c2) : 0;
    if (!EARLY) {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        WM_PDL_EARLY_M();
        WM_TL_BEGIN(P.tl);
    }
    fdev::CombCin cin;
    if (live) fdev::comb_cin_fetch<false>(P, r, j, cin);
    if (EARLY) {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        WM_PDL_EARLY_M();
        WM_TL_BEGIN(P.tl);
    }
    if (live) fdev::comb_pair<false>(P, r, j, cin);
    WM_TL_END(P.tl);
    WM_PDL_LATE_M();
}

template <class K, class Prm>
cudaError_t launch_pdl(K kern, const Prm& P, std::uint64_t threads, cudaStream_t s,
                       unsigned block = 128) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((threads + block - 1) / block));
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, P);
}

}  // namespace

cudaError_t launch_frame_prep(const FramePrepParams& P, cudaStream_t s) {
    if (P.limbs) {
        if (P.c > 2048) return cudaErrorInvalidValue;
        const unsigned rows = static_cast<unsigned>(g_prep_rows > 0 && P.c / 2 * g_prep_rows <= 1024
                                                         ? g_prep_rows : 1);
        const std::uint64_t n = static_cast<std::uint64_t>(P.c) * (P.c / 2);
        if (rows * (P.c / 2) <= 128)
            return P.early ? launch_pdl(k_frame_prep_limbs<256, true, true>, P, n, s, rows * (P.c / 2))
                           : launch_pdl(k_frame_prep_limbs<256, true, false>, P, n, s, rows * (P.c / 2));
        return P.early ? launch_pdl(k_frame_prep_limbs<1024, false, true>, P, n, s, rows * (P.c / 2))
                       : launch_pdl(k_frame_prep_limbs<1024, false, false>, P, n, s, rows * (P.c / 2));
    }
    return launch_pdl(k_frame_prep, P, static_cast<std::uint64_t>(P.c) * (P.c / 2), s);
}

cudaError_t launch_frame_comb(const FrameCombParams& P, cudaStream_t s) {
    const std::uint64_t n = static_cast<std::uint64_t>(P.c) * (P.c / 2);
    return P.early ? launch_pdl(k_frame_comb<true>, P, n, s, g_comb_block)
                   : launch_pdl(k_frame_comb<false>, P, n, s, g_comb_block);
}

bool frame_kernel_available() { return true; }

}  // namespace wm
