// Thin inline-PTX helpers for sm_100a: tcgen05 (UMMA / TMEM), mbarrier and
// proxy fences.  Descriptor bit layouts follow the sm_100 UMMA encodings
// (shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), layout [61,64); instruction descriptor for kind::i8:
// D format S32 [4,6), A/B format U8 [7,10)/[10,13), K-major A/B [15]/[16],
// N>>3 [17,23), M>>4 [24,29)).
#pragma once

#include <cstdint>

namespace wm {
namespace tc {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no-swizzle operand tile: core matrices of 8 rows x 16 bytes;
// lbo = byte distance between the two 16-B K halves of one MMA step,
// sbo = byte distance between consecutive 8-row groups.
__device__ __forceinline__ std::uint64_t smem_desc(std::uint32_t saddr, std::uint32_t lbo,
                                                   std::uint32_t sbo) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100)
    return d;         // base offset 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr std::uint32_t idesc_i8(int M, int N) {
    return (2u << 4)                                  // D: s32
           | (0u << 7) | (0u << 10)                   // A, B: u8
           | (0u << 15) | (0u << 16)                  // K-major A and B
           | (static_cast<std::uint32_t>(N >> 3) << 17)
           | (static_cast<std::uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(std::uint32_t tmem_d, std::uint64_t adesc,
                                       std::uint64_t bdesc, std::uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<std::uint32_t>(acc)));
}

__device__ __forceinline__ void commit(std::uint64_t* mbar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void tmem_alloc(std::uint32_t* dst_smem, std::uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(std::uint32_t taddr, std::uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr),
                 "r"(ncols)
                 : "memory");
}

__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_init(std::uint64_t* mbar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ bool mbar_try_wait(std::uint64_t* mbar, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(mbar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// bounded wait: a lost arrival traps (a launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(std::uint64_t* mbar, std::uint32_t parity) {
    std::uint32_t spins = 0;
    while (!mbar_try_wait(mbar, parity))
        if (++spins > (1u << 26)) __trap();
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* mbar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
                 "r"(bytes)
                 : "memory");
}
// bulk global -> shared copy completing `bytes` of transaction on mbar (size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes,
                                         std::uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

}  // namespace tc
}  // namespace wm
