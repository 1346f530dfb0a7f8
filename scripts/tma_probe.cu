// Microbenchmark: per-SM TMA delivery rate versus box shape (diagnostic only).
// One producer thread per CTA streams boxes of a uint16 matrix resident in L2
// into a 4-deep ring; a consumer thread releases each stage as soon as it
// lands.  Reports GB/s aggregate and ns per box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);       \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra W;\n}\n" ::"r"(su32(b)),
        "r"(ph));
}
__device__ __forceinline__ void mb_spin(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n .reg .pred P;\n W: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra W;\n}\n" ::"r"(su32(b)),
        "r"(ph));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes));
}

struct Cfg {
    int mode;          // 0 tensor 2D, 1 bulk 1D
    int box_c, box_r;  // tensor box (elements, rows)
    int bytes;         // bytes per load
    int loads;         // loads per stage
    int iters;         // stages per CTA
    int depth;         // ring depth (<= 16)
    int spin;          // 1: test_wait polling instead of try_wait
};

__global__ void __launch_bounds__(64) k_probe(const __grid_constant__ CUtensorMap map,
                                              const uint16_t* src, Cfg c, unsigned long long* t) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    const int per = c.bytes * c.loads;
    if (threadIdx.x == 0) {
        for (int s = 0; s < c.depth; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        for (int i = 0; i < c.iters; ++i) {
            const int s = i % c.depth;
            if (i >= c.depth) {
                if (c.spin) mb_spin(&empty[s], ((i / c.depth) - 1) & 1);
                else mb_wait(&empty[s], ((i / c.depth) - 1) & 1);
            }
            mb_expect(&full[s], per);
            for (int l = 0; l < c.loads; ++l) {
                uint8_t* dst = sm + s * per + l * c.bytes;
                const int it = i * c.loads + l;
                if (c.mode == 0) {
                    // walk K (x) inside a 256-wide strip, rows per CTA tile
                    const int x = (it * c.box_c) % 256 + 256 * ((blockIdx.x / 16) % 14);
                    const int y = (blockIdx.x % 16) * 256 + ((it * c.box_c) / 256 * c.box_r) % 256;
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::"
                        "bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
                        "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(y), "r"(su32(&full[s]))
                        : "memory");
                } else {
                    const uint8_t* g = reinterpret_cast<const uint8_t*>(src) +
                                       (static_cast<uint64_t>(blockIdx.x) * 1048576 +
                                        static_cast<uint64_t>(it) * c.bytes) % (32u << 20);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                        "%2, [%3];" ::"r"(su32(dst)),
                        "l"(g), "r"(c.bytes), "r"(su32(&full[s]))
                        : "memory");
                }
            }
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < c.iters; ++i) {
            const int s = i % c.depth;
            if (c.spin) mb_spin(&full[s], (i / c.depth) & 1);
            else mb_wait(&full[s], (i / c.depth) & 1);
            mb_arrive(&empty[s]);
        }
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}

__global__ void k_spin(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const uint64_t R = 4096, C = 4096;  // uint16 matrix, 32 MB (L2-resident after warm-up)
    uint16_t* src;
    CK(cudaMalloc(&src, R * C * 2));
    CK(cudaMemset(src, 1, R * C * 2));
    unsigned long long* t;
    CK(cudaMalloc(&t, 4096 * 8));
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_spin<<<148, 32>>>(300000000ull);  // 300 ms at load: let the SM clocks ramp
    CK(cudaDeviceSynchronize());
    struct Case {
        const char* name;
        int mode, box_c, box_r, loads, sw, depth, spin;
    } cases[] = {
        {"1d 8KB x1 d4 trywait", 1, 0, 0, 1, 0, 4, 0},
        {"1d 4KB x2 d4 trywait", 1, 0, 0, 2, 0, 4, 0},
        {"1d 2KB x4 d4 trywait", 1, 0, 0, 4, 0, 4, 0},
        {"1d 8KB x1 d8 trywait", 1, 0, 0, 1, 0, 8, 0},
        {"1d 8KB x1 d16 trywait", 1, 0, 0, 1, 0, 16, 0},
        {"1d 8KB x4 d4 trywait", 1, 0, 0, 4, 0, 4, 0},
        {"1d 32KB x1 d4 trywait", 1, 0, 0, 1, 0, 4, 0},
        {"2d 32x128 d4 trywait", 0, 32, 128, 1, 2, 4, 0},
        {"2d 32x128 x4 d4 trywait", 0, 32, 128, 4, 2, 4, 0},
        {"2d 64x128 x2 d4 trywait", 0, 64, 128, 2, 3, 4, 0},
    };
    const int sizes1d[] = {8192, 4096, 2048, 8192, 8192, 8192, 32768};
    int i1 = 0;
    for (const Case& k : cases) {
        Cfg c;
        c.mode = k.mode;
        c.box_c = k.box_c;
        c.box_r = k.box_r;
        c.loads = k.loads;
        c.bytes = k.mode == 0 ? k.box_c * k.box_r * 2 : sizes1d[i1++];
        c.iters = 64;
        c.depth = k.depth;
        c.spin = k.spin;
        CUtensorMap map;
        if (k.mode == 0) {
            cuuint64_t dims[2] = {C, R};
            cuuint64_t str[1] = {C * 2};
            cuuint32_t box[2] = {static_cast<cuuint32_t>(k.box_c), static_cast<cuuint32_t>(k.box_r)};
            cuuint32_t es[2] = {1, 1};
            CUtensorMapSwizzle sw = k.sw == 0   ? CU_TENSOR_MAP_SWIZZLE_NONE
                                    : k.sw == 1 ? CU_TENSOR_MAP_SWIZZLE_32B
                                    : k.sw == 2 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_128B;
            if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, src, dims, str, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("encode failed %s\n", k.name);
                continue;
            }
        } else {
            memset(&map, 0, sizeof(map));
        }
        const int smem = c.depth * c.bytes * c.loads;
        for (int grid : {8, 16, 32, 64, 112, 148}) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                k_probe<<<grid, 64, smem>>>(map, src, c, t);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            unsigned long long h[4096];
            CK(cudaMemcpy(h, t, grid * 8, cudaMemcpyDeviceToHost));
            double mean = 0;
            for (int i = 0; i < grid; ++i) mean += h[i];
            mean /= grid;
            const double bytes = static_cast<double>(c.bytes) * c.loads * c.iters;
            printf("%-30s grid %3d: per-CTA %.0f ns/stage (%.1f GB/s/SM), aggregate %.0f GB/s (event %.1f us)\n",
                   k.name, grid, mean / c.iters, bytes / mean, bytes * grid / (best * 1e6), best * 1e3);
        }
    }
    return 0;
}
