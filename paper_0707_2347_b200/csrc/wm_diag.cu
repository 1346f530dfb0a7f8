// Diagnostics used by scripts/microbench.py to calibrate the design (not on
// the multiplication path): dependent-launch latency inside a CUDA graph with
// and without programmatic dependent launch, and streaming bandwidth of a
// one-CTA-per-SM copy (what one SM can pull from L2 / HBM).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/winomem_b200.h"

namespace {

__global__ void k_tiny(double* p, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1.0;
    if (pdl) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__global__ void k_stream(const double2* __restrict__ src, double2* __restrict__ dst,
                         std::uint64_t n2, int write) {
    double2 acc = make_double2(0, 0);
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        double2 v = __ldg(src + i);
        if (write) dst[i] = v;
        else {
            acc.x += v.x;
            acc.y += v.y;
        }
    }
    if (!write && acc.x == 12345.678) dst[0] = acc;
}

// one chained "prep-like" step: every thread reads `nin` 16-B words (strided by
// the grid) and writes `nout` 16-B words
__global__ void k_chain(const double2* __restrict__ src, double2* __restrict__ dst, int nin,
                        int nout, std::uint64_t stride) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const std::uint64_t t = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    double2 acc = make_double2(0, 0);
    for (int i = 0; i < nin; ++i) {
        const double2 v = src[t + i * stride];
        acc.x += v.x;
        acc.y += v.y;
    }
    for (int i = 0; i < nout; ++i) dst[t + i * stride] = make_double2(acc.x + i, acc.y);
}

// the same step with a counter handoff instead of griddepcontrol.wait: thread 0
// spins until the predecessor's CTAs have all signalled, every CTA signals its
// own completion (release) after its stores
__global__ void k_chain_flag(const double2* __restrict__ src, double2* __restrict__ dst, int nin,
                             int nout, std::uint64_t stride, const unsigned* wait_ctr,
                             unsigned target, unsigned* done_ctr) {
    if (wait_ctr) {
        if (threadIdx.x == 0) {
            unsigned v;
            unsigned long long t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wait_ctr) : "memory");
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 2000000000ull) __trap();
            } while (v < target);
        }
        __syncthreads();
    } else {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
    }
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const std::uint64_t t = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    double2 acc = make_double2(0, 0);
    for (int i = 0; i < nin; ++i) {
        const double2 v = src[t + i * stride];
        acc.x += v.x;
        acc.y += v.y;
    }
    for (int i = 0; i < nout; ++i) dst[t + i * stride] = make_double2(acc.x + i, acc.y);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done_ctr) : "memory");
    }
}

}  // namespace

extern "C" {

// Host -> device copy rate of a pinned rows x cols u32 matrix: mode 0 one
// contiguous copy, 1 four quadrant 2-D copies, 2 two contiguous row halves.
// Returns GB/s.
int wm_diag_h2d(const void* host, unsigned long long rows, unsigned long long cols, int mode,
                int reps, double* gbs) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 12;
    void* dev = nullptr;
    const std::size_t bytes = rows * cols * 4;
    if (cudaMalloc(&dev, bytes) != cudaSuccess) return 12;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto once = [&]() {
        const char* h = static_cast<const char*>(host);
        char* d = static_cast<char*>(dev);
        if (mode == 0) {
            cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
        } else if (mode == 1) {
            for (int q = 0; q < 4; ++q) {
                const std::size_t off = ((q / 2) * (rows / 2) * cols + (q % 2) * (cols / 2)) * 4;
                cudaMemcpy2DAsync(d + off, cols * 4, h + off, cols * 4, cols / 2 * 4, rows / 2,
                                  cudaMemcpyHostToDevice, s);
            }
        } else {
            cudaMemcpyAsync(d, h, bytes / 2, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(d + bytes / 2, h + bytes / 2, bytes / 2, cudaMemcpyHostToDevice, s);
        }
    };
    once();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) once();
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *gbs = static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e9;
    cudaFree(dev);
    cudaStreamDestroy(s);
    return cudaGetLastError() == cudaSuccess ? 0 : 12;
}

// wm_diag_chain with the counter handoff (k_chain_flag)
int wm_diag_chain_flag(int threads, int block, int nin, int nout, int n, int nbuf, double* us) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 12;
    const std::uint64_t stride = static_cast<std::uint64_t>(threads);
    const std::uint64_t words = stride * (nin > nout ? nin : nout);
    double2* buf = nullptr;
    unsigned* ctr = nullptr;
    if (cudaMalloc(&buf, 2 * nbuf * words * sizeof(double2) + 16) != cudaSuccess) return 12;
    if (cudaMalloc(&ctr, (n + 1) * sizeof(unsigned)) != cudaSuccess) return 12;
    cudaMemset(buf, 0, 2 * nbuf * words * sizeof(double2));
    const unsigned nblk = static_cast<unsigned>((threads + block - 1) / block);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaMemsetAsync(ctr, 0, (n + 1) * sizeof(unsigned), s);
    for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nblk);
        cfg.blockDim = dim3(block);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = i > 0 ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int b = i % nbuf;
        cudaLaunchKernelEx(&cfg, k_chain_flag, static_cast<const double2*>(buf + 2 * b * words),
                           buf + (2 * b + 1) * words, nin, nout, stride,
                           static_cast<const unsigned*>(i > 0 ? ctr + i : nullptr), nblk, ctr + i + 1);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return 12;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *us = 1000.0 * ms / (reps * n);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(buf);
    cudaFree(ctr);
    cudaStreamDestroy(s);
    return cudaGetLastError() == cudaSuccess ? 0 : 12;
}

// Microseconds per kernel of a PDL chain of `n` k_chain launches (graph replay):
// `threads` threads each reading nin and writing nout 16-B words, rotating over
// `nbuf` buffer pairs (L2-resident when small).
int wm_diag_chain(int threads, int block, int nin, int nout, int n, int nbuf, double* us) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 12;
    const std::uint64_t stride = static_cast<std::uint64_t>(threads);
    const std::uint64_t words = stride * (nin > nout ? nin : nout);
    double2* buf = nullptr;
    if (cudaMalloc(&buf, 2 * nbuf * words * sizeof(double2)) != cudaSuccess) return 12;
    cudaMemset(buf, 0, 2 * nbuf * words * sizeof(double2));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((threads + block - 1) / block);
        cfg.blockDim = dim3(block);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int b = i % nbuf;
        cudaLaunchKernelEx(&cfg, k_chain, buf + 2 * b * words, buf + (2 * b + 1) * words, nin, nout,
                           stride);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return 12;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *us = 1000.0 * ms / (reps * n);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(buf);
    cudaStreamDestroy(s);
    return cudaGetLastError() == cudaSuccess ? 0 : 12;
}

// Average microseconds per kernel of `n` dependent single-CTA kernels replayed as
// one CUDA graph (pdl=1: launched with programmatic stream serialization).
int wm_diag_launch_latency(int n, int pdl, int blocks, double* us_per_kernel) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 12;
    double* d = nullptr;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(128);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_tiny, d, pdl);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return 12;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *us_per_kernel = 1000.0 * ms / (reps * n);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(d);
    cudaStreamDestroy(s);
    return cudaGetLastError() == cudaSuccess ? 0 : 12;
}

// GB/s of a grid of `blocks` x 256 threads streaming `bytes` (read-only when write=0).
int wm_diag_stream(std::uint64_t bytes, int blocks, int write, int reps, double* gbs) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double2 *a = nullptr, *b = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) return 12;
    cudaMemset(a, 0, bytes);
    const std::uint64_t n2 = bytes / 16;
    k_stream<<<blocks, 256, 0, s>>>(a, b, n2, write);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) k_stream<<<blocks, 256, 0, s>>>(a, b, n2, write);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *gbs = (write ? 2.0 : 1.0) * bytes * reps / (ms * 1e-3) / 1e9;
    cudaFree(a);
    cudaFree(b);
    cudaStreamDestroy(s);
    return cudaGetLastError() == cudaSuccess ? 0 : 12;
}

}  // extern "C"
