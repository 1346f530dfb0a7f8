// Multi-GPU product partition behind the C-ABI (wm_dist_*): the protocol of
// paper_0707_2347_b200/dist.py for C / C++ callers of run_variant
// (drivers.hpp:213-222), one process (or thread) per GPU.
//
//   1. the root broadcasts A and B over NCCL (one collective each);
//   2. every rank forms its own operands S_t, T_t with the one-pass combination
//      kernel (wm_lincomb) and multiplies them with the single-GPU memory-lean
//      plan (wm_run_variant: `ip` on square operands -- they are scratch copies,
//      so the local product needs no temporaries);
//   3. products go to the root with ncclSend on a communication stream (the
//      rank's compute stream moves on to its next product); the root receives
//      them in product order into a ring of `window` buffers and folds
//      alpha * coef * P_t straight into the C blocks on a fold stream -- after
//      scaling C by beta once, with no full-size accumulator.
// Each pair of ranks sees its point-to-point messages in the same order on both
// sides (product order), so the exchange cannot cross-deadlock.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, RTLD_LOCAL) so the
// library keeps no link-time dependency on it and never clashes with the copy
// a host framework may already have loaded.
#include <dlfcn.h>

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/winomem_b200.h"
#include "wm_types.h"

namespace wm {
namespace {

struct NcclApi {
    void* so = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.so) return api;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        api.so = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        if (api.so) break;
    }
    if (!api.so) fail(E_NCCL, "libnccl.so.2 not found");
    auto sym = [&](const char* n) {
        void* p = dlsym(api.so, n);
        if (!p) fail(E_NCCL, std::string("NCCL symbol missing: ") + n);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}
void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void wck(int rc) {
    if (rc != WM_OK) fail(rc, wm_last_error());
}

// Table-1 quadrant coefficients over (11, 12, 21, 22): S_i, T_i, and the C
// quadrants each P_i folds into (dist.py holds the same tables)
constexpr int S_COEF[7][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {1, 1, -1, -1}, {0, 0, 0, 1},
                              {0, 0, 1, 1}, {-1, 0, 1, 1}, {1, 0, -1, 0}};
constexpr int T_COEF[7][4] = {{1, 0, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}, {1, -1, -1, 1},
                              {-1, 1, 0, 0}, {1, -1, 0, 1}, {0, -1, 0, 1}};
constexpr int C_COEF[7][4] = {{1, 1, 1, 1}, {1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, -1, 0},
                              {0, 1, 0, 1}, {0, 1, 1, 1}, {0, 0, 1, 1}};

wm_dmat quad(const wm_dmat& v, int q) {
    const std::uint64_t r = v.rows / 2, c = v.cols / 2;
    return {v.ptr + (q >> 1) * r * v.ld + (q & 1) * c, r, c, v.ld};
}

double makespan(int world, std::uint64_t products) {
    const std::uint64_t per = (products + world - 1) / world;
    return static_cast<double>(products) / static_cast<double>(per);
}

}  // namespace
}  // namespace wm

struct wm_dist {
    wm_ctx* ctx = nullptr;
    int rank = 0, world = 1, device = 0;
    std::uint32_t p = 65521;
    int field = WM_FIELD_MODP;
    ncclComm_t comm = nullptr;
    cudaStream_t main = nullptr, comm_s = nullptr, fold_s = nullptr;
    std::uint64_t live = 0, peak = 0;  // device bytes this call holds
    void hold(std::uint64_t b, std::uint64_t transient = 0) {
        live += b;
        peak = std::max(peak, live + transient);
    }
    void release(std::uint64_t b) { live -= b; }
};

namespace wm {
namespace {

thread_local std::string g_dist_err;

template <class F>
int dguard(F&& fn) {
    try {
        fn();
        return WM_OK;
    } catch (const Error& e) {
        g_dist_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_dist_err = e.what();
        return E_INVALID;
    }
}

double* dalloc(wm_dist* D, std::uint64_t words, cudaStream_t s) {
    void* p = nullptr;
    cck(cudaMallocAsync(&p, words * sizeof(double), s), "cudaMallocAsync");
    D->hold(words * sizeof(double));
    return static_cast<double*>(p);
}
void dfree(wm_dist* D, double* p, std::uint64_t words, cudaStream_t s) {
    cck(cudaFreeAsync(p, s), "cudaFreeAsync");
    D->release(words * sizeof(double));
}

// the uint32 scalar wm_lincomb takes for s * coef: a residue (MODP), or the
// signed value reinterpreted (REAL64 reads it as an int32)
std::uint32_t scalar(const wm_dist* D, std::uint32_t s, int coef) {
    if (D->field == WM_FIELD_REAL64)
        return static_cast<std::uint32_t>(static_cast<std::int32_t>(s) * coef);
    const std::int64_t p = D->p, v = static_cast<std::int64_t>(s % D->p) * coef;
    return static_cast<std::uint32_t>(((v % p) + p) % p);
}

// S_idx(A) / T_idx(B): one combination of at most four quadrants per level, each
// level's block freed once the next one exists (stream-ordered on `s`)
wm_dmat operand(wm_dist* D, const wm_dmat& M, const std::vector<int>& idx, const int (*table)[4],
                cudaStream_t s) {
    wm_dmat X = M;
    bool owned = false;
    for (int i : idx) {
        wm_dmat src[4];
        std::uint32_t coef[4];
        int n = 0;
        for (int q = 0; q < 4; ++q)
            if (table[i][q]) {
                src[n] = quad(X, q);
                coef[n] = scalar(D, 1, table[i][q]);
                ++n;
            }
        wm_dmat Y{dalloc(D, (X.rows / 2) * (X.cols / 2), s), X.rows / 2, X.cols / 2, X.cols / 2};
        wck(wm_lincomb(D->ctx, Y, n, src, coef));
        if (owned) dfree(D, X.ptr, X.rows * X.cols, s);
        X = Y;
        owned = true;
    }
    return X;
}

// (block of C, coefficient) pairs product idx folds into
std::vector<std::pair<wm_dmat, int>> targets(const wm_dmat& C, const std::vector<int>& idx) {
    std::vector<std::pair<wm_dmat, int>> out = {{C, 1}};
    for (int i : idx) {
        std::vector<std::pair<wm_dmat, int>> next;
        for (const auto& [blk, coef] : out)
            for (int q = 0; q < 4; ++q)
                if (C_COEF[i][q]) next.push_back({quad(blk, q), coef * C_COEF[i][q]});
        out.swap(next);
    }
    return out;
}

}  // namespace
}  // namespace wm

extern "C" {

const char* wm_dist_last_error(void) { return wm::g_dist_err.c_str(); }

int wm_dist_unique_id(unsigned char id[128]) {
    return wm::dguard([&] {
        ncclUniqueId u;
        wm::nck(wm::nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, sizeof(u.internal));
    });
}

int wm_dist_create(wm_ctx* ctx, int rank, int world, const unsigned char id[128], wm_dist** out) {
    return wm::dguard([&] {
        if (!ctx || !out || world < 1 || rank < 0 || rank >= world) wm::fail(wm::E_INVALID, "bad dist arguments");
        auto D = std::make_unique<wm_dist>();
        D->ctx = ctx;
        D->rank = rank;
        D->world = world;
        void* stream = nullptr;
        wm::wck(wm_ctx_info(ctx, &D->device, &D->p, &D->field, &stream));
        D->main = static_cast<cudaStream_t>(stream);
        wm::cck(cudaSetDevice(D->device), "cudaSetDevice");
        wm::cck(cudaStreamCreateWithFlags(&D->comm_s, cudaStreamNonBlocking), "stream");
        wm::cck(cudaStreamCreateWithFlags(&D->fold_s, cudaStreamNonBlocking), "stream");
        ncclUniqueId u;
        std::memcpy(u.internal, id, sizeof(u.internal));
        wm::nck(wm::nccl().CommInitRank(&D->comm, world, u, rank), "ncclCommInitRank");
        *out = D.release();
    });
}

int wm_dist_destroy(wm_dist* D) {
    if (!D) return WM_OK;
    cudaStreamSynchronize(D->main);
    cudaStreamSynchronize(D->comm_s);
    cudaStreamSynchronize(D->fold_s);
    if (D->comm) wm::nccl().CommDestroy(D->comm);
    cudaStreamDestroy(D->comm_s);
    cudaStreamDestroy(D->fold_s);
    delete D;
    return WM_OK;
}

int wm_dist_choose_levels(int world, uint64_t n, int cutoff) {
    int best_l = 1;
    double best = 0.0;
    for (int L = 1; L <= 3; ++L)
        if ((n >> L) >= std::max<std::uint64_t>(2 * static_cast<std::uint64_t>(cutoff), 2))
            best = std::max(best, wm::makespan(world, static_cast<std::uint64_t>(std::pow(7, L))));
    for (int L = 1; L <= 3; ++L)
        if ((n >> L) >= std::max<std::uint64_t>(2 * static_cast<std::uint64_t>(cutoff), 2) &&
            wm::makespan(world, static_cast<std::uint64_t>(std::pow(7, L))) >= 0.98 * best) {
            best_l = L;
            break;
        }
    return best_l;
}

int wm_dist_run_variant(wm_dist* D, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                        uint32_t alpha, uint32_t beta, int cutoff, int levels, int window,
                        wm_dist_report* report) {
    (void)variant;
    return wm::dguard([&] {
        using namespace wm;
        const bool root = D->rank == 0;
        const bool real = D->field == WM_FIELD_REAL64;
        D->live = D->peak = 0;
        window = std::max(1, window);
        // 1. shapes from the root
        std::uint64_t* meta = nullptr;
        cck(cudaMallocAsync(reinterpret_cast<void**>(&meta), 3 * sizeof(std::uint64_t), D->main), "meta");
        if (root) {
            if (A.ld != A.cols || B.ld != B.cols)
                fail(E_INVALID, "wm_dist_run_variant: A and B must be contiguous (ld == cols)");
            const std::uint64_t h[3] = {A.rows, A.cols, B.cols};
            cck(cudaMemcpyAsync(meta, h, sizeof(h), cudaMemcpyHostToDevice, D->main), "meta");
        }
        nck(nccl().Broadcast(meta, meta, 3, ncclUint64, 0, D->comm, D->main), "broadcast shapes");
        std::uint64_t shp[3];
        cck(cudaMemcpyAsync(shp, meta, sizeof(shp), cudaMemcpyDeviceToHost, D->main), "meta");
        cck(cudaStreamSynchronize(D->main), "sync");
        cck(cudaFreeAsync(meta, D->main), "meta");
        const std::uint64_t m = shp[0], k = shp[1], n = shp[2];
        const int L = levels > 0 ? levels : wm_dist_choose_levels(D->world, std::min({m, k, n}), cutoff);
        const std::uint64_t f = 1ull << L;
        if (m % f || k % f || n % f) fail(E_DIMENSION, "shape does not split into the partition's blocks");
        // 2. A and B to every rank
        if (!root) {
            A = {dalloc(D, m * k, D->main), m, k, k};
            B = {dalloc(D, k * n, D->main), k, n, n};
        }
        nck(nccl().Broadcast(A.ptr, A.ptr, m * k, ncclFloat64, 0, D->comm, D->main), "broadcast A");
        nck(nccl().Broadcast(B.ptr, B.ptr, k * n, ncclFloat64, 0, D->comm, D->main), "broadcast B");
        // the products, outer level first, product t on rank t mod G
        std::vector<std::vector<int>> prods = {{}};
        for (int l = 0; l < L; ++l) {
            std::vector<std::vector<int>> next;
            for (const auto& t : prods)
                for (int i = 0; i < 7; ++i) {
                    auto u = t;
                    u.push_back(i);
                    next.push_back(u);
                }
            prods.swap(next);
        }
        const std::uint64_t bm = m / f, bk = k / f, bn = n / f, pw = bm * bn;
        const char* local = (bm == bk && bk == bn) ? "ip" : "std2";
        cudaEvent_t ev;
        cck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        auto after = [&](cudaStream_t from, cudaStream_t to) {
            cck(cudaEventRecord(ev, from), "event");
            cck(cudaStreamWaitEvent(to, ev, 0), "event");
        };
        if (root) {  // C <- beta * C once, on the fold stream
            after(D->main, D->fold_s);
            const std::uint32_t b = scalar(D, beta, 1);
            wm_ctx_set_stream(D->ctx, D->fold_s);
            wck(wm_lincomb(D->ctx, C, 1, &C, &b));
            wm_ctx_set_stream(D->ctx, D->main);
        }
        auto fold = [&](std::size_t t, const wm_dmat& P) {  // on the fold stream
            wm_ctx_set_stream(D->ctx, D->fold_s);
            for (const auto& [blk, coef] : targets(C, prods[t])) {
                const wm_dmat src[2] = {blk, P};
                const std::uint32_t cf[2] = {1, scalar(D, alpha, coef)};
                wck(wm_lincomb(D->ctx, blk, 2, src, cf));
            }
            wm_ctx_set_stream(D->ctx, D->main);
        };
        std::uint64_t products = 0, sent = 0, received = 0;
        std::vector<double*> ring(root ? static_cast<std::size_t>(window) : 0, nullptr);
        std::vector<cudaEvent_t> ring_free(ring.size());
        for (std::size_t w = 0; w < ring.size(); ++w) {
            ring[w] = dalloc(D, pw, D->comm_s);
            cck(cudaEventCreateWithFlags(&ring_free[w], cudaEventDisableTiming), "event");
            cck(cudaEventRecord(ring_free[w], D->comm_s), "event");
        }
        std::size_t slot = 0;
        after(D->main, D->comm_s);  // the broadcasts precede every send / receive
        for (std::size_t t = 0; t < prods.size(); ++t) {
            const int owner = static_cast<int>(t % static_cast<std::size_t>(D->world));
            if (owner == D->rank) {
                const wm_dmat X = operand(D, A, prods[t], S_COEF, D->main);
                const wm_dmat Y = operand(D, B, prods[t], T_COEF, D->main);
                wm_dmat P{dalloc(D, pw, D->main), bm, bn, bn};
                wm_report rep{};
                const int rc = real ? wm_run_variant_real(D->ctx, local, X, Y, P, 1.0, 0.0, cutoff, &rep)
                                    : wm_run_variant(D->ctx, local, X, Y, P, 1, 0, cutoff, &rep);
                wck(rc);
                D->hold(0, rep.peak_extra_bytes);
                dfree(D, X.ptr, bm * bk, D->main);
                dfree(D, Y.ptr, bk * bn, D->main);
                ++products;
                if (root) {
                    after(D->main, D->fold_s);
                    fold(t, P);
                    after(D->fold_s, D->main);
                    dfree(D, P.ptr, pw, D->main);
                } else {
                    after(D->main, D->comm_s);
                    nck(nccl().Send(P.ptr, pw, ncclFloat64, 0, D->comm, D->comm_s), "send product");
                    dfree(D, P.ptr, pw, D->comm_s);
                    sent += pw * sizeof(double);
                }
            } else if (root) {
                double* buf = ring[slot];
                cck(cudaStreamWaitEvent(D->comm_s, ring_free[slot], 0), "event");
                nck(nccl().Recv(buf, pw, ncclFloat64, owner, D->comm, D->comm_s), "receive product");
                received += pw * sizeof(double);
                after(D->comm_s, D->fold_s);
                fold(t, {buf, bm, bn, bn});
                cck(cudaEventRecord(ring_free[slot], D->fold_s), "event");
                slot = (slot + 1) % ring.size();
            }
        }
        after(D->fold_s, D->main);
        after(D->comm_s, D->main);
        for (std::size_t w = 0; w < ring.size(); ++w) {
            dfree(D, ring[w], pw, D->main);
            cudaEventDestroy(ring_free[w]);
        }
        if (!root) {
            dfree(D, A.ptr, m * k, D->main);
            dfree(D, B.ptr, k * n, D->main);
        }
        cck(cudaStreamSynchronize(D->main), "sync");
        cudaEventDestroy(ev);
        if (report) {
            report->levels = L;
            report->products = products;
            report->peak_extra_bytes = D->peak;
            report->bytes_sent = sent;
            report->bytes_received = received + (root ? 0 : (m * k + k * n) * sizeof(double));
        }
    });
}

}  // extern "C"
