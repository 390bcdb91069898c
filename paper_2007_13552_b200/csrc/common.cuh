// common.cuh -- shared runtime pieces of libdndc (the C-ABI in include/dndc.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dndc.h"

namespace dndc {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void value_error(const std::string& what) { throw Error(DNDC_EVALUE, what); }

void set_last_error(const std::string& what);

#define DNDC_CUDA(expr)                                                                     \
    do {                                                                                    \
        cudaError_t e__ = (expr);                                                           \
        if (e__ != cudaSuccess)                                                             \
            throw ::dndc::Error(DNDC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
    } while (0)

#define DNDC_NCCL(expr)                                                                     \
    do {                                                                                    \
        ncclResult_t r__ = (expr);                                                          \
        if (r__ != ncclSuccess)                                                             \
            throw ::dndc::Error(DNDC_ETRANSPORT, std::string(#expr) + ": " + ncclGetErrorString(r__)); \
    } while (0)

#define DNDC_LAUNCHED(ctx)                                                                  \
    do {                                                                                    \
        DNDC_CUDA(cudaGetLastError());                                                      \
        (ctx)->launches++;                                                                  \
    } while (0)

template <typename F>
int guard(F&& fn) {
    try {
        fn();
        return DNDC_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return DNDC_EINTERNAL;
    }
}

// ---------------------------------------------------------------- k-means
// Device-resident Lloyd state (one per context); see kmeans.cu.
struct KMeansState;
void destroy_kmeans_state(KMeansState*);

}  // namespace dndc

// --------------------------------------------------------------- context
struct dndc_group;  // loopback.cu: ranks that share GPUs

struct dndc_ctx {
    int device = 0, rank = 0, world = 1;
    dndc_group* group = nullptr;        // host-staged transport (world > #GPUs), not owned
    int num_sms = 148;
    cudaStream_t stream = nullptr;      // work stream (user's or own)
    cudaStream_t own_stream = nullptr;  // created by dndc_create
    cudaStream_t comm_stream = nullptr; // ring exchanges overlap compute here
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    ncclComm_t comm = nullptr;
    dndc_counters counters{};
    uint64_t launches = 0;
    int64_t last_refined = 0;
    const char* last_kernel = "";  // the k-means loop kernel of the last fit (kmeans.cu)
    int64_t persist_trace_len = 0;  // DNDC_PERSIST_TRACE marks of the last persistent fit
    int persist_trace_grid = 0;
    int km_slot = 0;  // constant-memory centroid table slot (kmeans.cu)

    // Growable device workspace, carved by named slots so repeated calls reuse
    // the same addresses (CUDA-graph friendly).
    std::map<std::string, std::pair<void*, size_t>> slots;
    void* slot(const std::string& name, size_t bytes);
    uint64_t slot_gen = 0;  // bumped when a slot moves (reallocation): captured graphs key on it

    // stream-ordered pool behind dndc_alloc/dndc_free (hostio.cu): arrays the
    // host layer allocates per call (cdist outputs, results) reuse memory
    // instead of paying cudaMalloc/cudaFree each time; trimmed on OOM
    cudaMemPool_t pool = nullptr;
    void trim_pool();

    // file <-> HBM streaming (dataio.cu): per I/O thread two pinned chunks,
    // one in flight on the copy engine while the thread reads/writes the other
    std::vector<void*> io_buf;
    std::vector<cudaEvent_t> io_ev;

    // LASSO: the instantiated one-sweep graph of the last fit and its key (lasso.cu)
    cudaGraphExec_t ls_exec = nullptr;
    std::string ls_key;

    // pinned host staging for small results
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    void* host_staging(size_t bytes);

    dndc::KMeansState* km = nullptr;

    // NVLink peer exchange (world > 1): a small region per rank, mapped into
    // every other rank through CUDA IPC (runtime.cu setup_peer_exchange); the
    // fused k-means kernel writes its stats straight into every peer's region.
    bool p2p = false;
    std::string p2p_status = "world == 1";
    void* xchg = nullptr;              // own region (cudaMalloc)
    std::vector<void*> peer_bases;     // every rank's region as mapped here (own = xchg)
    void** peer_bases_dev = nullptr;   // the same table in device memory
};

namespace dndc {
// Layout of one rank's exchange region: [2 slots][world][XCHG_STATS] f64
// receive buffers, then [world] u64 arrival flags, then one u64 epoch.
constexpr int XCHG_STATS = 4096;
inline size_t xchg_bytes(int world) {
    return sizeof(double) * 2 * world * XCHG_STATS + sizeof(unsigned long long) * (world + 1);
}
__host__ __device__ inline double* xchg_recv(void* base, int slot, int world, int r) {
    return static_cast<double*>(base) + (static_cast<size_t>(slot) * world + r) * XCHG_STATS;
}
__host__ __device__ inline unsigned long long* xchg_flags(void* base, int world) {
    return reinterpret_cast<unsigned long long*>(static_cast<double*>(base) + 2 * static_cast<size_t>(world) * XCHG_STATS);
}
}  // namespace dndc

namespace dndc {

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

void chunk_map(int64_t n, int p, std::vector<int64_t>& off, std::vector<int64_t>& ext);

// Collective helpers over the context's NCCL communicator, on `stream`.
void allgather_f64(dndc_ctx* ctx, const double* send, double* recv, size_t count,
                   cudaStream_t stream);
void allreduce_sum_f64(dndc_ctx* ctx, double* buf, size_t count, cudaStream_t stream);

// Transport primitives (loopback.cu): NCCL over NVLink when every rank owns a
// GPU, host-staged through the rank group when ranks share GPUs.  Device
// buffers, ordered on `s` (the group path synchronises).
enum XportKind { XK_ALLGATHER = 1, XK_ALLREDUCE = 2, XK_BARRIER = 3 };
struct XSend {
    int peer;
    const void* buf;
    size_t bytes;
};
struct XRecv {
    int peer;
    void* buf;
    size_t bytes;
};
void xport_allgather(dndc_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s);
void xport_allreduce_sum_f64(dndc_ctx* ctx, double* buf, size_t count, cudaStream_t s);
void xport_exchange(dndc_ctx* ctx, const std::vector<XSend>& sends, const std::vector<XRecv>& recvs, cudaStream_t s);
void xport_barrier(dndc_ctx* ctx);

// ------------------------------------------------------------ device math
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__host__ __device__ inline double uniform01(uint64_t seed, uint64_t counter) {
    const uint64_t z = splitmix64(seed ^ splitmix64(counter));
    return static_cast<double>(z >> 11) * 0x1.0p-53;
}

// The reference's f64 arithmetic without contraction: every product is
// rounded before the add (it is compiled for baseline x86-64, no FMA).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// distance_block's per-entry formula (pairwise.cpp:26-31), bit-exact.
__device__ __forceinline__ double ref_distance(double na, double nb, double g) {
    const double sq = sub_rn(add_rn(na, nb), mul_rn(2.0, g));
    return __dsqrt_rn(sq > 0.0 ? sq : 0.0);
}

__device__ __forceinline__ float sqrt_approx(float v) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// Packed fp32 FMA / add (sm_100 FFMA2 / FADD2): two independent fmaf's in one
// instruction.  The CUDA intrinsics, not inline asm: the asm's 64-bit operand
// packing cost ~30 extra moves per row in the k-means scores (ncu, r2).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }

__device__ __forceinline__ void st_stream(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_stream4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace dndc
