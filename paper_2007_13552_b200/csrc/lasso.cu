// lasso.cu -- F4: LASSO by cyclic coordinate descent on the HBM shards.
//
// Reference: lasso_fit / lasso_predict / soft_threshold (regression.cpp:19-127).
// Per coordinate j the reference sums rho = x_j . (r + w_j x_j) over its rows,
// allreduces that scalar, takes the exact coordinate minimiser and updates
// its rank-local residual r.  Here:
//  * the shard is transposed once into column-major xt (m x rows), so a
//    coordinate streams one contiguous column; the residual lives in HBM (and
//    mostly in L2: 8 bytes per row);
//  * one kernel per coordinate: every thread first applies the previous
//    coordinate's pending residual shift, then accumulates rho for column j
//    in the same pass; CTA partials are folded in a fixed order by the last
//    CTA to arrive, which also does the cross-GPU sum and the update -- so a
//    coordinate is one launch and no host round trip;
//  * across GPUs the scalar goes through the NVLink peer-exchange region of
//    the k-means kernel (CUDA IPC, release/acquire flags, epoch parity slots)
//    and is summed in rank order on every rank -- the "m scalar allreduces
//    per sweep" as peer stores instead of NCCL launches; without peer access
//    the tail leaves rho_local for an in-stream NCCL allreduce and a 1-thread
//    update kernel;
//  * one sweep (m coordinate kernels + the objective kernel) is captured as a
//    CUDA graph and replayed `sweeps` times; after convergence (max change <
//    tol) every kernel returns at once.
// predict is the reference's row loop, multiply then add without FMA
// contraction, so its output is bit-identical.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace dndc {

constexpr int LS_THREADS = 256;

struct LassoCtl {
    double shift;       // w_old - w_new of coordinate jprev, not yet applied to r
    double max_change;  // this sweep
    double rho_local;   // NCCL fallback: this rank's sum, allreduced in place
    double rho_pending_wold;
    int jprev;          // -1: nothing pending
    int done;
    int sweep;          // sweeps completed
    int pending_j;      // NCCL fallback: coordinate whose update waits for the allreduce
    int timeout;        // a peer never arrived at the NVLink sum: every later step is a no-op
};

struct LassoArgs {
    const double* xt;
    double* r;
    int64_t rows;
    int m;
    double* w;
    const double* sq;
    LassoCtl* ctl;
    double* partials;
    unsigned* counter;
    double lambda, tol;
    double* trace;
    void* const* peers;  // NVLink exchange bases (world > 1 with peer access) or null
    int rank, world;
};

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__host__ __device__ inline double soft_threshold(double rho, double t) {
    if (rho > t) return rho - t;
    if (rho < -t) return rho + t;
    return 0.0;
}

// fixed-order block sum (warp shuffles, then the warps in order)
static __device__ double ls_block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < LS_THREADS / 32; ++w) t += sh[w];
    __syncthreads();
    return t;  // valid in thread 0
}

// every rank's value, summed in rank order 0..world-1 (allreduce(plus),
// transport.hpp:140-146), via the peer regions; one CTA, all its threads
static __device__ double peer_sum(const LassoArgs& a, double v, unsigned long long* s_epoch) {
    const int world = a.world;
    if (threadIdx.x == 0) {
        unsigned long long* ep = xchg_flags(a.peers[a.rank], world) + world;
        *s_epoch = *ep + 1;
        *ep = *s_epoch;
    }
    __syncthreads();
    const unsigned long long epoch = *s_epoch;
    const int slot = static_cast<int>(epoch & 1);
    if (threadIdx.x < world) xchg_recv(a.peers[threadIdx.x], slot, world, a.rank)[0] = v;  // NVLink store
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < world) {
        st_release_sys_u64(xchg_flags(a.peers[threadIdx.x], world) + a.rank, epoch);
        const unsigned long long* mine = xchg_flags(a.peers[a.rank], world) + threadIdx.x;
        const long long t0 = clock64();
        while (ld_acquire_sys_u64(mine) < epoch) {
            __nanosleep(64);
            if (clock64() - t0 > 40000000000ll) {  // a peer never arrived (~20 s): TimeoutError, no trap
                a.ctl->timeout = 1;
                a.ctl->done = 1;
                break;
            }
        }
    }
    __syncthreads();
    __threadfence();
    double t = 0.0;
    for (int r = 0; r < world; ++r) t += xchg_recv(a.peers[a.rank], slot, world, r)[0];
    return t;
}

// coordinate update from the global rho (regression.cpp:80-90); thread 0
static __device__ void apply_update(const LassoArgs& a, int j, double rho, double w_old) {
    LassoCtl* c = a.ctl;
    if (a.sq[j] == 0.0) {  // degenerate column: skipped, keeps its weight
        c->shift = 0.0;
        c->jprev = -1;
        return;
    }
    const double w_new = j == 0 ? rho / a.sq[0] : soft_threshold(rho, a.lambda / 2.0) / a.sq[j];
    c->shift = w_old - w_new;
    c->jprev = j;
    a.w[j] = w_new;
    c->max_change = fmax(c->max_change, fabs(w_new - w_old));
}

// end of a sweep (regression.cpp:92-101); thread 0
static __device__ void finish_sweep(const LassoArgs& a, double ssr) {
    LassoCtl* c = a.ctl;
    double pen = 0.0;
    for (int j = 1; j < a.m; ++j) pen += fabs(a.w[j]);
    a.trace[c->sweep] = ssr + a.lambda * pen;
    c->sweep += 1;
    if (c->max_change < a.tol) c->done = 1;
    c->max_change = 0.0;
    c->shift = 0.0;
    c->jprev = -1;
}

// j < m: coordinate j; j == m: the objective of the sweep
__global__ void __launch_bounds__(LS_THREADS) lasso_step_kernel(LassoArgs a, int j) {
    __shared__ double sh[LS_THREADS / 32];
    __shared__ int s_last;
    __shared__ unsigned long long s_epoch;
    LassoCtl* c = a.ctl;
    if (c->done) return;
    const double shift = c->shift;
    const int jp = c->jprev;
    const bool apply = jp >= 0 && shift != 0.0;
    const bool obj = j == a.m;
    const double w_old = obj ? 0.0 : a.w[j];
    const double* xp = a.xt + static_cast<int64_t>(apply ? jp : 0) * a.rows;
    const double* xj = a.xt + static_cast<int64_t>(obj ? 0 : j) * a.rows;
    double acc = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * LS_THREADS;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(LS_THREADS) + threadIdx.x; i < a.rows; i += stride) {
        double ri = a.r[i];
        if (apply) {
            ri += shift * xp[i];
            a.r[i] = ri;
        }
        if (obj) {
            acc += ri * ri;
        } else {
            const double x = xj[i];
            acc += x * (ri + w_old * x);
        }
    }
    const double part = ls_block_sum(acc, sh);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = part;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.counter, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // CTA partials in CTA order (thread-strided, then the fixed block tree)
    double t = 0.0;
    for (int g = threadIdx.x; g < static_cast<int>(gridDim.x); g += LS_THREADS) t += a.partials[g];
    const double local = ls_block_sum(t, sh);
    if (threadIdx.x == 0) *a.counter = 0u;
    double total = local;
    if (a.world > 1) {
        if (!a.peers) {  // NCCL fallback: the allreduce and update follow in-stream
            if (threadIdx.x == 0) {
                c->rho_local = local;
                c->pending_j = j;
                c->rho_pending_wold = w_old;
            }
            return;
        }
        __shared__ double s_local;
        if (threadIdx.x == 0) s_local = local;
        __syncthreads();
        total = peer_sum(a, s_local, &s_epoch);
    }
    if (threadIdx.x != 0) return;
    if (obj) finish_sweep(a, total);
    else apply_update(a, j, total, w_old);
}

// NCCL fallback: after the in-place allreduce of ctl->rho_local
__global__ void lasso_update_kernel(LassoArgs a) {
    LassoCtl* c = a.ctl;
    if (c->done) return;
    if (c->pending_j == a.m) finish_sweep(a, c->rho_local);
    else apply_update(a, c->pending_j, c->rho_local, c->rho_pending_wold);
}

// rows x m (row-major) -> m x rows, 32 x 32 tiles through shared memory;
// counts rows whose bias column is not exactly 1.0
__global__ void lasso_transpose_kernel(const double* __restrict__ x, int64_t rows, int m, double* __restrict__ xt,
                                       unsigned long long* bad_bias) {
    __shared__ double tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int c0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k;
        const int c = c0 + threadIdx.x;
        if (r < rows && c < m) {
            const double v = x[r * m + c];
            tile[k][threadIdx.x] = v;
            if (c == 0 && v != 1.0) atomicAdd(bad_bias, 1ull);
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k;
        const int64_t r = r0 + threadIdx.x;
        if (r < rows && c < m) xt[static_cast<int64_t>(c) * rows + r] = tile[threadIdx.x][k];
    }
}

// column sums of squares: CTA (j, b) sums slice b of column j into
// part[j][b]; lasso_sq_final_kernel adds the LS_SQ_SLICES slices in order
constexpr int LS_SQ_SLICES = 64;
__global__ void __launch_bounds__(LS_THREADS) lasso_sq_kernel(const double* __restrict__ xt, int64_t rows,
                                                              double* __restrict__ part) {
    __shared__ double sh[LS_THREADS / 32];
    const double* col = xt + static_cast<int64_t>(blockIdx.x) * rows;
    const int64_t per = (rows + LS_SQ_SLICES - 1) / LS_SQ_SLICES;
    const int64_t lo = blockIdx.y * per, hi = min(rows, lo + per);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += LS_THREADS) acc += col[i] * col[i];
    const double t = ls_block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x * LS_SQ_SLICES + blockIdx.y] = t;
}

__global__ void lasso_sq_final_kernel(const double* __restrict__ part, int m, double* __restrict__ sq) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double t = 0.0;
    for (int b = 0; b < LS_SQ_SLICES; ++b) t += part[j * LS_SQ_SLICES + b];
    sq[j] = t;
}

// Xw per row in column order, products rounded before the add
// (regression.cpp:116-121)
__global__ void lasso_predict_kernel(const double* __restrict__ x, int64_t rows, int m, const double* __restrict__ w,
                                     double* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows) return;
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, __dmul_rn(x[i * m + j], w[j]));
    out[i] = acc;
}

static void lasso_fit(dndc_ctx* ctx, const double* x, int64_t rows, int64_t n_global, int64_t m64, const double* y,
                      double lambda, int sweeps, double tol, double* w_host, double* trace_host, int* sweeps_run) {
    if (n_global < 1) value_error("lasso_fit: need at least one sample");
    if (m64 < 1) value_error("lasso_fit: design matrix needs at least the bias column");
    if (!(lambda >= 0.0)) value_error("lasso_fit: lambda must be nonnegative");
    if (sweeps < 1) value_error("lasso_fit: sweeps must be positive");
    if (rows < 0) value_error("lasso_fit: negative row count");
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    static const bool trace_on = std::getenv("DNDC_LASSO_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace_on) return;
        DNDC_CUDA(cudaDeviceSynchronize());
        std::fprintf(stderr, "lasso rank %d %-12s %.3f ms\n", ctx->rank, what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    const int64_t R = std::max<int64_t>(rows, 1);
    double* xt = static_cast<double*>(ctx->slot("ls_xt", sizeof(double) * R * m));
    double* r = static_cast<double*>(ctx->slot("ls_r", sizeof(double) * R));
    double* w = static_cast<double*>(ctx->slot("ls_w", sizeof(double) * m));
    double* sq = static_cast<double*>(ctx->slot("ls_sq", sizeof(double) * (m + 1)));
    double* trace = static_cast<double*>(ctx->slot("ls_trace", sizeof(double) * sweeps));
    LassoCtl* ctl = static_cast<LassoCtl*>(ctx->slot("ls_ctl", sizeof(LassoCtl)));
    unsigned* counter = static_cast<unsigned*>(ctx->slot("ls_counter", 64));
    const int G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 4, ceil_div(R, LS_THREADS))));
    double* partials = static_cast<double*>(ctx->slot("ls_partials", sizeof(double) * G));
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(counter + 8);

    DNDC_CUDA(cudaMemsetAsync(counter, 0, 64, s));
    DNDC_CUDA(cudaMemsetAsync(sq, 0, sizeof(double) * (m + 1), s));
    if (rows > 0) {
        lasso_transpose_kernel<<<dim3(static_cast<unsigned>(ceil_div(rows, 32)), (m + 31) / 32), dim3(32, 8), 0, s>>>(
            x, rows, m, xt, bad);
        DNDC_LAUNCHED(ctx);
        double* sq_part = static_cast<double*>(ctx->slot("ls_sq_part", sizeof(double) * m * LS_SQ_SLICES));
        lasso_sq_kernel<<<dim3(m, LS_SQ_SLICES), LS_THREADS, 0, s>>>(xt, rows, sq_part);
        DNDC_LAUNCHED(ctx);
        lasso_sq_final_kernel<<<(m + 127) / 128, 128, 0, s>>>(sq_part, m, sq);
        DNDC_LAUNCHED(ctx);
        DNDC_CUDA(cudaMemcpyAsync(r, y, sizeof(double) * rows, cudaMemcpyDeviceToDevice, s));  // r = y - X0
    }
    // the bias-column count rides along with the norms: sq[m] (exact in f64)
    {
        std::vector<unsigned long long> hb(1);
        DNDC_CUDA(cudaMemcpyAsync(hb.data(), bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaStreamSynchronize(s));
        const double nb = static_cast<double>(hb[0]);
        DNDC_CUDA(cudaMemcpyAsync(sq + m, &nb, sizeof(double), cudaMemcpyHostToDevice, s));
        DNDC_CUDA(cudaStreamSynchronize(s));
    }
    mark("norms");
    if (ctx->world > 1) {
        const int rc = dndc_allreduce_f64(ctx, sq, m + 1);  // rank-order fold (regression.cpp:61-62)
        if (rc != DNDC_OK) throw Error(rc, dndc_last_error());
    }
    double bad_total = 0.0;
    DNDC_CUDA(cudaMemcpyAsync(&bad_total, sq + m, sizeof(double), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    if (bad_total != 0.0) value_error("lasso_fit: column 0 must be the all-ones bias column");
    mark("allreduce");

    LassoCtl c0{0.0, 0.0, 0.0, 0.0, -1, 0, 0, 0, 0};
    DNDC_CUDA(cudaMemcpyAsync(ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
    DNDC_CUDA(cudaMemsetAsync(w, 0, sizeof(double) * m, s));
    DNDC_CUDA(cudaMemsetAsync(trace, 0, sizeof(double) * sweeps, s));

    LassoArgs a{xt, r, rows, m, w, sq, ctl, partials, counter, lambda, tol, trace,
                ctx->world > 1 && ctx->p2p ? ctx->peer_bases_dev : nullptr, ctx->rank, ctx->world};
    const bool nccl = ctx->world > 1 && !ctx->p2p;
    double* rho = &reinterpret_cast<LassoCtl*>(ctl)->rho_local;
    auto sweep = [&](cudaStream_t st) {
        for (int j = 0; j <= m; ++j) {
            lasso_step_kernel<<<G, LS_THREADS, 0, st>>>(a, j);
            if (nccl) {
                xport_allreduce_sum_f64(ctx, rho, 1, st);
                lasso_update_kernel<<<1, 1, 0, st>>>(a);
            }
        }
    };
    if (ctx->group) {
        // ranks sharing GPUs: host-staged scalar sums cannot sit in a graph
        for (int sw = 0; sw < sweeps; ++sw) {
            sweep(s);
            ctx->launches += static_cast<uint64_t>(2 * (m + 1));
        }
        LassoCtl ch;
        DNDC_CUDA(cudaMemcpyAsync(&ch, ctl, sizeof(ch), cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaMemcpyAsync(w_host, w, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaMemcpyAsync(trace_host, trace, sizeof(double) * sweeps, cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaStreamSynchronize(s));
        if (ch.timeout) throw Error(DNDC_ETIMEOUT, "lasso_fit: a peer rank did not arrive at the coordinate sum");
        *sweeps_run = ch.sweep;
        return;
    }
    // one sweep as a graph, replayed (launch cost of m+1 kernels -> one);
    // instantiated once per (buffers, shape, lambda, tol, transport) and kept
    cudaStream_t gs = ctx->own_stream;
    cudaEvent_t ev = ctx->ev_a;
    DNDC_CUDA(cudaEventRecord(ev, s));
    DNDC_CUDA(cudaStreamWaitEvent(gs, ev, 0));
    char keybuf[256];
    std::snprintf(keybuf, sizeof(keybuf), "%p/%p/%lld/%d/%.17g/%.17g/%d/%d/%d/%llu", (const void*)xt, (void*)r,
                  (long long)rows, m, lambda, tol, G, ctx->world, nccl ? 1 : 0,
                  static_cast<unsigned long long>(ctx->slot_gen));
    if (!ctx->ls_exec || ctx->ls_key != keybuf) {
        if (ctx->ls_exec) cudaGraphExecDestroy(ctx->ls_exec);
        ctx->ls_exec = nullptr;
        cudaGraph_t graph;
        DNDC_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        try {
            sweep(gs);
        } catch (...) {
            cudaStreamEndCapture(gs, &graph);
            throw;
        }
        DNDC_CUDA(cudaStreamEndCapture(gs, &graph));
        DNDC_CUDA(cudaGraphInstantiate(&ctx->ls_exec, graph, 0));
        DNDC_CUDA(cudaGraphDestroy(graph));
        ctx->ls_key = keybuf;
    }
    cudaGraphExec_t exec = ctx->ls_exec;
    mark("instantiate");
    for (int sw = 0; sw < sweeps; ++sw) {
        DNDC_CUDA(cudaGraphLaunch(exec, gs));
        ctx->launches += static_cast<uint64_t>(m + 1);
    }
    DNDC_CUDA(cudaEventRecord(ev, gs));
    DNDC_CUDA(cudaStreamWaitEvent(s, ev, 0));
    LassoCtl ch;
    DNDC_CUDA(cudaMemcpyAsync(&ch, ctl, sizeof(ch), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(w_host, w, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(trace_host, trace, sizeof(double) * sweeps, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    mark("sweeps");
    if (ch.timeout)
        throw Error(DNDC_ETIMEOUT, "lasso_fit: a peer rank did not arrive at the NVLink coordinate sum within the "
                                   "deadlock timeout (transport.cpp:76-93)");
    *sweeps_run = ch.sweep;
}

}  // namespace dndc

extern "C" {

int dndc_lasso_fit_f64(dndc_ctx* ctx, const double* x_local, int64_t rows, int64_t n_global, int64_t m,
                       const double* y_local, double lambda, int sweeps, double tol, double* weights_out,
                       double* trace_out, int* sweeps_run) {
    return dndc::guard([&] {
        DNDC_CUDA(cudaSetDevice(ctx->device));
        dndc::lasso_fit(ctx, x_local, rows, n_global, m, y_local, lambda, sweeps, tol, weights_out, trace_out,
                        sweeps_run);
    });
}

int dndc_lasso_predict_f64(dndc_ctx* ctx, const double* x_local, int64_t rows, int64_t m, const double* weights,
                           double* out_local) {
    return dndc::guard([&] {
        if (rows < 0 || m < 1) dndc::value_error("lasso_predict: bad extents");
        if (rows == 0) return;
        DNDC_CUDA(cudaSetDevice(ctx->device));
        double* w = static_cast<double*>(ctx->slot("lp_w", sizeof(double) * m));
        DNDC_CUDA(cudaMemcpyAsync(w, weights, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
        dndc::lasso_predict_kernel<<<static_cast<unsigned>(dndc::ceil_div(rows, 256)), 256, 0, ctx->stream>>>(
            x_local, rows, static_cast<int>(m), w, out_local);
        DNDC_LAUNCHED(ctx);
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
