// resplit.cu -- F1: move an N-D array between split axes (or to/from full
// replication) with its shards in HBM.
//
// Reference: resplit (ndarray.hpp:340-386) -- slice locally when the source is
// replicated, allgather_varying when the target is, alltoall_varying of the
// intersection blocks between two split axes -- and its helpers extract_chunk
// / place_chunk.  Here every case is one rule: rank r's source box (its chunk
// of the source split axis, every other axis whole) intersected with rank q's
// target box is the block r sends q.  Blocks are packed into a contiguous
// staging buffer by a strided box-copy kernel, exchanged with one grouped
// NCCL send/recv round (NVLink), and unpacked into the target shard; the
// block a rank keeps is copied shard to shard directly.  A replicated source
// sends nothing (every rank already holds its target box).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace dndc {

constexpr int RS_MAX_DIMS = 8;

struct BoxCopy {
    int nd;
    int64_t ext[RS_MAX_DIMS];  // box extents, row-major
    int64_t src_st[RS_MAX_DIMS], dst_st[RS_MAX_DIMS];  // element strides
    int64_t total;
};

template <typename E>
__global__ void box_copy_kernel(const E* __restrict__ src, E* __restrict__ dst, BoxCopy b) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < b.total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t rem = e, so = 0, doff = 0;
        for (int d = b.nd - 1; d >= 0; --d) {
            const int64_t i = rem % b.ext[d];
            rem /= b.ext[d];
            so += i * b.src_st[d];
            doff += i * b.dst_st[d];
        }
        dst[doff] = src[so];
    }
}

struct Box {
    std::vector<int64_t> lo, hi;
    int64_t numel() const {
        int64_t n = 1;
        for (size_t d = 0; d < lo.size(); ++d) n *= std::max<int64_t>(0, hi[d] - lo[d]);
        return n;
    }
};

// the global box rank r holds under `split` (-1 = replicated)
static Box owned_box(const std::vector<int64_t>& shape, int split, int r, int world) {
    Box b{std::vector<int64_t>(shape.size(), 0), shape};
    if (split >= 0) {
        std::vector<int64_t> off, ext;
        chunk_map(shape[split], world, off, ext);
        b.lo[split] = off[r];
        b.hi[split] = off[r] + ext[r];
    }
    return b;
}

static Box intersect(const Box& a, const Box& b) {
    Box o = a;
    for (size_t d = 0; d < a.lo.size(); ++d) {
        o.lo[d] = std::max(a.lo[d], b.lo[d]);
        o.hi[d] = std::max(o.lo[d], std::min(a.hi[d], b.hi[d]));
    }
    return o;
}

// row-major element strides of a shard whose global box is `owner`
static std::vector<int64_t> strides_of(const Box& owner) {
    const size_t nd = owner.lo.size();
    std::vector<int64_t> st(nd, 1);
    for (size_t d = nd; d-- > 1;) st[d - 1] = st[d] * (owner.hi[d] - owner.lo[d]);
    return st;
}

static int64_t offset_in(const Box& owner, const std::vector<int64_t>& st, const Box& blk) {
    int64_t o = 0;
    for (size_t d = 0; d < st.size(); ++d) o += (blk.lo[d] - owner.lo[d]) * st[d];
    return o;
}

// copy `blk` (global coordinates) from a buffer laid out as `sbox` to one laid
// out as `dbox`; a null box means "contiguous block" (staging)
static void copy_box(dndc_ctx* ctx, const char* src, const Box* sbox, char* dst, const Box* dbox, const Box& blk,
                     int64_t esz) {
    const int64_t total = blk.numel();
    if (total == 0) return;
    const int nd = static_cast<int>(blk.lo.size());
    BoxCopy b{};
    b.nd = nd;
    b.total = total;
    const Box& sref = sbox ? *sbox : blk;
    const Box& dref = dbox ? *dbox : blk;
    const auto sst = strides_of(sref), dst_st = strides_of(dref);
    for (int d = 0; d < nd; ++d) {
        b.ext[d] = blk.hi[d] - blk.lo[d];
        b.src_st[d] = sst[d];
        b.dst_st[d] = dst_st[d];
    }
    src += offset_in(sref, sst, blk) * esz;
    dst += offset_in(dref, dst_st, blk) * esz;
    const int threads = 256;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(total, threads), ctx->num_sms * 16));
    cudaStream_t s = ctx->stream;
    switch (esz) {
        case 1: box_copy_kernel<uint8_t><<<grid, threads, 0, s>>>(reinterpret_cast<const uint8_t*>(src), reinterpret_cast<uint8_t*>(dst), b); break;
        case 2: box_copy_kernel<uint16_t><<<grid, threads, 0, s>>>(reinterpret_cast<const uint16_t*>(src), reinterpret_cast<uint16_t*>(dst), b); break;
        case 4: box_copy_kernel<uint32_t><<<grid, threads, 0, s>>>(reinterpret_cast<const uint32_t*>(src), reinterpret_cast<uint32_t*>(dst), b); break;
        case 8: box_copy_kernel<uint64_t><<<grid, threads, 0, s>>>(reinterpret_cast<const uint64_t*>(src), reinterpret_cast<uint64_t*>(dst), b); break;
        default: value_error("resplit: element size must be 1, 2, 4 or 8 bytes");
    }
    DNDC_LAUNCHED(ctx);
}

static void resplit(dndc_ctx* ctx, const void* src_local, int ndim, const int64_t* shape_in, int64_t esz,
                    int src_split, int dst_split, void* dst_local) {
    if (ndim < 1 || ndim > RS_MAX_DIMS) value_error("resplit: 1 to 8 dimensions");
    if (esz != 1 && esz != 2 && esz != 4 && esz != 8) value_error("resplit: element size must be 1, 2, 4 or 8 bytes");
    if (src_split < -1 || src_split >= ndim || dst_split < -1 || dst_split >= ndim)
        value_error("resplit: split axis out of range");
    std::vector<int64_t> shape(shape_in, shape_in + ndim);
    for (int64_t e : shape)
        if (e < 0) value_error("resplit: negative extent");
    const int W = ctx->world, r = ctx->rank;
    const Box mine_src = owned_box(shape, src_split, r, W), mine_dst = owned_box(shape, dst_split, r, W);
    const char* src = static_cast<const char*>(src_local);
    char* dst = static_cast<char*>(dst_local);
    // the block this rank keeps
    copy_box(ctx, src, &mine_src, dst, &mine_dst, intersect(mine_src, mine_dst), esz);
    if (W == 1 || src_split < 0) return;

    std::vector<Box> send(W), recv(W);
    int64_t send_total = 0, recv_total = 0;
    for (int q = 0; q < W; ++q) {
        if (q == r) continue;
        send[q] = intersect(mine_src, owned_box(shape, dst_split, q, W));
        recv[q] = intersect(owned_box(shape, src_split, q, W), mine_dst);
        send_total += send[q].numel();
        recv_total += recv[q].numel();
    }
    char* sbuf = static_cast<char*>(ctx->slot("rs_send", static_cast<size_t>(send_total * esz)));
    char* rbuf = static_cast<char*>(ctx->slot("rs_recv", static_cast<size_t>(recv_total * esz)));
    int64_t so = 0;
    for (int q = 0; q < W; ++q) {
        if (q == r) continue;
        copy_box(ctx, src, &mine_src, sbuf + so * esz, nullptr, send[q], esz);
        so += send[q].numel();
    }
    std::vector<XSend> xs;
    std::vector<XRecv> xr;
    so = 0;
    int64_t ro = 0;
    for (int q = 0; q < W; ++q) {
        if (q == r) continue;
        const int64_t ns = send[q].numel() * esz, nr = recv[q].numel() * esz;
        if (ns) xs.push_back({q, sbuf + so * esz, static_cast<size_t>(ns)});
        if (nr) xr.push_back({q, rbuf + ro * esz, static_cast<size_t>(nr)});
        so += send[q].numel();
        ro += recv[q].numel();
    }
    xport_exchange(ctx, xs, xr, ctx->stream);
    ro = 0;
    for (int q = 0; q < W; ++q) {
        if (q == r) continue;
        copy_box(ctx, rbuf + ro * esz, nullptr, dst, &mine_dst, recv[q], esz);
        ro += recv[q].numel();
    }
}

}  // namespace dndc

extern "C" {

int dndc_resplit(dndc_ctx* ctx, const void* src_local, int ndim, const int64_t* shape, int64_t elem_bytes,
                 int src_split, int dst_split, void* dst_local) {
    return dndc::guard([&] {
        dndc::resplit(ctx, src_local, ndim, shape, elem_bytes, src_split, dst_split, dst_local);
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
