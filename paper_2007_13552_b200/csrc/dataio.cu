// dataio.cu -- F2: DNB payload ranges streamed between a file and HBM.
//
// Reference: dnb_load / dnb_save (dataio.hpp:61-142) read and write each
// rank's byte range `header + offset(r) * row_bytes` with positioned stream
// I/O into a host tile.  Here the range goes straight to (or from) the HBM
// shard: the host reads chunk i+1 with pread while the copy engine moves
// chunk i, through two pinned buffers, so a 360 MB shard (the SUSY-sized
// cfg1 input) costs about one file read.  Header parsing and validation stay
// in the host layer (cpp/include/dnd/dataio.hpp), as in the reference.
// Reads fan out over DNDC_IO_THREADS (default 8) threads, each with its own
// pair of pinned chunks, all copying on the context's stream.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace dndc {

constexpr size_t IO_CHUNK = size_t(8) << 20;

[[noreturn]] static void data_error(const std::string& what) { throw Error(DNDC_EDATA, what); }

// reader/writer threads: a single pread stream out of the page cache tops out
// near 11 GB/s, well under PCIe; DNDC_IO_THREADS overrides
static int io_threads() {
    const char* e = std::getenv("DNDC_IO_THREADS");
    return std::max(1, std::min(16, e ? std::atoi(e) : 8));
}

static void io_buffers(dndc_ctx* ctx, int threads) {
    while (static_cast<int>(ctx->io_buf.size()) < 2 * threads) {
        void* p = nullptr;
        cudaEvent_t ev = nullptr;
        DNDC_CUDA(cudaMallocHost(&p, IO_CHUNK));
        DNDC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        ctx->io_buf.push_back(p);
        ctx->io_ev.push_back(ev);
    }
}

struct Fd {
    int fd;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

// thread t streams its contiguous slice [lo, hi) of the range through its
// own two pinned chunks: pread chunk i+1 while the copy engine moves chunk i
static void read_slice(dndc_ctx* ctx, int fd, const char* path, uint64_t off, size_t lo, size_t hi, char* dst,
                       int t) {
    cudaStream_t s = ctx->stream;
    for (size_t done = lo, i = 0; done < hi; done += IO_CHUNK, ++i) {
        const int b = 2 * t + static_cast<int>(i & 1);
        const size_t len = std::min(IO_CHUNK, hi - done);
        DNDC_CUDA(cudaEventSynchronize(ctx->io_ev[b]));  // the copy out of this buffer two chunks ago
        char* h = static_cast<char*>(ctx->io_buf[b]);
        for (size_t got = 0; got < len;) {
            const ssize_t r = pread(fd, h + got, len - got, static_cast<off_t>(off + done + got));
            if (r < 0 && errno == EINTR) continue;
            if (r <= 0) data_error(std::string("short read from ") + path);
            got += static_cast<size_t>(r);
        }
        DNDC_CUDA(cudaMemcpyAsync(dst + done, h, len, cudaMemcpyHostToDevice, s));
        DNDC_CUDA(cudaEventRecord(ctx->io_ev[b], s));
    }
}

static void read_to_device(dndc_ctx* ctx, const char* path, uint64_t off, size_t bytes, void* dst) {
    Fd f{open(path, O_RDONLY | O_CLOEXEC)};
    if (f.fd < 0) data_error(std::string("cannot open ") + path + " for reading: " + std::strerror(errno));
    if (!bytes) return;
    const int T = static_cast<int>(std::min<size_t>(io_threads(), (bytes + IO_CHUNK - 1) / IO_CHUNK));
    io_buffers(ctx, T);
    // slices in whole chunks so every thread's copies stay chunk-aligned
    const size_t chunks = (bytes + IO_CHUNK - 1) / IO_CHUNK, per = (chunks + T - 1) / T;
    std::vector<std::thread> th;
    std::vector<std::string> err(T);
    std::vector<int> code(T, DNDC_OK);
    for (int t = 0; t < T; ++t) {
        const size_t lo = std::min(bytes, t * per * IO_CHUNK), hi = std::min(bytes, (t + 1) * per * IO_CHUNK);
        th.emplace_back([&, t, lo, hi] {
            try {
                DNDC_CUDA(cudaSetDevice(ctx->device));
                read_slice(ctx, f.fd, path, off, lo, hi, static_cast<char*>(dst), t);
            } catch (const Error& e) {
                err[t] = e.what();
                code[t] = e.code;
            } catch (const std::exception& e) {
                err[t] = e.what();
                code[t] = DNDC_EINTERNAL;
            }
        });
    }
    for (auto& x : th) x.join();
    DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int t = 0; t < T; ++t)
        if (code[t] != DNDC_OK) throw Error(code[t], err[t]);
}

static void write_from_device(dndc_ctx* ctx, const char* path, uint64_t off, const void* src, size_t bytes) {
    Fd f{open(path, O_WRONLY | O_CLOEXEC)};
    if (f.fd < 0) data_error(std::string("cannot open ") + path + " for writing: " + std::strerror(errno));
    if (!bytes) return;
    io_buffers(ctx, 1);
    cudaStream_t s = ctx->stream;
    const size_t n = (bytes + IO_CHUNK - 1) / IO_CHUNK;
    auto issue = [&](size_t i) {
        const size_t len = std::min(IO_CHUNK, bytes - i * IO_CHUNK);
        DNDC_CUDA(cudaMemcpyAsync(ctx->io_buf[i & 1], static_cast<const char*>(src) + i * IO_CHUNK, len,
                                  cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaEventRecord(ctx->io_ev[i & 1], s));
    };
    issue(0);
    for (size_t i = 0; i < n; ++i) {
        DNDC_CUDA(cudaEventSynchronize(ctx->io_ev[i & 1]));
        if (i + 1 < n) issue(i + 1);  // next chunk crosses PCIe while this one is written
        const size_t len = std::min(IO_CHUNK, bytes - i * IO_CHUNK);
        const char* h = static_cast<const char*>(ctx->io_buf[i & 1]);
        for (size_t put = 0; put < len;) {
            const ssize_t w = pwrite(f.fd, h + put, len - put, static_cast<off_t>(off + i * IO_CHUNK + put));
            if (w < 0 && errno == EINTR) continue;
            if (w <= 0) data_error(std::string("write to ") + path + " failed: " + std::strerror(errno));
            put += static_cast<size_t>(w);
        }
    }
}

}  // namespace dndc

extern "C" {

int dndc_file_read_to_device(dndc_ctx* ctx, const char* path, uint64_t byte_offset, size_t bytes, void* dev_dst) {
    return dndc::guard([&] {
        DNDC_CUDA(cudaSetDevice(ctx->device));
        dndc::read_to_device(ctx, path, byte_offset, bytes, dev_dst);
    });
}

int dndc_file_write_from_device(dndc_ctx* ctx, const char* path, uint64_t byte_offset, const void* dev_src,
                                size_t bytes) {
    return dndc::guard([&] {
        DNDC_CUDA(cudaSetDevice(ctx->device));
        dndc::write_from_device(ctx, path, byte_offset, dev_src, bytes);
    });
}

}  // extern "C"
