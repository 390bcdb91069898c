// dnd -- GPU bench / verify CLI over the C++ drop-in API.
//
// Mirrors the reference's tools/main.cpp subcommands `bench` and `verify`
// (tools/bench.cpp:84-130, tools/verify.cpp:20-193) for the hot-path
// algorithms, with the same protocol: warmup runs, then timed runs bracketed by
// barriers with the slowest rank reported, synthetic random_uniform data.
//
//   dnd bench  --algo kmeans|cdist|moments --synthetic 5000000x18 [--k 8]
//              [--iters 20] [--ranks 1] [--warmup 1] [--runs 9] [--seed 42]
//   dnd verify --algo kmeans|cdist|moments --synthetic 20000x18 [--ranks 2] ...
//   (--data FILE.dnb instead of --synthetic loads a DNB container into HBM;
//    --algo load times that load itself, f32 containers)
//
// bench prints one JSON object (the reference's report keys plus GB/s, the
// fraction of p x the measured HBM copy peak, and NVML clocks);
// verify runs the algorithm on `ranks` GPUs and on one and reports the largest
// relative deviation |a-b|/max(1,|b|) against the gate (distances/centroids
// 1e-5, moments 1e-12), exit status 1 when it fails.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dnd/dnd.hpp"

namespace {

struct Options {
    std::string cmd, algo = "kmeans", data;  // data: DNB path (else synthetic)
    dnd::index_t rows = 20000, cols = 18;
    int k = 8, iters = 20, ranks = 1, warmup = 1, runs = 9;
    std::uint64_t seed = 42;
    double peak_gbs = 6538.9;  // MEASURED_PEAKS.json hbm_gbs (copy bandwidth)
};

[[noreturn]] void usage(const char* why) {
    std::fprintf(stderr,
                 "dnd: %s\nusage: dnd bench|verify --algo kmeans|cdist|moments|load|lasso --synthetic ROWSxCOLS | --data FILE.dnb [--k K] "
                 "[--iters N] [--ranks P] [--warmup W] [--runs R] [--seed S] [--peak-gbs G]\n",
                 why);
    std::exit(2);
}

Options parse(int argc, char** argv) {
    if (argc < 2) usage("missing subcommand");
    Options o;
    o.cmd = argv[1];
    if (o.cmd != "bench" && o.cmd != "verify") usage("unknown subcommand");
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (i + 1 >= argc) usage(("missing value for " + a).c_str());
        const std::string v = argv[++i];
        if (a == "--algo") o.algo = v;
        else if (a == "--data") o.data = v;
        else if (a == "--synthetic") {
            const auto x = v.find('x');
            if (x == std::string::npos) usage("--synthetic takes ROWSxCOLS");
            o.rows = std::atoll(v.substr(0, x).c_str());
            o.cols = std::atoll(v.substr(x + 1).c_str());
        } else if (a == "--k") o.k = std::atoi(v.c_str());
        else if (a == "--iters") o.iters = std::atoi(v.c_str());
        else if (a == "--ranks") o.ranks = std::atoi(v.c_str());
        else if (a == "--warmup") o.warmup = std::atoi(v.c_str());
        else if (a == "--runs") o.runs = std::atoi(v.c_str());
        else if (a == "--seed") o.seed = std::strtoull(v.c_str(), nullptr, 10);
        else if (a == "--peak-gbs") o.peak_gbs = std::atof(v.c_str());
        else usage(("unknown option " + a).c_str());
    }
    if (o.algo != "kmeans" && o.algo != "cdist" && o.algo != "moments" && o.algo != "load" && o.algo != "lasso")
        usage("unknown --algo");
    if (o.algo == "load" && o.data.empty()) usage("--algo load times dnb_load of --data");
    if (!o.data.empty()) {  // shape from the container header (options.hpp:71-90)
        const auto h = dnd::dnb_read_header(o.data);
        if (h.extents.size() != 2) usage("--data needs a 2-D DNB container");
        o.rows = static_cast<dnd::index_t>(h.extents[0]);
        o.cols = static_cast<dnd::index_t>(h.extents[1]);
    }
    if (o.rows < 1 || o.cols < 1 || o.ranks < 1 || o.runs < 1 || o.warmup < 0) usage("bad sizes");
    return o;
}

using LassoData = std::pair<dnd::DndArray<double>, dnd::DndArray<double>>;

// LASSO input built once per rank from x: column 0 ones, the rest x widened
// to f64, y = a fixed sparse linear model of the row plus a little of x[:,0]
LassoData make_lasso(const Options& o, const dnd::DndArray<float>& xin) {
    const auto xf = dnd::gather(xin);
    std::vector<double> x(xf.begin(), xf.end()), y(static_cast<std::size_t>(o.rows));
    for (dnd::index_t i = 0; i < o.rows; ++i) {
        double acc = 0.0;
        for (dnd::index_t j = 1; j < o.cols; ++j) acc += (j % 3 == 0 ? 0.0 : 1.0 / j) * x[i * o.cols + j];
        y[i] = 0.5 + acc + 0.01 * (x[i * o.cols] - 0.5);
        x[i * o.cols] = 1.0;
    }
    return {dnd::from_global(x, {o.rows, o.cols}, 0, xin.comm()), dnd::from_global(y, {o.rows}, 0, xin.comm())};
}

// one run of the algorithm; returns a scalar that depends on the result
// (kept, like the reference's sink, so nothing is optimised away) and fills
// `out` with the replicated result for verify
double run_algo(const Options& o, const dnd::DndArray<float>& x, const LassoData* ld, std::vector<double>* out) {
    const dnd::Communicator& comm = x.comm();
    if (o.algo == "load") {  // the DNB container into the HBM shards (dataio.hpp:102-142)
        const auto y = dnd::dnb_load<float>(o.data, 0, comm);
        if (out) {
            const auto g = dnd::gather(y);
            out->assign(g.begin(), g.end());
        }
        return y.numel_local() > 0 ? 1.0 : 0.0;
    }
    if (o.algo == "lasso") {  // --iters sweeps, lambda 1 (regression.cpp:25-102)
        const auto model = dnd::lasso_fit(ld->first, ld->second, 1.0, o.iters, 0.0);
        if (out) *out = model.weights;
        return model.objective_trace.back();
    }
    if (o.algo == "kmeans") {
        const auto model = dnd::kmeans_fit(x, o.k, o.iters, 0.0, o.seed);
        if (out) *out = model.centroids;
        return model.inertia_trace.back();
    }
    if (o.algo == "cdist") {
        const auto d = dnd::cdist(x);
        if (out) {
            const auto g = dnd::gather(d);
            out->assign(g.begin(), g.end());
        }
        float first = 0.f;
        if (d.numel_local() > 1)
            dnd::detail::check(dndc_memcpy(comm.handle(), &first, d.device_data() + 1, sizeof(float), DNDC_COPY_D2H));
        return first;
    }
    const auto mu = dnd::gather(dnd::mean_axis(x, 0));
    const auto var = dnd::gather(dnd::var_axis(x, 0));
    if (out) {
        *out = mu;
        out->insert(out->end(), var.begin(), var.end());
    }
    return mu[0] + var[0];
}

// SM clock and throttle reasons of GPU 0 sampled every 5 ms during the timed
// runs through NVML (dlopen'ed: the driver ships it; absent -> "clocks": null)
class ClockSampler {
  public:
    ClockSampler() {
        lib_ = dlopen("libnvidia-ml.so.1", RTLD_NOW);
        if (!lib_) return;
        auto init = reinterpret_cast<int (*)()>(dlsym(lib_, "nvmlInit_v2"));
        auto get = reinterpret_cast<int (*)(unsigned, void**)>(dlsym(lib_, "nvmlDeviceGetHandleByIndex_v2"));
        clock_ = reinterpret_cast<int (*)(void*, int, unsigned*)>(dlsym(lib_, "nvmlDeviceGetClockInfo"));
        maxclock_ = reinterpret_cast<int (*)(void*, int, unsigned*)>(dlsym(lib_, "nvmlDeviceGetMaxClockInfo"));
        reasons_ = reinterpret_cast<int (*)(void*, unsigned long long*)>(
            dlsym(lib_, "nvmlDeviceGetCurrentClocksThrottleReasons"));
        ok_ = init && get && clock_ && maxclock_ && reasons_ && init() == 0 && get(0, &dev_) == 0;
    }
    void start() {
        if (!ok_) return;
        run_ = true;
        th_ = std::thread([this] {
            while (run_) {
                unsigned mhz = 0;
                unsigned long long r = 0;
                if (clock_(dev_, 1 /*NVML_CLOCK_SM*/, &mhz) == 0) mhz_.push_back(mhz);
                if (reasons_(dev_, &r) == 0) seen_ |= r;
                std::this_thread::sleep_for(std::chrono::milliseconds(5));
            }
        });
    }
    void stop() {
        if (!th_.joinable()) return;
        run_ = false;
        th_.join();
    }
    std::string json() {
        if (!ok_ || mhz_.empty()) return "null";
        std::sort(mhz_.begin(), mhz_.end());
        unsigned mx = 0;
        maxclock_(dev_, 1, &mx);
        static const std::pair<unsigned long long, const char*> names[] = {
            {0x4, "sw_power_cap"}, {0x8, "hw_slowdown"}, {0x20, "sw_thermal_slowdown"},
            {0x40, "hw_thermal_slowdown"}, {0x80, "hw_power_brake_slowdown"}};
        std::string rs;
        for (const auto& [bit, name] : names)
            if (seen_ & bit) rs += std::string(rs.empty() ? "" : ", ") + "\"" + name + "\"";
        return "{\"sm_mhz\": " + std::to_string(mhz_[mhz_.size() / 2]) + ", \"sm_max_mhz\": " + std::to_string(mx) +
               ", \"reasons\": [" + rs + "], \"samples\": " + std::to_string(mhz_.size()) + "}";
    }
    ~ClockSampler() { stop(); }

  private:
    void* lib_ = nullptr;
    void* dev_ = nullptr;
    bool ok_ = false;
    std::atomic<bool> run_{false};
    std::thread th_;
    std::vector<unsigned> mhz_;
    unsigned long long seen_ = 0;
    int (*clock_)(void*, int, unsigned*) = nullptr;
    int (*maxclock_)(void*, int, unsigned*) = nullptr;
    int (*reasons_)(void*, unsigned long long*) = nullptr;
};

// the input: a DNB file loaded straight into the HBM shards (f64 files are
// narrowed to the fp32 hot path), or random_uniform<float>
dnd::DndArray<float> make_input(const Options& o, const dnd::Communicator& comm) {
    if (o.data.empty()) return dnd::random_uniform<float>({o.rows, o.cols}, 0, o.seed, comm);
    if (dnd::dnb_read_header(o.data).dtype == dnd::DnbDtype::f32) return dnd::dnb_load<float>(o.data, 0, comm);
    return dnd::astype<float>(dnd::dnb_load<double>(o.data, 0, comm));
}

double bytes_per_run(const Options& o) {
    const double xb = 4.0 * o.rows * o.cols;
    if (o.algo == "kmeans") return xb * o.iters;
    if (o.algo == "cdist") return 4.0 * o.rows * o.rows + xb;
    if (o.algo == "load") return static_cast<double>(std::filesystem::file_size(o.data));
    if (o.algo == "lasso") return 8.0 * o.rows * o.cols * o.iters;  // X (f64) once per sweep
    return xb;
}

int bench(const Options& o) {
    std::vector<double> secs;
    std::mutex mu;
    ClockSampler clocks;
    dnd::run_world(o.ranks, [&](const dnd::Communicator& comm) {
        const auto x = make_input(o, comm);
        std::unique_ptr<LassoData> ld;
        if (o.algo == "lasso") ld = std::make_unique<LassoData>(make_lasso(o, x));
        double sink = 0.0;
        for (int w = 0; w < o.warmup; ++w) sink += run_algo(o, x, ld.get(), nullptr);
        if (comm.rank() == 0) clocks.start();
        // slowest rank per run (bench.cpp:102-112): the ranks are threads of
        // this process, so the max is taken under a mutex after the runs
        std::vector<double> mine;
        for (int r = 0; r < o.runs; ++r) {
            comm.barrier();
            const auto t0 = std::chrono::steady_clock::now();
            sink += run_algo(o, x, ld.get(), nullptr);
            comm.barrier();
            mine.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        if (comm.rank() == 0) clocks.stop();
        if (!std::isfinite(sink)) throw dnd::ValueError("benchmark produced non-finite results");
        std::lock_guard<std::mutex> lock(mu);
        if (secs.empty()) secs.assign(mine.size(), 0.0);
        for (size_t i = 0; i < mine.size(); ++i) secs[i] = std::max(secs[i], mine[i]);
    });
    const auto st = dnd::local_moments(dnd::Tile<double>{{static_cast<dnd::index_t>(secs.size())}, secs});
    std::string runs;
    for (double t : secs) runs += (runs.empty() ? "" : ", ") + std::to_string(t);
    const double mean = st.mean[0], sd = std::sqrt(st.m2[0] / static_cast<double>(st.count));
    std::printf("{\"algo\": \"%s\", \"ranks\": %d, \"split\": 0, \"params\": {\"rows\": %lld, \"cols\": %lld, "
                "\"k\": %d, \"iters\": %d, \"seed\": %llu}, \"warmup_runs\": %d, \"timed_runs\": %d, "
                "\"mean_seconds\": %.9g, \"std_seconds\": %.9g, \"GB_per_s\": %.6g, \"roofline_frac\": %.4f, "
                "\"peak_gbs_per_gpu\": %.1f, \"clocks\": %s, \"device\": \"B200 (libdndc)\", \"run_seconds\": [%s]}\n",
                o.algo.c_str(), o.ranks, static_cast<long long>(o.rows), static_cast<long long>(o.cols), o.k, o.iters,
                static_cast<unsigned long long>(o.seed), o.warmup, o.runs, mean, sd, bytes_per_run(o) / mean / 1e9,
                bytes_per_run(o) / mean / 1e9 / (o.peak_gbs * o.ranks), o.peak_gbs, clocks.json().c_str(), runs.c_str());
    return 0;
}

int verify(const Options& o) {
    std::vector<double> dist_res, single_res;
    std::mutex mu;
    auto collect = [&](int ranks, std::vector<double>& dst) {
        dnd::run_world(ranks, [&](const dnd::Communicator& comm) {
            const auto x = make_input(o, comm);
            std::unique_ptr<LassoData> ld;
            if (o.algo == "lasso") ld = std::make_unique<LassoData>(make_lasso(o, x));
            std::vector<double> r;
            run_algo(o, x, ld.get(), &r);
            std::lock_guard<std::mutex> lock(mu);
            if (comm.rank() == 0) dst = r;
        });
    };
    collect(o.ranks, dist_res);
    collect(1, single_res);
    if (dist_res.size() != single_res.size()) {
        std::printf("{\"algo\": \"%s\", \"ranks\": %d, \"pass\": false, \"error\": \"size mismatch\"}\n",
                    o.algo.c_str(), o.ranks);
        return 1;
    }
    double dev = 0.0;
    for (size_t i = 0; i < dist_res.size(); ++i)
        dev = std::max(dev, std::abs(dist_res[i] - single_res[i]) / std::max(1.0, std::abs(single_res[i])));
    const double gate = o.algo == "moments" ? 1e-12 : 1e-5;  // tools/verify.cpp:20-33 + BASELINE.json
    const bool pass = dev <= gate;
    std::printf("{\"algo\": \"%s\", \"ranks\": %d, \"max_rel_dev\": %.3e, \"gate\": %.0e, \"pass\": %s}\n",
                o.algo.c_str(), o.ranks, dev, gate, pass ? "true" : "false");
    return pass ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options o = parse(argc, argv);
        return o.cmd == "bench" ? bench(o) : verify(o);
    } catch (const dnd::Error& e) {
        std::fprintf(stderr, "dnd: %s\n", e.what());
        return 1;
    }
}
