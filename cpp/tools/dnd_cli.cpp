// dnd -- GPU bench / verify / convert CLI over the C++ drop-in API (SURVEY.md
// 8(f) F3), with the reference's command line (tools/main.cpp:12-83):
//
//   dnd convert SRC.csv DST.dnb [--dtype f32|f64] [--skip-header]
//   dnd bench  ALGO [--ranks P] [--data F.dnb | --synthetic RxC | --samples N]
//              [--seed S] [--split 0|1|none] [--axis 0|1|none] [--k K] [--iters N]
//              [--lambda L] [--ddof D] [--warmup W] [--runs R] [--out json]
//   dnd verify ALGO [same data/algorithm flags] [--tol T] [--inject-combiner-fault]
//
// ALGO is moments | cdist | kmeans | lasso, plus `load` (times dnb_load of
// --data into the HBM shards).  --algo ALGO is accepted too.  Defaults follow
// tools/options.hpp:22-98 (ranks = $DND_RANKS or 1, per-algorithm default
// shapes, 30 k-means / 20 lasso iterations, lambda 0.1, tol 1e-10).  The
// reference's float64 data become fp32 on the B200 hot path (BASELINE: fp32),
// so verify's default gate is BASELINE's (1e-5 distances/centroids/weights,
// 1e-12 moments) unless --tol is given.
//
// bench prints one JSON object: the reference's report keys (bench.cpp:120-129)
// plus GB/s, the fraction of p x the measured HBM copy peak and NVML clocks.
// verify prints the reference's gate lines (verify.cpp:35-50, :283-300) and
// exits 1 on a failed gate.  A dnd::Error exits 2 (main.cpp:78-82), a usage
// error 2 as CLI11 does.
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
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "dnd/dnd.hpp"

namespace {

int ranks_from_env() {
    if (const char* e = std::getenv("DND_RANKS")) {
        const int v = std::atoi(e);
        if (v >= 1) return v;
    }
    return 1;
}

struct Options {
    std::string cmd, algo, data;  // data: DNB path (else synthetic)
    dnd::index_t rows = 0, cols = 0, samples = 0;
    int k = 8, iters = 0, ranks = ranks_from_env(), warmup = 1, runs = 9;
    std::int64_t ddof = 0;
    double lambda = 0.1, tol = -1.0;  // tol < 0: BASELINE's gate for the algorithm
    bool inject_combiner_fault = false;
    std::string split = "0", axis = "none", out = "json";
    std::uint64_t seed = 42;
    double peak_gbs = 6451.8;  // MEASURED_PEAKS.json hbm_gbs (copy bandwidth)
    // convert
    std::string src, dst, dtype = "f64";
    bool skip_header = false;
    std::optional<int> split_axis() const {
        if (split == "none") return std::nullopt;
        return split == "1" ? 1 : 0;
    }
};

[[noreturn]] void usage(const std::string& why) {
    std::fprintf(stderr,
                 "dnd: %s\nusage: dnd convert SRC DST [--dtype f32|f64] [--skip-header]\n"
                 "       dnd bench|verify ALGO [--ranks P] [--data F.dnb | --synthetic RxC | --samples N] "
                 "[--seed S] [--split 0|1|none] [--axis 0|1|none] [--k K] [--iters N] [--lambda L] [--ddof D] "
                 "[--warmup W] [--runs R] [--out json] [--tol T] [--inject-combiner-fault] [--peak-gbs G]\n"
                 "       ALGO: moments | cdist | kmeans | lasso | load\n",
                 why.c_str());
    std::exit(2);
}

Options parse(int argc, char** argv) {
    if (argc < 2) usage("a subcommand is required");
    Options o;
    o.cmd = argv[1];
    if (o.cmd != "bench" && o.cmd != "verify" && o.cmd != "convert") usage("unknown subcommand " + o.cmd);
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--", 0) != 0) {
            pos.push_back(a);
            continue;
        }
        if (a == "--skip-header") { o.skip_header = true; continue; }
        if (a == "--inject-combiner-fault") { o.inject_combiner_fault = true; continue; }
        if (i + 1 >= argc) usage("missing value for " + a);
        const std::string v = argv[++i];
        if (a == "--algo") o.algo = v;
        else if (a == "--data") o.data = v;
        else if (a == "--synthetic") {
            const auto x = v.find('x');
            if (x == std::string::npos) usage("--synthetic expects ROWSxCOLS, got \"" + v + "\"");
            o.rows = std::atoll(v.substr(0, x).c_str());
            o.cols = std::atoll(v.substr(x + 1).c_str());
            if (o.rows < 0 || o.cols < 0) usage("--synthetic extents must be nonnegative");
        } else if (a == "--samples") o.samples = std::atoll(v.c_str());
        else if (a == "--k") o.k = std::atoi(v.c_str());
        else if (a == "--iters") o.iters = std::atoi(v.c_str());
        else if (a == "--ranks") o.ranks = std::atoi(v.c_str());
        else if (a == "--warmup") o.warmup = std::atoi(v.c_str());
        else if (a == "--runs") o.runs = std::atoi(v.c_str());
        else if (a == "--seed") o.seed = std::strtoull(v.c_str(), nullptr, 10);
        else if (a == "--split") o.split = v;
        else if (a == "--axis") o.axis = v;
        else if (a == "--lambda") o.lambda = std::atof(v.c_str());
        else if (a == "--ddof") o.ddof = std::atoll(v.c_str());
        else if (a == "--tol") o.tol = std::atof(v.c_str());
        else if (a == "--out") o.out = v;
        else if (a == "--dtype") o.dtype = v;
        else if (a == "--peak-gbs") o.peak_gbs = std::atof(v.c_str());
        else usage("unknown option " + a);
    }
    if (o.cmd == "convert") {
        if (pos.size() != 2) usage("convert takes SRC and DST");
        if (o.dtype != "f32" && o.dtype != "f64") usage("--dtype must be f32 or f64");
        o.src = pos[0];
        o.dst = pos[1];
        return o;
    }
    if (o.algo.empty()) {
        if (pos.size() != 1) usage("bench/verify take one ALGO");
        o.algo = pos[0];
    } else if (!pos.empty()) {
        usage("unexpected argument " + pos[0]);
    }
    if (o.algo != "kmeans" && o.algo != "cdist" && o.algo != "moments" && o.algo != "load" && o.algo != "lasso")
        usage("ALGO must be moments, cdist, kmeans, lasso or load, got " + o.algo);
    if (o.split != "0" && o.split != "1" && o.split != "none") usage("--split must be 0, 1 or none");
    if (o.axis != "0" && o.axis != "1" && o.axis != "none") usage("--axis must be 0, 1 or none");
    if (o.algo == "load" && o.data.empty()) usage("load times dnb_load of --data");
    if (!o.data.empty()) {  // shape from the container header (options.hpp:71-90)
        const auto h = dnd::dnb_read_header(o.data);
        if (h.extents.size() != 2) throw dnd::ValueError("--data needs a 2-D DNB container");
        o.rows = static_cast<dnd::index_t>(h.extents[0]);
        o.cols = static_cast<dnd::index_t>(h.extents[1]);
    } else if (o.samples > 0) {
        o.rows = o.samples;
        o.cols = 18;
    } else if (o.rows == 0 && o.cols == 0) {  // per-algorithm defaults (options.hpp:84-96)
        if (o.algo == "moments") { o.rows = 300; o.cols = 1000; }
        else if (o.algo == "cdist") { o.rows = 2000; o.cols = 18; }
        else if (o.algo == "kmeans") { o.rows = 600; o.cols = 8; }
        else { o.rows = 1000; o.cols = 21; }
    }
    if (o.iters == 0) o.iters = o.algo == "lasso" ? 20 : 30;
    if (o.iters < 1) throw dnd::ValueError("--iters must be positive");
    if (o.runs < 1) throw dnd::ValueError("--runs must be at least 1");
    if (o.warmup < 0) throw dnd::ValueError("--warmup must be nonnegative");
    if (o.out != "json") throw dnd::ValueError("--out supports only \"json\", got \"" + o.out + "\"");
    if (o.ranks < 1) throw dnd::ValueError("--ranks must be positive");
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

// Deliberately broken combiner of `verify --inject-combiner-fault`
// (verify.cpp:57-73): drops the between-chunk term of M2, so distributed
// variances come out wrong whenever chunk means differ -- proves the gate bites.
dnd::MomentState corrupt_combine(dnd::MomentState a, const dnd::MomentState& b) {
    if (a.count == 0) return b;
    if (b.count == 0) return a;
    dnd::MomentState out;
    out.count = a.count + b.count;
    out.mean.resize(a.arity());
    out.m2.resize(a.arity());
    const double na = static_cast<double>(a.count), nb = static_cast<double>(b.count);
    for (std::size_t i = 0; i < a.arity(); ++i) {
        out.mean[i] = (na * a.mean[i] + nb * b.mean[i]) / (na + nb);
        out.m2[i] = a.m2[i] + b.m2[i];
    }
    return out;
}

// what verify compares (rank 0's replicated results)
struct Result {
    std::vector<double> values, trace, extra;
    std::vector<std::int32_t> labels;
    bool rounds_ok = true;
};

// one run of the algorithm; returns a scalar that depends on the result
// (kept, like the reference's sink, so nothing is optimised away) and fills
// `out` with the replicated result for verify
double run_algo(const Options& o, const dnd::DndArray<float>& x, const LassoData* ld, Result* out) {
    const dnd::Communicator& comm = x.comm();
    if (o.algo == "load") {  // the DNB container into the HBM shards (dataio.hpp:102-142)
        const auto y = dnd::dnb_load<float>(o.data, o.split_axis(), comm);
        if (out) {
            const auto g = dnd::gather(y);
            out->values.assign(g.begin(), g.end());
        }
        return y.numel_local() > 0 ? 1.0 : 0.0;
    }
    if (o.algo == "lasso") {  // --iters sweeps at --lambda (regression.cpp:25-102)
        const auto model = dnd::lasso_fit(ld->first, ld->second, o.lambda, o.iters, 0.0);
        if (out) {
            out->values = model.weights;
            out->trace = model.objective_trace;
        }
        return model.objective_trace.back();
    }
    if (o.algo == "kmeans") {
        const auto model = dnd::kmeans_fit(x, o.k, o.iters, 0.0, o.seed);
        if (out) {
            out->values = model.centroids;
            out->trace = model.inertia_trace;
            out->labels = dnd::gather(dnd::kmeans_predict(model, x.split() && *x.split() != 0 ? dnd::resplit(x, 0) : x));
        }
        return model.inertia_trace.back();
    }
    if (o.algo == "cdist") {
        const auto before = comm.counters().sendrecvs;
        const auto d = dnd::cdist(x);
        if (out) {
            out->rounds_ok = comm.counters().sendrecvs - before ==
                             static_cast<std::uint64_t>(x.split() == std::optional<int>(0) ? comm.size() - 1 : 0);
            const auto g = dnd::gather(d);
            out->values.assign(g.begin(), g.end());
        }
        float first = 0.f;
        if (d.numel_local() > 1)
            dnd::detail::check(dndc_memcpy(comm.handle(), &first, d.device_data() + 1, sizeof(float), DNDC_COPY_D2H));
        return first;
    }
    // moments: the scalars (flattened) and the axis-0 columns (moments.cpp:126-140)
    double mean = 0.0, var = 0.0;
    if (o.inject_combiner_fault && comm.size() > 1) {
        const auto t = x.tile();
        dnd::Tile<double> td{t.extents, std::vector<double>(t.data.begin(), t.data.end())};
        const auto st = comm.allreduce(dnd::local_moments(td), corrupt_combine, dnd::MomentState::identity(1));
        mean = st.mean[0];
        var = st.m2[0] / static_cast<double>(st.count - o.ddof);
    } else {
        mean = dnd::mean(x);
        var = dnd::var(x, o.ddof);
    }
    if (out) {
        out->values = {mean, var, std::sqrt(var)};
        if (o.axis == "0" || !o.inject_combiner_fault) {
            out->extra = dnd::gather(dnd::mean_axis(x, 0));
            const auto sd = dnd::gather(dnd::stddev_axis(x, 0, o.ddof));
            out->extra.insert(out->extra.end(), sd.begin(), sd.end());
        }
    } else if (o.axis == "0") {
        const auto mu = dnd::mean_axis(x, 0);
        const auto sd = dnd::stddev_axis(x, 0, o.ddof);
        return mean + static_cast<double>(mu.numel_global()) + static_cast<double>(sd.numel_global());
    }
    return mean + var;
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
// narrowed to the fp32 hot path), or random_uniform<float>, on --split
dnd::DndArray<float> make_input(const Options& o, const dnd::Communicator& comm) {
    const auto split = o.split_axis();
    if (o.data.empty()) return dnd::random_uniform<float>({o.rows, o.cols}, split, o.seed, comm);
    if (dnd::dnb_read_header(o.data).dtype == dnd::DnbDtype::f32) return dnd::dnb_load<float>(o.data, split, comm);
    return dnd::astype<float>(dnd::dnb_load<double>(o.data, split, comm));
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
        if (o.algo == "kmeans" && static_cast<dnd::index_t>(o.k) > x.shape()[0])
            throw dnd::ValueError("kmeans: k=" + std::to_string(o.k) + " exceeds " + std::to_string(x.shape()[0]) +
                                  " samples");
        if (o.algo == "cdist" && x.shape()[0] == 0) throw dnd::ValueError("cdist: data has no rows");
        std::unique_ptr<LassoData> ld;
        if (o.algo == "lasso") ld = std::make_unique<LassoData>(make_lasso(o, x));
        double sink = 0.0;
        for (int w = 0; w < o.warmup; ++w) sink += run_algo(o, x, ld.get(), nullptr);
        if (comm.rank() == 0) clocks.start();
        // slowest rank per run (bench.cpp:102-112)
        std::vector<double> mine;
        for (int r = 0; r < o.runs; ++r) {
            comm.barrier();
            const auto t0 = std::chrono::steady_clock::now();
            sink += run_algo(o, x, ld.get(), nullptr);
            comm.barrier();
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            mine.push_back(comm.allreduce(el, [](double a, double b) { return a > b ? a : b; }, 0.0));
        }
        if (comm.rank() == 0) clocks.stop();
        if (!std::isfinite(sink)) throw dnd::ValueError("benchmark produced non-finite results");
        std::lock_guard<std::mutex> lock(mu);
        if (comm.rank() == 0) secs = mine;
    });
    const auto st = dnd::local_moments(dnd::Tile<double>{{static_cast<dnd::index_t>(secs.size())}, secs});
    std::string runs;
    for (double t : secs) runs += (runs.empty() ? "" : ", ") + std::to_string(t);
    const double mean = st.mean[0], sd = std::sqrt(st.m2[0] / static_cast<double>(st.count));
    std::string params = "\"seed\": " + std::to_string(o.seed) + ", \"rows\": " + std::to_string(o.rows) +
                         ", \"cols\": " + std::to_string(o.cols);
    if (o.algo == "moments")
        params += ", \"axis\": " + std::string(o.axis == "none" ? "null" : o.axis) + ", \"ddof\": " + std::to_string(o.ddof);
    else if (o.algo == "kmeans")
        params += ", \"k\": " + std::to_string(o.k) + ", \"iters\": " + std::to_string(o.iters);
    else if (o.algo == "lasso")
        params += ", \"lambda\": " + std::to_string(o.lambda) + ", \"iters\": " + std::to_string(o.iters);
    const std::string split = o.split == "none" ? "\"none\"" : o.split;
    std::printf("{\"algo\": \"%s\", \"ranks\": %d, \"split\": %s, \"params\": {%s}, \"warmup_runs\": %d, "
                "\"timed_runs\": %d, \"mean_seconds\": %.9g, \"std_seconds\": %.9g, \"GB_per_s\": %.6g, "
                "\"roofline_frac\": %.4f, \"peak_gbs_per_gpu\": %.1f, \"clocks\": %s, \"device\": \"B200 (libdndc)\", "
                "\"run_seconds\": [%s]}\n",
                o.algo.c_str(), o.ranks, split.c_str(), params.c_str(), o.warmup, o.runs, mean, sd,
                bytes_per_run(o) / mean / 1e9, bytes_per_run(o) / mean / 1e9 / (o.peak_gbs * std::min(o.ranks, 8)),
                o.peak_gbs, clocks.json().c_str(), runs.c_str());
    return 0;
}

// the reference's gate printer (verify.cpp:20-50): |a-b| / max(1, |ref|)
struct Gate {
    bool ok = true;
    void deviation(const char* what, const std::vector<double>& a, const std::vector<double>& ref, double tol) {
        double mabs = 0.0, mrel = 0.0;
        bool same = a.size() == ref.size();
        for (std::size_t i = 0; same && i < a.size(); ++i) {
            const double d = std::fabs(a[i] - ref[i]);
            mabs = std::max(mabs, d);
            mrel = std::max(mrel, d / std::max(1.0, std::fabs(ref[i])));
        }
        const bool pass = same && mrel <= tol;
        std::printf("  %-18s max_abs=%.3e max_rel=%.3e  %s\n", what, mabs, mrel, pass ? "OK" : "FAIL");
        ok = ok && pass;
    }
    void flag(const char* what, bool pass) {
        std::printf("  %-18s %s\n", what, pass ? "OK" : "FAIL");
        ok = ok && pass;
    }
};

bool nonincreasing(const std::vector<double>& t, double slack) {
    for (std::size_t i = 1; i < t.size(); ++i)
        if (t[i] > t[i - 1] + slack * std::max(1.0, std::fabs(t[i - 1]))) return false;
    return true;
}

int verify(const Options& o) {
    auto collect = [&](int ranks) {
        Result res;
        std::mutex mu;
        dnd::run_world(ranks, [&](const dnd::Communicator& comm) {
            const auto x = make_input(o, comm);
            std::unique_ptr<LassoData> ld;
            if (o.algo == "lasso") ld = std::make_unique<LassoData>(make_lasso(o, x));
            Result r;
            run_algo(o, x, ld.get(), &r);
            const bool all_ok = comm.allreduce(r.rounds_ok, [](bool a, bool b) { return a && b; }, true);
            std::lock_guard<std::mutex> lock(mu);
            if (comm.rank() == 0) {
                res = std::move(r);
                res.rounds_ok = all_ok;
            }
        });
        return res;
    };
    // fp32 hot path: BASELINE's gates unless --tol (the reference's 1e-10 is for f64 end to end)
    const double tol = o.tol >= 0 ? o.tol : (o.algo == "moments" ? 1e-12 : (o.algo == "lasso" ? 1e-9 : 1e-5));
    std::printf("verify %s ranks=%d split=%s rows=%lld cols=%lld seed=%llu tol=%.1e\n", o.algo.c_str(), o.ranks,
                o.split.c_str(), static_cast<long long>(o.rows), static_cast<long long>(o.cols),
                static_cast<unsigned long long>(o.seed), tol);
    const Result dist = collect(o.ranks), ref = collect(1);
    Gate gate;
    if (o.algo == "moments") {
        gate.deviation("mean/var/std", dist.values, ref.values, tol);
        if (!dist.extra.empty()) gate.deviation("axis-0 moments", dist.extra, ref.extra, tol);
    } else if (o.algo == "cdist") {
        gate.deviation("distances", dist.values, ref.values, tol);
        const dnd::index_t n = o.rows;
        bool diag = true, sym = true, nonneg = true;
        for (dnd::index_t i = 0; i < n; ++i)
            for (dnd::index_t j = 0; j < n; ++j) {
                const double dij = dist.values[static_cast<std::size_t>(i * n + j)];
                const double dji = dist.values[static_cast<std::size_t>(j * n + i)];
                if (i == j) diag = diag && dij == 0.0;
                sym = sym && std::fabs(dij - dji) <= 1e-5 * std::max(1.0, std::fabs(dij));
                nonneg = nonneg && dij >= 0.0;
            }
        gate.flag("zero diagonal", diag);
        gate.flag("symmetry", sym);
        gate.flag("nonnegativity", nonneg);
        gate.flag("ring rounds p-1", dist.rounds_ok);
    } else if (o.algo == "kmeans") {
        gate.deviation("centroids", dist.values, ref.values, tol);
        gate.deviation("inertia trace", dist.trace, ref.trace, tol);
        gate.flag("labels identical", dist.labels == ref.labels);
        gate.flag("inertia monotone", nonincreasing(dist.trace, 1e-9));
    } else if (o.algo == "lasso") {
        gate.deviation("weights", dist.values, ref.values, tol);
        gate.flag("objective monotone", nonincreasing(dist.trace, 1e-9));
    } else {
        gate.deviation("loaded values", dist.values, ref.values, 0.0);
    }
    std::printf("result: %s\n", gate.ok ? "OK" : "FAIL");
    return gate.ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options o = parse(argc, argv);
        if (o.cmd == "convert") {  // main.cpp:66-73
            dnd::csv_to_dnb(o.src, o.dst, o.dtype == "f32" ? dnd::DnbDtype::f32 : dnd::DnbDtype::f64, o.skip_header);
            const auto h = dnd::dnb_read_header(o.dst);
            std::fprintf(stderr, "wrote %s (%lldx%lld, %s)\n", o.dst.c_str(), static_cast<long long>(h.extents[0]),
                         static_cast<long long>(h.extents.size() > 1 ? h.extents[1] : 1), o.dtype.c_str());
            return 0;
        }
        return o.cmd == "bench" ? bench(o) : verify(o);
    } catch (const dnd::Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
