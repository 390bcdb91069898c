// C++ drop-in tests: the reference's own test cases (proj/tests/test_pairwise.cpp,
// test_cluster.cpp, test_moments.cpp, test_chunking.cpp) written against the
// B200 dnd API, run with one rank per visible GPU (up to 2).
//
//     make -C cpp test && cpp/build/test_dnd
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "dnd/dnd.hpp"

using dnd::Communicator;
using dnd::index_t;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)          \
    do {                                     \
        bool thrown = false;                 \
        try {                                \
            (void)(expr);                    \
        } catch (const type&) {              \
            thrown = true;                   \
        }                                    \
        CHECK(thrown&& #expr " throws " #type); \
    } while (0)

static bool close_rel(double a, double b, double tol) { return std::abs(a - b) <= tol * std::max(1.0, std::abs(b)); }

// naive_cdist (oracles.hpp:61-73): the reference formula, f64, no FMA
static std::vector<double> naive_cdist(const std::vector<double>& x, index_t n, const std::vector<double>& y,
                                       index_t ny, index_t m) {
    std::vector<double> nx(n), nyv(ny), out(n * ny);
    auto sq = [&](const std::vector<double>& a, index_t i) {
        volatile double acc = 0.0;
        for (index_t f = 0; f < m; ++f) {
            volatile double p = a[i * m + f] * a[i * m + f];
            acc = acc + p;
        }
        return static_cast<double>(acc);
    };
    for (index_t i = 0; i < n; ++i) nx[i] = sq(x, i);
    for (index_t j = 0; j < ny; ++j) nyv[j] = sq(y, j);
    for (index_t i = 0; i < n; ++i)
        for (index_t j = 0; j < ny; ++j) {
            volatile double g = 0.0;
            for (index_t f = 0; f < m; ++f) {
                volatile double p = x[i * m + f] * y[j * m + f];
                g = g + p;
            }
            volatile double s = nx[i] + nyv[j];
            volatile double t = 2.0 * g;
            const double d = s - t;
            out[i * ny + j] = std::sqrt(d > 0.0 ? d : 0.0);
        }
    return out;
}

static void each_world(const std::function<void(const Communicator&)>& body) {
    int ndev = 0;
    dnd::detail::check(dndc_device_count(&ndev));
    for (int p = 1; p <= std::min(ndev, 2); ++p) dnd::run_world(p, body);
}

int main() {
    // chunking (test_chunking.cpp:10-14)
    {
        const auto m = dnd::chunk_map(5, 3);
        CHECK((m.extents == std::vector<index_t>{2, 2, 1}));
        CHECK((m.offsets == std::vector<index_t>{0, 2, 4}));
    }
    each_world([](const Communicator& comm) {
        // (0,0),(3,4) -> [[0,5],[5,0]] exactly (test_pairwise.cpp:23-28)
        auto x64 = dnd::from_global<double>({0, 0, 3, 4}, {2, 2}, 0, comm);
        CHECK((dnd::gather(dnd::cdist(x64)) == std::vector<double>{0, 5, 5, 0}));
        auto x32 = dnd::from_global<float>({0, 0, 3, 4}, {2, 2}, 0, comm);
        CHECK((dnd::gather(dnd::cdist(x32)) == std::vector<float>{0, 5, 5, 0}));

        // repeated rows -> 0 (test_pairwise.cpp:16-21)
        std::vector<double> rep;
        for (int i = 0; i < 5; ++i) rep.insert(rep.end(), {1.0, 2.0, 3.0});
        const auto d_rep = dnd::gather(dnd::cdist(dnd::from_global<double>(rep, {5, 3}, 0, comm)));
        CHECK(std::all_of(d_rep.begin(), d_rep.end(), [](double v) { return v == 0.0; }));

        // cdist f64 bit-exact against the naive oracle; cdist_xy too
        const index_t n = 37, ny = 11, m = 6;
        auto xa = dnd::random_uniform<double>({n, m}, 0, 7, comm);
        auto ya = dnd::random_uniform<double>({ny, m}, std::nullopt, 8, comm);
        const auto xh = dnd::gather(xa), yh = dnd::gather(ya);
        CHECK(dnd::gather(dnd::cdist(xa)) == naive_cdist(xh, n, xh, n, m));
        CHECK(dnd::gather(dnd::cdist_xy(xa, ya)) == naive_cdist(xh, n, yh, ny, m));
        const auto c0 = comm.counters();
        dnd::cdist_xy(xa, ya);
        CHECK(comm.counters().sendrecvs == c0.sendrecvs);  // communication-free (test_pairwise.cpp:146-166)

        // fp32 within the parity gate (1e-5 rel)
        auto xf = dnd::random_uniform<float>({n, m}, 0, 7, comm);
        const auto df = dnd::gather(dnd::cdist(xf));
        const auto ref = naive_cdist(xh, n, xh, n, m);  // same values: random_uniform<float> == f32(f64)
        double dev = 0.0;
        const auto xfh = dnd::gather(xf);
        const auto ref32 = naive_cdist(std::vector<double>(xfh.begin(), xfh.end()), n,
                                       std::vector<double>(xfh.begin(), xfh.end()), n, m);
        for (std::size_t i = 0; i < df.size(); ++i)
            dev = std::max(dev, std::abs(df[i] - ref32[i]) / std::max(1.0, std::abs(ref32[i])));
        CHECK(dev <= 1e-5);
        (void)ref;

        // distance to a zero row = sqrt(|x|^2) (test_pairwise.cpp:116-133)
        dnd::Tile<double> a{{2, 3}, {1, 2, 2, 0, 3, 4}};
        dnd::Tile<double> z{{1, 3}, {0, 0, 0}};
        const auto blk = dnd::detail::distance_block(a, dnd::detail::row_norms(a), z, dnd::detail::row_norms(z));
        CHECK(blk.data[0] == 3.0 && blk.data[1] == 5.0);

        // predict (test_cluster.cpp:221-241)
        dnd::KMeansModel model;
        model.k = 3;
        model.n_features = 2;
        model.centroids = {0, 0, 5, 5, 9, 0};
        auto xp = dnd::from_global<double>({0, 0, 5, 5, 9, 0}, {3, 2}, 0, comm);
        CHECK((dnd::gather(dnd::kmeans_predict(model, xp)) == std::vector<std::int32_t>{0, 1, 2}));
        dnd::KMeansModel tie;
        tie.k = 2;
        tie.n_features = 1;
        tie.centroids = {0.0, 2.0};
        auto xt = dnd::from_global<double>({1.0, 1.0}, {2, 1}, 0, comm);
        CHECK((dnd::gather(dnd::kmeans_predict(tie, xt)) == std::vector<std::int32_t>{0, 0}));

        // k = 1 -> the global mean (test_cluster.cpp:119-132)
        auto xk = dnd::random_uniform<double>({101, 4}, 0, 3, comm);
        const auto xkh = dnd::gather(xk);
        const auto m1 = dnd::kmeans_fit(xk, 1, 3, 0.0, 5);
        for (int f = 0; f < 4; ++f) {
            double s = 0.0;
            for (int i = 0; i < 101; ++i) s += xkh[i * 4 + f];
            CHECK(close_rel(m1.centroids[f], s / 101.0, 1e-12));
        }

        // two clouds -> their exact means (test_cluster.cpp:83-117)
        std::vector<float> cl;
        for (int i = 0; i < 40; ++i) cl.insert(cl.end(), {0.0f + 0.01f * (i % 7), 0.0f + 0.02f * (i % 5)});
        for (int i = 0; i < 40; ++i) cl.insert(cl.end(), {10.0f + 0.01f * (i % 3), 10.0f + 0.03f * (i % 4)});
        auto xc = dnd::from_global<float>(cl, {80, 2}, 0, comm);
        const auto mc = dnd::kmeans_fit(xc, 2, 10, 0.0, 1);
        double mean_a[2] = {0, 0}, mean_b[2] = {0, 0};
        for (int i = 0; i < 40; ++i)
            for (int f = 0; f < 2; ++f) {
                mean_a[f] += static_cast<double>(cl[i * 2 + f]) / 40.0;
                mean_b[f] += static_cast<double>(cl[(40 + i) * 2 + f]) / 40.0;
            }
        const bool a_first = mc.centroids[0] < 5.0;
        const double* ca = a_first ? &mc.centroids[0] : &mc.centroids[2];
        const double* cb = a_first ? &mc.centroids[2] : &mc.centroids[0];
        if (!close_rel(ca[0], mean_a[0], 1e-12))
            std::fprintf(stderr, "p=%d clouds: %.17g %.17g | %.17g %.17g vs %.17g %.17g | %.17g %.17g (iters %d)\n",
                         comm.size(), mc.centroids[0], mc.centroids[1], mc.centroids[2], mc.centroids[3], mean_a[0],
                         mean_a[1], mean_b[0], mean_b[1], mc.iterations_run);
        CHECK(close_rel(ca[0], mean_a[0], 1e-12) && close_rel(ca[1], mean_a[1], 1e-12));
        CHECK(close_rel(cb[0], mean_b[0], 1e-12) && close_rel(cb[1], mean_b[1], 1e-12));
        for (std::size_t i = 1; i < mc.inertia_trace.size(); ++i)
            CHECK(mc.inertia_trace[i] <= mc.inertia_trace[i - 1] * (1 + 1e-12));

        // validation (test_cluster.cpp:285-300)
        auto xv = dnd::from_global<double>({1, 2, 3, 4}, {2, 2}, 0, comm);
        CHECK_THROWS_AS(dnd::kmeans_fit(xv, 3, 5, 0.0, 1), dnd::ValueError);
        CHECK_THROWS_AS(dnd::kmeans_fit(xv, 1, 0, 0.0, 1), dnd::ValueError);
        auto xnan = dnd::from_global<double>({1, NAN, 3, 4}, {2, 2}, 0, comm);
        CHECK_THROWS_AS(dnd::kmeans_fit(xnan, 1, 2, 0.0, 1), dnd::ValueError);
        auto v1 = dnd::from_global<double>({1, 2, 3}, {3}, 0, comm);
        CHECK_THROWS_AS(dnd::cdist(v1), dnd::ValueError);

        // moments: [1,2,3,4] -> mean 2.5, var 1.25 / 5/3 (test_moments.cpp:46-56, :182-192)
        auto mv = dnd::from_global<double>({1, 2, 3, 4}, {4, 1}, 0, comm);
        CHECK(dnd::mean(mv) == 2.5);
        CHECK(close_rel(dnd::var(mv), 1.25, 1e-15));
        CHECK(close_rel(dnd::var(mv, 1), 5.0 / 3.0, 1e-15));
        CHECK(close_rel(dnd::gather(dnd::var_axis(mv, 0, 1))[0], 5.0 / 3.0, 1e-15));
        // the 1e8 offset (test_moments.cpp:160-180): single pass stays accurate
        std::vector<double> off;
        for (int i = 0; i < 1000; ++i) off.push_back(1e8 + (i % 10));
        auto xo = dnd::from_global<double>(off, {1000, 1}, 0, comm);
        CHECK(close_rel(dnd::var(xo), 8.25, 1e-9));
        // combine with the identity returns the operand exactly
        auto st = dnd::local_moments(dnd::Tile<double>{{3}, {1, 5, 9}});
        const auto st2 = dnd::combine(st, dnd::MomentState::identity(1));
        CHECK(st2.count == st.count && st2.mean == st.mean && st2.m2 == st.m2);
        // random_uniform is split- and rank-count independent (A1)
        auto r1 = dnd::random_uniform<float>({53, 5}, 0, 42, comm);
        auto r2 = dnd::random_uniform<float>({53, 5}, std::nullopt, 42, comm);
        CHECK(dnd::gather(r1) == dnd::gather(r2));
    });

    // resplit (test_ndarray.cpp:205-260, acceptance.cpp:70-89): every split
    // transition preserves the content bitwise, lands on the requested axis,
    // and balances the new axis per its chunk map; ranks 1..visible GPUs
    {
        std::vector<double> data3(5 * 7 * 3);
        for (std::size_t i = 0; i < data3.size(); ++i) data3[i] = std::sin(0.37 * static_cast<double>(i)) * 100.0;
        const std::vector<std::optional<int>> splits{std::nullopt, 0, 1, 2};
        each_world([&](const Communicator& comm) {
            for (const auto& from : splits)
                for (const auto& to : splits) {
                    auto a = dnd::from_global(data3, {5, 7, 3}, from, comm);
                    auto r = dnd::resplit(a, to);
                    CHECK(r.split() == to);
                    CHECK(dnd::gather(r) == data3);
                    if (to) CHECK(r.lshape()[static_cast<std::size_t>(*to)] == r.split_chunks().extent(comm.rank()));
                }
            auto a0 = dnd::from_global(data3, {5, 7, 3}, 0, comm);
            CHECK(dnd::resplit(dnd::resplit(a0, 1), 0).tile().data == a0.tile().data);
            // 2 x 4, split=1 -> none on every rank
            const std::vector<double> mat{1, 2, 3, 4, 5, 6, 7, 8};
            auto r = dnd::resplit(dnd::from_global(mat, {2, 4}, 1, comm), std::nullopt);
            CHECK(!r.split() && r.lshape() == std::vector<index_t>({2, 4}) && r.tile().data == mat);
            // f32 through the same machinery (test_ndarray.cpp:290-300)
            std::vector<float> f(24);
            for (int i = 0; i < 24; ++i) f[i] = static_cast<float>(i) * 0.25f;
            CHECK(dnd::gather(dnd::resplit(dnd::from_global(f, {4, 6}, 1, comm), 0)) == f);
            // random_uniform with split=1 equals split=0 content
            CHECK(dnd::gather(dnd::random_uniform<float>({37, 9}, 1, 42, comm)) ==
                  dnd::gather(dnd::random_uniform<float>({37, 9}, 0, 42, comm)));
        });
        // cdist of inputs with other splits (test_pairwise.cpp:47-58)
        const index_t n = 23, m = 5;
        std::vector<double> data(n * m);
        for (std::size_t i = 0; i < data.size(); ++i) data[i] = std::cos(0.91 * static_cast<double>(i));
        const auto expected = naive_cdist(data, n, data, n, m);
        each_world([&](const Communicator& comm) {
            for (auto split : {std::optional<int>(1), std::optional<int>()}) {
                auto x = dnd::from_global(data, {n, m}, split, comm);
                const auto d = dnd::gather(dnd::cdist(x));
                double dev = 0.0;
                for (std::size_t i = 0; i < d.size(); ++i) dev = std::max(dev, std::abs(d[i] - expected[i]));
                CHECK(dev <= 1e-8);
                // kmeans_fit and moments on the same layouts match split=0
                auto x0 = dnd::from_global(data, {n, m}, 0, comm);
                const auto ma = dnd::kmeans_fit(x, 3, 10, 0.0, 7), mb = dnd::kmeans_fit(x0, 3, 10, 0.0, 7);
                CHECK(ma.centroids == mb.centroids && ma.iterations_run == mb.iterations_run);
                const auto va = dnd::gather(dnd::var_axis(x, 0)), vb = dnd::gather(dnd::var_axis(x0, 0));
                for (index_t c = 0; c < m; ++c) CHECK(close_rel(va[c], vb[c], 1e-14));
            }
            CHECK_THROWS_AS(dnd::kmeans_predict(dnd::kmeans_fit(dnd::from_global(data, {n, m}, 0, comm), 2, 3, 0.0, 1),
                                                dnd::from_global(data, {n, m}, 1, comm)),
                            dnd::ValueError);
        });
    }

    // DNB containers (test_dataio.cpp:26-220), loaded straight into HBM
    {
        namespace fs = std::filesystem;
        const fs::path dir = fs::temp_directory_path() / ("dnd_dataio_" + std::to_string(::getpid()));
        fs::create_directories(dir);
        auto write_text = [&](const std::string& name, const std::string& text) {
            std::ofstream(dir / name) << text;
            return (dir / name).string();
        };
        std::vector<double> d60(60);
        for (std::size_t i = 0; i < d60.size(); ++i) d60[i] = std::sin(1.7 * static_cast<double>(i) + 0.3);
        const std::vector<index_t> shape{5, 4, 3};
        const std::vector<std::optional<int>> splits{std::nullopt, 0, 1, 2};
        each_world([&](const Communicator& comm) {
            const auto path = (dir / ("rt" + std::to_string(comm.size()))).string();
            for (const auto& ss : splits)
                for (const auto& ls : splits) {
                    dnd::dnb_save(dnd::from_global(d60, shape, ss, comm), path);
                    auto b = dnd::dnb_load<double>(path, ls, comm);
                    CHECK(b.shape() == shape && b.split() == ls && dnd::gather(b) == d60);
                }
            // f32 round trip; loading as f64 names the dtype_code
            std::vector<float> f24(24);
            for (int i = 0; i < 24; ++i) f24[i] = static_cast<float>(i) / 7.0f;
            const auto fpath = (dir / ("f" + std::to_string(comm.size()))).string();
            dnd::dnb_save(dnd::from_global(f24, {6, 4}, 0, comm), fpath);
            CHECK(dnd::gather(dnd::dnb_load<float>(fpath, 0, comm)) == f24);
            CHECK_THROWS_AS(dnd::dnb_load<double>(fpath, 0, comm), dnd::DataError);
            CHECK(dnd::dnb_read_header(fpath).dtype == dnd::DnbDtype::f32);
            // chunked loads slice like the chunk map; replicated == gathered chunks
            const auto apath = (dir / ("a" + std::to_string(comm.size()))).string();
            dnd::dnb_save(dnd::from_global<double>({0, 1, 2, 3, 4}, {5}, std::nullopt, comm), apath);
            const auto part = dnd::dnb_load<double>(apath, 0, comm).tile().data;
            const auto map = dnd::chunk_map(5, comm.size());
            std::vector<double> want;
            for (index_t i = map.offset(comm.rank()); i < map.end(comm.rank()); ++i) want.push_back(double(i));
            CHECK(part == want);
            CHECK(dnd::dnb_load<double>(apath, std::nullopt, comm).tile().data ==
                  dnd::gather(dnd::dnb_load<double>(apath, 0, comm)));
            // an empty array gives a header-only file
            const auto epath = (dir / ("e" + std::to_string(comm.size()))).string();
            dnd::dnb_save(dnd::from_global<double>({}, {0, 7}, 0, comm), epath);
            auto e = dnd::dnb_load<double>(epath, 0, comm);
            CHECK(e.shape() == std::vector<index_t>({0, 7}) && e.numel_local() == 0);
            CHECK(fs::file_size(epath) == 6 + 8 * 2);
        });
        // header law: 6 + 8 ndim + 8 numel bytes
        dnd::run_world(1, [&](const Communicator& comm) {
            const std::vector<std::vector<index_t>> shapes{{3}, {2, 5}, {4, 1, 6}};
            for (const auto& sh : shapes) {
                const auto path = (dir / "law").string();
                dnd::dnb_save(dnd::random_uniform<double>(sh, std::nullopt, 3, comm), path);
                CHECK(fs::file_size(path) == 6 + 8 * sh.size() + 8 * static_cast<std::uint64_t>(dnd::detail::product(sh)));
            }
        });
        // malformed containers name the field
        const auto good = (dir / "good.dnb").string();
        dnd::run_world(1, [&](const Communicator& comm) {
            dnd::dnb_save(dnd::from_global<double>({0, 1, 2, 3}, {4}, std::nullopt, comm), good);
        });
        auto clone = [&](const std::string& name, std::size_t cut, long at, char v) {
            std::ifstream in(good, std::ios::binary);
            std::vector<char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
            bytes.resize(bytes.size() - cut);
            if (at >= 0) bytes[static_cast<std::size_t>(at)] = v;
            std::ofstream(dir / name, std::ios::binary).write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
            return (dir / name).string();
        };
        auto throws_with = [](auto&& fn, const std::string& needle) {
            try {
                fn();
            } catch (const dnd::DataError& e) {
                return std::string(e.what()).find(needle) != std::string::npos;
            }
            return false;
        };
        CHECK(throws_with([&] { dnd::dnb_read_header(clone("magic.dnb", 0, 0, 'X')); }, "magic"));
        CHECK(throws_with([&] { dnd::dnb_read_header(clone("dtype.dnb", 0, 4, 9)); }, "dtype_code"));
        const auto trunc = clone("short.dnb", 8, -1, 0);
        dnd::run_world(1, [&](const Communicator& comm) {
            CHECK(throws_with([&] { dnd::dnb_load<double>(trunc, std::nullopt, comm); }, "truncated"));
        });
        CHECK_THROWS_AS(dnd::dnb_read_header((dir / "missing.dnb").string()), dnd::DataError);
        // CSV conversion
        const auto m_dnb = (dir / "m.dnb").string();
        dnd::csv_to_dnb(write_text("m.csv", "1,2\n3,4\n"), m_dnb);
        std::string text;
        std::vector<double> expect;
        for (int i = 0; i < 7; ++i)
            for (int j = 0; j < 4; ++j) {
                const double v = std::cos(0.1 * (i * 4 + j)) * 100.0 - 50.0;
                expect.push_back(v);
                char buf[64];
                std::snprintf(buf, sizeof buf, "%.17g", v);
                text += buf;
                text += j + 1 < 4 ? "," : "\n";
            }
        const auto r_dnb = (dir / "r.dnb").string();
        dnd::csv_to_dnb(write_text("r.csv", text), r_dnb);
        const auto h_dnb = (dir / "h.dnb").string();
        dnd::csv_to_dnb(write_text("h.csv", "a,b\n1.5,2.5\n3.5, 4.5\n"), h_dnb, dnd::DnbDtype::f32, true);
        each_world([&](const Communicator& comm) {
            auto a = dnd::dnb_load<double>(m_dnb, std::nullopt, comm);
            CHECK(a.shape() == std::vector<index_t>({2, 2}) && a.tile().data == std::vector<double>({1, 2, 3, 4}));
            CHECK(dnd::gather(dnd::dnb_load<double>(r_dnb, 0, comm)) == expect);
            auto hf = dnd::dnb_load<float>(h_dnb, std::nullopt, comm);
            CHECK(hf.tile().data == std::vector<float>({1.5f, 2.5f, 3.5f, 4.5f}));
        });
        CHECK(throws_with([&] { dnd::csv_to_dnb(write_text("rag.csv", "1,2\n3\n"), (dir / "o").string()); }, "line 2"));
        CHECK(throws_with([&] { dnd::csv_to_dnb(write_text("gar.csv", "1,2\n3,x\n"), (dir / "o").string()); },
                          "line 2"));
        CHECK_THROWS_AS(dnd::csv_to_dnb(write_text("empty.csv", "\n"), (dir / "o").string()), dnd::DataError);
        fs::remove_all(dir);
    }

    // LASSO (test_regression.cpp:83-230) against a sequential restatement of
    // regression.cpp:25-102 (one rank, row order)
    {
        struct Problem {
            index_t n, m;
            std::vector<double> x, y;
        };
        auto make_problem = [](index_t n, index_t m, int seed) {
            Problem p{n, m, std::vector<double>(n * m), std::vector<double>(n)};
            std::vector<double> beta(m);
            for (index_t j = 0; j < m; ++j) beta[j] = std::sin(1.3 * (j + seed)) * 3.0;
            for (index_t i = 0; i < n; ++i) {
                double yi = 0.0;
                for (index_t j = 0; j < m; ++j) {
                    // hash-style pseudo-random features (independent columns)
                    const double h = std::sin(12.9898 * static_cast<double>(i) + 78.233 * static_cast<double>(j) +
                                              static_cast<double>(seed)) * 43758.5453;
                    const double v = j == 0 ? 1.0 : h - std::floor(h) - 0.5;
                    p.x[i * m + j] = v;
                    yi += v * beta[j];
                }
                p.y[i] = yi + 0.05 * std::cos(3.1 * i + seed);
            }
            return p;
        };
        auto naive = [](const Problem& p, double lam, int sweeps, double tol, std::vector<double>& trace) {
            std::vector<double> sq(p.m, 0.0), w(p.m, 0.0), r = p.y;
            for (index_t i = 0; i < p.n; ++i)
                for (index_t j = 0; j < p.m; ++j) sq[j] += p.x[i * p.m + j] * p.x[i * p.m + j];
            trace.clear();
            for (int s = 0; s < sweeps; ++s) {
                double mc = 0.0;
                for (index_t j = 0; j < p.m; ++j) {
                    if (sq[j] == 0.0) continue;
                    double rho = 0.0;
                    for (index_t i = 0; i < p.n; ++i) {
                        const double x = p.x[i * p.m + j];
                        rho += x * (r[i] + w[j] * x);
                    }
                    const double wn = j == 0 ? rho / sq[0] : dnd::soft_threshold(rho, lam / 2.0) / sq[j];
                    if (wn != w[j])
                        for (index_t i = 0; i < p.n; ++i) r[i] += (w[j] - wn) * p.x[i * p.m + j];
                    mc = std::max(mc, std::abs(wn - w[j]));
                    w[j] = wn;
                }
                double ssr = 0.0, pen = 0.0;
                for (double v : r) ssr += v * v;
                for (index_t j = 1; j < p.m; ++j) pen += std::abs(w[j]);
                trace.push_back(ssr + lam * pen);
                if (mc < tol) break;
            }
            return w;
        };
        CHECK(dnd::soft_threshold(0.5, 1.0) == 0.0 && dnd::soft_threshold(2.0, 0.5) == 1.5);
        CHECK(dnd::soft_threshold(-2.0, 0.5) == -1.5 && dnd::soft_threshold(3.0, 0.0) == 3.0);
        const auto p1 = make_problem(300, 20, 151), p2 = make_problem(2000, 7, 3);
        auto zc = make_problem(40, 6, 167);
        for (index_t i = 0; i < zc.n; ++i) zc.x[i * zc.m + 3] = 0.0;
        each_world([&](const Communicator& comm) {
            for (const Problem* pp : {&p1, &p2, static_cast<const Problem*>(&zc)}) {
                const Problem& p = *pp;
                for (double lam : {0.0, 1.0, 30.0}) {
                    std::vector<double> tr;
                    const auto want = naive(p, lam, 25, 0.0, tr);
                    auto x = dnd::from_global(p.x, {p.n, p.m}, 0, comm);
                    auto y = dnd::from_global(p.y, {p.n}, 0, comm);
                    const auto model = dnd::lasso_fit(x, y, lam, 25);
                    CHECK(model.sweeps_run == 25 && model.objective_trace.size() == 25);
                    bool ok = true;
                    for (index_t j = 0; j < p.m; ++j) ok &= close_rel(model.weights[j], want[j], 1e-9);
                    for (int t = 0; t < 25; ++t) ok &= close_rel(model.objective_trace[t], tr[t], 1e-10);
                    for (int t = 1; t < 25; ++t) ok &= model.objective_trace[t] <= model.objective_trace[t - 1] + 1e-9;
                    CHECK(ok);
                }
            }
            CHECK(dnd::lasso_fit(dnd::from_global(zc.x, {zc.n, zc.m}, 0, comm),
                                 dnd::from_global(zc.y, {zc.n}, 0, comm), 0.5, 50)
                      .weights[3] == 0.0);
            // tol stops early, the same sweep as the restatement
            std::vector<double> tr;
            naive(p2, 1.0, 500, 1e-10, tr);
            const auto mt = dnd::lasso_fit(dnd::from_global(p2.x, {p2.n, p2.m}, 0, comm),
                                           dnd::from_global(p2.y, {p2.n}, 0, comm), 1.0, 500, 1e-10);
            CHECK(mt.sweeps_run < 500 && std::abs(mt.sweeps_run - static_cast<int>(tr.size())) <= 1);
            // replicated / split=1 inputs give the split=0 fit
            const auto ms = dnd::lasso_fit(dnd::from_global(p2.x, {p2.n, p2.m}, 1, comm),
                                           dnd::from_global(p2.y, {p2.n}, std::nullopt, comm), 1.0, 20);
            const auto m0 = dnd::lasso_fit(dnd::from_global(p2.x, {p2.n, p2.m}, 0, comm),
                                           dnd::from_global(p2.y, {p2.n}, 0, comm), 1.0, 20);
            CHECK(ms.weights == m0.weights);
            // y = 1 + 2x on 3 samples (more ranks than samples on 2+ GPUs)
            const auto tiny = dnd::lasso_fit(dnd::from_global<double>({1, 0.0, 1, 1.0, 1, 2.0}, {3, 2}, 0, comm),
                                             dnd::from_global<double>({1.0, 3.0, 5.0}, {3}, 0, comm), 0.0, 200,
                                             1e-15);
            CHECK(std::abs(tiny.weights[0] - 1.0) <= 1e-10 && std::abs(tiny.weights[1] - 2.0) <= 1e-10);
            // predict: bit-identical to the row loop
            auto xp = dnd::from_global(p1.x, {p1.n, p1.m}, 0, comm);
            dnd::LassoModel dense;
            for (index_t j = 0; j < p1.m; ++j) dense.weights.push_back(0.25 * j - 1.0);
            const auto got = dnd::gather(dnd::lasso_predict(dense, xp));
            bool exact = true;
            for (index_t i = 0; i < p1.n; ++i) {
                volatile double acc = 0.0;
                for (index_t j = 0; j < p1.m; ++j) {
                    volatile double prod = p1.x[i * p1.m + j] * dense.weights[j];
                    acc = acc + prod;
                }
                exact &= got[i] == acc;
            }
            CHECK(exact);
            // validation (test_regression.cpp:214-230): every rank raises
            auto x4 = dnd::from_global<double>({1, 1, 1, 1, 1, 1, 1, 1}, {4, 2}, 0, comm);
            auto y4 = dnd::from_global<double>({1, 1, 1, 1}, {4}, 0, comm);
            auto y3 = dnd::from_global<double>({1, 1, 1}, {3}, 0, comm);
            CHECK_THROWS_AS(dnd::lasso_fit(x4, y3, 0.1, 5), dnd::ValueError);
            CHECK_THROWS_AS(dnd::lasso_fit(x4, y4, -1.0, 5), dnd::ValueError);
            CHECK_THROWS_AS(dnd::lasso_fit(x4, y4, 0.1, 0), dnd::ValueError);
            CHECK_THROWS_AS(dnd::lasso_fit(y4, y4, 0.1, 5), dnd::ValueError);
            auto xbad = dnd::from_global<double>({1, 1, 1, 1, 1, 1, 2, 1}, {4, 2}, 0, comm);
            CHECK_THROWS_AS(dnd::lasso_fit(xbad, y4, 0.1, 5), dnd::ValueError);
        });
    }
    std::printf("test_dnd: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
