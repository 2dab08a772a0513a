// C++ drop-in check: the reference's own unit-test cases (proj/tests/
// test_music.cpp, test_gsvd.cpp) written against include/sslgpu/ssl.hpp and
// run on the GPU engine.  Prints "ok <n>" and exits 0 when every check holds.
#include <sslgpu/ssl.hpp>

#include <cmath>
#include <cstdio>
#include <random>

static int failures = 0, checks = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        ++checks;                                                     \
        if (!(c)) {                                                   \
            ++failures;                                               \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
        }                                                             \
    } while (0)

static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol * (1 + std::fabs(b)); }

int main() {
    // test_music.cpp:110-146 — worked two-channel example
    {
        ssl::SteeringField steer;
        steer.m = 2;
        steer.directions = {{0, 0}, {90, 0}};
        steer.vectors = {{1, 0}, {1, 0}, {0, 1}, {0, -1}};
        ssl::GsvdBatch<float> basis;
        basis.bins.resize(1);
        basis.bins[0].e = ssl::CMatrix<float>(2, 2);
        basis.bins[0].e(0, 0) = 1.0f;
        basis.bins[0].e(1, 1) = 0.5f;
        ssl::MusicConfig cfg;
        const auto s = ssl::calc_average_power<float>(basis, steer, cfg, true);
        CHECK(near(s.power[0], 4.0, 1e-12) && near(s.power[1], 4.0, 1e-12));
        CHECK(near(s.bin_power[0][0], 4.0, 1e-12));
        cfg.squared_denominator = true;
        CHECK(near(ssl::calc_average_power<float>(basis, steer, cfg).power[0], 8.0, 1e-12));
    }
    // test_music.cpp:240-316 — topology and peak search on the 72-azimuth ring
    {
        std::vector<ssl::Direction> dirs;
        for (int i = 0; i < 72; ++i) dirs.push_back({i * 5.0, 0.0});
        const auto topo = ssl::DirectionTopology::build(dirs, 11.0);
        for (const auto& n : topo.neighbors) CHECK(n.size() == 4);
        std::vector<double> p(72, 1.0);
        p[7] = 5.0;
        p[6] = p[8] = 2.0;
        auto est = ssl::peak_search(p, dirs, topo, ssl::MusicConfig{});
        CHECK(est.size() == 1 && est[0].direction_index == 7 && !est[0].low_power);
        std::vector<double> flat(72, 2.0);
        est = ssl::peak_search(flat, dirs, topo, ssl::MusicConfig{});
        CHECK(est.size() == 1 && est[0].direction_index == 0 && est[0].low_power);
    }
    // test_gsvd.cpp:120-131 — 2x2 closed form; 191-204 — K = 2I halves values
    {
        std::mt19937_64 rng(121);
        std::normal_distribution<double> nd;
        for (int trial = 0; trial < 10; ++trial) {
            ssl::CorrelationSet r;
            r.m = 2;
            r.bins.assign(1, ssl::CMatrix<float>(2, 2));
            for (auto& z : r.bins[0].data) z = {float(nd(rng)), float(nd(rng))};
            const auto& a = r.bins[0];
            const double s = std::norm(std::complex<double>(a(0, 0))) + std::norm(std::complex<double>(a(0, 1))) +
                             std::norm(std::complex<double>(a(1, 0))) + std::norm(std::complex<double>(a(1, 1)));
            const auto det = std::complex<double>(a(0, 0)) * std::complex<double>(a(1, 1)) -
                             std::complex<double>(a(0, 1)) * std::complex<double>(a(1, 0));
            const double disc = std::sqrt(std::max(0.0, s * s - 4 * std::norm(det)));
            const auto got = ssl::gsvd_reference(ssl::NoiseModel::identity(2, 1), r);
            CHECK(near(got.bins[0].singular_values[0], std::sqrt((s + disc) / 2), 1e-10));
            CHECK(std::fabs(got.bins[0].singular_values[1] - std::sqrt(std::max(0.0, (s - disc) / 2))) <=
                  1e-10 * std::sqrt((s + disc) / 2));
        }
        ssl::CorrelationSet r;
        r.m = 4;
        r.bins.assign(1, ssl::CMatrix<float>(4, 4));
        for (std::size_t i = 0; i < 4; ++i)
            for (std::size_t j = 0; j < 4; ++j) r.bins[0](i, j) = float(1.0 / (1 + i + j));
        auto k2 = ssl::NoiseModel::identity(4, 1);
        for (std::size_t i = 0; i < 4; ++i) k2.k.bins[0](i, i) = 2.0f;
        const auto plain = ssl::gsvd_reference(ssl::NoiseModel::identity(4, 1), r);
        const auto white = ssl::gsvd_reference(k2, r);
        for (int i = 0; i < 4; ++i)
            CHECK(near(white.bins[0].singular_values[i], plain.bins[0].singular_values[i] / 2, 1e-12));
    }
    // test_gsvd.cpp:57-65 / 292-302 — error taxonomy
    {
        auto sing = ssl::NoiseModel::identity(3, 2);
        sing.k.bins[1] = ssl::CMatrix<float>(3, 3);
        ssl::CorrelationSet r;
        r.m = 3;
        r.bins.assign(2, ssl::CMatrix<float>::identity(3));
        bool threw = false;
        try {
            ssl::gsvd_reference(sing, r);
        } catch (const ssl::NumericalError& e) {
            threw = std::string(e.what()).find("1") != std::string::npos;
        }
        CHECK(threw);
        ssl::NoiseModel ind;
        ind.k.m = 2;
        ind.k.bins.assign(1, ssl::CMatrix<float>(2, 2));
        ind.k.bins[0](0, 0) = 1;
        ind.k.bins[0](0, 1) = 3;
        ind.k.bins[0](1, 0) = 3;
        ind.k.bins[0](1, 1) = 1;
        threw = false;
        try {
            ind.check_positive_definite();
        } catch (const ssl::NumericalError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // pipeline.hpp:71-75 — run_locate on a SampleBlock (device STFT) gives the
    // estimates run_locate gives on that block's STFT frames
    {
        const std::uint32_t m = 4, nsamp = 4000;
        ssl::StftConfig sc;
        sc.bin_min = 10;
        sc.bin_max = 40;
        ssl::SteeringField st;
        st.m = m;
        st.bin_min = sc.bin_min;
        st.bin_max = sc.bin_max;
        for (int a = 0; a < 36; ++a) st.directions.push_back({10.0 * a, 0.0});
        const double pi = 3.14159265358979323846;
        for (const auto& d : st.directions)
            for (std::uint32_t b = sc.bin_min; b <= sc.bin_max; ++b)
                for (std::uint32_t i = 0; i < m; ++i) {
                    const double ang = 2 * pi * i / m, az = d.azimuth_deg * pi / 180;
                    const double tau = -0.05 * (std::cos(az) * std::cos(ang) + std::sin(az) * std::sin(ang)) / 343.0;
                    const double ph = -2 * pi * (b * 16000.0 / 512) * tau;
                    st.vectors.push_back({float(std::cos(ph)), float(std::sin(ph))});
                }
        ssl::SampleBlock blk;
        std::mt19937_64 rng(5);
        std::normal_distribution<double> nd;
        blk.channels.assign(m, std::vector<float>(nsamp));
        for (std::uint32_t n = 0; n < nsamp; ++n) {
            const double s0 = nd(rng);
            for (std::uint32_t i = 0; i < m; ++i) blk.channels[i][n] = float(s0 + 0.3 * nd(rng));
        }
        const auto noise = ssl::NoiseModel::identity(m, sc.bin_count());
        ssl::MusicConfig mc;
        mc.num_sources = 1;
        std::vector<ssl::FrameEstimates> a, b;
        const auto na = ssl::run_locate(blk, sc, 8, noise, st, ssl::SolverConfig{}, mc, ssl::SolvePath::batched, 4,
                                        [&](const ssl::FrameEstimates& fe) { a.push_back(fe); });
        // frames of the same block through the stage entry point
        ssl::Engine e(m, sc.bin_count(), 8, mc, ssl::SolverConfig{});
        sslg_stft_config c{sc.frame_length, sc.shift, 0, sc.bin_min, sc.bin_max};
        ssl::check(sslg_set_stft(e.get(), &c));
        std::vector<float> pcm;
        for (const auto& ch : blk.channels) pcm.insert(pcm.end(), ch.begin(), ch.end());
        std::uint32_t nf = 0;
        ssl::check(sslg_stft(e.get(), pcm.data(), nsamp, nullptr, 0, &nf));
        std::vector<float> fr(std::size_t(nf) * m * sc.bin_count() * 2);
        ssl::check(sslg_stft(e.get(), pcm.data(), nsamp, fr.data(), nf, &nf));
        std::vector<ssl::SpectrumFrame> frames(nf);
        for (std::uint32_t f = 0; f < nf; ++f) {
            frames[f].frame_index = f;
            frames[f].spectra.assign(m, std::vector<ssl::cfloat>(sc.bin_count()));
            for (std::uint32_t i = 0; i < m; ++i)
                for (std::uint32_t k = 0; k < sc.bin_count(); ++k) {
                    const std::size_t o = ((std::size_t(f) * m + i) * sc.bin_count() + k) * 2;
                    frames[f].spectra[i][k] = {fr[o], fr[o + 1]};
                }
        }
        const auto nb = ssl::run_locate(frames, 8, noise, st, ssl::SolverConfig{}, mc, 4,
                                        [&](const ssl::FrameEstimates& fe) { b.push_back(fe); });
        CHECK(na == nb && na == nf - 7 && a.size() == b.size());
        for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) {
            CHECK(a[i].frame_index == b[i].frame_index);
            CHECK(a[i].estimates.size() == b[i].estimates.size());
            for (std::size_t j = 0; j < a[i].estimates.size() && j < b[i].estimates.size(); ++j) {
                CHECK(a[i].estimates[j].direction_index == b[i].estimates[j].direction_index);
                CHECK(a[i].estimates[j].power == b[i].estimates[j].power);
            }
        }
    }
    // test_correlation.cpp:67-120 -- CorrelationWindow against brute force,
    // the rebuild cadence, underfill and shape changes
    {
        auto random_frame = [](std::uint32_t index, std::size_t m, std::size_t bins, std::mt19937_64& rng) {
            std::normal_distribution<double> nd;
            ssl::SpectrumFrame f;
            f.frame_index = index;
            f.spectra.assign(m, std::vector<ssl::cfloat>(bins));
            for (auto& ch : f.spectra)
                for (auto& v : ch) v = ssl::cfloat(float(nd(rng)), float(nd(rng)));
            return f;
        };
        const std::size_t m = 3, bins = 4, t = 5;
        std::mt19937_64 rng(23);
        ssl::CorrelationWindow window(t);
        std::vector<ssl::SpectrumFrame> hist;
        for (std::uint32_t i = 0; i < 17; ++i) {
            hist.push_back(random_frame(i, m, bins, rng));
            window.push(hist.back());
            if (i + 1 < t) {
                CHECK(!window.filled());
                continue;
            }
            CHECK(window.filled());
            const auto got = window.normalized();
            CHECK(got.frame_index == i);
            for (std::size_t b = 0; b < bins; ++b)
                for (std::size_t r = 0; r < m; ++r)
                    for (std::size_t c = 0; c < m; ++c) {
                        ssl::cdouble want(0, 0);
                        for (std::size_t k = hist.size() - t; k < hist.size(); ++k)
                            want += ssl::cdouble(hist[k].spectra[r][b]) * std::conj(ssl::cdouble(hist[k].spectra[c][b]));
                        want /= double(t);
                        CHECK(std::abs(ssl::cdouble(got.bins[b](r, c)) - want) <= 1e-6 * (1.0 + std::abs(want)));
                    }
        }
        ssl::CorrelationWindow frequent(4, 3), rare(4, 1000000);
        std::mt19937_64 rng2(31);
        for (std::uint32_t i = 0; i < 40; ++i) {
            const auto f = random_frame(i, 2, 2, rng2);
            frequent.push(f);
            rare.push(f);
            if (!frequent.filled()) continue;
            const auto a = frequent.normalized(), b = rare.normalized();
            for (std::size_t bin = 0; bin < 2; ++bin)
                for (std::size_t q = 0; q < 4; ++q) CHECK(std::abs(a.bins[bin].data[q] - b.bins[bin].data[q]) <= 1e-6f);
        }
        ssl::CorrelationWindow small(3);
        std::mt19937_64 rng3(5);
        small.push(random_frame(0, 2, 2, rng3));
        bool threw = false;
        try {
            small.normalized();
        } catch (const ssl::ValidationError&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            small.push(random_frame(1, 3, 2, rng3));
        } catch (const ssl::ValidationError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // test_gsvd.cpp:36-76 -- inverses, pivot-free elimination
    {
        ssl::NoiseModel piv;
        piv.k.m = 2;
        piv.k.bins.assign(1, ssl::CMatrix<float>(2, 2));
        piv.k.bins[0](0, 1) = 1;
        piv.k.bins[0](1, 0) = 1;
        piv.prepare_inverses(ssl::Pivoting::partial);
        const auto inv = piv.inverse_double(0);
        CHECK(std::abs(inv(0, 1) - ssl::cdouble(1, 0)) <= 1e-14 && std::abs(inv(0, 0)) <= 1e-14);
        bool threw = false;
        try {
            piv.prepare_inverses(ssl::Pivoting::none);
        } catch (const ssl::NumericalError&) {
            threw = true;
        }
        CHECK(threw);
        std::mt19937_64 rng(101);
        std::normal_distribution<double> nd;
        for (std::size_t n : {1, 2, 5, 8}) {
            ssl::NoiseModel nm;
            nm.k.m = std::uint32_t(n);
            nm.k.bins.assign(1, ssl::CMatrix<float>(n, n));
            ssl::CMatrix<double> a(n, n);
            for (auto& z : a.data) z = {nd(rng), nd(rng)};
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) {
                    ssl::cdouble v(0, 0);
                    for (std::size_t q = 0; q < n; ++q) v += a(i, q) * std::conj(a(j, q));
                    nm.k.bins[0](i, j) = ssl::cfloat(float(v.real() / n + (i == j ? 0.5 : 0)), float(v.imag() / n));
                }
            nm.prepare_inverses(ssl::Pivoting::partial);
            const auto ki = nm.inverse_double(0);
            double err = 0;
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) {
                    ssl::cdouble v(0, 0);
                    for (std::size_t q = 0; q < n; ++q) v += ssl::cdouble(nm.k.bins[0](i, q)) * ki(q, j);
                    err = std::max(err, std::abs(v - ssl::cdouble(i == j ? 1 : 0, 0)));
                }
            CHECK(err <= 1e-12);
        }
    }
    // test_gsvd.cpp:159-223 -- E_r, the residual, budgets
    {
        std::mt19937_64 rng(127);
        std::normal_distribution<double> nd;
        ssl::CorrelationSet r;
        r.m = 5;
        r.bins.assign(1, ssl::CMatrix<float>(5, 5));
        for (auto& z : r.bins[0].data) z = {float(nd(rng)), float(nd(rng))};
        ssl::SolverConfig cfg;
        cfg.compute_residual = true;
        const auto noise = ssl::NoiseModel::identity(5, 1);
        const auto got = ssl::gsvd_reference(noise, r, cfg);
        const auto& g = got.bins[0];
        CHECK(g.recon_residual >= 0.0 && g.recon_residual <= 1e-12);
        double err = 0, ref = 0, def = 0;
        for (std::size_t i = 0; i < 5; ++i)
            for (std::size_t j = 0; j < 5; ++j) {
                ssl::cdouble v(0, 0), u(0, 0);
                for (std::size_t q = 0; q < 5; ++q) {
                    v += g.e(i, q) * g.singular_values[q] * g.e_r(q, j);
                    u += std::conj(g.e_r(q, i)) * g.e_r(q, j);  // E_r^H E_r
                }
                err += std::norm(v - ssl::cdouble(r.bins[0](i, j)));
                ref += std::norm(ssl::cdouble(r.bins[0](i, j)));
                def += std::norm(u - ssl::cdouble(i == j ? 1 : 0, 0));
            }
        CHECK(std::sqrt(err / ref) <= 1e-12 && std::sqrt(def) <= 1e-10);
        ssl::SolverConfig tight;
        tight.max_qr_sweeps = 1;
        ssl::CorrelationSet r12;
        r12.m = 12;
        r12.bins.assign(1, ssl::CMatrix<float>(12, 12));
        for (auto& z : r12.bins[0].data) z = {float(nd(rng)), float(nd(rng))};
        CHECK(!ssl::gsvd(ssl::NoiseModel::identity(12, 1), r12, tight).bins[0].converged);
        CHECK(ssl::gsvd(ssl::NoiseModel::identity(12, 1), r12).bins[0].converged);
        // repeated solves reuse the noise model's device context
        const auto again = ssl::gsvd_reference(noise, r, cfg);
        CHECK(again.bins[0].singular_values == g.singular_values);
        bool threw = false;
        try {
            ssl::SolverConfig bad;
            bad.tolerance_scale = 0;
            ssl::gsvd(noise, r, bad);
        } catch (const ssl::ValidationError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // files: save/load round trips, NoiseModel::from_file, JSONL records
    {
        ssl::CorrelationSet k;
        k.m = 2;
        k.bins.assign(3, ssl::CMatrix<float>::identity(2));
        k.bins[1](0, 1) = {0.25f, -0.5f};
        k.bins[1](1, 0) = {0.25f, 0.5f};
        ssl::save_correlation("/tmp/sslg_dropin_k.sslc", k, 7);
        std::uint32_t t = 0;
        const auto back = ssl::load_correlation("/tmp/sslg_dropin_k.sslc", &t);
        CHECK(t == 7 && back.m == 2 && back.bins.size() == 3 && back.bins[1](0, 1) == k.bins[1](0, 1));
        const auto nm = ssl::NoiseModel::from_file("/tmp/sslg_dropin_k.sslc");
        CHECK(nm.k.bins[1](1, 0) == k.bins[1](1, 0));
        ssl::SteeringField st;
        st.m = 2;
        st.bin_min = 3;
        st.bin_max = 4;
        st.directions = {{0, 0}, {90, 10.5}};
        st.vectors = {{1, 0}, {0, 1}, {1, 1}, {0, -1}, {2, 0}, {0, 2}, {3, 3}, {-1, 0}};
        ssl::save_steering(st, "/tmp/sslg_dropin_h.steer");
        const auto s2 = ssl::load_steering("/tmp/sslg_dropin_h.steer");
        CHECK(s2.m == 2 && s2.bin_min == 3 && s2.bin_max == 4 && s2.directions.size() == 2 &&
              s2.directions[1].elevation_deg == 10.5 && s2.vectors == st.vectors);
        bool threw = false;
        try {
            ssl::load_correlation("/tmp/sslg_dropin_missing.sslc");
        } catch (const ssl::IoError&) {
            threw = true;
        }
        CHECK(threw);
        ssl::FrameEstimates fe;
        fe.frame_index = 49;
        fe.estimates.push_back({8, {40.0, 0.0}, 12.5, false});
        fe.estimates.push_back({30, {150.0, 0.0}, 3.0, true});
        CHECK(ssl::format_estimates_json(fe) ==
              "{\"estimates\":[{\"azimuth_deg\":40.0,\"direction\":8,\"elevation_deg\":0.0,\"low_power\":false,"
              "\"power\":12.5},{\"azimuth_deg\":150.0,\"direction\":30,\"elevation_deg\":0.0,\"low_power\":true,"
              "\"power\":3.0}],\"frame\":49}");
    }
    if (failures) {
        std::fprintf(stderr, "%d of %d checks failed\n", failures, checks);
        return 1;
    }
    std::printf("ok %d\n", checks);
    return 0;
}
