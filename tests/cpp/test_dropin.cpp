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
    if (failures) {
        std::fprintf(stderr, "%d of %d checks failed\n", failures, checks);
        return 1;
    }
    std::printf("ok %d\n", checks);
    return 0;
}
