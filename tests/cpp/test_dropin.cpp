// The reference's hot-path unit tests (proj/tests/test_denoise.cpp and
// test_parallel.cpp), restated as plain checks and compiled against the
// drop-in headers in include/phgrms/ -- i.e. code written for the reference
// API, unchanged, now running on the B200 kernels.  Built by
// __graft_entry__.build(); run by tests/test_dropin_gpu.py on a GPU.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <limits>
#include <sstream>
#include <string>
#include <random>
#include <stdexcept>

#include "phgrms/bench.hpp"
#include "phgrms/pgm_gpu.hpp"
#include "phgrms/denoise.hpp"
#include "phgrms/image.hpp"
#include "phgrms/metrics.hpp"
#include "phgrms/noise.hpp"
#include "phgrms/pgm.hpp"

using namespace phgrms;

static int g_fail = 0, g_checks = 0;
static std::string g_golden_dir = "tests/golden";
#define CHECK(x)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(x)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #x); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, ex)    \
    do {                             \
        bool thrown_ = false;        \
        try {                        \
            (void)(expr);            \
        } catch (const ex&) {        \
            thrown_ = true;          \
        }                            \
        CHECK(thrown_);              \
    } while (0)

static GrayImage random_image(std::mt19937& rng, int w, int h) {
    GrayImage img(w, h);
    for (auto& p : img.pixels) p = static_cast<std::uint8_t>(rng() & 0xFF);
    return img;
}

int main(int argc, char** argv) {
    if (argc > 1) g_golden_dir = argv[1];
    {  // cardinality of a constant image equals the in-bounds window size
        const auto card = compute_cardinality(GrayImage(3, 3, 100), 20, 1);
        CHECK((card.counts == std::vector<std::int32_t>{4, 6, 4, 6, 9, 6, 4, 6, 4}));
    }
    {  // cardinality isolates a centre impulse
        GrayImage img(3, 3, 100);
        img.at(1, 1) = 255;
        CHECK((compute_cardinality(img, 20, 1).counts == std::vector<std::int32_t>{3, 5, 3, 5, 1, 5, 3, 5, 3}));
        const auto [out, st] = denoise_pass(img, compute_cardinality(img, 20, 1), DenoiseParams{});
        CHECK(out == GrayImage(3, 3, 100));
        CHECK(st.flagged == 1 && st.replaced == 1);
    }
    {  // border mode forks the corner behaviour
        GrayImage img(4, 4, 50);
        img.at(0, 0) = 255;
        const auto card = compute_cardinality(img, 20, 1);
        CHECK(card.at(0, 0) == 1);
        const auto [kept, ks] = denoise_pass(img, card, DenoiseParams{});
        CHECK(kept == img && ks.flagged == 1 && ks.replaced == 0);
        DenoiseParams inb;
        inb.border = BorderMode::InBounds;
        const auto [fixed, fs] = denoise_pass(img, card, inb);
        CHECK(fixed == GrayImage(4, 4, 50) && fs.replaced == 1);
    }
    {  // two adjacent impulses clear in pass 1 and stop in pass 2
        GrayImage img(7, 7, 100);
        img.at(3, 3) = img.at(3, 4) = 255;
        const auto r = denoise(img, DenoiseParams{});
        CHECK(r.image == GrayImage(7, 7, 100));
        CHECK(r.stats.size() == 2 && r.stats[0].replaced == 2 && r.stats[1].replaced == 0);
    }
    {  // driver stops after one clean pass on a constant image
        const auto r = denoise(GrayImage(64, 64, 77), DenoiseParams{});
        CHECK(r.stats.size() == 1 && r.stats[0].iteration == 1 && r.stats[0].replaced == 0);
    }
    {  // an isolated interior impulse is restored exactly in one pass
        std::mt19937 rng(105);
        for (int i = 0; i < 30; ++i) {
            const int v = static_cast<int>(rng() % 256);
            DenoiseParams p;
            p.alpha = 1 + static_cast<int>(rng() % 100);
            const int imp = static_cast<int>(rng() % 256);
            if (std::abs(imp - v) < p.alpha) continue;
            GrayImage img(5, 5, static_cast<std::uint8_t>(v));
            img.at(2, 2) = static_cast<std::uint8_t>(imp);
            const auto r = denoise(img, p);
            CHECK(r.stats.front().replaced == 1);
            CHECK(r.image == GrayImage(5, 5, static_cast<std::uint8_t>(v)));
        }
    }
    {  // faithful borders never rewrite beta=1 corners; C >= thr untouched
        std::mt19937 rng(104);
        for (int i = 0; i < 20; ++i) {
            const GrayImage img = random_image(rng, 7, 7);
            DenoiseParams p;
            p.alpha = 1 + static_cast<int>(rng() % 255);
            const auto card = compute_cardinality(img, p.alpha, p.beta);
            const auto [out, st] = denoise_pass(img, card, p);
            for (int r : {0, 6})
                for (int c : {0, 6}) CHECK(out.at(r, c) == img.at(r, c));
            for (std::size_t j = 0; j < img.size(); ++j)
                if (card.counts[j] >= p.card_threshold) CHECK(out.pixels[j] == img.pixels[j]);
            CHECK(st.replaced <= st.flagged);
        }
    }
    {  // parallel output is bit-identical to serial for any worker count
        std::mt19937 rng(201);
        for (int i = 0; i < 25; ++i) {
            const GrayImage img = random_image(rng, 1 + static_cast<int>(rng() % 32), 1 + static_cast<int>(rng() % 32));
            DenoiseParams p;
            p.alpha = 1 + static_cast<int>(rng() % 60);
            p.beta = 1 + static_cast<int>(rng() % 2);
            p.border = (rng() & 1) ? BorderMode::InBounds : BorderMode::Faithful;
            const auto serial = denoise(img, p, EngineSpec::serial());
            for (const int w : {2, 3, 8}) {
                const auto par = denoise(img, p, EngineSpec::parallel(w));
                CHECK(par.image == serial.image);
                CHECK(par.stats.size() == serial.stats.size());
                for (std::size_t s = 0; s < par.stats.size() && s < serial.stats.size(); ++s)
                    CHECK(par.stats[s].flagged == serial.stats[s].flagged &&
                          par.stats[s].replaced == serial.stats[s].replaced);
            }
        }
    }
    {  // PHGRMS_DEVICES: Parallel(W) bands spread over GPUs (device 0 listed twice)
        setenv("PHGRMS_DEVICES", "0,0", 1);
        std::mt19937 rng(202);
        for (int i = 0; i < 10; ++i) {
            const GrayImage img = random_image(rng, 16 + static_cast<int>(rng() % 600), 8 + static_cast<int>(rng() % 300));
            DenoiseParams p;
            p.beta = 1 + static_cast<int>(rng() % 2);
            p.max_iterations = 1 + static_cast<int>(rng() % 9);
            const auto serial = denoise(img, p, EngineSpec::serial());
            for (const int w : {2, 5}) {
                const auto par = denoise(img, p, EngineSpec::parallel(w));
                CHECK(par.image == serial.image);
                CHECK(par.stats.size() == serial.stats.size());
                for (std::size_t s = 0; s < par.stats.size() && s < serial.stats.size(); ++s)
                    CHECK(par.stats[s].flagged == serial.stats[s].flagged &&
                          par.stats[s].replaced == serial.stats[s].replaced);
            }
        }
        unsetenv("PHGRMS_DEVICES");
    }
    {  // a zero-replacement pass is a fixed point
        std::mt19937 rng(106);
        for (int i = 0; i < 10; ++i) {
            const GrayImage img = random_image(rng, 12, 12);
            DenoiseParams p;
            p.alpha = 1 + static_cast<int>(rng() % 120);
            p.max_iterations = 8;
            const auto r = denoise(img, p);
            if (r.stats.back().replaced == 0) {
                const auto [again, st] = denoise_pass(r.image, compute_cardinality(r.image, p.alpha, p.beta), p);
                CHECK(again == r.image && st.replaced == 0);
            }
        }
    }
    {  // parameter validation + rms rounding + row blocks
        const GrayImage img(4, 4, 1);
        DenoiseParams p;
        p.alpha = 0;
        CHECK_THROWS_AS(denoise(img, p), std::invalid_argument);
        p = {};
        p.beta = 0;
        CHECK_THROWS_AS(denoise(img, p), std::invalid_argument);
        p = {};
        p.max_iterations = 0;
        CHECK_THROWS_AS(denoise(img, p), std::invalid_argument);
        CHECK_THROWS_AS(denoise_pass(img, compute_cardinality(GrayImage(3, 3, 1), 20, 1), DenoiseParams{}),
                        std::invalid_argument);
        using detail::rms_replacement;
        CHECK(rms_replacement(0, 1) == 0 && rms_replacement(2, 1) == 1 && rms_replacement(9, 4) == 2);
        CHECK(rms_replacement(25, 4) == 3 && rms_replacement(65025ULL, 1) == 255 &&
              rms_replacement(65025ULL * 8, 8) == 255);
        CHECK(row_blocks(5, 8).size() == 5);
    }
    {  // noise fixture (test_noise.cpp:43-62) through the drop-in generator
        const auto [noisy, mask] = inject_sp_noise(GrayImage(10, 10, 100), {0.2, 0.5, 77});
        CHECK(noisy.pixels[4] == 255 && noisy.pixels[2] == 0 && mask.count() == 20);
    }
    {  // metrics.hpp: test_cli.cpp:76-95 fixture and acceptance.cpp:305-320
        const GrayImage a(8, 8, 40);
        GrayImage b = a;
        for (auto& p : b.pixels) p += 16;
        CHECK(mse(a, a) == 0.0 && psnr(a, a).infinite() && format_db(psnr(a, a)) == "inf");
        CHECK(mse(a, b) == 256.0 && format_db(psnr(a, b)) == "24.048");
        CHECK_THROWS_AS(mse(GrayImage(4, 4, 1), GrayImage(4, 5, 1)), std::invalid_argument);
        CHECK(format_db(psnr(GrayImage(1, 1, 0), GrayImage(1, 1, 255))) == "0.000");
        std::mt19937 rng(7);
        const GrayImage x = random_image(rng, 333, 77), y = random_image(rng, 333, 77);
        std::uint64_t s = 0;
        for (std::size_t i = 0; i < x.size(); ++i) {
            const int d = int(x.pixels[i]) - int(y.pixels[i]);
            s += std::uint64_t(d * d);
        }
        CHECK(mse(x, y) == double(s) / double(x.size()));
    }
    {  // residual_noise_count == count of C < thr of compute_cardinality (metrics.hpp:52-59)
        std::mt19937 rng(9);
        for (int i = 0; i < 20; ++i) {
            const GrayImage img = random_image(rng, 1 + static_cast<int>(rng() % 700), 1 + static_cast<int>(rng() % 60));
            const int alpha = 1 + static_cast<int>(rng() % 80), beta = 1 + static_cast<int>(rng() % 3);
            const int thr = 1 + static_cast<int>(rng() % 6);
            const auto card = compute_cardinality(img, alpha, beta);
            std::size_t n = 0;
            for (auto c : card.counts) n += c < thr;
            CHECK(residual_noise_count(img, alpha, beta, thr) == n);
        }
    }
    {  // cardmap P2 text (test_cli.cpp:113-131)
        const auto c1 = compute_cardinality(GrayImage(3, 3, 100), 20, 1);
        CHECK(write_p2(c1.width, c1.height, c1.counts, 9) == "P2\n3 3\n9\n4 6 4\n6 9 6\n4 6 4\n");
        GrayImage imp(3, 3, 100);
        imp.at(1, 1) = 255;
        const auto c2 = compute_cardinality(imp, 20, 1);
        CHECK(write_p2(c2.width, c2.height, c2.counts, 9) == "P2\n3 3\n9\n3 5 3\n5 1 5\n3 5 3\n");
        const auto c3 = compute_cardinality(GrayImage(3, 3, 100), 20, 2);
        CHECK(write_p2(c3.width, c3.height, c3.counts, 25).substr(0, 9) == "P2\n3 3\n25");
    }
    {  // pgm.hpp codec (test_pgm.cpp)
        const auto img = read_pgm("P2\n2 2\n255\n0 64 128 255");
        CHECK(img.width == 2 && img.height == 2 && (img.pixels == std::vector<std::uint8_t>{0, 64, 128, 255}));
        CHECK(write_pgm(GrayImage(1, 1, 200)) == std::string("P5\n1 1\n255\n") + '\xC8');
        CHECK(write_pgm(GrayImage(2, 3, 9)).size() == std::string("P5\n2 3\n255\n").size() + 6);
        std::mt19937 rng(7);
        for (int i = 0; i < 25; ++i) {
            const GrayImage r = random_image(rng, 1 + static_cast<int>(rng() % 20), 1 + static_cast<int>(rng() % 20));
            CHECK(read_pgm(write_pgm(r, false)) == r && read_pgm(write_pgm(r, true)) == r);
        }
        CHECK((read_pgm("P2\n# produced by hand\n2 1 # dims\n# maxval next\n255\n3 4").pixels ==
               std::vector<std::uint8_t>{3, 4}));
        CHECK((read_pgm("P5\n# note\n1 1\n255\n" + std::string(1, '\x05')).pixels == std::vector<std::uint8_t>{5}));
        CHECK((read_pgm("P2\n2 1\n15\n0 15").pixels == std::vector<std::uint8_t>{0, 15}));
        auto msg = [](const std::string& s) {
            try {
                (void)read_pgm(s);
            } catch (const PgmError& e) {
                return std::string(e.what());
            }
            return std::string("no error");
        };
        CHECK(msg("P2\n2 1\n15\n0 16") == "PGM pixel value exceeds maxval");
        CHECK(msg("P2\n1 1\n65535\n1234") == "16-bit PGM unsupported");
        CHECK(msg(std::string("P5\n1 1\n256\n") + '\0') == "16-bit PGM unsupported");
        CHECK(msg("P6\n1 1\n255\nxxx") == "not a PGM stream (expected P2 or P5 magic)");
        CHECK(msg("") == "not a PGM stream (expected P2 or P5 magic)");
        CHECK(msg("P2\n1\n255\n0") != "no error" && msg("P2\n0 1\n255\n") == "malformed PGM header");
        CHECK(msg("P5\n2 2\n255\nab") == "truncated PGM pixel data");
        CHECK(msg("P2\n2 2\n255\n1 2 3") == "truncated PGM pixel data");
    }
    {  // bench.hpp grid + CSV (test_bench.cpp)
        const std::string hdr =
            "image_id,width,height,noise_pct,engine,workers,iterations_run,"
            "total_ms,psnr_noisy_db,psnr_denoised_db,replaced_total\n";
        CHECK(write_csv({}) == hdr);
        BenchRecord rec;
        rec.image_id = "smooth-16";
        rec.width = rec.height = 16;
        rec.noise_pct = 5.0;
        rec.engine = "serial";
        rec.workers = 1;
        rec.iterations_run = 2;
        rec.total_ms = 1.2345;
        rec.psnr_noisy_db = 18.7;
        rec.psnr_denoised_db = std::numeric_limits<double>::infinity();
        rec.replaced_total = 12;
        CHECK(write_csv({rec}) == hdr + "smooth-16,16,16,5.000,serial,1,2,1.234,18.700,inf,12\n");
        BenchConfig cfg;
        cfg.synth_sizes = {24};
        cfg.densities = {0.10};
        cfg.repetitions = 1;
        cfg.engines = {EngineSpec::serial(), EngineSpec::parallel(2), EngineSpec::parallel(3)};
        const auto res = run_benchmark(cfg);
        CHECK(res.records.size() == 3);
        if (res.records.size() == 3) {
            const auto& s0 = res.records[0];
            CHECK(s0.engine == "serial" && s0.workers == 1 && s0.total_ms > 0.0);
            CHECK(s0.iterations_run >= 1 && s0.iterations_run <= cfg.params.max_iterations);
            for (const auto& r : res.records)
                CHECK(r.psnr_denoised_db == s0.psnr_denoised_db && r.psnr_noisy_db == s0.psnr_noisy_db &&
                      r.replaced_total == s0.replaced_total && r.total_ms > 0.0);
        }
        BenchConfig g2;
        g2.synth_sizes = {8, 12};
        g2.densities = {0.05, 0.20};
        g2.repetitions = 1;
        g2.engines = {EngineSpec::serial(), EngineSpec::parallel(2)};
        const auto r2 = run_benchmark(g2);
        CHECK(r2.records.size() == 8 && r2.warnings.empty());
        BenchConfig g3;
        g3.corpus_files = {"/nonexistent/missing.pgm"};
        g3.synth_sizes = {8};
        g3.densities = {0.1};
        g3.repetitions = 1;
        g3.engines = {EngineSpec::serial()};
        const auto r3 = run_benchmark(g3);
        CHECK(r3.warnings.size() == 1 && r3.warnings[0].find("missing.pgm") != std::string::npos &&
              r3.records.size() == 1);
        BenchConfig g4;
        g4.synth_sizes = {};
        CHECK_THROWS_AS(run_benchmark(g4), std::invalid_argument);
        // the reference harness's own output for a 3 x 3 x 2 grid
        // (tests/golden/bench_grid.csv, make_bench_golden.cpp): every column
        // but the wall time must match
        BenchConfig g5;
        g5.synth_sizes = {24, 64, 200};
        g5.densities = {0.05, 0.30, 0.70};
        g5.engines = {EngineSpec::serial(), EngineSpec::parallel(3)};
        g5.repetitions = 1;
        g5.seed = 5;
        auto r5 = run_benchmark(g5);
        for (auto& r : r5.records) r.total_ms = 0.0;
        std::string got;
        {
            std::istringstream in(write_csv(r5.records));
            std::string line;
            while (std::getline(in, line)) {
                std::string out, cur;
                std::istringstream ls(line);
                for (int f = 0; std::getline(ls, cur, ','); ++f) out += (out.empty() ? "" : ",") + (f == 7 ? "-" : cur);
                got += out + "\n";
            }
        }
        std::ifstream gf(g_golden_dir + "/bench_grid.csv");
        const std::string want((std::istreambuf_iterator<char>(gf)), std::istreambuf_iterator<char>());
        CHECK(!want.empty() && got == want);
        // GPU columns (opt-in CSV): device time, rate and roofline fraction
        const std::string gcsv = write_csv_gpu(r5.records);
        CHECK(gcsv.rfind(hdr.substr(0, hdr.size() - 1) + ",device_ms,mpix_it_per_s,hbm_roofline_frac\n", 0) == 0);
        for (const auto& r : r5.records)
            CHECK(r.device_ms > 0.0 && r.mpix_it_per_s > 0.0 && r.hbm_roofline_frac > 0.0 &&
                  std::abs(r.mpix_it_per_s - double(r.width) * r.height * r.iterations_run / (r.device_ms * 1e3)) <
                      1e-6 * r.mpix_it_per_s);
    }
    {  // pgm_gpu.hpp: file -> device -> file equals save_pgm(denoise(load_pgm))
        const auto clean = synth_image(700, 300, 3, SynthKind::SmoothRandom);
        NoiseSpec spec;
        spec.density = 0.3;
        spec.seed = 9;
        const auto noisy = inject_sp_noise(clean, spec).first;
        for (const bool ascii : {false, true}) {
            const std::string in = std::string("/tmp/phg_dropin_in") + (ascii ? "2" : "5") + ".pgm";
            const std::string out = "/tmp/phg_dropin_out.pgm", want = "/tmp/phg_dropin_want.pgm";
            save_pgm(in, noisy, ascii);
            const auto st = denoise_pgm_file(in, out);
            const auto ref = denoise(noisy, DenoiseParams{});
            save_pgm(want, ref.image);
            std::ifstream a(out, std::ios::binary), b(want, std::ios::binary);
            const std::string ga((std::istreambuf_iterator<char>(a)), std::istreambuf_iterator<char>());
            const std::string gb((std::istreambuf_iterator<char>(b)), std::istreambuf_iterator<char>());
            CHECK(!ga.empty() && ga == gb && st.size() == ref.stats.size());
        }
        CHECK_THROWS_AS(denoise_pgm_file("/nonexistent/x.pgm", "/tmp/phg_x.pgm"), PgmError);
    }
    std::printf("dropin: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
