// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers in place
// (-I /root/reference/proj/include -I /root/reference/proj/tests) and exposes
// them through a C ABI so the Python tests can (1) pin the C restatement in
// oracle/phgrms_oracle.c against the reference itself and (2) time the
// reference's own CPU path as bench.py's cpu_baseline ("kind": "reference").
// Output: oracle/_ref/libphgrms_ref.so (git-ignored, travels with gpurun).
// No reference source is copied into this repository.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "phgrms/denoise.hpp"
#include "phgrms/image.hpp"
#include "phgrms/noise.hpp"
#include "support/oracles.hpp"

using namespace phgrms;

namespace {

DenoiseParams to_params(int alpha, int beta, int k, int thr, int border) {
    DenoiseParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.max_iterations = k;
    p.card_threshold = thr;
    p.border = border ? BorderMode::InBounds : BorderMode::Faithful;
    return p;
}

EngineSpec to_engine(int workers) {
    return workers <= 1 ? EngineSpec::serial() : EngineSpec::parallel(workers);
}

GrayImage wrap(const uint8_t* img, int w, int h) {
    return GrayImage(w, h, std::vector<uint8_t>(img, img + static_cast<size_t>(w) * h));
}

}  // namespace

extern "C" {

int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

int ref_synth_image(int w, int h, uint32_t seed, int kind, uint8_t* out) {
    try {
        const auto img = synth_image(w, h, seed, static_cast<SynthKind>(kind));
        std::memcpy(out, img.pixels.data(), img.size());
        return 0;
    } catch (...) {
        return -1;
    }
}

long long ref_inject_sp_noise(const uint8_t* img, int w, int h, double density,
                              double salt_ratio, uint32_t seed, uint8_t* out,
                              uint8_t* mask) {
    try {
        const auto [noisy, m] = inject_sp_noise(wrap(img, w, h), {density, salt_ratio, seed});
        std::memcpy(out, noisy.pixels.data(), noisy.size());
        if (mask) std::memcpy(mask, m.flags.data(), m.flags.size());
        return static_cast<long long>(m.count());
    } catch (...) {
        return -1;
    }
}

int ref_compute_cardinality(const uint8_t* img, int w, int h, int alpha, int beta,
                            int workers, int32_t* counts) {
    try {
        const auto card = compute_cardinality(wrap(img, w, h), alpha, beta, to_engine(workers));
        std::memcpy(counts, card.counts.data(), card.counts.size() * sizeof(int32_t));
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int ref_cardinality_scatter(const uint8_t* img, int w, int h, int alpha, int beta,
                            int workers, int32_t* counts) {
    const auto c = oracle::cardinality_scatter(wrap(img, w, h), alpha, beta, workers);
    std::memcpy(counts, c.data(), c.size() * sizeof(int32_t));
    return 0;
}

int ref_denoise_pass(const uint8_t* img, const int32_t* card, int w, int h, int alpha,
                     int beta, int k, int thr, int border, int workers, uint8_t* out,
                     int64_t* flagged, int64_t* replaced) {
    try {
        CardinalityMap cm{w, h, std::vector<int32_t>(card, card + static_cast<size_t>(w) * h)};
        const auto [o, st] = denoise_pass(wrap(img, w, h), cm, to_params(alpha, beta, k, thr, border),
                                          to_engine(workers));
        std::memcpy(out, o.pixels.data(), o.size());
        *flagged = st.flagged;
        *replaced = st.replaced;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int ref_oracle_removal_pass(const uint8_t* img, const int32_t* card, int w, int h, int alpha,
                            int beta, int thr, int border, uint8_t* out) {
    const auto o = oracle::removal_pass(wrap(img, w, h),
                                        std::vector<int32_t>(card, card + static_cast<size_t>(w) * h),
                                        to_params(alpha, beta, 1, thr, border));
    std::memcpy(out, o.pixels.data(), o.size());
    return 0;
}

int ref_denoise(const uint8_t* img, int w, int h, int alpha, int beta, int k, int thr,
                int border, int workers, uint8_t* out, int64_t* flagged, int64_t* replaced,
                int* iterations_run) {
    try {
        const auto res = denoise(wrap(img, w, h), to_params(alpha, beta, k, thr, border),
                                 to_engine(workers));
        std::memcpy(out, res.image.pixels.data(), res.image.size());
        for (size_t i = 0; i < res.stats.size(); ++i) {
            flagged[i] = res.stats[i].flagged;
            replaced[i] = res.stats[i].replaced;
        }
        *iterations_run = static_cast<int>(res.stats.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// Image-level parallelism over a packed batch [n][h][w]: `threads` host
// threads each run the reference's Serial engine on whole images (the
// strongest CPU arrangement for the batch config).
int ref_denoise_batch(const uint8_t* imgs, int n, int w, int h, int alpha, int beta, int k,
                      int thr, int border, int threads, uint8_t* out, int* iterations_run) {
    const size_t px = static_cast<size_t>(w) * h;
    const auto p = to_params(alpha, beta, k, thr, border);
    auto work = [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) {
            const auto res = denoise(wrap(imgs + px * i, w, h), p, EngineSpec::serial());
            std::memcpy(out + px * i, res.image.pixels.data(), px);
            iterations_run[i] = static_cast<int>(res.stats.size());
        }
    };
    if (threads <= 1) {
        work(0, n);
        return 0;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int lo = static_cast<int>(static_cast<int64_t>(n) * t / threads);
        const int hi = static_cast<int>(static_cast<int64_t>(n) * (t + 1) / threads);
        if (hi > lo) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    return 0;
}

// Same as ref_denoise_batch, plus the per-iteration counters [n][k] (rows
// past iterations_run[i] are left as they are).
int ref_denoise_batch_stats(const uint8_t* imgs, int n, int w, int h, int alpha, int beta, int k, int thr,
                            int border, int threads, uint8_t* out, int64_t* flagged, int64_t* replaced,
                            int* iterations_run) {
    const size_t px = static_cast<size_t>(w) * h;
    const auto p = to_params(alpha, beta, k, thr, border);
    auto work = [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) {
            const auto res = denoise(wrap(imgs + px * i, w, h), p, EngineSpec::serial());
            std::memcpy(out + px * i, res.image.pixels.data(), px);
            iterations_run[i] = static_cast<int>(res.stats.size());
            for (size_t j = 0; j < res.stats.size(); ++j) {
                flagged[static_cast<size_t>(i) * k + j] = res.stats[j].flagged;
                replaced[static_cast<size_t>(i) * k + j] = res.stats[j].replaced;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) {
        const int lo = static_cast<int>(static_cast<int64_t>(n) * t / std::max(1, threads));
        const int hi = static_cast<int>(static_cast<int64_t>(n) * (t + 1) / std::max(1, threads));
        if (hi > lo) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    return 0;
}

// One row band of a tall image, for golden digests of images too large to
// denoise whole (C5, 2^32 px).  Band rows [0, bh) hold consecutive image
// rows; the owned band rows [own_lo, own_hi) are at least beta*k rows from
// every band edge that is not an image edge, so k passes of the reference
// (compute_cardinality + detail::removal_rows, denoise.hpp:139-223) on the
// band alone give their exact values: a fake edge corrupts one more row per
// pass.  Runs all k passes (a zero-replacement pass is a fixed point, so
// truncating after the global first zero is exact) and counts flagged /
// replaced over the owned rows only.
int ref_denoise_band(const uint8_t* band, int w, int bh, int own_lo, int own_hi, int alpha, int beta, int k,
                     int thr, int border, uint8_t* out_owned, int64_t* flagged, int64_t* replaced) {
    try {
        const auto p = to_params(alpha, beta, k, thr, border);
        GrayImage cur = wrap(band, w, bh);
        for (int i = 0; i < k; ++i) {
            const auto card = compute_cardinality(cur, alpha, beta, EngineSpec::serial());
            GrayImage next = cur;
            detail::removal_rows(cur, card, p, next.pixels.data(), 0, own_lo);
            const auto c = detail::removal_rows(cur, card, p, next.pixels.data(), own_lo, own_hi);
            detail::removal_rows(cur, card, p, next.pixels.data(), own_hi, bh);
            flagged[i] = c.flagged;
            replaced[i] = c.replaced;
            cur = std::move(next);
        }
        std::memcpy(out_owned, cur.pixels.data() + static_cast<size_t>(own_lo) * w,
                    static_cast<size_t>(own_hi - own_lo) * w);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

}  // extern "C"
