#pragma once
// Drop-in for phgrms/denoise.hpp of the reference
// (proj/include/phgrms/denoise.hpp:25-311): identical types, defaults,
// signatures and exception texts, with every pass executed by the sm_100a
// kernels behind the C ABI (include/phgrms_b200.h, libphgrms_cuda.so).
//
//   compute_cardinality  denoise.hpp:227-241  -> phg_cardinality
//   denoise_pass         denoise.hpp:243-283  -> phg_denoise_pass
//   denoise              denoise.hpp:292-311  -> phg_denoise
//
// EngineSpec keeps its meaning as a partition request: Serial runs the
// whole image as one device pipeline; Parallel(W) splits the rows into the
// same row_blocks bands the reference hands to W threads, and the bands run
// as separate device buffers with halo exchange -- bit-identical either way.
// With PHGRMS_DEVICES set (e.g. "0,1,2,3"), Parallel(W)'s W bands are spread
// over those GPUs in contiguous groups (phg_denoise_sharded): the
// reference's own call scales across an NVSwitch node unchanged.
// row_blocks / parallel_for_rows / similar / detail::rms_replacement remain
// host utilities with the reference's contracts.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "phgrms/image.hpp"
#include "phgrms_b200.h"

namespace phgrms {

enum class BorderMode { Faithful, InBounds };
enum class EngineMode { Serial, Parallel };

struct DenoiseParams {
    int alpha = 20;
    int beta = 1;
    int max_iterations = 5;
    int card_threshold = 3;
    BorderMode border = BorderMode::Faithful;

    phg_params c() const {
        return {alpha, beta, max_iterations, card_threshold, border == BorderMode::InBounds ? 1 : 0};
    }
    void validate() const {
        const phg_params p = c();
        if (phg_validate_params(&p) != PHG_OK) throw std::invalid_argument(phg_last_error());
    }
    int window_cells() const { return (2 * beta + 1) * (2 * beta + 1); }
};

struct EngineSpec {
    EngineMode mode = EngineMode::Serial;
    int workers = 0;

    static EngineSpec serial() { return {EngineMode::Serial, 1}; }
    static EngineSpec parallel(int workers = 0) { return {EngineMode::Parallel, workers}; }
    int resolved_workers() const {
        if (mode == EngineMode::Serial) return 1;
        if (workers >= 1) return workers;
        const unsigned hw = std::thread::hardware_concurrency();
        return hw ? static_cast<int>(hw) : 1;
    }
};

struct PassStats {
    int iteration = 0;
    std::int64_t flagged = 0;
    std::int64_t replaced = 0;
    double elapsed_ms = 0.0;
};

struct CardinalityMap {
    int width = 0;
    int height = 0;
    std::vector<std::int32_t> counts;
    std::int32_t at(int r, int c) const { return counts[static_cast<std::size_t>(r) * width + c]; }
};

inline bool similar(int a, int b, int alpha) { return std::abs(a - b) < alpha; }

struct RowBlock {
    int begin = 0;
    int end = 0;
};

inline std::vector<RowBlock> row_blocks(int height, int workers) {
    if (height < 0 || workers < 1) throw std::invalid_argument("row_blocks: bad height or worker count");
    std::vector<RowBlock> out;
    for (int k = 0; k < workers; ++k) {
        const int b = static_cast<int>(static_cast<std::int64_t>(height) * k / workers);
        const int e = static_cast<int>(static_cast<std::int64_t>(height) * (k + 1) / workers);
        if (e > b) out.push_back({b, e});
    }
    return out;
}

template <typename Fn>
void parallel_for_rows(int height, int workers, Fn&& fn) {
    const auto blocks = row_blocks(height, workers);
    if (blocks.size() <= 1) {
        for (const auto& b : blocks) fn(b.begin, b.end);
        return;
    }
    std::vector<std::exception_ptr> err(blocks.size());
    std::vector<std::thread> pool;
    for (std::size_t i = 0; i < blocks.size(); ++i)
        pool.emplace_back([&, i] {
            try {
                fn(blocks[i].begin, blocks[i].end);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

namespace detail {
// llround(sqrt(sum/flag)) clamped to [0,255] -- evaluated with the exact
// integer rule the kernels use (largest u with (2u-1)^2 * flag <= 4 sum).
inline std::uint8_t rms_replacement(std::uint64_t sum_sq, int flag) {
    std::uint64_t u = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(sum_sq) / flag)) + 2;
    while (u >= 1 && (2 * u - 1) * (2 * u - 1) * static_cast<std::uint64_t>(flag) > 4 * sum_sq) --u;
    return static_cast<std::uint8_t>(std::min<std::uint64_t>(u, 255));
}

// PHGRMS_DEVICES: comma-separated device ordinals; empty when unset.
inline std::vector<int> engine_devices() {
    std::vector<int> d;
    const char* e = std::getenv("PHGRMS_DEVICES");
    if (!e) return d;
    const std::string s(e);
    std::size_t i = 0;
    while (i < s.size()) {
        const std::size_t j = std::min(s.find(',', i), s.size());
        if (j > i) d.push_back(std::stoi(s.substr(i, j - i)));
        i = j + 1;
    }
    return d;
}

inline void throw_on(int rc) {
    if (rc == PHG_OK) return;
    if (rc == PHG_EINVAL) throw std::invalid_argument(phg_last_error());
    throw std::runtime_error(std::string("phgrms_b200: ") + phg_last_error());
}
}  // namespace detail

inline CardinalityMap compute_cardinality(const GrayImage& img, int alpha, int beta,
                                          const EngineSpec& = EngineSpec::serial()) {
    CardinalityMap m{img.width, img.height, std::vector<std::int32_t>(img.size())};
    detail::throw_on(phg_cardinality(img.pixels.data(), img.width, img.height, alpha, beta, m.counts.data()));
    return m;
}

inline std::pair<GrayImage, PassStats> denoise_pass(const GrayImage& img, const CardinalityMap& card,
                                                    const DenoiseParams& params,
                                                    const EngineSpec& = EngineSpec::serial()) {
    params.validate();
    if (card.width != img.width || card.height != img.height)
        throw std::invalid_argument("cardinality map does not match image");
    GrayImage out(img.width, img.height);
    phg_pass_stats st{};
    const phg_params p = params.c();
    detail::throw_on(phg_denoise_pass(img.pixels.data(), img.width, img.height, card.counts.data(), card.width,
                                      card.height, &p, out.pixels.data(), &st));
    return {std::move(out), PassStats{1, st.flagged, st.replaced, st.elapsed_ms}};
}

struct DenoiseResult {
    GrayImage image;
    std::vector<PassStats> stats;
};

inline DenoiseResult denoise(const GrayImage& img, const DenoiseParams& params,
                             const EngineSpec& engine = EngineSpec::serial()) {
    params.validate();
    const phg_params p = params.c();
    std::vector<phg_pass_stats> st(static_cast<std::size_t>(params.max_iterations));
    int iters = 0;
    DenoiseResult r{GrayImage(img.width, img.height), {}};
    const int workers = engine.resolved_workers();
    const std::vector<int> devs = engine.mode == EngineMode::Parallel ? detail::engine_devices() : std::vector<int>{};
    if (!devs.empty()) {
        std::vector<int> band_dev(static_cast<std::size_t>(workers));
        for (int g = 0; g < workers; ++g)
            band_dev[g] = devs[static_cast<std::size_t>(static_cast<std::int64_t>(g) * devs.size() / workers)];
        detail::throw_on(phg_denoise_sharded(img.pixels.data(), 1, img.width, img.height, &p, band_dev.data(),
                                             workers, r.image.pixels.data(), st.data(), &iters));
    } else {
        detail::throw_on(phg_denoise(img.pixels.data(), img.width, img.height, &p, workers, r.image.pixels.data(),
                                     st.data(), &iters));
    }
    for (int i = 0; i < iters; ++i) r.stats.push_back({st[i].iteration, st[i].flagged, st[i].replaced, st[i].elapsed_ms});
    return r;
}

}  // namespace phgrms
