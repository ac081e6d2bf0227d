#pragma once
// Drop-in for phgrms/noise.hpp of the reference (proj/include/phgrms/
// noise.hpp:24-89): exact-count salt & pepper injection, delegated to
// phg_inject_sp_noise (same mt19937 / rejection / partial Fisher-Yates
// contract, so fixtures reproduce).

#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "phgrms/image.hpp"
#include "phgrms_b200.h"

namespace phgrms {

struct NoiseSpec {
    double density = 0.0;
    double salt_ratio = 0.5;
    std::uint32_t seed = 0;

    void validate() const {
        if (!(density >= 0.0 && density <= 1.0)) throw std::invalid_argument("density must be in [0, 1]");
        if (!(salt_ratio >= 0.0 && salt_ratio <= 1.0)) throw std::invalid_argument("salt_ratio must be in [0, 1]");
    }
};

struct CorruptionMask {
    int width = 0;
    int height = 0;
    std::vector<std::uint8_t> flags;
    std::size_t count() const {
        std::size_t n = 0;
        for (auto f : flags) n += f;
        return n;
    }
};

inline std::pair<GrayImage, CorruptionMask> inject_sp_noise(const GrayImage& img, const NoiseSpec& spec) {
    spec.validate();
    GrayImage out(img.width, img.height);
    CorruptionMask mask{img.width, img.height, std::vector<std::uint8_t>(img.size())};
    if (phg_inject_sp_noise(img.pixels.data(), img.width, img.height, spec.density, spec.salt_ratio, spec.seed,
                            out.pixels.data(), mask.flags.data()) < 0)
        throw std::invalid_argument(phg_last_error());
    return {std::move(out), std::move(mask)};
}

}  // namespace phgrms
