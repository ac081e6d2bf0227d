#pragma once
// Drop-in for phgrms/image.hpp of the reference (proj/include/phgrms/
// image.hpp:16-106): the same GrayImage value type and synth_image entry
// point.  Pixel generation is delegated to libphgrms_cuda (phg_synth_image),
// which restates the reference generator bit for bit.

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "phgrms_b200.h"

namespace phgrms {

// uint8 raster, row-major, pixel (r, c) at r * width + c, no padding.
struct GrayImage {
    int width = 0;
    int height = 0;
    std::vector<std::uint8_t> pixels;

    GrayImage() = default;
    GrayImage(int w, int h, std::uint8_t fill = 0) : width(w), height(h) {
        check(w, h);
        pixels.assign(static_cast<std::size_t>(w) * h, fill);
    }
    GrayImage(int w, int h, std::vector<std::uint8_t> px) : width(w), height(h), pixels(std::move(px)) {
        check(w, h);
        if (pixels.size() != static_cast<std::size_t>(w) * h)
            throw std::invalid_argument("pixel count does not match dimensions");
    }

    std::size_t size() const { return pixels.size(); }
    std::size_t index(int r, int c) const { return static_cast<std::size_t>(r) * width + c; }
    std::uint8_t at(int r, int c) const { return pixels[index(r, c)]; }
    std::uint8_t& at(int r, int c) { return pixels[index(r, c)]; }
    bool same_shape(const GrayImage& o) const { return width == o.width && height == o.height; }
    friend bool operator==(const GrayImage&, const GrayImage&) = default;

private:
    static void check(int w, int h) {
        if (w < 1 || h < 1) throw std::invalid_argument("image dimensions must be >= 1");
    }
};

enum class SynthKind { Gradient, Checker, SmoothRandom };

inline GrayImage synth_image(int width, int height, std::uint32_t seed, SynthKind kind) {
    if (width < 1 || height < 1) throw std::invalid_argument("image dimensions must be >= 1");
    GrayImage img(width, height);
    if (phg_synth_image(width, height, seed, static_cast<int>(kind), img.pixels.data()) != PHG_OK)
        throw std::invalid_argument(phg_last_error());
    return img;
}

}  // namespace phgrms
