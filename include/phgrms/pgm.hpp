#pragma once
// The cardinality-map writer of the reference's codec
// (proj/include/phgrms/pgm.hpp:123-136, used by `phgrms cardmap`,
// tools/phgrms_main.cpp:151-168): an ASCII P2 raster with an arbitrary
// maxval, one text row per image row, single spaces, trailing newline.
// The rest of the PGM codec (P5/P2 parsing, file helpers) is host I/O
// outside the accelerated path.

#include <cstdint>
#include <cstdio>
#include <span>
#include <string>

namespace phgrms {

inline std::string write_p2(int width, int height, std::span<const std::int32_t> values, int maxval) {
    std::string out = "P2\n" + std::to_string(width) + ' ' + std::to_string(height) + '\n' +
                      std::to_string(maxval) + '\n';
    out.reserve(out.size() + static_cast<std::size_t>(width) * height * 3);
    char num[16];
    for (int r = 0; r < height; ++r) {
        const std::int32_t* row = values.data() + static_cast<std::size_t>(r) * width;
        for (int c = 0; c < width; ++c) {
            if (c) out.push_back(' ');
            const int n = std::snprintf(num, sizeof(num), "%d", row[c]);
            out.append(num, static_cast<std::size_t>(n));
        }
        out.push_back('\n');
    }
    return out;
}

}  // namespace phgrms
