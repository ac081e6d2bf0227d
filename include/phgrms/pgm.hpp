#pragma once
// Drop-in for phgrms/pgm.hpp of the reference (proj/include/phgrms/pgm.hpp:
// 18-176): the netpbm P5/P2 codec (maxval <= 255, '#' comments in the
// header) and the P2 writer of `phgrms cardmap` (pgm.hpp:123-136,
// tools/phgrms_main.cpp:151-168), with the reference's PgmError texts.
// Host I/O around the accelerated path; nothing here runs on the device.

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "phgrms/image.hpp"

namespace phgrms {

struct PgmError : std::runtime_error {
    explicit PgmError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {

// Cursor over a PGM byte stream.
class PgmCursor {
public:
    explicit PgmCursor(std::string_view s) : s_(s) {}

    static bool space(char ch) {
        return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f';
    }
    static bool digit(char ch) { return ch >= '0' && ch <= '9'; }
    bool done() const { return i_ >= s_.size(); }
    char peek() const { return s_[i_]; }
    std::size_t pos() const { return i_; }
    std::size_t left() const { return s_.size() - i_; }
    void advance(std::size_t n = 1) { i_ += n; }

    // header token: whitespace and '#'-to-end-of-line comments may precede it
    long header_int() {
        for (;;) {
            if (done()) break;
            if (space(peek())) {
                advance();
            } else if (peek() == '#') {
                while (!done() && peek() != '\n') advance();
            } else {
                break;
            }
        }
        return number("malformed PGM header");
    }
    // P2 raster token: whitespace only
    long body_int() {
        while (!done() && space(peek())) advance();
        if (done()) throw PgmError("truncated PGM pixel data");
        return number("malformed PGM pixel data");
    }

private:
    long number(const char* err) {
        if (done() || !digit(peek())) throw PgmError(err);
        long v = 0;
        for (; !done() && digit(peek()); advance()) {
            v = 10 * v + (peek() - '0');
            if (v > 1000000000L) throw PgmError(err);
        }
        return v;
    }
    std::string_view s_;
    std::size_t i_ = 0;
};

inline std::string pgm_header(char kind, int w, int h, int maxval) {
    return std::string("P") + kind + '\n' + std::to_string(w) + ' ' + std::to_string(h) + '\n' +
           std::to_string(maxval) + '\n';
}

template <class Get>
void append_p2_rows(std::string& out, int width, int height, Get get) {
    char num[16];
    for (int r = 0; r < height; ++r) {
        for (int c = 0; c < width; ++c) {
            if (c) out.push_back(' ');
            const int n = std::snprintf(num, sizeof(num), "%d", static_cast<int>(get(r, c)));
            out.append(num, static_cast<std::size_t>(n));
        }
        out.push_back('\n');
    }
}

}  // namespace detail

inline GrayImage read_pgm(std::string_view bytes) {
    if (bytes.size() < 2 || bytes[0] != 'P' || (bytes[1] != '2' && bytes[1] != '5'))
        throw PgmError("not a PGM stream (expected P2 or P5 magic)");
    detail::PgmCursor cur(bytes);
    cur.advance(2);
    const long w = cur.header_int(), h = cur.header_int(), maxval = cur.header_int();
    if (w < 1 || h < 1 || maxval < 1) throw PgmError("malformed PGM header");
    if (maxval > 255) throw PgmError("16-bit PGM unsupported");
    const std::size_t n = static_cast<std::size_t>(w) * static_cast<std::size_t>(h);
    std::vector<std::uint8_t> px(n);
    if (bytes[1] == '2') {
        for (auto& p : px) {
            const long v = cur.body_int();
            if (v > maxval) throw PgmError("PGM pixel value exceeds maxval");
            p = static_cast<std::uint8_t>(v);
        }
    } else {
        // one whitespace byte -- or a comment through its newline -- ends the header
        if (!cur.done() && cur.peek() == '#') {
            while (!cur.done() && cur.peek() != '\n') cur.advance();
            if (cur.done()) throw PgmError("truncated PGM pixel data");
        } else if (cur.done() || !detail::PgmCursor::space(cur.peek())) {
            throw PgmError("malformed PGM header");
        }
        cur.advance();
        if (cur.left() < n) throw PgmError("truncated PGM pixel data");
        const auto* raw = reinterpret_cast<const std::uint8_t*>(bytes.data() + cur.pos());
        for (std::size_t i = 0; i < n; ++i) {
            if (raw[i] > maxval) throw PgmError("PGM pixel value exceeds maxval");
            px[i] = raw[i];
        }
    }
    return GrayImage(static_cast<int>(w), static_cast<int>(h), std::move(px));
}

// P2 raster with an arbitrary maxval (cardinality dumps: counts exceed 255)
inline std::string write_p2(int width, int height, std::span<const std::int32_t> values, int maxval) {
    std::string out = detail::pgm_header('2', width, height, maxval);
    out.reserve(out.size() + static_cast<std::size_t>(width) * height * 3);
    detail::append_p2_rows(out, width, height,
                           [&](int r, int c) { return values[static_cast<std::size_t>(r) * width + c]; });
    return out;
}

inline std::string write_pgm(const GrayImage& img, bool ascii = false) {
    std::string out = detail::pgm_header(ascii ? '2' : '5', img.width, img.height, 255);
    if (ascii) {
        detail::append_p2_rows(out, img.width, img.height, [&](int r, int c) { return img.at(r, c); });
    } else {
        out.append(reinterpret_cast<const char*>(img.pixels.data()), img.pixels.size());
    }
    return out;
}

inline GrayImage load_pgm(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw PgmError("cannot open " + path);
    const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return read_pgm(bytes);
}

inline void save_bytes(const std::string& path, std::string_view bytes) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw PgmError("cannot open " + path + " for writing");
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw PgmError("write failed for " + path);
}

inline void save_pgm(const std::string& path, const GrayImage& img, bool ascii = false) {
    save_bytes(path, write_pgm(img, ascii));
}

}  // namespace phgrms
