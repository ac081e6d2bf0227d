/*
 * phgrms_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the P-HGRMS CPU reference (arXiv 1306.5390
 * artifact, /root/reference/proj) used as the parity CHECKER for the CUDA
 * product path.  Nothing in the product package links, imports or executes
 * this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * Parity pinning: every function here is checked (tests/test_oracle.py)
 * against (a) the reference's own golden vectors and known-answer tests
 * (test_denoise.cpp, test_noise.cpp, acceptance.cpp crit 3) and (b) the
 * reference compiled from its own headers (oracle/_ref/libphgrms_ref.so,
 * built by oracle/Makefile from /root/reference/proj/include) through
 * fixtures committed under tests/golden/.
 *
 * Citations are path:line relative to /root/reference/proj.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* std::mt19937 (ISO C++ [rand.eng.mers]); the reference relies on its  */
/* standardised output sequence: include/phgrms/image.hpp:91-96,        */
/* include/phgrms/noise.hpp:78.                                        */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t mt[624];
    int idx;
} orc_mt19937;

static void mt_seed(orc_mt19937* g, uint32_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

static uint32_t mt_next(orc_mt19937* g) {
    if (g->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
            uint32_t v = g->mt[(i + 397) % 624] ^ (y >> 1);
            if (y & 1u) v ^= 0x9908b0dfu;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint32_t y = g->mt[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

uint32_t orc_mt19937_nth(uint32_t seed, uint64_t n) {
    orc_mt19937 g;
    mt_seed(&g, seed);
    uint32_t v = 0;
    for (uint64_t i = 0; i < n; ++i) v = mt_next(&g);
    return v;
}

/* ------------------------------------------------------------------ */
/* Input generators (out of the hot path; used to build parity inputs) */
/* ------------------------------------------------------------------ */

/* synth_image(..., SmoothRandom): include/phgrms/image.hpp:77-103.
 * kind: 0 Gradient (:63-70), 1 Checker (:72-76), 2 SmoothRandom. */
int orc_synth_image(int w, int h, uint32_t seed, int kind, uint8_t* out) {
    if (w < 1 || h < 1) return -1;
    const size_t n = (size_t)w * (size_t)h;
    if (kind == 0) {
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c)
                out[(size_t)r * w + c] = (uint8_t)(w == 1 ? 0 : (int)(255LL * c / (w - 1)));
        return 0;
    }
    if (kind == 1) {
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c)
                out[(size_t)r * w + c] = ((r / 8 + c / 8) % 2 == 0) ? 64 : 192;
        return 0;
    }
    uint8_t* field = (uint8_t*)malloc(n);
    if (!field) return -2;
    orc_mt19937 g;
    mt_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) field[i] = (uint8_t)(mt_next(&g) & 0xFFu);
    for (int r = 0; r < h; ++r) {
        const int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
        for (int c = 0; c < w; ++c) {
            const int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
            int sum = 0, cnt = 0;
            for (int i = r0; i <= r1; ++i)
                for (int j = c0; j <= c1; ++j) {
                    sum += field[(size_t)i * w + j];
                    ++cnt;
                }
            int v = (sum + cnt / 2) / cnt;
            out[(size_t)r * w + c] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
        }
    }
    free(field);
    return 0;
}

/* detail::bounded_rand: include/phgrms/noise.hpp:52-58 (rejection of the
 * top 2^32 mod bound values). */
static uint32_t bounded_rand(orc_mt19937* g, uint32_t bound) {
    const uint32_t threshold = (0u - bound) % bound;
    for (;;) {
        const uint32_t r = mt_next(g);
        if (r >= threshold) return r % bound;
    }
}

/* inject_sp_noise: include/phgrms/noise.hpp:62-89.  Exact-count salt and
 * pepper via a partial Fisher-Yates over uint32 pixel indices.  `mask` may
 * be NULL.  Returns the number of corrupted pixels. */
long long orc_inject_sp_noise(const uint8_t* img, int w, int h, double density,
                              double salt_ratio, uint32_t seed, uint8_t* out,
                              uint8_t* mask) {
    if (!(density >= 0.0 && density <= 1.0)) return -1;
    if (!(salt_ratio >= 0.0 && salt_ratio <= 1.0)) return -1;
    const size_t total = (size_t)w * (size_t)h;
    const size_t n = (size_t)llround(density * (double)total);
    const size_t salt = (size_t)llround(salt_ratio * (double)n);
    memcpy(out, img, total);
    if (mask) memset(mask, 0, total);
    if (n == 0) return 0;
    uint32_t* order = (uint32_t*)malloc(total * sizeof(uint32_t));
    if (!order) return -2;
    for (size_t i = 0; i < total; ++i) order[i] = (uint32_t)i;
    orc_mt19937 g;
    mt_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) {
        const size_t j = i + bounded_rand(&g, (uint32_t)(total - i));
        const uint32_t t = order[i];
        order[i] = order[j];
        order[j] = t;
        const uint32_t pos = order[i];
        out[pos] = i < salt ? 255 : 0;
        if (mask) mask[pos] = 1;
    }
    free(order);
    return (long long)n;
}

/* ------------------------------------------------------------------ */
/* The hot path                                                        */
/* ------------------------------------------------------------------ */

/* similar(): include/phgrms/denoise.hpp:88 -- |a-b| < alpha, strict. */
static inline int similar(int a, int b, int alpha) { return abs(a - b) < alpha; }

/* detail::cardinality_rows + compute_cardinality:
 * include/phgrms/denoise.hpp:139-160, 227-241.  Gather form; OOB cells are
 * excluded (not padded); the centre counts itself. */
int orc_cardinality(const uint8_t* img, int w, int h, int alpha, int beta,
                    int32_t* counts) {
    if (alpha < 1 || alpha > 255) return -1;
    if (beta < 1) return -1;
    for (int r = 0; r < h; ++r) {
        const int r0 = r - beta < 0 ? 0 : r - beta;
        const int r1 = r + beta > h - 1 ? h - 1 : r + beta;
        for (int c = 0; c < w; ++c) {
            const int c0 = c - beta < 0 ? 0 : c - beta;
            const int c1 = c + beta > w - 1 ? w - 1 : c + beta;
            const int center = img[(size_t)r * w + c];
            int32_t n = 0;
            for (int i = r0; i <= r1; ++i)
                for (int j = c0; j <= c1; ++j)
                    n += similar(img[(size_t)i * w + j], center, alpha);
            counts[(size_t)r * w + c] = n;
        }
    }
    return 0;
}

/* The paper's Algorithm 1 as a scatter, i.e. the test
 * oracle tests/support/oracles.hpp:43-75 run on one thread: every pixel
 * bumps the count of each in-bounds window cell it is similar to. */
int orc_cardinality_scatter(const uint8_t* img, int w, int h, int alpha,
                            int beta, int32_t* counts) {
    memset(counts, 0, (size_t)w * h * sizeof(int32_t));
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c)
            for (int i = r - beta; i <= r + beta; ++i)
                for (int j = c - beta; j <= c + beta; ++j) {
                    if (i < 0 || i >= h || j < 0 || j >= w) continue;
                    if (similar(img[(size_t)i * w + j], img[(size_t)r * w + c], alpha))
                        counts[(size_t)i * w + j] += 1;
                }
    return 0;
}

/* detail::rms_replacement: include/phgrms/denoise.hpp:163-169 --
 * llround(sqrt(double(sum)/flag)) clamped to [0,255]. */
int orc_rms_replacement(uint64_t sum_sq, int flag) {
    const double rms = sqrt((double)sum_sq / flag);
    long long v = llround(rms);
    if (v < 0) v = 0;
    if (v > 255) v = 255;
    return (int)v;
}

typedef struct {
    int alpha, beta, max_iterations, card_threshold, border; /* border: 0 Faithful, 1 InBounds */
} orc_params;

/* DenoiseParams::validate: include/phgrms/denoise.hpp:41-49.
 * 0 ok, 1 alpha, 2 beta, 3 iterations, 4 card_threshold. */
int orc_validate(const orc_params* p) {
    if (p->alpha < 1 || p->alpha > 255) return 1;
    if (p->beta < 1) return 2;
    if (p->max_iterations < 1) return 3;
    if (p->card_threshold < 1) return 4;
    return 0;
}

/* detail::removal_rows + denoise_pass: include/phgrms/denoise.hpp:176-223,
 * 243-283.  Reads only `img`/`card`, writes a fresh `out`. */
int orc_removal_pass(const uint8_t* img, const int32_t* card, int w, int h,
                     const orc_params* p, uint8_t* out, int64_t* flagged,
                     int64_t* replaced) {
    if (orc_validate(p)) return -1;
    const int full_window = (2 * p->beta + 1) * (2 * p->beta + 1);
    int64_t nf = 0, nr = 0;
    for (int r = 0; r < h; ++r) {
        const int r0 = r - p->beta < 0 ? 0 : r - p->beta;
        const int r1 = r + p->beta > h - 1 ? h - 1 : r + p->beta;
        for (int c = 0; c < w; ++c) {
            const size_t idx = (size_t)r * w + c;
            const int center = img[idx];
            uint8_t value = (uint8_t)center;
            if (card[idx] < p->card_threshold) {
                ++nf;
                const int c0 = c - p->beta < 0 ? 0 : c - p->beta;
                const int c1 = c + p->beta > w - 1 ? w - 1 : c + p->beta;
                const int in_bounds = (r1 - r0 + 1) * (c1 - c0 + 1);
                const int pix_count = p->border == 0 ? full_window : in_bounds;
                uint64_t sum_sq = 0;
                int flag = 0;
                for (int i = r0; i <= r1; ++i)
                    for (int j = c0; j <= c1; ++j) {
                        const int v = img[(size_t)i * w + j];
                        if (!similar(v, center, p->alpha)) {
                            sum_sq += (uint64_t)v * (uint64_t)v;
                            ++flag;
                        }
                    }
                if (flag > pix_count - 3 && flag > 0) {
                    value = (uint8_t)orc_rms_replacement(sum_sq, flag);
                    ++nr;
                }
            }
            out[idx] = value;
        }
    }
    *flagged = nf;
    *replaced = nr;
    return 0;
}

/* denoise(): include/phgrms/denoise.hpp:292-311.  Iterates cardinality +
 * removal up to max_iterations, stopping after the first iteration that
 * replaced nothing.  flagged/replaced hold one entry per executed
 * iteration (capacity max_iterations). */
int orc_denoise(const uint8_t* img, int w, int h, const orc_params* p,
                uint8_t* out, int64_t* flagged, int64_t* replaced,
                int* iterations_run) {
    if (orc_validate(p)) return -1;
    const size_t n = (size_t)w * h;
    uint8_t* cur = (uint8_t*)malloc(n);
    uint8_t* nxt = (uint8_t*)malloc(n);
    int32_t* card = (int32_t*)malloc(n * sizeof(int32_t));
    if (!cur || !nxt || !card) {
        free(cur);
        free(nxt);
        free(card);
        return -2;
    }
    memcpy(cur, img, n);
    int it = 0;
    for (int k = 1; k <= p->max_iterations; ++k) {
        orc_cardinality(cur, w, h, p->alpha, p->beta, card);
        orc_removal_pass(cur, card, w, h, p, nxt, &flagged[k - 1], &replaced[k - 1]);
        uint8_t* t = cur;
        cur = nxt;
        nxt = t;
        it = k;
        if (replaced[k - 1] == 0) break;
    }
    memcpy(out, cur, n);
    *iterations_run = it;
    free(cur);
    free(nxt);
    free(card);
    return 0;
}

/* row_blocks: include/phgrms/denoise.hpp:97-107.  Writes up to `workers`
 * (begin,end) pairs; returns the number of non-empty blocks. */
int orc_row_blocks(int height, int workers, int* begins, int* ends) {
    if (height < 0 || workers < 1) return -1;
    int nb = 0;
    for (int wk = 0; wk < workers; ++wk) {
        const int lo = (int)((int64_t)height * wk / workers);
        const int hi = (int)((int64_t)height * (wk + 1) / workers);
        if (hi > lo) {
            begins[nb] = lo;
            ends[nb] = hi;
            ++nb;
        }
    }
    return nb;
}

/* One iteration on a row band held in a buffer (the global-coordinate form
 * of cardinality_rows + removal_rows, denoise.hpp:139-160 / 176-223).
 * Buffer row b holds global image row b + row_base of an image `height`
 * rows tall.  Global rows [y_lo, y_hi) are computed into dst (same layout);
 * flagged/replaced are counted only over global rows [c_lo, c_hi).  Window
 * cells outside the IMAGE are excluded exactly as in the reference; the
 * caller guarantees every in-image row within beta of [y_lo, y_hi) is held
 * by the buffer.  Test infrastructure for the multi-rank band exchange. */
int orc_band_pass(const uint8_t* src, uint8_t* dst, int w, int buf_rows, int row_base, int height,
                  int y_lo, int y_hi, int c_lo, int c_hi, const orc_params* p, int64_t* flagged,
                  int64_t* replaced) {
    if (orc_validate(p)) return -1;
    const int full_window = (2 * p->beta + 1) * (2 * p->beta + 1);
    int64_t nf = 0, nr = 0;
    for (int r = y_lo; r < y_hi; ++r) {
        const int r0 = r - p->beta < 0 ? 0 : r - p->beta;
        const int r1 = r + p->beta > height - 1 ? height - 1 : r + p->beta;
        if (r0 - row_base < 0 || r1 - row_base >= buf_rows) return -2;
        for (int c = 0; c < w; ++c) {
            const int c0 = c - p->beta < 0 ? 0 : c - p->beta;
            const int c1 = c + p->beta > w - 1 ? w - 1 : c + p->beta;
            const int center = src[(size_t)(r - row_base) * w + c];
            int card = 0, flag = 0;
            uint64_t sum_sq = 0;
            for (int i = r0; i <= r1; ++i)
                for (int j = c0; j <= c1; ++j) {
                    const int v = src[(size_t)(i - row_base) * w + j];
                    if (similar(v, center, p->alpha))
                        ++card;
                    else {
                        sum_sq += (uint64_t)v * (uint64_t)v;
                        ++flag;
                    }
                }
            uint8_t value = (uint8_t)center;
            const int counted = r >= c_lo && r < c_hi;
            if (card < p->card_threshold) {
                nf += counted;
                const int in_bounds = (r1 - r0 + 1) * (c1 - c0 + 1);
                const int pix_count = p->border == 0 ? full_window : in_bounds;
                if (flag > pix_count - 3 && flag > 0) {
                    value = (uint8_t)orc_rms_replacement(sum_sq, flag);
                    nr += counted;
                }
            }
            dst[(size_t)(r - row_base) * w + c] = value;
        }
    }
    *flagged = nf;
    *replaced = nr;
    return 0;
}
