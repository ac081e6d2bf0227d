// kernels.cuh -- sm_100a kernels of the P-HGRMS hot path.
//
// fused_tb_kernel<BETA, T>: T fused iterations of
//   cardinality (denoise.hpp:139-160) + removal (denoise.hpp:176-223)
// per launch on one tile.  A tile of 496 x TH output pixels plus an 8-px /
// BETA*T-row halo is staged into shared memory with two TMA box loads, the
// T iterations ping-pong between two shared buffers (the reference's
// "temporary matrix", denoise.hpp:250), and only the final iteration's
// owned rows are stored to HBM: 2 B of HBM traffic per pixel per launch.
//
// scalar_kernel<MODE>: one-pixel-per-thread global-memory kernels used for
// the standalone compute_cardinality / denoise_pass entry points and for
// window radii without a fused kernel (beta >= 3).
#pragma once
#include <cuda.h>
#include <cstdint>
#include <type_traits>

#include "swar.cuh"

// build-time switches for A/B experiments (defaults = product)

namespace phg {

// ------------------------------------------------------------ geometry
// A tile stages region columns [x0, x0+528) with x0 = tile*496 - 16 into one
// dense shared buffer [SH][528]: a 16-px left apron (TMA tile boxes need a
// 16-byte aligned innermost start coordinate, so the apron cannot be
// narrower), 496 output px and a 16-px right apron.  The image is viewed by
// the tensor map as [images][rows][chunks][16 px], so ONE 4-D box
// {16, 33, SH, 1} lands as the dense [SH][528] tile.  The 128 threads of a
// row group compute region words 2..129 (8 px either side of the output,
// so beta*T <= 8).
constexpr int kLeftPx = 16;
constexpr int kOutPx = 496;
constexpr int kRP = kLeftPx + kOutPx + 16;  // 528 = shared row pitch
constexpr int kChunk = 16;
constexpr int kChunks = kRP / kChunk;       // 33
constexpr int kCompWords = 128;             // region words 2..129
constexpr int kFirstWord = 2;
constexpr int kOutWordLo = kLeftPx / 4;     // 4
constexpr int kOutWordHi = kOutWordLo + kOutPx / 4;  // 128
constexpr int kGroups = 2;                  // row groups per CTA
constexpr int kThreads = kCompWords * kGroups;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxHaloPx = 8;
constexpr int kRing = 64 + kCompWords * 4;  // per-warp candidate list: < 64 leftovers + one row

// bytes of one staged buffer of sh rows (rounded for 128-B alignment)
__host__ __device__ constexpr int buf_bytes(int sh) { return (kRP * sh + 127) / 128 * 128; }
// two staged buffers + candidate bitmap (one nibble-byte per word and row)
// + per-warp candidate lists
__host__ __device__ constexpr int smem_bytes(int sh) {
    return 2 * buf_bytes(sh) + (kCompWords * sh + 127) / 128 * 128 + kWarps * kRing * 2;
}

// Halo mirrors for row-band sharding (phg_denoise_sharded): owned output
// rows that lie in a neighbour band's halo are also stored into that band's
// next buffer -- a peer pointer over NVLink when the band lives on another
// device -- so no exchange step runs between launches.  Unused: lo == hi.
struct HaloPeers {
    uint8_t* ptr[2];  // peer band buffer, same pitch; buffer row 0 = global row row0[i]
    int row0[2];
    int lo[2], hi[2];  // global rows mirrored to peer i
};

__device__ __forceinline__ void mirror_row16(const HaloPeers& hp, int gy, int64_t pitch, int col, uint4 v) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
        if (gy >= hp.lo[i] && gy < hp.hi[i])
            *reinterpret_cast<uint4*>(hp.ptr[i] + static_cast<int64_t>(gy - hp.row0[i]) * pitch + col) = v;
}

struct TileArgs {
    uint8_t* dst;
    int64_t pitch;
    int64_t image_stride;
    int width;
    int height;      // global image height
    int row_base;    // global row of buffer row 0
    int own_lo;      // first owned global row
    int own_hi;      // one past the last owned global row
    int th;          // output rows per tile
    uint32_t k7;     // ((256-alpha) & 0x7f) in every byte
    uint32_t k_thr;  // (128 - min(thr,127)) in every byte
    int alpha;
    int thr;
    int faithful;
    int it0;
    int kcap;
    unsigned long long* counters;  // [n_images][kcap][2]
    uint32_t one;                  // runtime 1 (keeps IMAD adds on the FMA pipe)
    int32_t* card_out;             // CARD mode: [n][rows][card_pitch] (rows from row_base)
    int64_t card_pitch;            // elements
    int64_t card_stride;           // elements per image
    HaloPeers peers;               // single-image bands only
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// 4-D tile load: coordinates {px-in-chunk, chunk, row, image}.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t lds32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }

// Loads the 2*BETA+1 column-shifted variants of a staged row around the
// thread's word (rowp points at the word): v[BETA+dc] holds, in byte j, the
// pixel at column 4w+j+dc.
template <int BETA>
__device__ __forceinline__ void load_row(const uint8_t* rowp, uint32_t (&v)[2 * BETA + 1]) {
    const uint32_t c = lds32(rowp);
    const uint32_t l = lds32(rowp - 4);
    const uint32_t r = lds32(rowp + 4);
#pragma unroll
    for (int dc = 1; dc <= BETA; ++dc) {
        v[BETA - dc] = __funnelshift_l(l, c, 8 * dc);
        v[BETA + dc] = __funnelshift_r(c, r, 8 * dc);
    }
    v[BETA] = c;
}

__device__ __forceinline__ uint32_t fma_add(uint32_t x, uint32_t one, uint32_t k);

// Vertical pair symmetry: the same-column pair (y, y+d) is tested once, at
// row y ("down", returned) and reused as the "up" neighbour of row y+d.
// up[d-1] must hold the mask of the pair (y-d, y); validity of a stored pair
// already includes both rows and the column.
template <int BETA, bool ALE, bool ROWS_OK>
__device__ __forceinline__ uint32_t count_similar_vs(const uint32_t (&win)[2 * BETA + 1][2 * BETA + 1],
                                                     const uint32_t (&colm)[2 * BETA + 1],
                                                     const uint32_t (&rowm)[2 * BETA + 1], uint32_t k7,
                                                     uint32_t one, const uint32_t (&up)[BETA],
                                                     uint32_t (&down)[BETA]);

__device__ __forceinline__ uint32_t rms_round32(uint32_t S, uint32_t f) {
    const float x = fmaxf(__fdividef(static_cast<float>(4u * S), static_cast<float>(f)), 1e-30f);
    const float r = x * rsqrtf(x);
    const int m = __float2int_rn(r);
    if (m & 1) return (static_cast<uint32_t>(m * m) * f <= 4u * S) ? (m + 1) >> 1 : (m - 1) >> 1;
    return static_cast<uint32_t>(m) >> 1;
}

// One candidate pixel: decide and compute the RMS replacement exactly as
// removal_rows (denoise.hpp:192-217).  Cells outside the image hold 0 in the
// staged tile, so they add nothing to the sum of squares and count as
// dissimilar exactly when p >= alpha; the in-bounds count corrects f.
// Returns 1 if an owned pixel was replaced (per-iteration counters).
template <int BETA>
__device__ __forceinline__ uint32_t process_pixel(int y, int px, uint32_t interior, const uint8_t* src,
                                                  uint8_t* dst, int gx0, int gy0, int own_y_lo, int own_y_hi,
                                                  const TileArgs& a) {
    constexpr int W2 = (2 * BETA + 1) * (2 * BETA + 1);
    const uint8_t* c = src + y * kRP + px;
    const int p = *c;
    uint32_t S = 0, fc = 0;
#pragma unroll
    for (int dy = -BETA; dy <= BETA; ++dy)
#pragma unroll
        for (int dx = -BETA; dx <= BETA; ++dx) {
            if (dy == 0 && dx == 0) continue;
            const uint32_t q = c[dy * kRP + dx];
            const bool dis = __vabsdiffu4(q, static_cast<uint32_t>(p)) >= static_cast<uint32_t>(a.alpha);
            S += dis ? q * q : 0u;
            fc += dis;
        }
    const int gr = gy0 + y, gc = gx0 + px;
    const int inb = (min(gr + BETA, a.height - 1) - max(gr - BETA, 0) + 1) *
                    (min(gc + BETA, a.width - 1) - max(gc - BETA, 0) + 1);
    const int f = static_cast<int>(fc) - (p >= a.alpha ? W2 - inb : 0);
    const int pix_count = a.faithful ? W2 : inb;
    if (f > pix_count - 3 && f > 0) {
        dst[y * kRP + px] = static_cast<uint8_t>(rms_round32(S, static_cast<uint32_t>(f)));
        if (interior) return 0u;  // counted by the sweep
        return (y >= own_y_lo && y < own_y_hi && px >= kLeftPx && px < kLeftPx + kOutPx && gc < a.width) ? 1u
                                                                                                         : 0u;
    }
    return 0;
}

// t = x + k as an IMAD (FMA pipe): `one` is an opaque runtime 1, so ptxas
// cannot fold the multiply into an ALU add.
__device__ __forceinline__ uint32_t fma_add(uint32_t x, uint32_t one, uint32_t k) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(k));
    return r;
}

template <int BETA, bool ALE, bool ROWS_OK>
__device__ __forceinline__ uint32_t count_similar_vs(const uint32_t (&win)[2 * BETA + 1][2 * BETA + 1],
                                                     const uint32_t (&colm)[2 * BETA + 1],
                                                     const uint32_t (&rowm)[2 * BETA + 1], uint32_t k7,
                                                     uint32_t one, const uint32_t (&up)[BETA],
                                                     uint32_t (&down)[BETA]) {
    const uint32_t p = win[BETA][BETA];
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < 2 * BETA + 1; ++i) {
#pragma unroll
        for (int j = 0; j < 2 * BETA + 1; ++j) {
            if (i == BETA && j == BETA) continue;
            if (j == BETA && i < BETA) {
                cnt += up[BETA - i - 1] >> 7;  // (y-d, y) tested at row y-d
                continue;
            }
            uint32_t valid = ROWS_OK ? colm[j] : (colm[j] & rowm[i]);
            if (j == BETA && i > BETA && !ROWS_OK) valid &= rowm[BETA];  // stored for row y+d
            const uint32_t d = __vabsdiffu4(p, win[i][j]);
            const uint32_t tt = fma_add(d & kLo7, one, k7);
            const uint32_t sm = valid & ~(ALE ? (d | tt) : (d & tt));
            if (j == BETA && i > BETA) down[i - BETA - 1] = sm;
            cnt += sm >> 7;
        }
    }
    return cnt;
}

// CARD = true: one cardinality pass (compute_cardinality, denoise.hpp:
// 227-241) -- the same staged sweep, the per-lane counts C written as int32
// for the owned in-image pixels, no removal.
template <int BETA, int T, bool ALE, bool CARD = false>
__global__ void __launch_bounds__(kThreads)
    fused_tb_kernel(const __grid_constant__ CUtensorMap src_map, const TileArgs a) {
    static_assert(BETA * T <= kMaxHaloPx, "halo exceeds the staged columns");
    constexpr int HALO = BETA * T;
    constexpr int NB = 2 * BETA + 1;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][2];

    const int sh = a.th + 2 * HALO;
    uint8_t* buf[2] = {smem, smem + buf_bytes(sh)};
    const int lane = threadIdx.x & 31;
    uint8_t* cmap = smem + 2 * buf_bytes(sh);  // [sh][128] candidate nibbles
    uint16_t* list = reinterpret_cast<uint16_t*>(cmap + (kCompWords * sh + 127) / 128 * 128) +
                     (threadIdx.x >> 5) * kRing;

    const int img = blockIdx.z;
    const int x0 = blockIdx.x * kOutPx - kLeftPx;  // global col of region px 0 (16-aligned)
    const int out_r0 = (a.own_lo - a.row_base) + blockIdx.y * a.th;  // buffer row
    const int out_rows = min(a.th, (a.own_hi - a.row_base) - out_r0);
    const int y0 = out_r0 - HALO;  // buffer row of region row 0
    const int gy0 = a.row_base + y0;  // global row of region row 0

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(kRP * sh));
        tma_load_4d(buf[0], &src_map, 0, x0 / kChunk, y0, img, &bar);
    }
    if (threadIdx.x < 2 * T) red[threadIdx.x >> 1][threadIdx.x & 1] = 0;

    const int w = kFirstWord + threadIdx.x % kCompWords;  // region word
    const int g = threadIdx.x / kCompWords;
    const int gcol = x0 + 4 * w;  // global col of lane 0

    uint32_t colm[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        uint32_t m = 0;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int c = gcol + l + j - BETA;
            if (c >= 0 && c < a.width) m |= 0x80u << (8 * l);
        }
        colm[j] = m;
    }
    const uint32_t inimg_col = colm[BETA];
    const uint32_t inimg_bytes = msb_to_bytes(inimg_col);  // 0xff per in-image lane
    const bool own_word = (w >= kOutWordLo) && (w < kOutWordHi);
    const uint32_t own_col = own_word ? inimg_col : 0u;
    const bool col_border = (gcol - BETA < 0) || (gcol + 3 + BETA > a.width - 1);

    uint32_t nfl[T], nrp[T];
#pragma unroll
    for (int t = 0; t < T; ++t) nfl[t] = nrp[t] = 0;

    __syncthreads();  // barrier init + counters visible
    mbar_wait(&bar, 0);
    {
        // The TMA box reads the whole 16-px chunk that holds column W-1; its
        // bytes past the image edge are pitch padding, not zeros.  Clear them
        // so every cell outside the image is 0 in the staged tile.
        const int zlo = a.width - x0, zhi = min((a.width + 15) / 16 * 16 - x0, kRP);
        if (zlo >= 0 && zlo < zhi) {
            const int nz = zhi - zlo;
            for (int i = threadIdx.x; i < sh * nz; i += kThreads) buf[0][(i / nz) * kRP + zlo + i % nz] = 0;
            __syncthreads();
        }
    }

    const int g_lo = g * sh / kGroups;
    const int g_hi = (g + 1) * sh / kGroups;

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const uint8_t* src = buf[t & 1];
        uint8_t* dstb = buf[(t + 1) & 1];
        const int ylo = max(g_lo, BETA * (t + 1));
        const int yhi = min(g_hi, sh - BETA * (t + 1));
        uint32_t win[NB][NB];
        const uint8_t* colp = src + 4 * w;
        if (ylo < yhi) {
#pragma unroll
            for (int i = 0; i < NB - 1; ++i) load_row<BETA>(colp + (ylo - BETA + i) * kRP, win[i]);
        }
        // rows with the whole window inside the image need no row masks
        const int yint_lo = min(max(ylo, BETA - gy0), yhi);
        const int yint_hi = max(min(yhi, a.height - BETA - gy0), yint_lo);
        uint32_t fl_acc = 0;  // per-lane flagged counts (bytes; < 256 rows per thread)
        // same-column pairs for the first rows: up[d-1] = (ylo-d, ylo);
        // pend[d-2][q] = (ylo+1+q-d, ylo+1+q) for rows ylo+1+q, q < d-1
        uint32_t up[BETA];
        uint32_t pend[BETA > 1 ? BETA - 1 : 1][BETA > 1 ? BETA - 1 : 1];
        if (ylo < yhi) {
            auto rv = [&](int yy) { const int g = gy0 + yy; return (g >= 0 && g < a.height) ? 0xffffffffu : 0u; };
#pragma unroll
            for (int d = 1; d <= BETA; ++d) {
                const uint32_t da = __vabsdiffu4(win[BETA][BETA], win[BETA - d][BETA]);
                const uint32_t ta = fma_add(da & kLo7, a.one, a.k7);
                up[d - 1] = colm[BETA] & rv(ylo) & rv(ylo - d) & ~(ALE ? (da | ta) : (da & ta));
            }
#pragma unroll
            for (int d = 2; d <= BETA; ++d)
#pragma unroll
                for (int q = 0; q < d - 1; ++q) {
                    // rows ylo+1+q and ylo+1+q-d are window rows BETA+1+q and BETA+1+q-d (< NB-1)
                    const uint32_t db = __vabsdiffu4(win[BETA + 1 + q][BETA], win[BETA + 1 + q - d][BETA]);
                    const uint32_t tb = fma_add(db & kLo7, a.one, a.k7);
                    pend[d - 2][q] = colm[BETA] & rv(ylo + 1 + q) & rv(ylo + 1 + q - d) & ~(ALE ? (db | tb) : (db & tb));
                }
        }
        auto row = [&](int y, auto rows_ok_tag) {
            constexpr bool ROWS_OK = decltype(rows_ok_tag)::value;
            load_row<BETA>(colp + (y + BETA) * kRP, win[NB - 1]);
            const int gr = gy0 + y;
            uint32_t rowm[NB];
            bool row_in = true;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int rr = gr + i - BETA;
                rowm[i] = ROWS_OK || (rr >= 0 && rr < a.height) ? 0xffffffffu : 0u;
            }
            if (!ROWS_OK) row_in = rowm[BETA] != 0;
            uint32_t down[BETA];
            const uint32_t cnt = count_similar_vs<BETA, ALE, ROWS_OK>(win, colm, rowm, a.k7, a.one, up, down);
            // rotate the pending same-column pairs: up[d-1] for row y+1
#pragma unroll
            for (int d = BETA; d >= 2; --d) up[d - 1] = pend[d - 2][0];
            if (BETA >= 2) {
#pragma unroll
                for (int d = 2; d <= BETA; ++d) {
#pragma unroll
                    for (int q = 0; q < d - 2; ++q) pend[d - 2][q] = pend[d - 2][q + 1];
                    pend[d - 2][d - 2] = down[d - 1];
                }
            }
            up[0] = down[0];
            const uint32_t card = cnt + 0x01010101u;
            if constexpr (CARD) {
                if (y >= HALO && y < HALO + out_rows && own_word && row_in) {
                    int32_t* o = a.card_out + img * a.card_stride +
                                 static_cast<int64_t>(gy0 + y - a.row_base) * a.card_pitch + gcol;
                    const int nv = min(4, a.width - gcol);
                    if (nv == 4 && (a.card_pitch & 3) == 0) {
                        *reinterpret_cast<int4*>(o) = make_int4(card & 0xff, (card >> 8) & 0xff, (card >> 16) & 0xff,
                                                               card >> 24);
                    } else {
                        for (int l = 0; l < nv; ++l) o[l] = (card >> (8 * l)) & 0xff;
                    }
                }
            } else {
                const uint32_t inimg = row_in ? inimg_col : 0u;
                const uint32_t flagged = lt_bits(card, a.k_thr) & inimg;
                // interior: in_bounds = pix_count = (2B+1)^2, so
                // flag > pix_count-3 <=> card < 3 (and flag > 0 holds); border
                // words defer the whole decision to the replacement pass.
                const bool interior = ROWS_OK && !col_border;
                const uint32_t cand = interior ? (flagged & lt_bits(card, rep4(125u))) : flagged;
                // pixels outside the image are kept at 0 (see process_pixel)
                *reinterpret_cast<uint32_t*>(dstb + y * kRP + 4 * w) =
                    win[BETA][BETA] & (row_in ? inimg_bytes : 0u);
                // bits 7,15,23,31 -> nibble (no carries: the shifted copies never overlap)
                cmap[y * kCompWords + (w - kFirstWord)] = static_cast<uint8_t>((cand * 0x00204081u) >> 28);
                if (y >= HALO && y < HALO + out_rows) fl_acc += (flagged & own_col) >> 7;
            }
#pragma unroll
            for (int i = 0; i < NB - 1; ++i)
#pragma unroll
                for (int j = 0; j < NB; ++j) win[i][j] = win[i + 1][j];
        };
        for (int y = ylo; y < yint_lo; ++y) row(y, std::false_type{});
#pragma unroll 3
        for (int y = yint_lo; y < yint_hi; ++y) row(y, std::true_type{});
        for (int y = yint_hi; y < yhi; ++y) row(y, std::false_type{});
        if constexpr (CARD) continue;  // T == 1: the map is written, nothing else
        nfl[t] += __dp4a(fl_acc, 0x01010101u, 0u);
        __syncthreads();
        // replacement pass.  Each warp takes rows rlo+warp, +kWarps, ...; a
        // row's candidates (16 px per lane) are compacted with one warp scan
        // into the warp's ring of u16 items (y << 10 | px).  Items carry over
        // between rows, and the ring is drained only in full rounds of 64 --
        // two independent candidates per lane, so both dependency chains
        // (window loads -> sum of squares -> RMS) are in flight together.
        {
            const int warp = threadIdx.x >> 5;
            const int rlo = BETA * (t + 1), rhi = sh - BETA * (t + 1);
            int pending = 0;  // warp-uniform: items waiting at list[0, pending)
            auto item_px = [&](uint32_t it, uint32_t& r) {
                const int yy = it >> 10, px = it & 1023;
                r = process_pixel<BETA>(yy, px, 0u, src, dstb, x0, gy0, HALO, HALO + out_rows, a);
            };
            // process list[h, h+n), n <= 64: two independent items per lane
            auto drain = [&](int h, int n) {
                const bool ok0 = lane < n, ok1 = lane + 32 < n;
                const uint32_t it0 = list[h + (ok0 ? lane : 0)], it1 = list[h + (ok1 ? lane + 32 : 0)];
                uint32_t r0, r1;
                if (n == 64) {
                    item_px(it0, r0);
                    item_px(it1, r1);
                } else {
                    r0 = r1 = 0;
                    if (ok0) item_px(it0, r0);
                    if (ok1) item_px(it1, r1);
                }
                nrp[t] += r0 + r1;
            };
            for (int y = rlo + warp; y < rhi; y += kWarps) {
                // this lane's 16 px (4 words x 4 lanes) as 16 contiguous bits
                const uint32_t e = *reinterpret_cast<const uint32_t*>(cmap + y * kCompWords + 4 * lane) & 0x0f0f0f0fu;
                const uint32_t e2 = e | (e >> 4);
                uint32_t m = __byte_perm(e2, 0, 0x0020) & 0xffffu;  // bytes 0 and 2
                const int n = __popc(m);
                int incl = n;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (total == 0) continue;
                int pos = pending + incl - n;
                const uint32_t base = (static_cast<uint32_t>(y) << 10) | (4 * (kFirstWord + 4 * lane));
                while (m) {
                    // loop-carried chain is two ALU ops; the bit index (XU) is off it
                    const uint32_t lb = m & (0u - m);
                    m ^= lb;
                    list[pos++] = static_cast<uint16_t>(base + __popc(lb - 1u));
                }
                pending += total;
                __syncwarp();
                int h = 0;
                for (; pending - h >= 64; h += 64) drain(h, 64);
                pending -= h;
                if (h && pending) {  // move the < 64 leftovers to the front
                    __syncwarp();
                    const uint16_t v = lane < pending ? list[h + lane] : 0;
                    const uint16_t v2 = lane + 32 < pending ? list[h + lane + 32] : 0;
                    __syncwarp();
                    if (lane < pending) list[lane] = v;
                    if (lane + 32 < pending) list[lane + 32] = v2;
                }
                __syncwarp();
            }
            if (pending > 0) drain(0, pending);
        }
        __syncthreads();
    }

    if constexpr (CARD) return;
    // owned output rows: shared -> global, 16-byte coalesced stores
    {
        const uint8_t* fin = buf[T & 1];
        constexpr int kOutChunks = kOutPx / 16;  // 31
        uint8_t* gbase = a.dst + img * a.image_stride + static_cast<int64_t>(y0) * a.pitch + (x0 + kLeftPx);
        for (int i = threadIdx.x; i < out_rows * kOutChunks; i += kThreads) {
            const int r = i / kOutChunks, ch = i - r * kOutChunks;
            if (x0 + kLeftPx + 16 * ch >= a.width) continue;
            const int y = HALO + r;
            const uint4 v = *reinterpret_cast<const uint4*>(fin + y * kRP + kLeftPx + 16 * ch);
            *reinterpret_cast<uint4*>(gbase + static_cast<int64_t>(y) * a.pitch + 16 * ch) = v;
            mirror_row16(a.peers, a.row_base + y0 + y, a.pitch, x0 + kLeftPx + 16 * ch, v);
        }
    }

    // counters: warp reduce -> smem -> one global atomic per CTA per value
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const unsigned f = __reduce_add_sync(0xffffffffu, nfl[t]);
        const unsigned r = __reduce_add_sync(0xffffffffu, nrp[t]);
        if (lane == 0) {
            if (f) atomicAdd(&red[t][0], f);
            if (r) atomicAdd(&red[t][1], r);
        }
    }
    __syncthreads();
    if (threadIdx.x < 2 * T) {
        const int t = threadIdx.x >> 1, which = threadIdx.x & 1;
        const unsigned v = red[t][which];
        if (v) atomicAdd(&a.counters[((int64_t)img * a.kcap + a.it0 + t) * 2 + which], (unsigned long long)v);
    }
}

// ----------------------------------------------------------- scalar path
enum ScalarMode { kModeCard = 0, kModeRemoval = 1, kModeFused = 2 };

struct ScalarArgs {
    const uint8_t* src;
    uint8_t* dst;
    const int32_t* card_in;
    int32_t* card_out;
    int64_t card_pitch;  // elements
    int64_t pitch;
    int64_t image_stride;
    int width;
    int height;
    int row_base;
    int own_lo;
    int own_hi;
    int alpha;
    int beta;
    int thr;
    int faithful;
    int it0;
    int kcap;
    unsigned long long* counters;
    HaloPeers peers;  // kModeFused on single-image bands
};

// One thread per pixel, global loads (L1/L2 serve the window re-reads).
// Card: counts (denoise.hpp:139-160).  Removal: flagged from the supplied
// map, flag/sum from the image (denoise.hpp:176-223).  Fused: both.
template <int MODE>
__global__ void __launch_bounds__(256) scalar_kernel(const ScalarArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int gr = a.own_lo + blockIdx.y;
    const int img = blockIdx.z;
    unsigned fl = 0, rp = 0;
    if (c < a.width && gr < a.own_hi) {
        const uint8_t* base = a.src + img * a.image_stride;
        const int64_t yb = gr - a.row_base;
        const int r0 = max(0, gr - a.beta), r1 = min(a.height - 1, gr + a.beta);
        const int c0 = max(0, c - a.beta), c1 = min(a.width - 1, c + a.beta);
        const int p = base[yb * a.pitch + c];
        int card = 0;
        if (MODE != kModeRemoval) {
            for (int i = r0; i <= r1; ++i) {
                const uint8_t* row = base + (int64_t)(i - a.row_base) * a.pitch;
                for (int j = c0; j <= c1; ++j) card += abs(row[j] - p) < a.alpha;
            }
        }
        if (MODE == kModeCard) {
            a.card_out[(int64_t)img * a.height * a.card_pitch + yb * a.card_pitch + c] = card;
        } else {
            if (MODE == kModeRemoval)
                card = a.card_in[(int64_t)img * a.height * a.card_pitch + yb * a.card_pitch + c];
            int out = p;
            if (card < a.thr) {
                fl = 1;
                const int inb = (r1 - r0 + 1) * (c1 - c0 + 1);
                const int pix_count = a.faithful ? (2 * a.beta + 1) * (2 * a.beta + 1) : inb;
                uint64_t S = 0;
                int flag = 0;
                for (int i = r0; i <= r1; ++i) {
                    const uint8_t* row = base + (int64_t)(i - a.row_base) * a.pitch;
                    for (int j = c0; j <= c1; ++j) {
                        const int q = row[j];
                        if (abs(q - p) >= a.alpha) {
                            S += static_cast<uint64_t>(q * q);
                            ++flag;
                        }
                    }
                }
                if (flag > pix_count - 3 && flag > 0) {
                    out = static_cast<int>(rms_round(S, flag));
                    rp = 1;
                }
            }
            a.dst[img * a.image_stride + yb * a.pitch + c] = static_cast<uint8_t>(out);
#pragma unroll
            for (int i = 0; i < 2; ++i)
                if (gr >= a.peers.lo[i] && gr < a.peers.hi[i])
                    a.peers.ptr[i][static_cast<int64_t>(gr - a.peers.row0[i]) * a.pitch + c] = static_cast<uint8_t>(out);
        }
    }
    if (MODE != kModeCard && a.counters) {
        fl = __reduce_add_sync(0xffffffffu, fl);
        rp = __reduce_add_sync(0xffffffffu, rp);
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* ctr = a.counters + ((int64_t)img * a.kcap + a.it0) * 2;
            if (fl) atomicAdd(ctr, (unsigned long long)fl);
            if (rp) atomicAdd(ctr + 1, (unsigned long long)rp);
        }
    }
}

}  // namespace phg
