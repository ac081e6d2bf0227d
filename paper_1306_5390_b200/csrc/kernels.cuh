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

#include "swar.cuh"

namespace phg {

// ------------------------------------------------------------ geometry
// A tile stages region columns [x0, x0+528) with x0 = tile*496 - 16: a
// 16-px left apron (TMA tile boxes need a 16-byte aligned innermost start
// coordinate, so the apron cannot be narrower), 496 output px and a 16-px
// right apron.  Three TMA boxes fill one shared buffer laid out as
// [SH][256] | [SH][256] | [SH][16].  The 128 threads of a row group compute
// region words 2..129 (8 px either side of the output, so beta*T <= 8).
constexpr int kLeftPx = 16;
constexpr int kOutPx = 496;
constexpr int kRegionPx = kLeftPx + kOutPx + 16;  // 528
constexpr int kCompWords = 128;                  // words 2..129
constexpr int kFirstWord = 2;
constexpr int kOutWordLo = kLeftPx / 4;          // 4
constexpr int kOutWordHi = kOutWordLo + kOutPx / 4;  // 128
constexpr int kGroups = 2;                       // row groups per CTA
constexpr int kThreads = kCompWords * kGroups;
constexpr int kHalfPx = 256;                     // wide TMA box
constexpr int kApronBox = 16;                    // narrow TMA box
constexpr int kMaxHaloPx = 8;

// bytes of one staged buffer of sh rows (rounded for 128-B alignment)
__host__ __device__ constexpr int buf_bytes(int sh) { return (kRegionPx * sh + 127) / 128 * 128; }

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

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// Shared-memory location of region word w: byte offset at row 0 and the
// row pitch of the segment it lives in.
struct WordLoc {
    int off;
    int pitch;
};

__device__ __forceinline__ WordLoc word_loc(int w, int sh) {
    const int px = 4 * w;
    if (px < kHalfPx) return {px, kHalfPx};
    if (px < 2 * kHalfPx) return {kHalfPx * sh + px - kHalfPx, kHalfPx};
    return {2 * kHalfPx * sh + px - 2 * kHalfPx, kApronBox};
}

__device__ __forceinline__ uint32_t lds_word(const uint8_t* buf, WordLoc l, int y) {
    return *reinterpret_cast<const uint32_t*>(buf + l.off + y * l.pitch);
}

// Loads the 2*BETA+1 column-shifted variants of region row y around the
// thread's word: v[BETA+dc] holds, in byte j, the pixel at column 4w+j+dc.
template <int BETA>
__device__ __forceinline__ void load_row(const uint8_t* buf, WordLoc ll, WordLoc lc, WordLoc lr,
                                         int y, uint32_t (&v)[2 * BETA + 1]) {
    const uint32_t c = lds_word(buf, lc, y);
    const uint32_t l = lds_word(buf, ll, y);
    const uint32_t r = lds_word(buf, lr, y);
#pragma unroll
    for (int dc = 1; dc <= BETA; ++dc) {
        v[BETA - dc] = __funnelshift_l(l, c, 8 * dc);
        v[BETA + dc] = __funnelshift_r(c, r, 8 * dc);
    }
    v[BETA] = c;
}

// Number of similar in-bounds neighbours per byte lane (centre excluded).
template <int BETA, bool ALE, bool ROWS_OK>
__device__ __forceinline__ uint32_t count_similar(const uint32_t (&win)[2 * BETA + 1][2 * BETA + 1],
                                                  const uint32_t (&colm)[2 * BETA + 1],
                                                  const uint32_t (&rowm)[2 * BETA + 1],
                                                  uint32_t k7) {
    const uint32_t p = win[BETA][BETA];
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < 2 * BETA + 1; ++i) {
#pragma unroll
        for (int j = 0; j < 2 * BETA + 1; ++j) {
            if (i == BETA && j == BETA) continue;
            const uint32_t valid = ROWS_OK ? colm[j] : (colm[j] & rowm[i]);
            cnt += sim_bits<ALE>(p, win[i][j], k7, valid) >> 7;
        }
    }
    return cnt;
}

// Decides one flagged lane exactly as removal_rows (denoise.hpp:192-217)
// and returns the replacement value, or -1 when the pixel is kept.
template <int BETA>
__device__ __forceinline__ int lane_replacement(const uint32_t (&win)[2 * BETA + 1][2 * BETA + 1],
                                                const uint32_t (&colm)[2 * BETA + 1],
                                                const uint32_t (&rowm)[2 * BETA + 1], int lane,
                                                int alpha, int faithful) {
    const int sh = 8 * lane;
    const int p = (win[BETA][BETA] >> sh) & 0xff;
    uint32_t S = 0;
    int flag = 0, inb = 0;
#pragma unroll
    for (int i = 0; i < 2 * BETA + 1; ++i) {
#pragma unroll
        for (int j = 0; j < 2 * BETA + 1; ++j) {
            const bool ok = ((colm[j] & rowm[i]) >> (sh + 7)) & 1u;
            if (i == BETA && j == BETA) {
                ++inb;
                continue;
            }
            const int q = (win[i][j] >> sh) & 0xff;
            const bool dis = ok && abs(q - p) >= alpha;
            inb += ok;
            flag += dis;
            S += dis ? static_cast<uint32_t>(q * q) : 0u;
        }
    }
    const int window = (2 * BETA + 1) * (2 * BETA + 1);
    const int pix_count = faithful ? window : inb;
    if (flag > pix_count - 3 && flag > 0) return static_cast<int>(rms_round(S, flag));
    return -1;
}

template <int BETA, int T, bool ALE>
__global__ void __launch_bounds__(kThreads)
    fused_tb_kernel(const __grid_constant__ CUtensorMap src_map,
                    const __grid_constant__ CUtensorMap apron_map, const TileArgs a) {
    static_assert(BETA * T <= kMaxHaloPx, "halo exceeds the staged columns");
    constexpr int HALO = BETA * T;
    constexpr int NB = 2 * BETA + 1;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][2];

    const int sh = a.th + 2 * HALO;
    uint8_t* buf[2] = {smem, smem + buf_bytes(sh)};

    const int img = blockIdx.z;
    const int x0 = blockIdx.x * kOutPx - kLeftPx;  // global col of region col 0 (16-aligned)
    const int out_r0 = (a.own_lo - a.row_base) + blockIdx.y * a.th;  // buffer row
    const int out_rows = min(a.th, (a.own_hi - a.row_base) - out_r0);
    const int y0 = out_r0 - HALO;  // buffer row of region row 0

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(kRegionPx * sh));
        tma_load_3d(buf[0], &src_map, x0, y0, img, &bar);
        tma_load_3d(buf[0] + kHalfPx * sh, &src_map, x0 + kHalfPx, y0, img, &bar);
        tma_load_3d(buf[0] + 2 * kHalfPx * sh, &apron_map, x0 + 2 * kHalfPx, y0, img, &bar);
    }
    if (threadIdx.x < 2 * T) red[threadIdx.x >> 1][threadIdx.x & 1] = 0;

    const int w = kFirstWord + threadIdx.x % kCompWords;  // region word
    const int g = threadIdx.x / kCompWords;
    const int gcol = x0 + 4 * w;  // global col of lane 0
    const WordLoc lc = word_loc(w, sh), ll = word_loc(w - 1, sh), lr = word_loc(w + 1, sh);

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
    const bool own_word = (w >= kOutWordLo) && (w < kOutWordHi);
    const uint32_t own_col = own_word ? inimg_col : 0u;
    const bool col_border = (gcol - BETA < 0) || (gcol + 3 + BETA > a.width - 1);

    uint32_t nfl[T], nrp[T];
#pragma unroll
    for (int t = 0; t < T; ++t) nfl[t] = nrp[t] = 0;

    __syncthreads();  // barrier init + counters visible
    mbar_wait(&bar, 0);

    const int g_lo = g * sh / kGroups;
    const int g_hi = (g + 1) * sh / kGroups;

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const uint8_t* src = buf[t & 1];
        uint8_t* dstb = buf[(t + 1) & 1];
        const int ylo = max(g_lo, BETA * (t + 1));
        const int yhi = min(g_hi, sh - BETA * (t + 1));
        uint32_t win[NB][NB];
        if (ylo < yhi) {
#pragma unroll
            for (int i = 0; i < NB - 1; ++i) load_row<BETA>(src, ll, lc, lr, ylo - BETA + i, win[i]);
        }
        for (int y = ylo; y < yhi; ++y) {
            load_row<BETA>(src, ll, lc, lr, y + BETA, win[NB - 1]);
            const int gr = a.row_base + y0 + y;  // global row
            const bool rows_ok = (gr - BETA >= 0) && (gr + BETA < a.height);
            const bool row_in = (gr >= 0) && (gr < a.height);
            uint32_t rowm[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int rr = gr + i - BETA;
                rowm[i] = (rr >= 0 && rr < a.height) ? 0xffffffffu : 0u;
            }
            const uint32_t cnt = rows_ok ? count_similar<BETA, ALE, true>(win, colm, rowm, a.k7)
                                         : count_similar<BETA, ALE, false>(win, colm, rowm, a.k7);
            const uint32_t card = cnt + 0x01010101u;
            const uint32_t inimg = row_in ? inimg_col : 0u;
            const uint32_t flagged = lt_bits(card, a.k_thr) & inimg;
            uint32_t out = win[BETA][BETA];
            uint32_t rep = 0;
            if (flagged) {
                if (rows_ok && !col_border) {
                    // interior: in_bounds = pix_count = (2B+1)^2, so
                    // flag > pix_count-3 <=> card < 3 (and flag > 0 holds).
                    rep = flagged & lt_bits(card, rep4(125u));
                    uint32_t m = rep;
                    while (m) {
                        const int lane = (__ffs(m) - 8) >> 3;
                        m &= m - 1;
                        const int v = lane_replacement<BETA>(win, colm, rowm, lane, a.alpha, a.faithful);
                        out = (out & ~(0xffu << (8 * lane))) | (static_cast<uint32_t>(v) << (8 * lane));
                    }
                } else {
                    uint32_t m = flagged;
                    while (m) {
                        const int lane = (__ffs(m) - 8) >> 3;
                        m &= m - 1;
                        const int v = lane_replacement<BETA>(win, colm, rowm, lane, a.alpha, a.faithful);
                        if (v >= 0) {
                            rep |= 0x80u << (8 * lane);
                            out = (out & ~(0xffu << (8 * lane))) | (static_cast<uint32_t>(v) << (8 * lane));
                        }
                    }
                }
            }
            const bool own_row = (y >= HALO) && (y < HALO + out_rows);
            if (own_row) {
                nfl[t] += __popc(flagged & own_col);
                nrp[t] += __popc(rep & own_col);
            }
            if (t == T - 1) {
                if (own_row && own_word && gcol < a.width) {
                    uint8_t* p = a.dst + img * a.image_stride + (int64_t)(y0 + y) * a.pitch + gcol;
                    *reinterpret_cast<uint32_t*>(p) = out;
                }
            } else {
                *reinterpret_cast<uint32_t*>(dstb + lc.off + y * lc.pitch) = out;
            }
#pragma unroll
            for (int i = 0; i < NB - 1; ++i)
#pragma unroll
                for (int j = 0; j < NB; ++j) win[i][j] = win[i + 1][j];
        }
        if (t + 1 < T) __syncthreads();
    }

    // counters: warp reduce -> smem -> one global atomic per CTA per value
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const unsigned f = __reduce_add_sync(0xffffffffu, nfl[t]);
        const unsigned r = __reduce_add_sync(0xffffffffu, nrp[t]);
        if ((threadIdx.x & 31) == 0) {
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
