// kernel_card.cuh -- the callers either side of the denoise loop
// (SURVEY.md 8(f) rows f1 and f4):
//
//   card_h2_kernel<MODE>  beta = 1 cardinality map (compute_cardinality,
//                         denoise.hpp:227-241, int32 C per pixel) or the count
//                         of pixels with C < thr (residual_noise_count,
//                         metrics.hpp:52-59) -- the fp16 two-tile sweep of
//                         kernel_h2.cuh with one iteration and no candidates.
//                         HBM-bound: 1 B in + 4 B out per pixel (map), 1 B in
//                         (count).
//   sse_kernel            exact sum of squared differences of two images
//                         (the uint64 numerator of mse, metrics.hpp:25-35):
//                         VABSDIFF4 + IDP.4A per 4 pixels; 2 B in per pixel.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "kernel_h2.cuh"

namespace phg {

enum CardMode { kCardMap = 0, kCardCount = 1 };

struct CardArgs {
    int32_t* card;         // kCardMap: [n][rows][card_pitch] (global rows row_base..)
    int64_t card_pitch;    // elements
    int64_t card_stride;   // elements per image
    int width;
    int height;            // global image height
    int row_base;          // global row of buffer row 0 (0 for whole images)
    int own_lo, own_hi;    // global rows written / counted
    int th;
    int tiles_x, tiles_y, n_tiles;
    uint32_t alpha2;       // half2(alpha, alpha)
    uint32_t thr_h2;       // half2(thr - 1) (kCardCount: C < thr <=> thr-1-cnt >= 1)
    unsigned long long* counts;  // kCardCount: [n_images]
};

__host__ __device__ constexpr int card_smem_bytes(int sh) { return 2 * h2_buf_bytes(sh); }

template <int MODE>
__global__ void __launch_bounds__(256, 2) card_h2_kernel(const __grid_constant__ CUtensorMap src_map,
                                                         const CardArgs a) {
    constexpr int HALO = 1;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[2];
    const int sh = a.th + 2 * HALO;
    const int bufb = h2_buf_bytes(sh);
    const int tid = threadIdx.x;
    const int lane = tid & 31;

    const int per_img = a.tiles_x * a.tiles_y;
    const int tA = 2 * blockIdx.x, tB = tA + 1;
    const bool hasB = tB < a.n_tiles;
    auto decode = [&](int t, int& img, int& x0, int& y0, int& out_rows) {
        img = t / per_img;
        const int r = t - img * per_img;
        const int ty = r / a.tiles_x, tx = r - ty * a.tiles_x;
        x0 = tx * kOutPx - kLeftPx;
        const int out_r0 = (a.own_lo - a.row_base) + ty * a.th;
        out_rows = min(a.th, (a.own_hi - a.row_base) - out_r0);
        y0 = out_r0 - HALO;
    };
    int imgA, x0A, y0A, outA, imgB, x0B, y0B, outB;
    decode(tA, imgA, x0A, y0A, outA);
    decode(hasB ? tB : tA, imgB, x0B, y0B, outB);
    if (!hasB) outB = 0;
    const int gyA = a.row_base + y0A, gyB = a.row_base + y0B;

    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(kRP * sh * (hasB ? 2 : 1)));
        tma_load_4d(smem + bufb, &src_map, 0, x0A / kChunk, y0A, imgA, &bar);
        if (hasB) tma_load_4d(smem + bufb + h2_stage_b(sh), &src_map, 0, x0B / kChunk, y0B, imgB, &bar);
    }
    if (tid < 2) red[tid] = 0;

    const int c = tid % kH2Cols;
    const int g = tid / kH2Cols;
    const int x = 8 + 4 * c;
    auto in_col = [&](int x0, bool has, int rc) {
        const int gx = x0 + rc;
        return has && gx >= 0 && gx < a.width;
    };
    uint32_t kc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rc = x - 2 + 2 * i;
        kc[i] = (in_col(x0A, true, rc) ? 0x64u : 0x74u) | (in_col(x0B, hasB, rc) ? 0x64u : 0x74u) << 8 |
                (in_col(x0A, true, rc + 1) ? 0x64u : 0x74u) << 16 | (in_col(x0B, hasB, rc + 1) ? 0x64u : 0x74u) << 24;
    }
    // owned & in-image columns of this thread, per tile
    const bool own_x = x >= kLeftPx && x < kLeftPx + kOutPx;  // 4-column groups never straddle
    uint32_t ocol[4];  // half2 1.0/0.0 (kCardCount)
    int nA = 0, nB = 0;  // owned in-image columns (kCardMap), a prefix of the 4
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool iA = own_x && in_col(x0A, true, x + j), iB = own_x && in_col(x0B, hasB, x + j);
        ocol[j] = (iA ? 0x3c00u : 0u) | (iB ? 0x3c000000u : 0u);
        nA += iA;
        nB += iB;
    }

    __syncthreads();
    mbar_wait(&bar, 0);
    {
        const uint8_t* sA = smem + bufb;
        const uint8_t* sB = smem + bufb + h2_stage_b(sh);
        for (int i = tid; i < sh * kChunks; i += 256) {
            const int r = i / kChunks, ch = i - r * kChunks;
            const uint4 va = *reinterpret_cast<const uint4*>(sA + r * kRP + 16 * ch);
            const uint4 vb = hasB ? *reinterpret_cast<const uint4*>(sB + r * kRP + 16 * ch) : make_uint4(0, 0, 0, 0);
            uint4 o0, o1;
            o0.x = prmt(va.x, vb.x, 0x5140); o0.y = prmt(va.x, vb.x, 0x7362);
            o0.z = prmt(va.y, vb.y, 0x5140); o0.w = prmt(va.y, vb.y, 0x7362);
            o1.x = prmt(va.z, vb.z, 0x5140); o1.y = prmt(va.z, vb.z, 0x7362);
            o1.z = prmt(va.w, vb.w, 0x5140); o1.w = prmt(va.w, vb.w, 0x7362);
            uint4* d = reinterpret_cast<uint4*>(smem + r * kH2RP + 32 * ch);
            d[0] = o0;
            d[1] = o1;
        }
    }
    __syncthreads();

    const int H = a.height;
    // owned rows only: [HALO, HALO + max(outA, outB)), split between the groups
    const int rows = max(outA, outB);
    const int ylo = HALO + g * rows / 2, yhi = HALO + (g + 1) * rows / 2;
    uint32_t flh = 0;
    if (ylo < yhi) {
        const uint32_t colp = smem_u32(smem) + 16 + 8 * c;
        auto row_oob = [&](int y) {
            const int ra = gyA + y, rb = gyB + y;
            return ((ra >= 0 && ra < H) ? 0u : 0x00100010u) | ((!hasB || (rb >= 0 && rb < H)) ? 0u : 0x10001000u);
        };
        uint32_t v[6], nv[6], up[4];
        uint2 raw, nraw;
        {
            uint32_t pv[6];
            uint2 praw;
            h2_load_row(colp + (ylo - 1) * kH2RP, kc, row_oob(ylo - 1), pv, praw);
            h2_load_row(colp + ylo * kH2RP, kc, row_oob(ylo), v, raw);
            uint32_t s[4], d[5], aa[5];
            h2_pairs_down(pv, v, a.alpha2, s, d, aa);
#pragma unroll
            for (int j = 0; j < 4; ++j) up[j] = h2add(h2add(s[j], d[j]), aa[j + 1]);
        }
        for (int y = ylo; y < yhi; ++y) {
            h2_load_row(colp + (y + 1) * kH2RP, kc, row_oob(y + 1), nv, nraw);
            uint32_t e[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) e[i] = h2sim(v[i], v[i + 1], a.alpha2);
            uint32_t s[4], d[5], aa[5];
            h2_pairs_down(v, nv, a.alpha2, s, d, aa);
            uint32_t cnt[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                cnt[j] = h2add(h2add(h2add(e[j], e[j + 1]), h2add(s[j], d[j + 1])), h2add(aa[j], up[j]));
                up[j] = h2add(h2add(s[j], d[j]), aa[j + 1]);
            }
            if (MODE == kCardMap) {
                // C = cnt + 1 as the low byte of half(1024 + C)
                uint32_t hv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) hv[j] = h2add(cnt[j], 0x64016401u);
                const int r = y - HALO;
                if (r < outA && nA > 0) {
                    int32_t* o = a.card + imgA * a.card_stride + (int64_t)(gyA + y - a.row_base) * a.card_pitch + (x0A + x);
                    const uint4 q = make_uint4(prmt(hv[0], 0, 0x4440), prmt(hv[1], 0, 0x4440), prmt(hv[2], 0, 0x4440),
                                               prmt(hv[3], 0, 0x4440));
                    if (nA == 4 && (a.card_pitch & 3) == 0) {
                        *reinterpret_cast<uint4*>(o) = q;
                    } else {
                        o[0] = q.x;
                        if (nA > 1) o[1] = q.y;
                        if (nA > 2) o[2] = q.z;
                        if (nA > 3) o[3] = q.w;
                    }
                }
                if (r < outB && nB > 0) {
                    int32_t* o = a.card + imgB * a.card_stride + (int64_t)(gyB + y - a.row_base) * a.card_pitch + (x0B + x);
                    const uint4 q = make_uint4(prmt(hv[0], 0, 0x4442), prmt(hv[1], 0, 0x4442), prmt(hv[2], 0, 0x4442),
                                               prmt(hv[3], 0, 0x4442));
                    if (nB == 4 && (a.card_pitch & 3) == 0) {
                        *reinterpret_cast<uint4*>(o) = q;
                    } else {
                        o[0] = q.x;
                        if (nB > 1) o[1] = q.y;
                        if (nB > 2) o[2] = q.z;
                        if (nB > 3) o[3] = q.w;
                    }
                }
            } else {
                const int r = y - HALO;
                const uint32_t om = (r < outA ? 0x0000ffffu : 0u) | (r < outB ? 0xffff0000u : 0u);
                uint32_t acc = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) acc = h2fma(h2sat_sub(a.thr_h2, cnt[j]), ocol[j], acc);
                flh = h2add(flh, acc & om);
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) v[i] = nv[i];
            raw = nraw;
        }
    }
    if (MODE == kCardCount) {
        // per-thread fp16 counts are exact (< 2048)
        unsigned cA = static_cast<unsigned>(__half2float(__ushort_as_half(static_cast<unsigned short>(flh & 0xffffu))));
        unsigned cB = static_cast<unsigned>(__half2float(__ushort_as_half(static_cast<unsigned short>(flh >> 16))));
        cA = __reduce_add_sync(0xffffffffu, cA);
        cB = __reduce_add_sync(0xffffffffu, cB);
        if (lane == 0) {
            if (cA) atomicAdd(&red[0], cA);
            if (cB) atomicAdd(&red[1], cB);
        }
        __syncthreads();
        if (tid == 0 && red[0]) atomicAdd(&a.counts[imgA], (unsigned long long)red[0]);
        if (tid == 1 && red[1]) atomicAdd(&a.counts[imgB], (unsigned long long)red[1]);
    }
}

// Exact sum of (a-b)^2 over [n][rows][width] pitched images (both with the
// same pitch/stride); one 16-byte chunk per thread step.
__global__ void __launch_bounds__(256) sse_kernel(const uint8_t* a, const uint8_t* b, int64_t pitch, int64_t stride,
                                                  int width, int rows, int n, unsigned long long* out) {
    const int chunks = (width + 15) / 16;
    const int64_t total = static_cast<int64_t>(n) * rows * chunks;
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t rr = i / chunks;
        const int ch = static_cast<int>(i - rr * chunks);
        const int img = static_cast<int>(rr / rows), r = static_cast<int>(rr - static_cast<int64_t>(img) * rows);
        const int64_t off = img * stride + r * pitch + 16 * ch;
        const uint4 va = *reinterpret_cast<const uint4*>(a + off);
        const uint4 vb = *reinterpret_cast<const uint4*>(b + off);
        const int valid = min(16, width - 16 * ch);
        uint32_t d[4] = {__vabsdiffu4(va.x, vb.x), __vabsdiffu4(va.y, vb.y), __vabsdiffu4(va.z, vb.z),
                         __vabsdiffu4(va.w, vb.w)};
        if (valid < 16) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int nb = min(max(valid - 4 * k, 0), 4);
                d[k] &= nb == 4 ? 0xffffffffu : ((1u << (8 * nb)) - 1u);
            }
        }
        uint32_t s = __dp4a(d[0], d[0], 0u);
        s = __dp4a(d[1], d[1], s);
        s = __dp4a(d[2], d[2], s);
        s = __dp4a(d[3], d[3], s);  // <= 16 * 65025 < 2^21
        acc += s;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Count of map entries below thr, per image ([n][rows][pitch] int32).
__global__ void __launch_bounds__(256) count_lt_kernel(const int32_t* card, int64_t pitch, int width, int rows, int n,
                                                       int thr, unsigned long long* counts) {
    const int img = blockIdx.y;
    const int64_t total = static_cast<int64_t>(rows) * width;
    unsigned cnt = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / width;
        cnt += card[img * rows * pitch + r * pitch + (i - r * width)] < thr;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&counts[img], (unsigned long long)cnt);
}

// ---------------------------------------------------------------------------
// denoise_pass with a caller-supplied cardinality map, beta = 1 or 2
// (removal_rows, denoise.hpp:171-223): flagged <=> map < thr (the map is
// honoured as given, never recomputed); a flagged pixel's 3x3 window gives
// the dissimilar count and sum of squares; replace if flag > pix_count - 3
// and flag > 0.  One thread per 4-pixel word of one row; the block stages
// its 256 x 16 tile plus a 1-row / 16-px apron in shared memory (zeros
// outside the image, corrected by the in-bounds count as in the fused
// kernel), reads the map as int4 and writes 4-byte words.  Per pixel: 1 B in,
// 4 B map in, 1 B out.
struct RemovalArgs {
    const uint8_t* src;
    uint8_t* dst;
    const int32_t* card;
    int64_t card_pitch;    // elements
    int64_t card_stride;   // elements per image
    int64_t pitch;         // image bytes per row (src and dst)
    int64_t image_stride;
    int width, height;
    int alpha, thr, faithful;
    uint32_t k7;           // ((256-alpha) & 0x7f) in every byte
    unsigned long long* counters;  // [n][1][2]
    int row0;              // first row of this launch's tile rows (grid.y <= 65535 per launch)
};

constexpr int kRmTW = 256;          // tile width (px)
constexpr int kRmTH = 16;           // tile height (rows)
constexpr int kRmSP = kRmTW + 32;   // staged row pitch: 16-px aprons

// dissimilar mask (bit 7 per byte) of four pixel pairs: |a - b| >= alpha
template <bool ALE>
__device__ __forceinline__ uint32_t dis4(uint32_t a, uint32_t b, uint32_t k7) {
    const uint32_t d = __vabsdiffu4(a, b);
    const uint32_t t = (d & kLo7) + k7;
    return (ALE ? (d | t) : (d & t)) & kHi;
}

// Flag count and sum of squares of the dissimilar cells among 4 window bytes.
template <bool ALE>
__device__ __forceinline__ void acc_window_word(uint32_t w, uint32_t p4, uint32_t k7, int& fc, uint32_t& S) {
    const uint32_t dis = dis4<ALE>(w, p4, k7);
    fc += __popc(dis);
    S = __dp4a(w & msb_to_bytes(dis), w, S);
}

template <bool ALE, bool VEC, int BETA = 1>
__global__ void __launch_bounds__(256) removal_tile_kernel(const RemovalArgs a) {
    static_assert(BETA == 1 || BETA == 2, "tiled removal covers beta 1 and 2");
    constexpr int W2 = (2 * BETA + 1) * (2 * BETA + 1);
    __shared__ __align__(16) uint8_t tile[(kRmTH + 2 * BETA) * kRmSP];
    const int img = blockIdx.z;
    const int x0 = blockIdx.x * kRmTW, y0 = a.row0 + blockIdx.y * kRmTH;
    const uint8_t* src = a.src + img * a.image_stride;
    // stage rows y0-BETA .. y0+kRmTH+BETA-1, columns x0-16 .. x0+kRmTW+16 (zeros outside)
    for (int i = threadIdx.x; i < (kRmTH + 2 * BETA) * (kRmSP / 16); i += 256) {
        const int r = i / (kRmSP / 16), ch = i - r * (kRmSP / 16);
        const int gy = y0 - BETA + r, gx = x0 - 16 + 16 * ch;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gy >= 0 && gy < a.height && gx >= 0 && gx < a.width) {
            v = *reinterpret_cast<const uint4*>(src + gy * a.pitch + gx);
            const int valid = a.width - gx;  // bytes past the width are pitch padding
            if (valid < 16) {
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int nb = min(max(valid - 4 * k, 0), 4);
                    w[k] &= nb == 4 ? 0xffffffffu : ((1u << (8 * nb)) - 1u);
                }
                v = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        *reinterpret_cast<uint4*>(tile + r * kRmSP + 16 * ch) = v;
    }
    __syncthreads();
    const int wcol = threadIdx.x & 63;   // word column
    const int rg = threadIdx.x >> 6;     // 4 row groups of 4 rows
    const int gx = x0 + 4 * wcol;
    unsigned fl = 0, rp = 0;
    if (gx < a.width) {
        const int nvalid = min(4, a.width - gx);
        for (int rr = 0; rr < kRmTH / 4; ++rr) {
            const int ly = rg * (kRmTH / 4) + rr;  // tile row
            const int gy = y0 + ly;
            if (gy >= a.height) break;
            const int32_t* cp = a.card + img * a.card_stride + gy * a.card_pitch + gx;
            int cv[4];
            if (VEC && nvalid == 4) {
                const int4 c4 = *reinterpret_cast<const int4*>(cp);
                cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) cv[j] = j < nvalid ? cp[j] : 0x7fffffff;
            }
            const uint8_t* c0 = tile + (ly + BETA) * kRmSP + 16 + 4 * wcol;  // this word, staged
            uint32_t out = *reinterpret_cast<const uint32_t*>(c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (cv[j] >= a.thr) continue;
                ++fl;
                int fc = 0;
                uint32_t S = 0, p;
                if (BETA == 1) {
                    // 3x3 window of lane j: three funnel-shifted row words
                    uint32_t R[3];
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        const uint8_t* rp0 = c0 + (r - 1) * kRmSP;
                        const uint32_t lo = *reinterpret_cast<const uint32_t*>(rp0 - 4);
                        const uint32_t mid = *reinterpret_cast<const uint32_t*>(rp0);
                        const uint32_t hi = *reinterpret_cast<const uint32_t*>(rp0 + 4);
                        // bytes j-1, j, j+1 of the word at lane 0
                        R[r] = j == 0 ? __funnelshift_l(lo, mid, 8) : __funnelshift_r(mid, hi, 8 * (j - 1));
                    }
                    const uint32_t p4 = prmt(R[1], 0, 0x1111);
                    acc_window_word<ALE>(prmt(R[0], R[1], 0x4210), p4, a.k7, fc, S);  // t0 t1 t2 m0
                    acc_window_word<ALE>(prmt(R[1], R[2], 0x6542), p4, a.k7, fc, S);  // m2 b0 b1 b2
                    p = (R[1] >> 8) & 0xff;
                } else {
                    // 5x5 window: per row, W = columns j-2..j+1 and X = column j+2
                    uint32_t Wr[5], Xr[5];
#pragma unroll
                    for (int r = 0; r < 5; ++r) {
                        const uint8_t* rp0 = c0 + (r - 2) * kRmSP;
                        const uint32_t lo = *reinterpret_cast<const uint32_t*>(rp0 - 4);
                        const uint32_t mid = *reinterpret_cast<const uint32_t*>(rp0);
                        const uint32_t hi = *reinterpret_cast<const uint32_t*>(rp0 + 4);
                        Wr[r] = j < 2 ? __funnelshift_l(lo, mid, 8 * (2 - j)) : __funnelshift_r(mid, hi, 8 * (j - 2));
                        Xr[r] = j < 2 ? (mid >> (8 * (j + 2))) : (hi >> (8 * (j - 2)));  // byte 0 = column j+2
                    }
                    const uint32_t p4 = prmt(Wr[2], 0, 0x2222);
                    acc_window_word<ALE>(Wr[0], p4, a.k7, fc, S);
                    acc_window_word<ALE>(Wr[1], p4, a.k7, fc, S);
                    acc_window_word<ALE>(Wr[3], p4, a.k7, fc, S);
                    acc_window_word<ALE>(Wr[4], p4, a.k7, fc, S);
                    // column j+2 of rows 0,1,3,4 and row 2 without its centre byte
                    const uint32_t x01 = prmt(Xr[0], Xr[1], 0x0040), x34 = prmt(Xr[3], Xr[4], 0x0040);
                    acc_window_word<ALE>(prmt(x01, x34, 0x5410), p4, a.k7, fc, S);
                    acc_window_word<ALE>(prmt(Wr[2], Xr[2], 0x4310), p4, a.k7, fc, S);
                    p = (Wr[2] >> 16) & 0xff;
                }
                const int gxj = gx + j;
                const int inr = min(gy + BETA, a.height - 1) - max(gy - BETA, 0) + 1;
                const int inc = min(gxj + BETA, a.width - 1) - max(gxj - BETA, 0) + 1;
                const int inb = inr * inc;
                // cells outside the image are 0 in the tile: dissimilar exactly when p >= alpha
                const int f = fc - (static_cast<int>(p) >= a.alpha ? W2 - inb : 0);
                const int pix_count = a.faithful ? W2 : inb;
                if (f > pix_count - 3 && f > 0) {
                    const uint32_t v = rms_round32(S, static_cast<uint32_t>(f));
                    out = (out & ~(0xffu << (8 * j))) | (v << (8 * j));
                    ++rp;
                }
            }
            uint8_t* dp = a.dst + img * a.image_stride + gy * a.pitch + gx;
            if (nvalid == 4) {
                *reinterpret_cast<uint32_t*>(dp) = out;
            } else {
                for (int j = 0; j < nvalid; ++j) dp[j] = static_cast<uint8_t>(out >> (8 * j));
            }
        }
    }
    fl = __reduce_add_sync(0xffffffffu, fl);
    rp = __reduce_add_sync(0xffffffffu, rp);
    if ((threadIdx.x & 31) == 0 && a.counters) {
        if (fl) atomicAdd(&a.counters[img * 2], (unsigned long long)fl);
        if (rp) atomicAdd(&a.counters[img * 2 + 1], (unsigned long long)rp);
    }
}

}  // namespace phg
