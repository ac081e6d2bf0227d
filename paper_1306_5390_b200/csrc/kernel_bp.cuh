// kernel_bp.cuh -- the beta = 1 hot path with packed-bit neighbour logic.
//
// fused_bp_kernel<T, ALE, WIDE>: T fused iterations of cardinality
// (denoise.hpp:139-160) + removal (denoise.hpp:176-223) for beta = 1,
// Faithful borders and card_threshold <= 3 (the reference defaults,
// denoise.hpp:34-39).
//
// What decides a pixel.  With beta = 1, Faithful borders and thr <= 3 a pixel
// is flagged iff it has at most thr-2 similar neighbours among its 8 in-bounds
// neighbours (C = 1 + that count, C < thr), and a flagged pixel is replaced
// iff its whole window is inside the image (an interior flagged pixel has
// flag = 8 - #similar >= 7 > 9 - 3; a border pixel has flag <= in_bounds - 1
// <= 5).  So the sweep only needs "at least one" / "at least two" similar
// neighbours per pixel, which is bit-parallel logic once the similarity tests
// are packed one bit per pixel.
//
// Sweep (one lane = a 32-px strip of a row, one warp = a 1024-px region row):
//   - the four unordered pair directions E, S, SE, SW are tested in byte-SIMD
//     (VABSDIFF4 + the carry trick of swar.cuh, 4 pairs per op), and each
//     test's dissimilar bits are packed into one 32-bit word per 32 px
//     (word i, byte j -> bit 8j + i: one shift-add per word);
//   - a pair credits both of its pixels; credits to the eastern end are a
//     one-pixel shift of the packed word (shE), the row below is carried in
//     registers;
//   - the 8 credits of a pixel are reduced to (o, w) = (>= 1 similar,
//     >= 2 similar) with 3-input majority / or LOP3s: 32 pixels per op.
// Replacement: each warp owns a band of rows.  A finalized row's replaced
// pixels (one 32-bit word per lane) are pushed into the warp's u16 list of
// buffer offsets (a warp scan of the per-lane counts, then a bfind loop,
// three items per trip); whenever a round of 96 is waiting, every lane
// replaces three: the exact RMS of the dissimilar cells of the 3x3 window
// (byte-SIMD masks + IDP.4A sums, h2_rms).
//
// Band boundaries: a warp's first band row lacks the credits of the pairs with
// the row above, which the warp above computes as the last step of its band
// and hands over in shared memory through a pairwise named barrier (warp 0
// computes its own from the row above).  Consecutive iterations synchronise
// only neighbouring warps when every band holds >= 3 rows.
//
// DIRECT / COUNT forms (T = 1, one staged buffer, up to 92-row tiles): see
// the template below.
//
// Tiles.  Narrow images (width <= 512): a CTA holds two consecutive tiles
// (image, row tile) side by side, one per half-warp (lanes 0-15 / 16-31),
// each the full image width -- no column halo at all.  Wide images: one
// 1024-px region per CTA, one column tile when width <= 1024, else 992 output
// columns with 16-px aprons (TMA start coordinates are 16-byte aligned).
// The image is staged once per launch by TMA, the T iterations ping-pong
// between two shared buffers, and only the last iteration's owned rows go to
// HBM (16-byte stores).
//
// Cells outside the image are masked out of every test (the reference's "out
// of bounds cells are not in the window", denoise.hpp:145-149).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "bp_launch.h"
#include "kernel_h2.cuh"

namespace phg {

constexpr int kBpWarps = 8;  // (band splits divide by 8 as a shift)
constexpr int kBpThreads = 32 * kBpWarps;
constexpr int kBpPad = 128;        // dynamic smem starts with a pad (window reads at region column -1)
#ifndef PHG_BP_DRAIN
#define PHG_BP_DRAIN 3  // 2: 974.6 K, 3: 994.4 K, 4: 975.4 K (C4, measured)
#endif
#ifndef PHG_BP_PUSH
#define PHG_BP_PUSH 3
#endif
constexpr int kBpDrain = PHG_BP_DRAIN;        // candidates per lane per drain round
constexpr int kBpPush = PHG_BP_PUSH;          // candidates per push-loop trip
constexpr int kBpRound = 32 * kBpDrain;
constexpr int kBpList = kBpRound + 1024;      // per-warp candidate list (u16 items): < one round + one row

__host__ __device__ constexpr int bp_buf_bytes(int sh) { return (1024 * sh + 64 + 127) / 128 * 128; }
// pad, two staged buffers (DIRECT: one), band-edge credits [warps][32][2],
// candidate lists [warps][kBpList]
__host__ __device__ constexpr int bp_smem_bytes(int sh, bool direct = false) {
    return kBpPad + (direct ? 1 : 2) * bp_buf_bytes(sh) + kBpWarps * 32 * 8 + kBpWarps * kBpList * 2;
}


// packed bit of strip pixel q (word q/4, byte q%4)
__host__ __device__ constexpr uint32_t bp_bit(int q) { return 8u * static_cast<uint32_t>(q & 3) + (q >> 2); }
// strip pixel of packed bit b
__device__ __forceinline__ uint32_t bp_px(uint32_t b) { return 4u * (b & 7u) + (b >> 3); }

// packed mask of the strip pixels q in [lo, hi) (clamped to [0, 32)): byte j
// holds pixels 4i + j, i.e. bits i in [ceil((lo-j)/4), ceil((hi-j)/4))
__device__ __forceinline__ uint32_t bp_range(int lo, int hi) {
    lo = max(lo, 0);
    hi = min(hi, 32);
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int il = (lo - j + 3) >> 2, ih = max(il, (hi - j + 3) >> 2);
        m |= (((1u << ih) - 1u) & ~((1u << il) - 1u)) << (8 * j);
    }
    return m;
}

// (a | b) & c and (a & b) & c as one opaque LOP3, so that the packing shift
// below stays a shift-add (LEA.HI) instead of being split into SHF + LOP3
__device__ __forceinline__ uint32_t lop_or_and(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xa8;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t lop_and_and(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// dissimilar bits of the 32 pairs (a[i] byte j, b[i] byte j), packed:
// VABSDIFF4, LOP3, IMAD (carry-trick add on the FMA pipe), LOP3, LEA.HI per word
template <bool ALE>
__device__ __forceinline__ uint32_t bp_dis(const uint32_t (&a)[8], const uint32_t (&b)[8], uint32_t k7,
                                           uint32_t one) {
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t d = __vabsdiffu4(a[i], b[i]);
        const uint32_t t = (d & kLo7) * one + k7;
        const uint32_t dis = ALE ? lop_or_and(d, t, kHi) : lop_and_and(d, t, kHi);
        acc += dis >> (7 - i);  // LEA.HI (as IMAD.HI on the FMA pipe: 942 -> 907 K, measured)
    }
    return acc;
}

// One pixel east: the bit of strip pixel q moves to pixel q+1; pixel 0 takes
// pixel 31 of the lane to the west (lane 0 takes lane 31's, whose pixel 31
// never has an eastern partner inside the region, so it is 0).
__device__ __forceinline__ uint32_t bp_shE(uint32_t P, int west) {
    const uint32_t prev = __shfl_sync(0xffffffffu, P, west);
    return (P << 8) | ((P >> 23) & 0xfeu) | (prev >> 31);
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

__device__ __forceinline__ uint4 lds128a(uint32_t a) {
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128a(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts32a(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// the lane's strip of one staged row: X[i] = pixels 4i..4i+3, EX[i] = pixels 4i+1..4i+4
__device__ __forceinline__ void bp_load(uint32_t a, uint32_t (&X)[8], uint32_t (&EX)[8]) {
    const uint4 u0 = lds128a(a), u1 = lds128a(a + 16);
    const uint32_t nx = lds32a(a + 32);
    X[0] = u0.x; X[1] = u0.y; X[2] = u0.z; X[3] = u0.w;
    X[4] = u1.x; X[5] = u1.y; X[6] = u1.z; X[7] = u1.w;
#pragma unroll
    for (int i = 0; i < 7; ++i) EX[i] = __funnelshift_r(X[i], X[i + 1], 8);
    EX[7] = __funnelshift_r(X[7], nx, 8);
}

// RMS replacement of one candidate (interior, Faithful, beta = 1), exactly as
// removal_rows (denoise.hpp:199-217); `o1` = shared address of the window's
// top-left cell, RP = staged row pitch.  Returns the new value.
template <bool ALE, int RP>
__device__ __forceinline__ uint32_t bp_replace(uint32_t o1, uint32_t k7) {
    const uint32_t b4 = o1 & ~3u;
    uint32_t R[3];  // bytes 0..2: the window row
#pragma unroll
    for (int r = 0; r < 3; ++r) R[r] = prmt_f4e(lds32a(b4 + r * RP), lds32a(b4 + r * RP + 4), o1);
    const uint32_t n1 = prmt(R[0], R[1], 0x4210);  // t0 t1 t2 m0
    const uint32_t n2 = prmt(R[1], R[2], 0x6542);  // m2 b0 b1 b2
    const uint32_t p4 = prmt(R[1], 0, 0x1111);     // centre x4
    const uint32_t d1 = __vabsdiffu4(n1, p4), d2 = __vabsdiffu4(n2, p4);
    const uint32_t t1 = (d1 & kLo7) + k7, t2 = (d2 & kLo7) + k7;
    const uint32_t dis1 = (ALE ? (d1 | t1) : (d1 & t1)) & kHi;
    const uint32_t dis2 = (ALE ? (d2 | t2) : (d2 & t2)) & kHi;
    const uint32_t f = __popc(dis1 | (dis2 >> 1));
    const uint32_t S = __dp4a(n2 & msb_to_bytes(dis2), n2, __dp4a(n1 & msb_to_bytes(dis1), n1, 0u));
    return h2_rms(S, f, rms_rcp<7>(f));  // f in {7, 8}
}

// DIRECT (T = 1, wide regions, no peer mirrors): one staged buffer; owned
// rows and replaced pixels are stored straight to HBM (see kernel_bp2.cuh).
// COUNT (T = 1, one staged buffer, either layout): the sweep alone -- the
// number of owned pixels with C < card_threshold per image goes to
// counters[image] (residual_noise_count, metrics.hpp:52-59); nothing is
// replaced or stored.
template <int T, bool ALE, bool WIDE, bool DIRECT = false, bool COUNT = false>
__global__ void __launch_bounds__(kBpThreads, 2)
    fused_bp_kernel(const __grid_constant__ CUtensorMap src_map, const BpArgs a) {
    static_assert(T >= 1 && T <= 8, "halo exceeds the aprons");
    static_assert(!DIRECT || (T == 1 && WIDE), "direct stores: one iteration, wide regions");
    static_assert(!COUNT || (T == 1 && !DIRECT), "count: one iteration");
    constexpr bool SINGLE = DIRECT || COUNT;  // one staged buffer
    constexpr int HALO = T;
    constexpr int RP = WIDE ? 1024 : 512;  // staged row pitch of one tile
    constexpr int NH = WIDE ? 1 : 2;       // tiles per CTA
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][4];  // flagged h0, flagged h1, replaced h0, replaced h1

    uint8_t* smem = smem_raw + kBpPad;
    const int sh = a.th + 2 * HALO;
    const int bufb = bp_buf_bytes(sh);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t down_a = s0 + (SINGLE ? 1 : 2) * bufb;  // [warps][32][2] u32 band-edge credits
    const uint32_t list_a = down_a + kBpWarps * 32 * 8 + warp * kBpList * 2;  // this warp's u16 list
    const uint32_t half_bytes = static_cast<uint32_t>(sh) * 512u;  // narrow: tile B offset

    // ---- the tiles of this CTA
    const int per_img = a.tiles_x * a.tiles_y;
    auto decode = [&](int t, int& img, int& x0, int& y0, int& out_rows) {
        img = t / per_img;
        const int r = t - img * per_img;
        const int ty = r / a.tiles_x, tx = r - ty * a.tiles_x;
        x0 = tx * a.x_step - a.x_apron;
        const int out_r0 = (a.own_lo - a.row_base) + ty * a.th;
        out_rows = min(a.th, (a.own_hi - a.row_base) - out_r0);
        y0 = out_r0 - HALO;
    };
    const int tA = NH * blockIdx.x;
    const int tB = tA + 1;
    const bool hasB = !WIDE && tB < a.n_tiles;
    int imgA, x0A, y0A, outA, imgB = 0, x0B = 0, y0B = 0, outB = 0;
    decode(tA, imgA, x0A, y0A, outA);
    if (hasB) decode(tB, imgB, x0B, y0B, outB);

    // device early exit: an image whose previous iteration replaced nothing is
    // at a fixed point (denoise.hpp:308); its iterations are plain copies
    bool convA = false, convB = !hasB;
    if (a.early && a.it0 > 0) {
        convA = a.counters[(static_cast<int64_t>(imgA) * a.kcap + a.it0 - 1) * 2 + 1] == 0ull;
        if (hasB) convB = a.counters[(static_cast<int64_t>(imgB) * a.kcap + a.it0 - 1) * 2 + 1] == 0ull;
    }
    const int nit = (convA && convB) ? 0 : T;

    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(RP * sh * (hasB ? 2 : 1)));
        tma_load_4d(smem, &src_map, 0, x0A / kChunk, y0A, imgA, &bar);
        if (hasB) tma_load_4d(smem + half_bytes, &src_map, 0, x0B / kChunk, y0B, imgB, &bar);
    }
    if (tid < 4 * T) (&red[0][0])[tid] = 0;

    // ---- per-lane constants: the lane's 32-px strip of its tile
    const int half = WIDE ? 0 : (lane >> 4);
    const int lw = WIDE ? lane : (lane & 15);
    auto lbase = [&](int l) -> uint32_t {  // byte offset of lane l's strip in a buffer row 0
        return WIDE ? static_cast<uint32_t>(l) * 32u
                    : static_cast<uint32_t>(l >> 4) * half_bytes + static_cast<uint32_t>(l & 15) * 32u;
    };
    const uint32_t cb = lbase(lane);
    const bool myhas = half ? hasB : true;
    const int myx0 = half ? x0B : x0A;
    const int gy0 = a.row_base + (half ? y0B : y0A);
    const int myout = half ? outB : outA;
    const bool myconv = half ? convB : convA;
    const int W = a.width, H = a.height;
    // column classes of the strip (packed masks): in the image, E pair inside
    // the image and the region, interior (whole window in the image), output
    const int gxs = myx0 + lw * 32;  // global column of strip pixel 0
    const int wr = max(min(W - gxs, 64), -64);  // clamped distances keep the ints small
    const int gl = max(min(-gxs, 64), -64);
    const uint32_t cIn = myhas ? bp_range(gl, wr) : 0u;
    const uint32_t cE = myhas ? bp_range(gl, min(wr - 1, RP - 1 - lw * 32)) : 0u;
    const uint32_t cInt = myhas ? bp_range(gl + 1, wr - 1) : 0u;
    const uint32_t cOwn = WIDE ? (cIn & bp_range(a.x_apron - lw * 32, a.x_apron + a.x_step - lw * 32)) : cIn;
    const uint32_t cF = myconv ? 0u : (cIn & a.enable);
    // row classes (buffer rows): valid [vlo, vhi), interior [ilo, ihi), owned [HALO, HALO + myout)
    const int vlo = myhas ? max(0, -gy0) : 0;
    const int vhi = myhas ? max(vlo, min(sh, H - gy0)) : 0;
    const int ilo = max(0, 1 - gy0);
    const int ihi = myhas ? max(ilo, min(sh, H - 1 - gy0)) : ilo;
    auto rowin = [&](int y) { return static_cast<unsigned>(y - vlo) < static_cast<unsigned>(vhi - vlo); };
    auto rowint = [&](int y) { return static_cast<unsigned>(y - ilo) < static_cast<unsigned>(ihi - ilo); };
    auto rowown = [&](int y) { return static_cast<unsigned>(y - HALO) < static_cast<unsigned>(myout); };
    const int west = (lane + 31) & 31;
    // DIRECT: global offset of the tile's buffer row 0, region column 0, and
    // which of the lane's two 16-px chunks are output columns
    const int64_t gtile = static_cast<int64_t>(imgA) * a.image_stride + static_cast<int64_t>(y0A) * a.pitch + x0A;
    const int px0 = lane * 32;
    const bool own0 = px0 >= a.x_apron && px0 < a.x_apron + a.x_step && x0A + px0 < W;
    const bool own1 = px0 + 16 >= a.x_apron && px0 + 16 < a.x_apron + a.x_step && x0A + px0 + 16 < W;

    __syncthreads();  // barrier init + counters visible
    mbar_wait(&bar, 0);

    for (int t = 0; t < nit; ++t) {
        const uint32_t src = s0 + ((t & 1) ? bufb : 0);
        const uint32_t dst = s0 + ((t & 1) ? 0 : bufb);
        const int lo = t + 1, n = sh - 2 - 2 * t;  // computed rows [lo, lo + n)
        const int nb = min(kBpWarps, n);
        // (nb == 8 whenever n >= 8: a shift instead of two integer divisions)
        const int b0 = lo + (nb == kBpWarps ? (n * warp) >> 3 : n * warp / nb);
        const int b1 = lo + (nb == kBpWarps ? (n * (warp + 1)) >> 3 : n * (warp + 1) / nb);
        const bool active = warp < nb;
        unsigned fl = 0, rp = 0;  // owned flagged / replaced (this lane's strip)
        uint32_t of = 0, wf = 0;  // the band's first row before its upper credits
        uint32_t Rh = 0;          // a finalized row held back to share the next row's push
        int yh = 0;
        bool held = false;        // warp-uniform
        uint32_t oM = 0, wM = 0;  // warp 0: the first row's upper credits

        // flagged (F) and replaced (R) pixels of row y from its (o, w) counts
        auto finalize = [&](int y, uint32_t o, uint32_t w) {
            const uint32_t F = ~(w | (o & a.sel2)) & (rowin(y) ? cF : 0u);
            const uint32_t R = F & (rowint(y) ? cInt : 0u);
            if (rowown(y)) {
                fl += __popc(F & cOwn);
                rp += __popc(R & cOwn);
            }
            // DIRECT: only owned candidates (nothing reads the others)
            return DIRECT ? (rowown(y) ? R & cOwn : 0u) : R;
        };
        unsigned pending = 0;  // warp-uniform: candidates waiting at list[0, pending)
        // replaces the candidates list[h, h + n), n <= kBpRound: kBpDrain per
        // lane, all loads first
        // DIRECT items are relative to the band's first row
        const uint32_t ibase = DIRECT ? static_cast<uint32_t>(b0) * RP : 0u;
        uint8_t* const gband = a.dst + gtile + static_cast<int64_t>(b0) * a.pitch;
        auto drain = [&](unsigned h, unsigned n) {
            uint32_t o[kBpDrain], v[kBpDrain];
#pragma unroll
            for (int u = 0; u < kBpDrain; ++u) {
                const unsigned i = lane + 32u * u;
                o[u] = lds16(list_a + 2 * (h + (i < n ? i : 0u)));
            }
#pragma unroll
            for (int u = 0; u < kBpDrain; ++u) v[u] = bp_replace<ALE, RP>(src + ibase + o[u] - RP - 1, a.k7);
#pragma unroll
            for (int u = 0; u < kBpDrain; ++u)
                if (lane + 32u * u < n) {
                    if constexpr (DIRECT)
                        gband[static_cast<int64_t>(o[u] >> 10) * a.pitch + (o[u] & 1023u)] = static_cast<uint8_t>(v[u]);
                    else
                        sts8a(dst + o[u], v[u]);
                }
        };
        // drains whole rounds once kBpRound candidates wait; the leftovers
        // (< kBpRound) move to the front of the list
        auto drain_full = [&]() {
            if (pending >= kBpRound) {
                __syncwarp();  // items and the destination row copies are visible
                unsigned h = 0;
                for (; pending - h >= kBpRound; h += kBpRound) drain(h, kBpRound);
                pending -= h;
                __syncwarp();
                if (pending) {
                    uint32_t l[kBpDrain];
#pragma unroll
                    for (int u = 0; u < kBpDrain; ++u)
                        l[u] = lane + 32u * u < pending ? lds16(list_a + 2 * (h + lane + 32u * u)) : 0u;
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < kBpDrain; ++u)
                        if (lane + 32u * u < pending) sts16(list_a + 2 * (lane + 32u * u), l[u]);
                }
                __syncwarp();
            }
        };
        // appends row y's candidates R (u16 buffer offsets) at the lane's
        // prefix `excl` (within the row) of the list tail, three per loop trip
        auto emit = [&](uint32_t mm, int y, unsigned excl) {
            const uint32_t rowoff = cb + static_cast<uint32_t>(y) * RP - ibase;
            uint32_t la = list_a + 2 * (pending + excl);
            while (mm) {
#pragma unroll
                for (int u = 0; u < kBpPush; ++u) {
                    uint32_t b, m1;
                    asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(mm));    // ~0 once mm is empty
                    asm("shl.b32 %0, 1, %1;" : "=r"(m1) : "r"(b));   // 0 for shifts >= 32
                    if (u == 0 || mm) sts16(la + 2 * u, rowoff + bp_px(b));
                    mm ^= m1;
                }
                la += 2 * kBpPush;
            }
        };
        // pushes the candidates RA of row yA and RB of row yB with ONE warp
        // scan (the two counts packed in 16-bit halves) and one drain check;
        // only when both rows would not fit behind the waiting items (dense
        // rows) is row A drained before row B is appended
        auto push = [&](uint32_t RA, int yA, uint32_t RB, int yB) {
            const unsigned cA = __popc(RA), cB = __popc(RB), c = cA | (cB << 16);
            unsigned incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) return;
            const unsigned tA = total & 0xffffu, tB = total >> 16;
            const bool split = pending + tA + tB > static_cast<unsigned>(kBpList);
            emit(RA, yA, (incl & 0xffffu) - cA);
            pending += tA;
            if (split) drain_full();
            emit(RB, yB, (incl >> 16) - cB);
            pending += tB;
            drain_full();
        };
        // one row per warp scan: the T > 1 kernels (the two-row form measured
        // C4 +-0, C2 -1.5%; the single-buffer T = 1 form C5 +1.6%)
        auto push1 = [&](uint32_t R, int y) {
            const unsigned c = __popc(R);
            unsigned incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) return;
            emit(R, y, incl - c);
            pending += total;
            drain_full();
        };

        if (active) {
            uint32_t X[8], EX[8], Xn[8], EXn[8];
            bp_load(src + cb + b0 * RP, X, EX);
            bool rv = rowin(b0);
            uint32_t e = ~bp_dis<ALE>(X, EX, a.k7, a.one) & (rv ? cE : 0u);
            uint32_t oP = 0, wP = 0, seP = 0;  // pairs with the row above: s|sw, s&sw, se
            if (warp == 0) {  // the row above the computed range is staged: credits from it
                bp_load(src + cb + (b0 - 1) * RP, Xn, EXn);
                const bool rp_ = rowin(b0 - 1) && rv;
                const uint32_t s_ = ~bp_dis<ALE>(Xn, X, a.k7, a.one) & (rp_ ? cIn : 0u);
                const uint32_t se_ = ~bp_dis<ALE>(Xn, EX, a.k7, a.one) & (rp_ ? cE : 0u);
                const uint32_t sw_ = ~bp_dis<ALE>(EXn, X, a.k7, a.one) & (rp_ ? cE : 0u);
                const uint32_t sse = bp_shE(se_, west);
                oM = s_ | sw_ | sse;
                wM = maj3(s_, sw_, sse);
            }
#pragma unroll 2
            for (int y = b0; y < b1; ++y) {
                bp_load(src + cb + (y + 1) * RP, Xn, EXn);
                const bool rvn = rowin(y + 1);
                const bool both = rv && rvn;
                const uint32_t s = ~bp_dis<ALE>(X, Xn, a.k7, a.one) & (both ? cIn : 0u);
                const uint32_t se = ~bp_dis<ALE>(X, EXn, a.k7, a.one) & (both ? cE : 0u);
                const uint32_t sw = ~bp_dis<ALE>(EX, Xn, a.k7, a.one) & (both ? cE : 0u);
                // unshifted credits of row y: s(y-1), sw(y-1) [oP, wP], e, s, se
                const uint32_t o2 = e | s | se, w2 = maj3(e, s, se);
                const uint32_t wA = wP | w2 | (oP & o2), oA = oP | o2;
                // credits to the eastern end: e(y), se(y-1), sw(y)
                const uint32_t oB = bp_shE(e | seP | sw, west);
                const uint32_t wB = bp_shE(maj3(e, seP, sw), west);
                const uint32_t w = wA | wB | (oA & oB), o = oA | oB;
                // the unchanged row goes to the destination (candidates are
                // overwritten by the replacement)
                if constexpr (COUNT) {
                } else if constexpr (DIRECT) {
                    if (rowown(y)) {
                        uint8_t* g = a.dst + gtile + static_cast<int64_t>(y) * a.pitch + px0;
                        if (own0) *reinterpret_cast<uint4*>(g) = make_uint4(X[0], X[1], X[2], X[3]);
                        if (own1) *reinterpret_cast<uint4*>(g + 16) = make_uint4(X[4], X[5], X[6], X[7]);
                    }
                } else {
                    const uint32_t da = dst + cb + y * RP;
                    sts128a(da, make_uint4(X[0], X[1], X[2], X[3]));
                    sts128a(da + 16, make_uint4(X[4], X[5], X[6], X[7]));
                }
                if (y == b0) {
                    of = o;
                    wf = w;
                } else if constexpr (COUNT) {
                    finalize(y, o, w);
                } else if constexpr (!SINGLE) {
                    push1(finalize(y, o, w), y);
                } else if (held) {
                    push(Rh, yh, finalize(y, o, w), y);
                    held = false;
                } else {
                    Rh = finalize(y, o, w);
                    yh = y;
                    held = true;
                }
                oP = s | sw;
                wP = s & sw;
                seP = se;
                if (y + 1 < b1) e = ~bp_dis<ALE>(Xn, EXn, a.k7, a.one) & (rvn ? cE : 0u);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    X[i] = Xn[i];
                    EX[i] = EXn[i];
                }
                rv = rvn;
            }
            // credits of the pairs (b1-1, b1) for the next band's first row
            // (handed over through named barrier 1 + warp: this warp arrives,
            // the warp below waits -- no CTA-wide barrier in mid-iteration)
            if (warp + 1 < nb) {
                const uint32_t sse = bp_shE(seP, west);
                const uint32_t dn = down_a + (warp * 32 + lane) * 8;
                sts32a(dn, oP | sse);
                sts32a(dn + 4, wP | (oP & sse));  // maj3(s, sw, sse)
                asm volatile("bar.arrive %0, 64;" ::"r"(1 + warp) : "memory");
            }
        }
        if (active) {
            if (warp > 0) {
                asm volatile("bar.sync %0, 64;" ::"r"(warp) : "memory");
                const uint32_t dn = down_a + ((warp - 1) * 32 + lane) * 8;
                oM = lds32a(dn);
                wM = lds32a(dn + 4);
            }
            if constexpr (COUNT)
                finalize(b0, of | oM, wf | wM | (of & oM));
            else
                if constexpr (SINGLE)
                    push(finalize(b0, of | oM, wf | wM | (of & oM)), b0, held ? Rh : 0u, yh);
                else
                    push1(finalize(b0, of | oM, wf | wM | (of & oM)), b0);
            if (pending) {
                __syncwarp();
                drain(0, pending);
            }
        }
        // per-tile counters of this iteration
        unsigned flA = (WIDE || lane < 16) ? fl : 0u, flB = fl - flA;
        unsigned rpA = (WIDE || lane < 16) ? rp : 0u, rpB = rp - rpA;
        flA = __reduce_add_sync(0xffffffffu, flA);
        rpA = __reduce_add_sync(0xffffffffu, rpA);
        if (!WIDE) {
            flB = __reduce_add_sync(0xffffffffu, flB);
            rpB = __reduce_add_sync(0xffffffffu, rpB);
        }
        if (lane == 0) {
            if (flA) atomicAdd(&red[t][0], flA);
            if (flB) atomicAdd(&red[t][1], flB);
            if (rpA) atomicAdd(&red[t][2], rpA);
            if (rpB) atomicAdd(&red[t][3], rpB);
        }
        // End of iteration t.  Iteration t+1 reads, around its band, rows at
        // most 3 above and 2 below it -- rows of this warp's two neighbours
        // when every band of both iterations holds >= 3 rows.  Then only the
        // neighbours are waited for (pairwise named barriers 8 + w for warps
        // w, w+1); otherwise, and before the output stores, the whole CTA.
        if (t + 1 < nit && n - 2 >= 3 * kBpWarps) {
            if (warp > 0) asm volatile("bar.sync %0, 64;" ::"r"(8 + warp - 1) : "memory");
            if (warp + 1 < kBpWarps) asm volatile("bar.sync %0, 64;" ::"r"(8 + warp) : "memory");
        } else {
            __syncthreads();
        }
    }

    // ---- owned output rows: 16-byte coalesced stores (DIRECT: only when
    // the iteration was skipped -- the staged rows are the result)
    if (!SINGLE || (DIRECT && nit == 0)) {
        const uint8_t* fin = smem + ((nit & 1) ? bufb : 0);
        constexpr int kChunksRow = RP / 16;
        const int c_lo = a.x_apron / 16;
        const int c_n = WIDE ? a.x_step / 16 : kChunksRow;
        // warps over (tile, row), lanes over the row's 16-byte chunks
        for (int hh = 0; hh < NH; ++hh) {
            const int out_h = hh ? outB : outA;
            const int x0h = hh ? x0B : x0A;
            uint8_t* gdst = a.dst + (hh ? imgB : imgA) * a.image_stride;
            const int y0h = hh ? y0B : y0A;
            for (int r = warp; r < out_h; r += kBpWarps) {
                const int y = HALO + r;
                for (int ch = c_lo + lane; ch < c_lo + c_n; ch += 32) {
                    if (x0h + 16 * ch >= a.width) break;
                    const uint4 v = *reinterpret_cast<const uint4*>(fin + hh * half_bytes + y * RP + 16 * ch);
                    *reinterpret_cast<uint4*>(gdst + static_cast<int64_t>(y0h + y) * a.pitch + x0h + 16 * ch) = v;
                    mirror_row16(a.peers, a.row_base + y0h + y, a.pitch, x0h + 16 * ch, v);
                }
            }
        }
    }
    if constexpr (COUNT) {
        if (tid < 2) {
            const unsigned v = red[0][tid];
            if (v) atomicAdd(&a.counters[tid ? imgB : imgA], static_cast<unsigned long long>(v));
        }
    } else if (tid < 4 * T && nit > 0) {
        const int t = tid >> 2, which = tid & 3;
        const unsigned v = red[t][which];
        const int img = (which & 1) ? imgB : imgA;
        if (v) atomicAdd(&a.counters[(static_cast<int64_t>(img) * a.kcap + a.it0 + t) * 2 + (which >> 1)],
                         static_cast<unsigned long long>(v));
    }
}

}  // namespace phg
