// kernel_h2b2.cuh -- the beta = 2 denoise on both integer pipes.
//
// fused_h2b2_kernel<T, ALE>: T fused iterations of cardinality
// (denoise.hpp:139-160) + removal (denoise.hpp:176-223) for beta = 2 (5x5
// windows), Faithful borders and card_threshold <= 3 -- the C3 configuration.
// Other beta = 2 parameter sets run fused_tb_kernel<2, T>.
//
// Why: fused_tb_kernel<2> tests all 24 neighbours of every word in
// byte-SIMD and keeps the ALU pipe 92% busy with the FMA pipe at 16%
// (profiles/r01_c3_tb_full.txt).  Here every unordered neighbour pair is
// tested once and credited to both ends (12 directions instead of 24), and
// the directions are split between the pipes by their column offset in the
// interleaved two-tile layout of fused_h2_kernel ([row][col][A,B], a 32-bit
// word = 2 columns x 2 tiles):
//   - odd column offsets -- E (0,1), SE (1,1), SW (1,-1), (2,1), (2,-1) --
//     and S (1,0) in packed fp16 on the FMA pipe (h2sim, as kernel_h2.cuh);
//   - even column offsets -- (0,2), (1,2), (1,-2), (2,0), (2,2), (2,-2) --
//     are whole words apart, so they run in byte-SIMD (VABSDIFF4 + carry
//     trick, swar.cuh) on the ALU pipe with no shifts: 17 word tests per
//     8 pixels.
// The byte counts join the fp16 counts as half(1024 + n) (one PRMT), and the
// candidate test is the sign of 1024 + total - (1025 + m).
//
// Borders without masks: a pixel within 2 of the image edge (a "border"
// pixel) is never replaced with Faithful borders (flag <= in_bounds - 1 <=
// 19 < 25 - 3), so only its flagged bit (C < thr) matters.  The sweep
// therefore ignores the image edges entirely -- cells outside the image hold
// whatever was staged (TMA zero fill) and only corrupt the counts of border
// pixels -- and candidates are masked to interior pixels.  The flagged
// border pixels a tile owns are counted exactly by a scalar pass at the end
// of every iteration (the <= 4 border rows / columns of edge tiles).
//
// Candidates (interior, <= m similar neighbours, m = min(thr - 2, 1)) are
// flagged and replaced: flag >= 23 > 22.  They are compacted into the
// per-warp rings of fused_h2_kernel and replaced two per lane per round with
// the exact RMS over the 5x5 window (f in {23, 24}).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "kernel_h2.cuh"

namespace phg {

#ifndef PHG_B2_PUSH_UNROLL
#define PHG_B2_PUSH_UNROLL 1
#endif
constexpr int kB2PushUnroll = PHG_B2_PUSH_UNROLL;  // candidates per push-loop trip

constexpr int kB2Round = 64;  // candidates drained per round: two per lane
static_assert(kB2Round <= kH2Round, "the b2 rings reuse the h2 ring layout");

// 0x80 per byte where |a-b| < alpha (swar.cuh), the add on the FMA pipe
template <bool ALE>
__device__ __forceinline__ uint32_t b2sim(uint32_t a, uint32_t b, uint32_t k7, uint32_t one) {
    const uint32_t d = __vabsdiffu4(a, b);
    const uint32_t t = fma_add(d & kLo7, one, k7);
    return ~(ALE ? (d | t) : (d & t)) & kHi;
}

// One staged row as seen by a thread: words w = cols (x-2,x-1), (x,x+1),
// (x+2,x+3), (x+4,x+5) (bytes [A,B] per col) and the 8 half2 of cols x-2..x+5.
struct B2Row {
    uint32_t w[4];
    uint32_t h[8];
};

__device__ __forceinline__ void b2_load_row(uint32_t rowa, B2Row& r) {
    const uint2 raw = lds64a(rowa);
    r.w[0] = lds32a(rowa - 4);
    r.w[1] = raw.x;
    r.w[2] = raw.y;
    r.w[3] = lds32a(rowa + 8);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r.h[2 * i] = prmt(r.w[i], 0x64646464u, 0x5140);
        r.h[2 * i + 1] = prmt(r.w[i], 0x64646464u, 0x7362);
    }
}

// Carries of credits to later rows: fp16 per own column (c1: row y+1,
// c2: row y+2) and byte counts per own word (b1, b2).
struct B2Carry {
    uint32_t c1[4], c2[4];
    uint32_t b1[2], b2[2];
};

// Pairs of row A (= y) with itself and with rows B (y+1) and C (y+2).
// OWN: also return row y's counts -- cnt[j] (fp16, odd-offset and S pairs)
// and own[0..1] (byte counts, even-offset pairs, per own word).
template <bool ALE, bool OWN>
__device__ __forceinline__ void b2_pairs(const B2Row& A, const B2Row& B, const B2Row& C, uint32_t alpha2,
                                         uint32_t k7, uint32_t one, B2Carry& cr, uint32_t (&cnt)[4],
                                         uint32_t (&own)[2]) {
    // ---- fp16: h index i = column x-2+i, own column j at i = j+2
    uint32_t e[5], s[4], d[5], aa[5], q1[5], q2[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (OWN) e[i] = h2sim(A.h[i + 1], A.h[i + 2], alpha2);    // (y,x-1+i)-(y,x+i)
        d[i] = h2sim(A.h[i + 1], B.h[i + 2], alpha2);             // (y,x-1+i)-(y+1,x+i)
        aa[i] = h2sim(A.h[i + 2], B.h[i + 1], alpha2);            // (y,x+i)-(y+1,x-1+i)
        q1[i] = h2sim(A.h[i + 1], C.h[i + 2], alpha2);            // (y,x-1+i)-(y+2,x+i)
        q2[i] = h2sim(A.h[i + 2], C.h[i + 1], alpha2);            // (y,x+i)-(y+2,x-1+i)
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = h2sim(A.h[j + 2], B.h[j + 2], alpha2);  // (y,x+j)-(y+1,x+j)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (OWN)
            cnt[j] = h2add(h2add(h2add(e[j], e[j + 1]), h2add(s[j], d[j + 1])),
                           h2add(h2add(aa[j], q1[j + 1]), h2add(q2[j], cr.c1[j])));
        cr.c1[j] = h2add(h2add(s[j], d[j]), h2add(aa[j + 1], cr.c2[j]));
        cr.c2[j] = h2add(q1[j], q2[j + 1]);
    }
    // ---- byte-SIMD: words k = 0..3 (WL, P0, P1, WR), own words 1 and 2
    uint32_t o0 = cr.b1[0], o1 = cr.b1[1];
    uint32_t n1a = cr.b2[0], n1b = cr.b2[1];  // credits to row y+1
    uint32_t n2a = 0, n2b = 0;                // credits to row y+2
    if (OWN) {  // (0,2) in row y
        const uint32_t ma = b2sim<ALE>(A.w[0], A.w[1], k7, one);
        const uint32_t mb = b2sim<ALE>(A.w[1], A.w[2], k7, one);
        const uint32_t mc = b2sim<ALE>(A.w[2], A.w[3], k7, one);
        o0 += (ma >> 7) + (mb >> 7);
        o1 += (mb >> 7) + (mc >> 7);
    }
    {  // (1,2): (A.w[k], B.w[k+1])
        const uint32_t m0 = b2sim<ALE>(A.w[0], B.w[1], k7, one);
        const uint32_t m1 = b2sim<ALE>(A.w[1], B.w[2], k7, one);
        const uint32_t m2 = b2sim<ALE>(A.w[2], B.w[3], k7, one);
        n1a += m0 >> 7;
        n1b += m1 >> 7;
        o0 += m1 >> 7;
        o1 += m2 >> 7;
    }
    {  // (1,-2): (A.w[k+1], B.w[k])
        const uint32_t m0 = b2sim<ALE>(A.w[1], B.w[0], k7, one);
        const uint32_t m1 = b2sim<ALE>(A.w[2], B.w[1], k7, one);
        const uint32_t m2 = b2sim<ALE>(A.w[3], B.w[2], k7, one);
        o0 += m0 >> 7;
        o1 += m1 >> 7;
        n1a += m1 >> 7;
        n1b += m2 >> 7;
    }
    {  // (2,0)
        const uint32_t m0 = b2sim<ALE>(A.w[1], C.w[1], k7, one);
        const uint32_t m1 = b2sim<ALE>(A.w[2], C.w[2], k7, one);
        o0 += m0 >> 7;
        o1 += m1 >> 7;
        n2a += m0 >> 7;
        n2b += m1 >> 7;
    }
    {  // (2,2): (A.w[k], C.w[k+1])
        const uint32_t m0 = b2sim<ALE>(A.w[0], C.w[1], k7, one);
        const uint32_t m1 = b2sim<ALE>(A.w[1], C.w[2], k7, one);
        const uint32_t m2 = b2sim<ALE>(A.w[2], C.w[3], k7, one);
        n2a += m0 >> 7;
        n2b += m1 >> 7;
        o0 += m1 >> 7;
        o1 += m2 >> 7;
    }
    {  // (2,-2): (A.w[k+1], C.w[k])
        const uint32_t m0 = b2sim<ALE>(A.w[1], C.w[0], k7, one);
        const uint32_t m1 = b2sim<ALE>(A.w[2], C.w[1], k7, one);
        const uint32_t m2 = b2sim<ALE>(A.w[3], C.w[2], k7, one);
        o0 += m0 >> 7;
        o1 += m1 >> 7;
        n2a += m1 >> 7;
        n2b += m2 >> 7;
    }
    own[0] = o0;
    own[1] = o1;
    cr.b1[0] = n1a;
    cr.b1[1] = n1b;
    cr.b2[0] = n2a;
    cr.b2[1] = n2b;
}

// The 5 bytes of one tile at columns c-2..c+2 of a staged row: `p` is the
// shared address of the word holding byte (o - 4) & ~3, sh = o & 3.
// Returns bytes (c-2, c-1, c+1, c+2) packed and the centre byte.
__device__ __forceinline__ void b2_gather_row(uint32_t p, uint32_t sh8, uint32_t& quad, uint32_t& mid) {
    const uint32_t w0 = lds32a(p), w1 = lds32a(p + 4), w2 = lds32a(p + 8);
    const uint32_t x = __funnelshift_r(w0, w1, sh8);  // bytes sh .. sh+3 -> cols c-2, (B), c-1, (B)
    const uint32_t y = __funnelshift_r(w1, w2, sh8);  // cols c, (B), c+1, (B)
    const uint32_t z = w2 >> sh8;                     // col c+2 in byte 0
    quad = prmt(prmt(x, y, 0x6420), z, 0x4310);       // c-2, c-1, c+1, c+2
    mid = y & 0xffu;
}

// One interior candidate: RMS of the dissimilar cells of its 5x5 window
// (removal_rows, denoise.hpp:199-217, f in {23, 24}); `o` = byte offset of
// the pixel in the interleaved tile.  Returns the new value.
template <bool ALE>
__device__ __forceinline__ uint32_t h2b2_replace(uint32_t src, int o, uint32_t k7, uint32_t one) {
    const int o0 = o - 2 * kH2RP - 4;
    const uint32_t b4 = static_cast<uint32_t>(o0 & ~3);
    const uint32_t sh8 = static_cast<uint32_t>(o0 & 3) * 8u;
    uint32_t q[5], m[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) b2_gather_row(src + b4 + r * kH2RP, sh8, q[r], m[r]);
    // 24 neighbours: the 4 side cells of every row + the 4 non-centre middles
    const uint32_t mids = m[0] | (m[1] << 8) | (m[3] << 16) | (m[4] << 24);
    const uint32_t p4 = m[2] * 0x01010101u;
    uint32_t f = 0, S = 0;
    const uint32_t nb[6] = {q[0], q[1], q[2], q[3], q[4], mids};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const uint32_t d = __vabsdiffu4(nb[i], p4);
        const uint32_t t = fma_add(d & kLo7, one, k7);
        const uint32_t dis = (ALE ? (d | t) : (d & t)) & kHi;
        f += __popc(dis);
        S = __dp4a(nb[i] & msb_to_bytes(dis), nb[i], S);
    }
    return h2_rms(S, f, rms_rcp<23>(f));  // f in {23, 24}
}

template <int T, bool ALE>
__global__ void __launch_bounds__(kH2Threads, 2)
    fused_h2b2_kernel(const __grid_constant__ CUtensorMap src_map, const H2Args a) {
    static_assert(T >= 1 && 2 * T <= 8, "halo exceeds the staged columns");
    constexpr int HALO = 2 * T;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][4];  // flagged A, flagged B, replaced A, replaced B

    const int sh = a.th + 2 * HALO;
    const int bufb = h2_buf_bytes(sh);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const uint32_t ring = smem_u32(smem + 2 * bufb) + warp * kH2Ring * 2;
    const uint32_t one = a.alpha2 != 0u ? 1u : 0u;  // opaque 1 (alpha2 is never 0)

    // ---- the two tiles (as fused_h2_kernel)
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
    if (tid < 4 * T) (&red[0][0])[tid] = 0;

    const int c = tid % kH2Cols;
    const int g = tid / kH2Cols;
    const int x = 8 + 4 * c;
    const int W = a.width, H = a.height;
    // interior (>= 2 from every image edge) and owned column slots, in the
    // candidate-word layout of fused_h2_kernel
    uint32_t colown = 0, colint = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int rc = x + j;
        const int gA = x0A + rc, gB = x0B + rc;
        const bool iA = gA >= 0 && gA < W, iB = hasB && gB >= 0 && gB < W;
        const bool nA = gA >= 2 && gA < W - 2, nB = hasB && gB >= 2 && gB < W - 2;
        const bool own_x = rc >= kLeftPx && rc < kLeftPx + kOutPx;
        const int bA = 8 * (2 * (j & 1)) + 4 * (j >> 1), bB = bA + 8;
        colown |= ((own_x && iA) ? 1u : 0u) << bA | ((own_x && iB) ? 1u : 0u) << bB;
        colint |= (nA ? 1u : 0u) << bA | (nB ? 1u : 0u) << bB;
    }
    // candidate <=> 1024 + total - (1025 + m) < 0
    const uint32_t ckh = f2h(1025.0f + static_cast<float>(a.m));
    const uint32_t ck2 = ckh | (ckh << 16);

    __syncthreads();
    mbar_wait(&bar, 0);
    {  // interleave the two staged tiles into buffer 0 (as fused_h2_kernel)
        const uint8_t* sA = smem + bufb;
        const uint8_t* sB = smem + bufb + h2_stage_b(sh);
        for (int i = tid; i < sh * kChunks; i += kH2Threads) {
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

    // rows whose pixels are interior for both tiles: no row mask
    const int f_lo = max(2 - gyA, hasB ? 2 - gyB : -1000000);
    const int f_hi = min(H - 2 - gyA, hasB ? H - 2 - gyB : 1000000);  // exclusive
    const int g_lo = g == 0 ? 2 : sh / 2;
    const int g_hi = g == 0 ? sh / 2 : sh - 2;

    for (int t = 0; t < T; ++t) {
        const uint32_t src = smem_u32(smem) + ((t & 1) ? bufb : 0);
        const uint32_t dst = smem_u32(smem) + ((t & 1) ? 0 : bufb);
        const int ylo = max(g_lo, 2 * (t + 1));
        const int yhi = min(g_hi, sh - 2 * (t + 1));
        uint32_t fl_n = 0;
        unsigned flA = 0, flB = 0;
        auto flush = [&]() {
            const uint32_t f = (fl_n & 0x0f0f0f0fu) + ((fl_n >> 4) & 0x0f0f0f0fu);
            flA += __dp4a(f, 0x00010001u, 0u);
            flB += __dp4a(f, 0x01000100u, 0u);
            fl_n = 0;
        };
        int pending = 0;
        auto drain = [&](int h, int n) {
            const int o0 = static_cast<int>(lds16(ring + 2 * (h + (lane < n ? lane : 0))));
            const int o1 = static_cast<int>(lds16(ring + 2 * (h + (lane + 32 < n ? lane + 32 : 0))));
            const uint32_t v0 = h2b2_replace<ALE>(src, o0, a.k7, one);
            const uint32_t v1 = h2b2_replace<ALE>(src, o1, a.k7, one);
            if (lane < n) sts8a(dst + o0, v0);
            if (lane + 32 < n) sts8a(dst + o1, v1);
        };
        if (ylo < yhi) {
            const uint32_t colp = src + 16 + 8 * c;
            B2Row A, B, C;
            B2Carry cr;
#pragma unroll
            for (int j = 0; j < 4; ++j) cr.c1[j] = cr.c2[j] = 0u;
            cr.b1[0] = cr.b1[1] = cr.b2[0] = cr.b2[1] = 0u;
            {  // prologue: carries into row ylo from rows ylo-2, ylo-1
                B2Row P0r, P1r;
                uint32_t cnt_[4], own_[2];
                b2_load_row(colp + (ylo - 2) * kH2RP, P0r);
                b2_load_row(colp + (ylo - 1) * kH2RP, P1r);
                b2_load_row(colp + ylo * kH2RP, A);
                b2_pairs<ALE, false>(P0r, P1r, A, a.alpha2, a.k7, one, cr, cnt_, own_);
                b2_load_row(colp + (ylo + 1) * kH2RP, B);
                b2_pairs<ALE, false>(P1r, A, B, a.alpha2, a.k7, one, cr, cnt_, own_);
            }
            uint32_t ownm = 0;
            int next_own = ylo;
            uint32_t R = 0;
            auto push = [&](int y0) {
                if (y0 & 4) flush();
                const int n = __popc(R);
                int incl = n;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const int vv = __shfl_up_sync(0xffffffffu, incl, dd);
                    if (lane >= dd) incl += vv;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (total) {
                    uint32_t addr = ring + 2 * (pending + incl - n);
                    const uint32_t base3 = static_cast<uint32_t>((y0 + 3) * kH2RP + 16 + 8 * c);
                    uint32_t mm = R;
                    // kB2PushUnroll items per loop trip (as in fused_h2_kernel's push)
                    while (mm) {
#pragma unroll
                        for (int u = 0; u < kB2PushUnroll; ++u) {
                            uint32_t b, m1;
                            asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(mm));
                            asm("shl.b32 %0, 1, %1;" : "=r"(m1) : "r"(b));
                            if (u == 0 || mm) sts16(addr + 2 * u, base3 - (b & 3u) * kH2RP + (b >> 3) + (b & 4u));
                            mm ^= m1;
                        }
                        addr += 2 * kB2PushUnroll;
                    }
                    pending += total;
                    if (pending >= kB2Round) {
                        __syncwarp();  // other lanes' ring items are read only by a drain
                        int h = 0;
                        for (; pending - h >= kB2Round; h += kB2Round) drain(h, kB2Round);
                        pending -= h;
                        __syncwarp();
                        if (pending) {  // move the leftovers (< kB2Round) to the front
                            const uint32_t l0 = lane < pending ? lds16(ring + 2 * (h + lane)) : 0;
                            const uint32_t l1 = lane + 32 < pending ? lds16(ring + 2 * (h + lane + 32)) : 0;
                            __syncwarp();
                            if (lane < pending) sts16(ring + 2 * lane, l0);
                            if (lane + 32 < pending) sts16(ring + 2 * (lane + 32), l1);
                        }
                        __syncwarp();
                    }
                }
                R = 0;
            };
            auto row = [&](int y, auto fast_tag) {
                constexpr bool FAST = decltype(fast_tag)::value;
                b2_load_row(colp + (y + 2) * kH2RP, C);
                uint32_t cnt[4], own[2];
                b2_pairs<ALE, true>(A, B, C, a.alpha2, a.k7, one, cr, cnt, own);
                // the centre row goes to the destination unchanged
                sts64a(dst + y * kH2RP + 16 + 8 * c, make_uint2(A.w[1], A.w[2]));
                uint32_t intm = colint;
                if (y == next_own) {
                    const uint32_t oa = (y >= HALO && y < HALO + outA) ? 0x00ff00ffu : 0u;
                    const uint32_t ob = (y >= HALO && y < HALO + outB) ? 0xff00ff00u : 0u;
                    ownm = colown & (oa | ob);
                    int nx = 1 << 30;
                    if (HALO > y) nx = min(nx, HALO);
                    if (HALO + outA > y) nx = min(nx, HALO + outA);
                    if (HALO + outB > y) nx = min(nx, HALO + outB);
                    next_own = nx;
                }
                if (!FAST) {
                    const int ra = gyA + y, rb = gyB + y;
                    const bool iA = ra >= 2 && ra < H - 2, iB = hasB && rb >= 2 && rb < H - 2;
                    intm &= (iA ? 0x00ff00ffu : 0u) | (iB ? 0xff00ff00u : 0u);
                }
                uint32_t vn[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t hb = prmt(own[j >> 1], 0x64646464u, (j & 1) ? 0x7362 : 0x5140);
                    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(vn[j]) : "r"(h2add(cnt[j], hb)), "r"(ck2));
                }
                const uint32_t s01 = prmt(vn[0], vn[1], 0xFDB9u);
                const uint32_t s23 = prmt(vn[2], vn[3], 0xFDB9u);
                const uint32_t Mi = ((s01 & 0x01010101u) | (s23 & 0x10101010u)) & intm;
                fl_n += Mi & ownm;
                R = (R << 1) | Mi;
                if ((y & 3) == 3) push(y - 3);
                A = B;
                B = C;
            };
            const int s0 = min(max(ylo, f_lo), yhi);
            const int s1 = max(min(yhi, f_hi), s0);
            for (int y = ylo; y < s0; ++y) row(y, std::false_type{});
#pragma unroll 3  // the A <- B <- C rotation becomes register renaming
            for (int y = s0; y < s1; ++y) row(y, std::true_type{});
            for (int y = s1; y < yhi; ++y) row(y, std::false_type{});
            if (yhi & 3) {
                R <<= 4 - (yhi & 3);
                push(yhi & ~3);
            }
        }
        if (pending > 0) drain(0, pending);
        flush();
        // interior candidates: flagged == replaced
        const unsigned rpA = flA, rpB = flB;
        // owned border pixels (within 2 of an image edge): flagged iff C < thr,
        // C over the in-bounds 5x5 window (denoise.hpp:145-160, 192-193)
        for (int tile = 0; tile < (hasB ? 2 : 1); ++tile) {
            const int gy0 = tile ? gyB : gyA, x0 = tile ? x0B : x0A, outr = tile ? outB : outA;
            const int cl = max(kLeftPx, -x0), ch = min(kLeftPx + kOutPx, W - x0);  // owned region cols
            const int rl = HALO, rh = HALO + outr;                                  // owned rows
            if (ch <= cl || rh <= rl) continue;
            // border rows: global rows < 2 or >= H-2; border cols likewise
            const int br_lo = min(max(rl, 2 - gy0), rh), br_hi = max(min(rh, H - 2 - gy0), br_lo);
            const int bc_lo = min(max(cl, 2 - x0), ch), bc_hi = max(min(ch, W - 2 - x0), bc_lo);
            const int ncol = ch - cl;
            const int top = br_lo - rl, bot = rh - br_hi;          // border rows above / below
            const int left = bc_lo - cl, right = ch - bc_hi;       // border cols left / right
            const int mid_rows = br_hi - br_lo;
            const int n_rows_items = (top + bot) * ncol;
            const int n_items = n_rows_items + mid_rows * (left + right);
            unsigned nf = 0;
            for (int i = tid; i < n_items; i += kH2Threads) {
                int yy, rc;
                if (i < n_rows_items) {
                    const int r = i / ncol;
                    rc = cl + (i - r * ncol);
                    yy = r < top ? rl + r : br_hi + (r - top);
                } else {
                    const int k = i - n_rows_items, nlr = left + right;
                    const int r = k / nlr, q = k - r * nlr;
                    yy = br_lo + r;
                    rc = q < left ? cl + q : bc_hi + (q - left);
                }
                const int gy = gy0 + yy, gx = x0 + rc;
                const uint8_t* base = smem + ((t & 1) ? bufb : 0) + tile;
                const int p = base[yy * kH2RP + 2 * rc];
                int C = 0;
                for (int dy = -2; dy <= 2; ++dy) {
                    if (gy + dy < 0 || gy + dy >= H) continue;
                    for (int dx = -2; dx <= 2; ++dx) {
                        if (gx + dx < 0 || gx + dx >= W) continue;
                        const int qv = base[(yy + dy) * kH2RP + 2 * (rc + dx)];
                        C += abs(qv - p) < static_cast<int>(a.alpha) ? 1 : 0;
                    }
                }
                nf += C < a.thr ? 1u : 0u;
            }
            nf = __reduce_add_sync(0xffffffffu, nf);
            if (lane == 0 && nf) atomicAdd(&red[t][tile], nf);
        }
        flA = __reduce_add_sync(0xffffffffu, flA);
        flB = __reduce_add_sync(0xffffffffu, flB);
        const unsigned rA = __reduce_add_sync(0xffffffffu, rpA);
        const unsigned rB = __reduce_add_sync(0xffffffffu, rpB);
        if (lane == 0) {
            if (flA) atomicAdd(&red[t][0], flA);
            if (flB) atomicAdd(&red[t][1], flB);
            if (rA) atomicAdd(&red[t][2], rA);
            if (rB) atomicAdd(&red[t][3], rB);
        }
        __syncthreads();
    }

    // ---- owned output rows: de-interleave, 16-byte coalesced stores
    {
        const uint8_t* fin = smem + ((T & 1) ? bufb : 0);
        constexpr int kOutChunks = kOutPx / 16;
        uint8_t* gA = a.dst + imgA * a.image_stride + static_cast<int64_t>(y0A) * a.pitch + (x0A + kLeftPx);
        uint8_t* gB = a.dst + imgB * a.image_stride + static_cast<int64_t>(y0B) * a.pitch + (x0B + kLeftPx);
        const int rows = max(outA, outB);
        for (int i = tid; i < rows * kOutChunks; i += kH2Threads) {
            const int r = i / kOutChunks, ch = i - r * kOutChunks;
            const int y = HALO + r;
            const uint4* s = reinterpret_cast<const uint4*>(fin + y * kH2RP + 2 * kLeftPx + 32 * ch);
            const uint4 u0 = s[0], u1 = s[1];
            if (r < outA && x0A + kLeftPx + 16 * ch < a.width) {
                uint4 o;
                o.x = prmt(u0.x, u0.y, 0x6420); o.y = prmt(u0.z, u0.w, 0x6420);
                o.z = prmt(u1.x, u1.y, 0x6420); o.w = prmt(u1.z, u1.w, 0x6420);
                *reinterpret_cast<uint4*>(gA + static_cast<int64_t>(y) * a.pitch + 16 * ch) = o;
                mirror_row16(a.peers, a.row_base + y0A + y, a.pitch, x0A + kLeftPx + 16 * ch, o);
            }
            if (r < outB && x0B + kLeftPx + 16 * ch < a.width) {
                uint4 o;
                o.x = prmt(u0.x, u0.y, 0x7531); o.y = prmt(u0.z, u0.w, 0x7531);
                o.z = prmt(u1.x, u1.y, 0x7531); o.w = prmt(u1.z, u1.w, 0x7531);
                *reinterpret_cast<uint4*>(gB + static_cast<int64_t>(y) * a.pitch + 16 * ch) = o;
                mirror_row16(a.peers, a.row_base + y0B + y, a.pitch, x0B + kLeftPx + 16 * ch, o);
            }
        }
    }
    if (tid < 4 * T) {
        const int t = tid >> 2, which = tid & 3;
        const unsigned v = red[t][which];
        const int img = (which & 1) ? imgB : imgA;
        if (v) atomicAdd(&a.counters[((int64_t)img * a.kcap + a.it0 + t) * 2 + (which >> 1)], (unsigned long long)v);
    }
}

}  // namespace phg
