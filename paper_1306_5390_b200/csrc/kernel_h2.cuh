// kernel_h2.cuh -- the beta=1 hot path on the FMA pipe: two tiles per CTA in
// the two fp16 lanes of every register.
//
// fused_h2_kernel<T, ALE>: T fused iterations of cardinality
// (denoise.hpp:139-160) + removal (denoise.hpp:176-223) for beta = 1,
// Faithful borders and card_threshold <= 3 (the reference defaults,
// denoise.hpp:34-39).  Other parameter sets run fused_tb_kernel.
//
// Why: the byte-SIMD sweep of fused_tb_kernel keeps the ALU pipe ~80% busy
// while the FMA pipe idles.  Here the similarity count runs in packed fp16:
//   a pixel v is the half 1024+v (bit pattern 0x64vv, exact, spacing 1),
//   similar(a,b) = sat(alpha - |a-b|)  -> one HADD2 + one HADD2.SAT (the
//   |.| folds into the operand), 1.0 or 0.0 per lane,
// and the counts are HADD2 sums.  Each unordered neighbour pair is tested
// once and credited to both ends (E, S, SE, SW pairs; 4 tests per pixel
// instead of 8).  The ALU pipe only converts bytes to halves (one PRMT per
// pair of pixels) and extracts candidate bits, so it is free for the RMS
// replacement of the ~13% candidate pixels (byte-SIMD, as before).  In rows
// whose window is inside the image the vertical (S) pairs, which are whole
// interleaved words apart, run in byte-SIMD on the ALU pipe instead, to
// balance the two pipes.
//
// Two tiles per CTA: lane 0 of every half2 holds tile A, lane 1 tile B (the
// next tile in the (image, row tile, column tile) order), so each lane is an
// independent 496-px-wide tile and nothing couples the halves.  The shared
// buffers interleave the two tiles byte by byte, [row][col][A,B], so one
// 32-bit load + one PRMT yields two half2 values.
//
// Cells outside the image: the byte is ignored and the exponent byte becomes
// 0x74 instead of 0x64 (value 16384+16v), so such a cell is never similar to
// an image pixel -- exactly the reference's "out-of-bounds cells are not in
// the window" (denoise.hpp:145-149).  Candidate bits are masked to pixels
// whose whole window is inside the image: with Faithful borders a border
// pixel is never replaced (flag <= in_bounds-1 < 9-2), so every candidate is
// an interior pixel with flag = 8 - #similar neighbours in {7, 8}, and its
// replacement needs no bounds logic.  Border pixels still count as flagged
// when C < thr (denoise.hpp:192-193); that count is accumulated in fp16.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "kernels.cuh"

namespace phg {

constexpr int kH2Threads = 256;           // 2 row groups x 128 column threads
constexpr int kH2Cols = 128;              // 4 columns (x 2 tiles) per thread: region cols [8, 520)
constexpr int kH2RP = 2 * kRP;            // 1056 interleaved bytes per staged row
constexpr int kH2MaxRows = 62;            // ring items are u16 byte offsets: sh * 1056 < 65536

// one interleaved buffer; buffer 1 first serves as the TMA staging area of
// the two [sh][528] tiles (B at a 128-byte aligned offset)
__host__ __device__ constexpr int h2_stage_b(int sh) { return (kRP * sh + 127) / 128 * 128; }
__host__ __device__ constexpr int h2_buf_bytes(int sh) { return (kH2RP * sh + 128 + 127) / 128 * 128; }
#ifndef PHG_PUSH_UNROLL
#define PHG_PUSH_UNROLL 3
#endif
constexpr int kH2PushUnroll = PHG_PUSH_UNROLL;  // candidates per push-loop trip
constexpr int kH2Round = 96;           // drained per round: three candidates per lane
constexpr int kH2Ring = kH2Round + 32 * 32;  // per-warp u16 items: leftovers + one row quad
__host__ __device__ constexpr int h2_smem_bytes(int sh) {
    return 2 * h2_buf_bytes(sh) + (kH2Threads / 32) * kH2Ring * 2;
}

struct H2Args {
    uint8_t* dst;
    int64_t pitch;
    int64_t image_stride;
    int width;
    int height;      // global image height
    int row_base;    // global row of buffer row 0
    int own_lo;      // first owned global row
    int own_hi;      // one past the last owned global row
    int th;          // output rows per tile
    int tiles_x;
    int tiles_y;
    int n_tiles;     // n_images * tiles_y * tiles_x
    uint32_t alpha2; // half2(alpha, alpha)
    uint32_t k7;     // ((256-alpha) & 0x7f) in every byte (candidate pass)
    int m;           // candidate <=> #similar neighbours <= m  (m = min(thr-2, 1))
    int thr;
    int alpha;       // integer alpha (border pass of fused_h2b2_kernel)
    int it0;
    int kcap;
    unsigned long long* counters;  // [n_images][kcap][2]
    HaloPeers peers;               // single-image bands only (kernels.cuh)
};

// ------------------------------------------------------------ fp16 helpers
__device__ __forceinline__ uint32_t h2sim(uint32_t a, uint32_t b, uint32_t alpha2) {
    uint32_t d, s;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    asm("{.reg .b32 t; abs.f16x2 t, %1; sub.sat.f16x2 %0, %2, t;}" : "=r"(s) : "r"(d), "r"(alpha2));
    return s;
}
__device__ __forceinline__ uint32_t h2add(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t h2sat_sub(uint32_t a, uint32_t b) {  // sat(a - b)
    uint32_t r;
    asm("sub.sat.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t h2fma(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
// bytes s .. s+3 of the 8-byte {b:a} with s = sel & 3 (PRMT's forward 4-extract
// mode: a byte funnel shift whose selector is the byte address itself)
__device__ __forceinline__ uint32_t prmt_f4e(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32.f4e %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t f2h(float f) {
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f)));
}
__device__ __forceinline__ uint32_t h2pack(float lo, float hi) { return f2h(lo) | (f2h(hi) << 16); }

// Shared-memory accesses by 32-bit shared address (no generic-address
// arithmetic in the row loop).  The "memory" clobber keeps them ordered with
// the barriers and the stores.
__device__ __forceinline__ uint32_t lds32a(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint2 lds64a(uint32_t a) {
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64a(uint32_t a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts8a(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// The per-thread view of one staged row: 6 half2 = columns x-1 .. x+4, lane 0
// tile A, lane 1 tile B.  kc[] holds the exponent bytes per column.
__device__ __forceinline__ void h2_load_row(uint32_t rowa, const uint32_t (&kc)[4], uint32_t row_oob,
                                            uint32_t (&v)[6], uint2& raw) {
    raw = lds64a(rowa);
    const uint32_t wl = lds32a(rowa - 4), wr = lds32a(rowa + 8);
    v[0] = prmt(wl, kc[0] | row_oob, 0x7362);
    v[1] = prmt(raw.x, kc[1] | row_oob, 0x5140);
    v[2] = prmt(raw.x, kc[1] | row_oob, 0x7362);
    v[3] = prmt(raw.y, kc[2] | row_oob, 0x5140);
    v[4] = prmt(raw.y, kc[2] | row_oob, 0x7362);
    v[5] = prmt(wr, kc[3] | row_oob, 0x5140);
}

// Credits to row y+1 from the pairs (row y, row y+1): up[j] for column j.
__device__ __forceinline__ void h2_pairs_down(const uint32_t (&v)[6], const uint32_t (&nv)[6], uint32_t alpha2,
                                              uint32_t (&s)[4], uint32_t (&d)[5], uint32_t (&a)[5]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = h2sim(v[j + 1], nv[j + 1], alpha2);   // (y,j)-(y+1,j)
#pragma unroll
    for (int i = 0; i < 5; ++i) d[i] = h2sim(v[i], nv[i + 1], alpha2);       // (y,i-1)-(y+1,i)
#pragma unroll
    for (int i = 0; i < 5; ++i) a[i] = h2sim(v[i + 1], nv[i], alpha2);       // (y,i)-(y+1,i-1)
}

// round(sqrt(S/f)) half away from zero (denoise.hpp:163-169), branch-free,
// for S < 2^23 and f in {7, 8} (beta = 1) or {23, 24} (beta = 2), rcp_f =
// fp32(1/f).  r ~ sqrt(S/f): one rounding in rcp_f, one in the product and
// MUFU.SQRT's own error, together a relative error below 2^-21.  Scaling r by
// 1 - 2^-20 inside the rounding FFMA puts it strictly below the exact root x
// (x > 0) and by less than 273 * 2^-19 < 1/2, so n = nearest(r (1 - 2^-20)) is
// the exact u = floor(x + 1/2) or u - 1 (and n >= 0), and u = n + [4S >= f
// (2n+1)^2] (an exact integer test, on the FMA pipe but for one compare).
// The FFMA's result is 0x4b400000 + n; the constant is carried through to
// the end (its low byte is 0).  Exhaustively checked on the GPU for every S
// up to 24 * 65025 (tests/test_parity_gpu.py, phg_debug_rms).
__device__ __forceinline__ uint32_t h2_rms(uint32_t S, uint32_t f, float rcp_f) {
    const float s = __int_as_float(0x4b000000 | S) - 8388608.0f;  // exact
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s * rcp_f));
    const uint32_t nb = __float_as_uint(fmaf(r, 0.99999904632568359375f, 12582912.0f));  // 0x4b400000 + n
    const uint32_t q = 2u * nb + (1u - 2u * 0x4b400000u);                                // 2n + 1
    return nb - 0x4b400000u + (q * (q * f) <= 4u * S ? 1u : 0u);
}

// fp32(1/f) for the two values f takes in a replacement, as one IMAD on the
// FMA pipe: f in {F0, F0 + 1} = {7, 8} (beta = 1) or {23, 24} (beta = 2)
template <int F0>
__device__ __forceinline__ float rms_rcp(uint32_t f) {
    static_assert(F0 == 7 || F0 == 23, "beta = 1 or 2");
    constexpr uint32_t b0 = F0 == 7 ? 0x3e124925u : 0x3d321643u;  // fp32(1/F0)
    constexpr uint32_t b1 = F0 == 7 ? 0x3e000000u : 0x3d2aaaabu;  // fp32(1/(F0 + 1))
    return __uint_as_float(b0 + static_cast<uint32_t>(F0) * (b0 - b1) - f * (b0 - b1));
}

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(static_cast<unsigned short>(v)) : "memory");
}
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
    return v;
}

// One candidate pixel (interior, Faithful, beta=1): RMS of the dissimilar
// cells of its 3x3 window, exactly as removal_rows (denoise.hpp:199-217).
// `o1` = byte offset of the window's top-left cell (the pixel's offset minus
// kH2RP + 2) in the interleaved tile; returns the new value (no store, so
// that several candidates' loads can be interleaved).
template <bool ALE>
__device__ __forceinline__ uint32_t h2_replace(uint32_t src, int o1, uint32_t k7) {
    const int b4 = o1 & ~3;
    const uint32_t sh = static_cast<uint32_t>(o1 & 3);
    const uint32_t sel = 0x0420u + sh * 0x0111u;  // bytes sh, sh+2, sh+4
    uint32_t R[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const uint32_t p = src + b4 + r * kH2RP;
        R[r] = prmt(lds32a(p), lds32a(p + 4), sel);
    }
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

template <int T, bool ALE>
__global__ void __launch_bounds__(kH2Threads, 2)
    fused_h2_kernel(const __grid_constant__ CUtensorMap src_map, const H2Args a) {
    static_assert(T >= 1 && T <= 8, "halo exceeds the staged columns");
    constexpr int HALO = T;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][4];  // flagged A, flagged B, replaced A, replaced B

    const int sh = a.th + 2 * HALO;
    const int bufb = h2_buf_bytes(sh);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const uint32_t ring = smem_u32(smem + 2 * bufb) + warp * kH2Ring * 2;  // shared address

    // ---- the two tiles
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
    const int gyA = a.row_base + y0A, gyB = a.row_base + y0B;  // global row of region row 0

    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(kRP * sh * (hasB ? 2 : 1)));
        tma_load_4d(smem + bufb, &src_map, 0, x0A / kChunk, y0A, imgA, &bar);
        if (hasB) tma_load_4d(smem + bufb + h2_stage_b(sh), &src_map, 0, x0B / kChunk, y0B, imgB, &bar);
    }
    if (tid < 4 * T) (&red[0][0])[tid] = 0;

    // ---- per-thread column constants (4 columns x 2 tiles = 8 slots)
    const int c = tid % kH2Cols;
    const int g = tid / kH2Cols;
    const int x = 8 + 4 * c;  // region column of this thread's column 0
    auto in_col = [&](int x0, bool has, int rc) {
        const int gx = x0 + rc;
        return has && gx >= 0 && gx < a.width;
    };
    auto int_col = [&](int x0, bool has, int rc) {
        const int gx = x0 + rc;
        return has && gx >= 1 && gx < a.width - 1;
    };
    uint32_t kc[4];  // exponent bytes (0x64 image, 0x74 outside) for columns x-2 .. x+5
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rc = x - 2 + 2 * i;
        kc[i] = (in_col(x0A, true, rc) ? 0x64u : 0x74u) | (in_col(x0B, hasB, rc) ? 0x64u : 0x74u) << 8 |
                (in_col(x0A, true, rc + 1) ? 0x64u : 0x74u) << 16 | (in_col(x0B, hasB, rc + 1) ? 0x64u : 0x74u) << 24;
    }
    // Candidate <=> cnt - ck < 0 (cnt = similar neighbours, centre excluded):
    //   interior pixel: ck = m + 1/2      (replace; flagged == replaced for thr <= 3)
    //   border pixel:   ck = thr - 3/2    (flagged only: C < thr, denoise.hpp:192)
    //   outside image:  ck = -64
    const float ck_int = static_cast<float>(a.m) + 0.5f, ck_bor = static_cast<float>(a.thr) - 1.5f;
    uint32_t ck[4];   // interior rows
    uint32_t ckb[4];  // border rows (every in-image column is a border pixel)
    // slot bits, layout of the per-row candidate word M: column j, tile t at
    // bit 8*(2*(j&1)+t) + 4*(j>>1)  (byte offset in the interleaved row = bit/8 + (bit&4))
    uint32_t colown = 0, colint = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int rc = x + j;
        const bool iA = in_col(x0A, true, rc), iB = in_col(x0B, hasB, rc);
        const bool nA = int_col(x0A, true, rc), nB = int_col(x0B, hasB, rc);
        const bool own_x = rc >= kLeftPx && rc < kLeftPx + kOutPx;
        ck[j] = h2pack(nA ? ck_int : (iA ? ck_bor : -64.0f), nB ? ck_int : (iB ? ck_bor : -64.0f));
        ckb[j] = h2pack(iA ? ck_bor : -64.0f, iB ? ck_bor : -64.0f);
        const int bA = 8 * (2 * (j & 1)) + 4 * (j >> 1), bB = bA + 8;
        colown |= ((own_x && iA) ? 1u : 0u) << bA | ((own_x && iB) ? 1u : 0u) << bB;
        colint |= (nA ? 1u : 0u) << bA | (nB ? 1u : 0u) << bB;
    }
    const uint32_t neg64 = 0xd400d400u;  // half2(-64, -64)
    uint32_t ckF[4];  // fast rows: counts carry -18 (two -9 credits)
#pragma unroll
    for (int j = 0; j < 4; ++j) ckF[j] = h2add(ck[j], 0xcc80cc80u);  // half2(-18)

    __syncthreads();  // barrier init + counters visible
    mbar_wait(&bar, 0);
    // ---- interleave the two staged tiles (buffer 1) into buffer 0: [row][col][A,B]
    {
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

    // rows whose whole window is in the image for both tiles: fast path
    const int H = a.height;
    const int f_lo = max(1 - gyA, hasB ? 1 - gyB : -1000000);
    const int f_hi = min(H - 1 - gyA, hasB ? H - 1 - gyB : 1000000);  // exclusive
    const int g_lo = g == 0 ? 1 : sh / 2;
    const int g_hi = g == 0 ? sh / 2 : sh - 1;

    for (int t = 0; t < T; ++t) {
        const uint32_t src = smem_u32(smem) + ((t & 1) ? bufb : 0);
        const uint32_t dst = smem_u32(smem) + ((t & 1) ? 0 : bufb);
        const int ylo = max(g_lo, t + 1);
        const int yhi = min(g_hi, sh - 1 - t);
        // per-byte nibble counters of own candidate bits (flushed every 15 rows)
        uint32_t fl_n = 0, rp_n = 0;
        unsigned flA = 0, flB = 0, rpA = 0, rpB = 0;
        auto flush = [&]() {
            const uint32_t f = (fl_n & 0x0f0f0f0fu) + ((fl_n >> 4) & 0x0f0f0f0fu);
            const uint32_t r = (rp_n & 0x0f0f0f0fu) + ((rp_n >> 4) & 0x0f0f0f0fu);
            flA += __dp4a(f, 0x00010001u, 0u); flB += __dp4a(f, 0x01000100u, 0u);
            rpA += __dp4a(r, 0x00010001u, 0u); rpB += __dp4a(r, 0x01000100u, 0u);
            fl_n = rp_n = 0;
        };
        int pending = 0;  // warp-uniform: items waiting at ring[0, pending)
        // process ring[h, h+n), n <= kH2Round: three independent candidates per
        // lane, all loads issued before any store.  Items are the byte offsets
        // of the candidates' window corners in the interleaved tile.
        auto drain = [&](int h, int n) {
            const int o0 = static_cast<int>(lds16(ring + 2 * (h + (lane < n ? lane : 0))));
            const int o1 = static_cast<int>(lds16(ring + 2 * (h + (lane + 32 < n ? lane + 32 : 0))));
            const int o2 = static_cast<int>(lds16(ring + 2 * (h + (lane + 64 < n ? lane + 64 : 0))));
            const uint32_t v0 = h2_replace<ALE>(src, o0, a.k7);
            const uint32_t v1 = h2_replace<ALE>(src, o1, a.k7);
            const uint32_t v2 = h2_replace<ALE>(src, o2, a.k7);
            const uint32_t dc = dst + kH2RP + 2;  // items are window corners
            if (lane < n) sts8a(dc + o0, v0);
            if (lane + 32 < n) sts8a(dc + o1, v1);
            if (lane + 64 < n) sts8a(dc + o2, v2);
        };
        if (ylo < yhi) {
            const uint32_t colp = src + 16 + 8 * c;
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
            // owned-pixel mask, recomputed only where it changes (rows HALO,
            // HALO + outA, HALO + outB; warp-uniform)
            uint32_t ownm = 0;
            int next_own = ylo;
            uint32_t R = 0;  // candidate bits of the current row quad (rows y0 .. y0+3, y0 % 4 == 0)
            // append the quad's interior candidates to the warp ring; drain full rounds
            auto push = [&](int y0) {
                if (y0 & 4) flush();  // every 8 rows: the nibble counters never exceed 8
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
                    // bit b = 8k + 4h + s: row y0 + 3 - s, column byte k + 4h
                    // items are window corners: pixel offset - kH2RP - 2
                    const uint32_t base3 = static_cast<uint32_t>((y0 + 2) * kH2RP + 14 + 8 * c);
                    uint32_t mm = R;
                    // kH2PushUnroll items per loop trip: the first store always
                    // has a bit, the others are predicated on a remaining bit
                    // (bfind of 0 is ~0u; shl.b32 by >= 32 gives 0)
                    while (mm) {
#pragma unroll
                        for (int u = 0; u < kH2PushUnroll; ++u) {
                            uint32_t b, m1;
                            asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(mm));
                            asm("shl.b32 %0, 1, %1;" : "=r"(m1) : "r"(b));
                            if (u == 0 || mm) sts16(addr + 2 * u, base3 - (b & 3u) * kH2RP + (b >> 3) + (b & 4u));
                            mm ^= m1;
                        }
                        addr += 2 * kH2PushUnroll;
                    }
                    pending += total;
                    if (pending >= kH2Round) {
                        __syncwarp();  // other lanes' ring items are read only by a drain
                        int h = 0;
                        for (; pending - h >= kH2Round; h += kH2Round) drain(h, kH2Round);
                        pending -= h;
                        __syncwarp();
                        if (pending) {  // move the leftovers (< kH2Round) to the front
                            const uint32_t l0 = lane < pending ? lds16(ring + 2 * (h + lane)) : 0;
                            const uint32_t l1 = lane + 32 < pending ? lds16(ring + 2 * (h + lane + 32)) : 0;
                            const uint32_t l2 = lane + 64 < pending ? lds16(ring + 2 * (h + lane + 64)) : 0;
                            __syncwarp();
                            if (lane < pending) sts16(ring + 2 * lane, l0);
                            if (lane + 32 < pending) sts16(ring + 2 * (lane + 32), l1);
                            if (lane + 64 < pending) sts16(ring + 2 * (lane + 64), l2);
                        }
                        __syncwarp();
                    }
                }
                R = 0;
            };
            auto row = [&](int y, auto fast_tag) {
                constexpr bool FAST = decltype(fast_tag)::value;
                h2_load_row(colp + (y + 1) * kH2RP, kc, FAST ? 0u : row_oob(y + 1), nv, nraw);
                uint32_t e[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) e[i] = h2sim(v[i], v[i + 1], a.alpha2);
                uint32_t cnt[4];
                if constexpr (FAST) {
                    // S pairs (y, j)-(y+1, j) on the ALU pipe: byte-SIMD test of
                    // the raw interleaved words, dissimilar bytes 0x80 become the
                    // halves 1024 + 128 dis (one PRMT), credited by
                    // fma(., -1/128, .) = -8 - dis = s - 9.  Counts in this loop
                    // carry -9 per credit (up[] too), compared against ckF = ck - 18.
                    const uint32_t d0 = __vabsdiffu4(raw.x, nraw.x), d1 = __vabsdiffu4(raw.y, nraw.y);
                    const uint32_t t0 = (d0 & kLo7) + a.k7, t1 = (d1 & kLo7) + a.k7;
                    const uint32_t x0 = (ALE ? (d0 | t0) : (d0 & t0)) & kHi;
                    const uint32_t x1 = (ALE ? (d1 | t1) : (d1 & t1)) & kHi;
                    const uint32_t sv[4] = {prmt(x0, 0x64646464u, 0x4140), prmt(x0, 0x64646464u, 0x4342),
                                            prmt(x1, 0x64646464u, 0x4140), prmt(x1, 0x64646464u, 0x4342)};
                    uint32_t d[5], aa[5];
#pragma unroll
                    for (int i = 0; i < 5; ++i) d[i] = h2sim(v[i], nv[i + 1], a.alpha2);
#pragma unroll
                    for (int i = 0; i < 5; ++i) aa[i] = h2sim(v[i + 1], nv[i], a.alpha2);
                    constexpr uint32_t m128 = 0xa000a000u;  // half2(-1/128)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        cnt[j] = h2add(h2add(h2add(e[j], e[j + 1]), h2fma(sv[j], m128, d[j + 1])), h2add(aa[j], up[j]));
                        up[j] = h2fma(sv[j], m128, h2add(d[j], aa[j + 1]));
                    }
                } else {  // rows with out-of-image cells: every pair in fp16
                    uint32_t s[4], d[5], aa[5];
                    h2_pairs_down(v, nv, a.alpha2, s, d, aa);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        cnt[j] = h2add(h2add(h2add(e[j], e[j + 1]), h2add(s[j], d[j + 1])), h2add(aa[j], up[j]));
                        up[j] = h2add(h2add(s[j], d[j]), aa[j + 1]);
                    }
                }
                // the centre row goes to the destination unchanged (candidates are
                // overwritten by the replacement pass)
                sts64a(dst + y * kH2RP + 16 + 8 * c, raw);
                // row classes (warp-uniform)
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
                uint32_t vn[4];
                if (FAST) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(vn[j]) : "r"(cnt[j]), "r"(ckF[j]));
                } else {
                    const int ra = gyA + y, rb = gyB + y;
                    const bool iA = ra >= 1 && ra < H - 1, iB = hasB && rb >= 1 && rb < H - 1;
                    const bool bA = ra == 0 || ra == H - 1, bB = hasB && (rb == 0 || rb == H - 1);
                    const uint32_t ki = (iA ? 0x0000ffffu : 0u) | (iB ? 0xffff0000u : 0u);
                    const uint32_t kb = (bA ? 0x0000ffffu : 0u) | (bB ? 0xffff0000u : 0u);
                    intm &= (iA ? 0x00ff00ffu : 0u) | (iB ? 0xff00ff00u : 0u);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t ckr = (ck[j] & ki) | (ckb[j] & kb) | (neg64 & ~(ki | kb));
                        asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(vn[j]) : "r"(cnt[j]), "r"(ckr));
                    }
                }
                // sign bits -> candidate word (see the slot layout above)
                const uint32_t s01 = prmt(vn[0], vn[1], 0xFDB9u);  // 0xff per candidate, cols 0/1
                const uint32_t s23 = prmt(vn[2], vn[3], 0xFDB9u);  // cols 2/3
                const uint32_t M = (s01 & 0x01010101u) | (s23 & 0x10101010u);
                const uint32_t Mi = M & intm;
                fl_n += M & ownm;
                rp_n += Mi & ownm;
                R = (R << 1) | Mi;
                if ((y & 3) == 3) push(y - 3);
#pragma unroll
                for (int i = 0; i < 6; ++i) v[i] = nv[i];
                raw = nraw;
            };
            const int s0 = min(max(ylo, f_lo), yhi);
            const int s1 = max(min(yhi, f_hi), s0);
            for (int y = ylo; y < s0; ++y) row(y, std::false_type{});
            constexpr uint32_t m9 = 0xc880c880u;  // half2(-9): the fast rows' credit offset
#pragma unroll
            for (int j = 0; j < 4; ++j) up[j] = h2add(up[j], m9);
#pragma unroll 2
            for (int y = s0; y < s1; ++y) row(y, std::true_type{});
#pragma unroll
            for (int j = 0; j < 4; ++j) up[j] = h2add(up[j], 0x48804880u);  // half2(+9)
            for (int y = s1; y < yhi; ++y) row(y, std::false_type{});
            if (yhi & 3) {  // a partial last quad: rows (yhi & ~3) .. yhi-1
                R <<= 4 - (yhi & 3);
                push(yhi & ~3);
            }
        }
        if (pending > 0) drain(0, pending);
        flush();
        flA = __reduce_add_sync(0xffffffffu, flA);
        flB = __reduce_add_sync(0xffffffffu, flB);
        rpA = __reduce_add_sync(0xffffffffu, rpA);
        rpB = __reduce_add_sync(0xffffffffu, rpB);
        if (lane == 0) {
            if (flA) atomicAdd(&red[t][0], flA);
            if (flB) atomicAdd(&red[t][1], flB);
            if (rpA) atomicAdd(&red[t][2], rpA);
            if (rpB) atomicAdd(&red[t][3], rpB);
        }
        __syncthreads();
    }

    // ---- owned output rows: de-interleave, 16-byte coalesced stores
    {
        const uint8_t* fin = smem + ((T & 1) ? bufb : 0);
        constexpr int kOutChunks = kOutPx / 16;  // 31
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
