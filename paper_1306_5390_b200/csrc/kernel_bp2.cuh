// kernel_bp2.cuh -- the beta = 2 hot path (config C3) with the packed-bit
// neighbour logic of kernel_bp.cuh.
//
// fused_bp2_kernel<T, ALE, WIDE>: T fused iterations of cardinality
// (denoise.hpp:139-160) + removal (denoise.hpp:176-223) for beta = 2,
// Faithful borders and card_threshold <= 3.  As for beta = 1, a pixel is
// flagged iff at most thr-2 of its 24 in-bounds neighbours are similar, and a
// flagged pixel is replaced iff its 5x5 window lies inside the image (an
// interior flagged pixel has flag = 24 - #similar >= 23 > 25 - 3; a border
// pixel has flag <= in_bounds - 1 <= 19).
//
// Sweep (lane = 32-px strip, warp = 1024-px region row).  Each step loads one
// NEW row r and tests every unordered pair whose lower pixel lies in row r:
//   T1[dx] = row r-1 against row r shifted by dx, T2[dx] = row r-2 against row
//   r shifted by dx (dx = -2..2, the shifted words of row r: W2 W1 X E1 E2),
//   R1, R2 = row r against itself shifted by 1, 2 (the in-row pairs),
// 12 byte-SIMD tests packed one bit per pixel, aligned at the UPPER (or
// western) pixel.  The upper pixel takes the credit as is; the lower pixel
// of T[dx] is dx columns away, so row r's credits are grouped by shift
// (0, +1, +2, -1, -2), reduced to (>= 1, >= 2 similar) per group and shifted
// once per group.  Row r-2 is complete after its T2 credits of step r.
//
// Band edges: warp w runs the steps r of its band (the rows whose pairs with
// the two rows above it computes), so its last two rows miss the credits of
// pairs with the first two rows of the next band.  Warp w+1 computes them in
// its first two steps and parks them in shared memory (named barrier w+1);
// warp w finishes those two rows after the handover.  The last warp runs two
// extra steps past the computed range instead.
//
// Candidates are replaced exactly as for beta = 1 (per-warp list, balanced
// rounds of 64) with the 5x5 window: f = 24 - #similar in {23, 24}.
//
// DIRECT (T = 1, wide regions, no peer mirrors): one iteration per launch
// needs no second staged buffer -- each owned row goes straight from the sweep
// to HBM (two 16-byte stores per lane) and each replaced pixel is stored to
// HBM by the drain (the warp's own rows; __syncwarp orders it after the row
// store).  One buffer doubles the tile height (90 staged rows), halving the
// per-tile halo and fixed costs, and the output store loop disappears.
// List items are then band-relative ((row - b0) * 1024 + column).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "kernel_bp.cuh"

namespace phg {

__host__ __device__ constexpr int bp2_smem_bytes(int sh, bool direct = false) {
    return kBpPad + (direct ? 1 : 2) * bp_buf_bytes(sh) + kBpWarps * 32 * 16 + kBpWarps * kBpList * 2;
}

// packed masks shifted by +-1, +-2 pixels along the strip (bit of pixel q
// moves to pixel q + d); pixels shifted across the strip edge come from the
// neighbouring lane (lane 0 / lane 31 pull from lanes whose outgoing bits are
// always 0, because the pair masks end at the region edges)
__device__ __forceinline__ uint32_t bp_shE1(uint32_t P, int west) { return bp_shE(P, west); }
__device__ __forceinline__ uint32_t bp_shE2(uint32_t P, int west) {
    const uint32_t prev = __shfl_sync(0xffffffffu, P, west);
    return (P << 16) | ((P >> 15) & 0xfefeu) | ((prev >> 23) & 0x101u);
}
__device__ __forceinline__ uint32_t bp_shW1(uint32_t P, int east) {
    const uint32_t next = __shfl_sync(0xffffffffu, P, east);
    return (P >> 8) | ((P & 0xfeu) << 23) | (next << 31);
}
__device__ __forceinline__ uint32_t bp_shW2(uint32_t P, int east) {
    const uint32_t next = __shfl_sync(0xffffffffu, P, east);
    return (P >> 16) | ((P & 0xfefeu) << 15) | ((next & 0x101u) << 23);
}

// (>= 1, >= 2) of a set of packed credit words
struct Om {
    uint32_t o, w;
};
__device__ __forceinline__ Om om2(uint32_t a, uint32_t b) { return {a | b, a & b}; }
__device__ __forceinline__ Om om3(uint32_t a, uint32_t b, uint32_t c) { return {a | b | c, maj3(a, b, c)}; }
__device__ __forceinline__ Om om4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const uint32_t t = a | b | c;
    return {t | d, maj3(a, b, c) | (t & d)};
}
__device__ __forceinline__ Om om5(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e) {
    const uint32_t t = a | b | c;
    return {t | d | e, maj3(a, b, c) | maj3(t, d, e)};
}
__device__ __forceinline__ Om om_add(Om x, Om y) { return {x.o | y.o, x.w | y.w | (x.o & y.o)}; }

// the strip of one staged row with its shifted copies: W2 W1 X E1 E2
// (byte j of S[d] = pixel 4i + j + d)
__device__ __forceinline__ void bp2_load(uint32_t a, uint32_t (&X)[8], uint32_t (&E1)[8], uint32_t (&E2)[8],
                                         uint32_t (&W1)[8], uint32_t (&W2)[8]) {
    const uint4 u0 = lds128a(a), u1 = lds128a(a + 16);
    const uint32_t nx = lds32a(a + 32), px = lds32a(a - 4);
    X[0] = u0.x; X[1] = u0.y; X[2] = u0.z; X[3] = u0.w;
    X[4] = u1.x; X[5] = u1.y; X[6] = u1.z; X[7] = u1.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t hi = i < 7 ? X[i + 1] : nx, lo = i > 0 ? X[i - 1] : px;
        E1[i] = __funnelshift_r(X[i], hi, 8);
        E2[i] = __funnelshift_r(X[i], hi, 16);
        W1[i] = __funnelshift_r(lo, X[i], 24);
        W2[i] = __funnelshift_r(lo, X[i], 16);
    }
}

// RMS replacement of one beta = 2 candidate (interior, Faithful) from its 5x5
// window, exactly as removal_rows (denoise.hpp:199-217); `o1` = shared
// address of the window's top-left cell.
template <bool ALE, int RP>
__device__ __forceinline__ uint32_t bp2_replace(uint32_t o1, uint32_t k7) {
    const uint32_t b4 = o1 & ~3u;
    uint32_t L[5], H[5];  // bytes 0..3 and byte 4 of each window row
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const uint32_t w0 = lds32a(b4 + r * RP), w1 = lds32a(b4 + r * RP + 4);
        L[r] = prmt_f4e(w0, w1, o1);
        H[r] = prmt_f4e(w1, 0u, o1);  // byte 4 of the window row in the low byte
    }
    const uint32_t c4 = prmt(L[2], 0, 0x2222);  // centre x4
    uint32_t n[6];
    n[0] = L[0];
    n[1] = L[1];
    n[2] = L[3];
    n[3] = L[4];
    n[4] = prmt(prmt(H[0], H[1], 0x0040), prmt(H[3], H[4], 0x0040), 0x5410);  // column 4 of rows 0,1,3,4
    n[5] = prmt(L[2], H[2], 0x4310);                                          // row 2: cells 0,1,3,4
    uint32_t packed = 0, S = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const uint32_t d = __vabsdiffu4(n[i], c4);
        const uint32_t t = (d & kLo7) + k7;
        const uint32_t dis = (ALE ? (d | t) : (d & t)) & kHi;
        packed |= dis >> i;
        S = __dp4a(n[i] & msb_to_bytes(dis), n[i], S);
    }
    const uint32_t f = __popc(packed);  // 23 or 24
    return h2_rms(S, f, rms_rcp<23>(f));  // f in {23, 24}
}

template <int T, bool ALE, bool WIDE, bool DIRECT = false>
__global__ void __launch_bounds__(kBpThreads, 2)
    fused_bp2_kernel(const __grid_constant__ CUtensorMap src_map, const BpArgs a) {
    static_assert(T >= 1 && T <= 8, "halo exceeds the aprons");
    static_assert(!DIRECT || (T == 1 && WIDE), "direct stores: one iteration, wide regions");
    constexpr int HALO = 2 * T;
    constexpr int RP = WIDE ? 1024 : 512;
    constexpr int NH = WIDE ? 1 : 2;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][4];

    uint8_t* smem = smem_raw + kBpPad;
    const int sh = a.th + 2 * HALO;
    const int bufb = bp_buf_bytes(sh);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t down_a = s0 + (DIRECT ? 1 : 2) * bufb;  // [warps][32][4] u32: rows b1-2, b1-1 of the band above, (o, w)
    const uint32_t list_a = down_a + kBpWarps * 32 * 16 + warp * kBpList * 2;
    const uint32_t half_bytes = static_cast<uint32_t>(sh) * 512u;

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

    const int half = WIDE ? 0 : (lane >> 4);
    const int lw = WIDE ? lane : (lane & 15);
    auto lbase = [&](int l) -> uint32_t {
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
    // column classes: in image; pairs (x, x+d) inside the image and the
    // region for d = -2, -1, 1, 2; interior (2-px margin); output columns
    const int gxs = myx0 + lw * 32;
    const int wr = max(min(W - gxs, 64), -64);
    const int gl = max(min(-gxs, 64), -64);
    const int rl = -lw * 32, rr = RP - lw * 32;  // region edges in strip pixels
    const uint32_t cIn = myhas ? bp_range(gl, wr) : 0u;
    const uint32_t cP1 = myhas ? bp_range(gl, min(wr, rr) - 1) : 0u;
    const uint32_t cP2 = myhas ? bp_range(gl, min(wr, rr) - 2) : 0u;
    const uint32_t cM1 = myhas ? bp_range(max(gl, rl) + 1, wr) : 0u;
    const uint32_t cM2 = myhas ? bp_range(max(gl, rl) + 2, wr) : 0u;
    const uint32_t cInt = myhas ? bp_range(gl + 2, wr - 2) : 0u;
    const uint32_t cOwn = WIDE ? (cIn & bp_range(a.x_apron - lw * 32, a.x_apron + a.x_step - lw * 32)) : cIn;
    const uint32_t cF = myconv ? 0u : (cIn & a.enable);
    const int vlo = myhas ? max(0, -gy0) : 0;
    const int vhi = myhas ? max(vlo, min(sh, H - gy0)) : 0;
    const int ilo = max(0, 2 - gy0);
    const int ihi = myhas ? max(ilo, min(sh, H - 2 - gy0)) : ilo;
    auto rowin = [&](int y) { return static_cast<unsigned>(y - vlo) < static_cast<unsigned>(vhi - vlo); };
    auto rowint = [&](int y) { return static_cast<unsigned>(y - ilo) < static_cast<unsigned>(ihi - ilo); };
    auto rowown = [&](int y) { return static_cast<unsigned>(y - HALO) < static_cast<unsigned>(myout); };
    const int west = (lane + 31) & 31, east = (lane + 1) & 31;
    // DIRECT: global offset of the tile's buffer row 0, region column 0, and
    // which of the lane's two 16-px chunks are output columns
    const int64_t gtile = static_cast<int64_t>(imgA) * a.image_stride + static_cast<int64_t>(y0A) * a.pitch + x0A;
    const int px0 = lane * 32;
    const bool own0 = px0 >= a.x_apron && px0 < a.x_apron + a.x_step && x0A + px0 < W;
    const bool own1 = px0 + 16 >= a.x_apron && px0 + 16 < a.x_apron + a.x_step && x0A + px0 + 16 < W;

    __syncthreads();
    mbar_wait(&bar, 0);

    for (int t = 0; t < nit; ++t) {
        const uint32_t src = s0 + ((t & 1) ? bufb : 0);
        const uint32_t dst = s0 + ((t & 1) ? 0 : bufb);
        const int lo = 2 * (t + 1), hi = sh - 2 * (t + 1);  // computed rows [lo, hi)
        const int n = hi - lo;
        // steps [lo, hi + 2) split over the warps, at least two per warp
        const int nb = min(kBpWarps, (n + 2) / 2);
        // (nb == 8 whenever n + 2 >= 16: a shift instead of two integer divisions)
        const int b0 = lo + (nb == kBpWarps ? ((n + 2) * warp) >> 3 : (n + 2) * warp / nb);
        const int b1 = lo + (nb == kBpWarps ? ((n + 2) * (warp + 1)) >> 3 : (n + 2) * (warp + 1) / nb);
        const bool active = warp < nb;
        const bool last = warp == nb - 1;
        unsigned fl = 0, rp = 0;

        auto finalize = [&](int y, Om c) {
            const uint32_t F = ~(c.w | (c.o & a.sel2)) & (rowin(y) ? cF : 0u);
            const uint32_t R = F & (rowint(y) ? cInt : 0u);
            if (rowown(y)) {
                fl += __popc(F & cOwn);
                rp += __popc(R & cOwn);
            }
            // DIRECT: nothing reads the value of a pixel this tile does not
            // own, so only owned candidates are replaced
            return DIRECT ? (rowown(y) ? R & cOwn : 0u) : R;
        };
        unsigned pending = 0;
        // DIRECT items are relative to the band's first row
        const uint32_t ibase = DIRECT ? static_cast<uint32_t>(b0) * RP : 0u;
        uint8_t* const gband = a.dst + gtile + static_cast<int64_t>(b0) * a.pitch;
        auto drain = [&](unsigned h, unsigned nn) {
            const bool a0 = lane < nn, a1 = lane + 32 < nn;
            const uint32_t o0 = lds16(list_a + 2 * (h + (a0 ? lane : 0u)));
            const uint32_t o1 = lds16(list_a + 2 * (h + (a1 ? lane + 32u : 0u)));
            const uint32_t v0 = bp2_replace<ALE, RP>(src + ibase + o0 - 2 * RP - 2, a.k7);
            const uint32_t v1 = bp2_replace<ALE, RP>(src + ibase + o1 - 2 * RP - 2, a.k7);
            if constexpr (DIRECT) {
                if (a0) gband[static_cast<int64_t>(o0 >> 10) * a.pitch + (o0 & 1023u)] = static_cast<uint8_t>(v0);
                if (a1) gband[static_cast<int64_t>(o1 >> 10) * a.pitch + (o1 & 1023u)] = static_cast<uint8_t>(v1);
            } else {
                if (a0) sts8a(dst + o0, v0);
                if (a1) sts8a(dst + o1, v1);
            }
        };
        auto push = [&](uint32_t R, int y) {
            const unsigned c = __popc(R);
            unsigned incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) return;
            uint32_t la = list_a + 2 * (pending + incl - c);
            const uint32_t rowoff = cb + static_cast<uint32_t>(y) * RP - ibase;
            uint32_t mm = R;
            while (mm) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    uint32_t b, m1;
                    asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(mm));
                    asm("shl.b32 %0, 1, %1;" : "=r"(m1) : "r"(b));
                    if (u == 0 || mm) sts16(la + 2 * u, rowoff + bp_px(b));
                    mm ^= m1;
                }
                la += 4;
            }
            pending += total;
            if (pending >= 64) {
                __syncwarp();
                unsigned h = 0;
                for (; pending - h >= 64; h += 64) drain(h, 64);
                pending -= h;
                __syncwarp();
                if (pending) {
                    const uint32_t l0 = lane < pending ? lds16(list_a + 2 * (h + lane)) : 0u;
                    const uint32_t l1 = lane + 32 < pending ? lds16(list_a + 2 * (h + lane + 32)) : 0u;
                    __syncwarp();
                    if (lane < pending) sts16(list_a + 2 * lane, l0);
                    if (lane + 32 < pending) sts16(list_a + 2 * (lane + 32), l1);
                }
                __syncwarp();
            }
        };

        Om accA{0, 0}, accB{0, 0};  // rows r-1 and r-2 of the coming step
        if (active) {
            uint32_t A[8], B[8];  // rows r-1 and r-2
            bp_load(src + cb + (b0 - 2) * RP, B, A);   // A: scratch E-shift, overwritten below
            {
                uint32_t tmp[8];
                bp_load(src + cb + (b0 - 1) * RP, A, tmp);
            }
            bool vA = rowin(b0 - 1), vB = rowin(b0 - 2);
            for (int r = b0; r < b1; ++r) {
                uint32_t X[8], E1[8], E2[8], W1[8], W2[8];
                bp2_load(src + cb + r * RP, X, E1, E2, W1, W2);
                const bool vX = rowin(r);
                const bool a1 = vA && vX, a2 = vB && vX;
                // pairs with row r-1 (T1) and r-2 (T2), aligned at the upper pixel
                const uint32_t t1m2 = ~bp_dis<ALE>(A, W2, a.k7, a.one) & (a1 ? cM2 : 0u);
                const uint32_t t1m1 = ~bp_dis<ALE>(A, W1, a.k7, a.one) & (a1 ? cM1 : 0u);
                const uint32_t t10 = ~bp_dis<ALE>(A, X, a.k7, a.one) & (a1 ? cIn : 0u);
                const uint32_t t1p1 = ~bp_dis<ALE>(A, E1, a.k7, a.one) & (a1 ? cP1 : 0u);
                const uint32_t t1p2 = ~bp_dis<ALE>(A, E2, a.k7, a.one) & (a1 ? cP2 : 0u);
                const uint32_t t2m2 = ~bp_dis<ALE>(B, W2, a.k7, a.one) & (a2 ? cM2 : 0u);
                const uint32_t t2m1 = ~bp_dis<ALE>(B, W1, a.k7, a.one) & (a2 ? cM1 : 0u);
                const uint32_t t20 = ~bp_dis<ALE>(B, X, a.k7, a.one) & (a2 ? cIn : 0u);
                const uint32_t t2p1 = ~bp_dis<ALE>(B, E1, a.k7, a.one) & (a2 ? cP1 : 0u);
                const uint32_t t2p2 = ~bp_dis<ALE>(B, E2, a.k7, a.one) & (a2 ? cP2 : 0u);
                const uint32_t r1 = ~bp_dis<ALE>(X, E1, a.k7, a.one) & (vX ? cP1 : 0u);
                const uint32_t r2 = ~bp_dis<ALE>(X, E2, a.k7, a.one) & (vX ? cP2 : 0u);
                // row r-2 is complete; row r-1 takes its T1 credits
                const Om cB = om_add(accB, om5(t2m2, t2m1, t20, t2p1, t2p2));
                const Om cA = om_add(accA, om5(t1m2, t1m1, t10, t1p1, t1p2));
                // row r: its pixel x + dx of each pair, grouped by dx
                const Om g0 = om4(t10, t20, r1, r2);
                const Om gp1 = om3(t1p1, t2p1, r1), gp2 = om3(t1p2, t2p2, r2);
                const Om gm1 = om2(t1m1, t2m1), gm2 = om2(t1m2, t2m2);
                Om cX = om_add(g0, Om{bp_shE1(gp1.o, west), bp_shE1(gp1.w, west)});
                cX = om_add(cX, Om{bp_shE2(gp2.o, west), bp_shE2(gp2.w, west)});
                cX = om_add(cX, Om{bp_shW1(gm1.o, east), bp_shW1(gm1.w, east)});
                cX = om_add(cX, Om{bp_shW2(gm2.o, east), bp_shW2(gm2.w, east)});
                // the unchanged row goes to the destination
                if constexpr (DIRECT) {
                    if (rowown(r)) {
                        uint8_t* g = a.dst + gtile + static_cast<int64_t>(r) * a.pitch + px0;
                        if (own0) *reinterpret_cast<uint4*>(g) = make_uint4(X[0], X[1], X[2], X[3]);
                        if (own1) *reinterpret_cast<uint4*>(g + 16) = make_uint4(X[4], X[5], X[6], X[7]);
                    }
                } else if (r < hi) {
                    const uint32_t da = dst + cb + r * RP;
                    sts128a(da, make_uint4(X[0], X[1], X[2], X[3]));
                    sts128a(da + 16, make_uint4(X[4], X[5], X[6], X[7]));
                }
                if (r - 2 >= b0) {
                    push(finalize(r - 2, cB), r - 2);
                } else if (warp > 0) {
                    // rows b0-2, b0-1 belong to the band above: hand over
                    const uint32_t dn = down_a + ((warp - 1) * 32 + lane) * 16 + (r - b0) * 8;
                    sts32a(dn, cB.o);
                    sts32a(dn + 4, cB.w);
                    if (r == b0 + 1) asm volatile("bar.arrive %0, 64;" ::"r"(warp) : "memory");
                }
                accB = cA;
                accA = cX;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    B[i] = A[i];
                    A[i] = X[i];
                }
                vB = vA;
                vA = vX;
            }
        }
        if (active) {
            if (!last) {
                // rows b1-2 (accB) and b1-1 (accA) take the credits of their
                // pairs with rows b1, b1+1 from the band below
                asm volatile("bar.sync %0, 64;" ::"r"(warp + 1) : "memory");
                const uint32_t dn = down_a + (warp * 32 + lane) * 16;
                const Om dB{lds32a(dn), lds32a(dn + 4)}, dA{lds32a(dn + 8), lds32a(dn + 12)};
                push(finalize(b1 - 2, om_add(accB, dB)), b1 - 2);
                push(finalize(b1 - 1, om_add(accA, dA)), b1 - 1);
            }
            if (pending) {
                __syncwarp();
                drain(0, pending);
            }
        }
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
        __syncthreads();
    }

    // the staged (DIRECT: only when the iteration was skipped) or final rows
    if (!DIRECT || nit == 0) {
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
    if (tid < 4 * T && nit > 0) {
        const int t = tid >> 2, which = tid & 3;
        const unsigned v = red[t][which];
        const int img = (which & 1) ? imgB : imgA;
        if (v) atomicAdd(&a.counters[(static_cast<int64_t>(img) * a.kcap + a.it0 + t) * 2 + (which >> 1)],
                         static_cast<unsigned long long>(v));
    }
}

}  // namespace phg
