// kernel_b1.cuh -- the beta = 1 fused kernel with pair-symmetric similarity.
//
// Same tile, staging and replacement pass as fused_tb_kernel (kernels.cuh);
// the cardinality part exploits the symmetry of similar() (SPEC.md
// "gather/scatter equivalence"): each unordered neighbour pair is tested
// once and credited to both pixels.  For centre row y the thread computes
// four pair masks per 4-px word,
//   E (y,c)~(y,c+1)   S (y,c)~(y+1,c)   SE (y,c)~(y+1,c+1)   SW (y,c)~(y+1,c-1)
// and the 8-neighbour count of (y,c) is
//   E + W + S + N + SE + NW + SW + NE,  with
//   W = E shifted one lane, N = S of row y-1, NW = SE of y-1 shifted one
//   lane, NE = SW of y-1 shifted back one lane.
// One thread covers 16 px (4 words) of a row, one warp covers a whole
// staged row (region px 8..519), so the cross-thread lane shifts are warp
// shuffles and the only lanes without a partner (warp edges) lie outside
// the dependency cone of the 496 output px.
#pragma once
#include "kernels.cuh"

namespace phg {

#ifndef PHG_B1_WARPS
#define PHG_B1_WARPS 8
#endif
constexpr int kB1Warps = PHG_B1_WARPS;  // row bands per CTA
constexpr int kB1Threads = kB1Warps * 32;
constexpr int kB1ListCap = 512;  // u16 items: one row of candidates

__host__ __device__ constexpr int b1_smem_bytes(int sh) {
    return 2 * buf_bytes(sh) + 128 * sh + kB1Warps * kB1ListCap * 2;
}

// similar(a, b) per byte lane as bit 7, restricted to `valid` (alpha <= 128
// or > 128 selects the carry form; see swar.cuh).
template <bool ALE>
__device__ __forceinline__ uint32_t sim4(uint32_t a, uint32_t b, uint32_t k7, uint32_t one, uint32_t valid) {
    const uint32_t d = __vabsdiffu4(a, b);
    const uint32_t t = fma_add(d & kLo7, one, k7);
    return valid & ~(ALE ? (d | t) : (d & t));
}

struct Row4 {
    uint32_t c[4];  // pixels 4i..4i+3 of the thread's 16
    uint32_t r[4];  // shifted one px right (column + 1)
    uint32_t l[4];  // shifted one px left  (column - 1)
};

// rowp points at the thread's first pixel (8-byte aligned)
__device__ __forceinline__ void load_row4(const uint8_t* rowp, Row4& R) {
    const uint2 a = *reinterpret_cast<const uint2*>(rowp);
    const uint2 b = *reinterpret_cast<const uint2*>(rowp + 8);
    const uint32_t lw = lds32(rowp - 4), rw = lds32(rowp + 16);
    R.c[0] = a.x;
    R.c[1] = a.y;
    R.c[2] = b.x;
    R.c[3] = b.y;
    R.l[0] = __funnelshift_l(lw, R.c[0], 8);
    R.r[3] = __funnelshift_r(R.c[3], rw, 8);
#pragma unroll
    for (int i = 1; i < 4; ++i) R.l[i] = __funnelshift_l(R.c[i - 1], R.c[i], 8);
#pragma unroll
    for (int i = 0; i < 3; ++i) R.r[i] = __funnelshift_r(R.c[i], R.c[i + 1], 8);
}

// Per-thread constants of the row sweep.
struct B1Ctx {
    uint32_t cin[4], vE[4], vSW[4], own[4], inb[4];
    bool interior_cols;
    uint32_t k7, k_thr, one;
    int height, gy0, own_lo, own_hi, lane;
    uint8_t* dst;         // this thread's first pixel in the destination buffer, row 0
    uint8_t* dst_tile;    // destination buffer, region origin
    const uint8_t* src_tile;  // source buffer, region origin
    uint16_t* list;       // this warp's candidate list
    uint32_t* cmap;       // this thread's slot in the candidate map, row 0
    const float* rcp;
    const TileArgs* args;
    int x0, px0;
};

// Sliding state: row y (pixels + shifted copies) and the pair masks
// between rows y-1 and y.
struct B1State {
    uint32_t c[4], r[4], l[4];
    uint32_t pS[4], pSE[4], pSW[4];
};

// Process centre row y: load row y+1 into `out`, form the four pair masks
// of row y, finish the counts of row y and emit its pixels + candidates.
// ROWS_OK: rows y-1, y, y+1 are all inside the image (no row masking).
template <bool ALE, bool ROWS_OK>
__device__ __forceinline__ void b1_step(const uint8_t* colp, int y, const B1State& in, B1State& out,
                                        const B1Ctx& x, uint32_t& fl_acc, uint32_t& rp_acc) {
    Row4 nx;
    load_row4(colp + (y + 1) * kRP, nx);
    const int g = x.gy0 + y;
    const bool row_in = ROWS_OK || (g >= 0 && g < x.height);
    const bool pair_in = ROWS_OK || (row_in && g + 1 < x.height);
    const uint32_t rv = row_in ? 0xffffffffu : 0u, pv = pair_in ? 0xffffffffu : 0u;
    uint32_t E[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        E[i] = sim4<ALE>(in.c[i], in.r[i], x.k7, x.one, ROWS_OK ? x.vE[i] : (x.vE[i] & rv));
        out.pS[i] = sim4<ALE>(in.c[i], nx.c[i], x.k7, x.one, ROWS_OK ? x.cin[i] : (x.cin[i] & pv));
        out.pSE[i] = sim4<ALE>(in.c[i], nx.r[i], x.k7, x.one, ROWS_OK ? x.vE[i] : (x.vE[i] & pv));
        out.pSW[i] = sim4<ALE>(in.c[i], nx.l[i], x.k7, x.one, ROWS_OK ? x.vSW[i] : (x.vSW[i] & pv));
    }
    const uint32_t El = __shfl_up_sync(0xffffffffu, E[3], 1);
    const uint32_t SEl = __shfl_up_sync(0xffffffffu, in.pSE[3], 1);
    const uint32_t SWr = __shfl_down_sync(0xffffffffu, in.pSW[0], 1);
    const bool interior = ROWS_OK && x.interior_cols;
    const bool own_row = y >= x.own_lo && y < x.own_hi;
    uint32_t cm = 0, o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t w_ = __funnelshift_l(i ? E[i - 1] : El, E[i], 1);
        const uint32_t nw = __funnelshift_l(i ? in.pSE[i - 1] : SEl, in.pSE[i], 1);
        const uint32_t ne = __funnelshift_r(in.pSW[i], i < 3 ? in.pSW[i + 1] : SWr, 15);
        uint32_t card = 0x01010101u + w_ + nw + ne;
        card += E[i] >> 7;
        card += in.pS[i] >> 7;
        card += out.pS[i] >> 7;
        card += out.pSE[i] >> 7;
        card += out.pSW[i] >> 7;
        const uint32_t flagged = lt_bits(card, x.k_thr) & (ROWS_OK ? x.cin[i] : (x.cin[i] & rv));
        // interior: in_bounds = pix_count = 9, so flag > 6 <=> card < 3
        const uint32_t cand = interior ? (flagged & lt_bits(card, rep4(125u))) : flagged;
        o[i] = in.c[i] & (ROWS_OK ? x.inb[i] : (x.inb[i] & rv));
        cm |= ((cand * 0x00204081u) >> 28) << (4 * i);
        if (own_row) fl_acc += (flagged & x.own[i]) >> 7;
        if (own_row && interior) rp_acc += (cand & x.own[i]) >> 7;
    }
    uint8_t* op = x.dst + y * kRP;
    *reinterpret_cast<uint2*>(op) = make_uint2(o[0], o[1]);
    *reinterpret_cast<uint2*>(op + 8) = make_uint2(o[2], o[3]);
    // candidate bits (low half) + "decided interior replacement" flag of the row
    x.cmap[y * 32] = cm | (interior ? 0x80000000u : 0u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        out.c[i] = nx.c[i];
        out.r[i] = nx.r[i];
        out.l[i] = nx.l[i];
    }
}

// Rows [y, end) of one kind, two rows per trip so the sliding state
// ping-pongs between A and B without register copies; returns with the
// current state in A.
template <bool ALE, bool ROWS_OK>
__device__ __forceinline__ void b1_sweep(const uint8_t* colp, int y, int end, B1State& A, B1State& B,
                                         const B1Ctx& x, uint32_t& fl_acc, uint32_t& rp_acc) {
    for (; y + 1 < end; y += 2) {
        b1_step<ALE, ROWS_OK>(colp, y, A, B, x, fl_acc, rp_acc);
        b1_step<ALE, ROWS_OK>(colp, y + 1, B, A, x, fl_acc, rp_acc);
    }
    if (y < end) {
        b1_step<ALE, ROWS_OK>(colp, y, A, B, x, fl_acc, rp_acc);
        A = B;
    }
}

template <int T, bool ALE>
__global__ void __launch_bounds__(kB1Threads)
    fused_b1_kernel(const __grid_constant__ CUtensorMap src_map, const TileArgs a, const uint32_t one) {
    static_assert(T <= kMaxHaloPx, "halo exceeds the staged columns");
    constexpr int HALO = T;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned int red[T][2];
    __shared__ float rcp[32];  // 1/f for the RMS rule

    const int sh = a.th + 2 * HALO;
    uint8_t* buf[2] = {smem, smem + buf_bytes(sh)};
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* cmap = reinterpret_cast<uint32_t*>(smem + 2 * buf_bytes(sh));  // [sh][32]
    uint16_t* list = reinterpret_cast<uint16_t*>(smem + 2 * buf_bytes(sh) + 128 * sh) + warp * kB1ListCap;

    const int img = blockIdx.z;
    const int x0 = blockIdx.x * kOutPx - kLeftPx;
    const int out_r0 = (a.own_lo - a.row_base) + blockIdx.y * a.th;
    const int out_rows = min(a.th, (a.own_hi - a.row_base) - out_r0);
    const int y0 = out_r0 - HALO;
    const int gy0 = a.row_base + y0;

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(kRP * sh));
        tma_load_4d(buf[0], &src_map, 0, x0 / kChunk, y0, img, &bar);
    }
    if (threadIdx.x < 2 * T) red[threadIdx.x >> 1][threadIdx.x & 1] = 0;
    if (threadIdx.x < 32) rcp[threadIdx.x] = threadIdx.x ? 1.0f / static_cast<float>(threadIdx.x) : 0.0f;

    // this thread's 16 px: region px px0 .. px0+15
    const int px0 = 8 + 16 * lane;
    const int gc0 = x0 + px0;
    uint32_t cin[4], vE[4], vSW[4], own[4], inb[4];
    bool interior_cols = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t m = 0, mr = 0, ml = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = gc0 + 4 * i + j;
            if (c >= 0 && c < a.width) m |= 0x80u << (8 * j);
            if (c + 1 >= 0 && c + 1 < a.width) mr |= 0x80u << (8 * j);
            if (c - 1 >= 0 && c - 1 < a.width) ml |= 0x80u << (8 * j);
        }
        cin[i] = m;
        vE[i] = m & mr;   // E and SE pairs: both columns in the image
        vSW[i] = m & ml;  // SW pairs
        const int p = px0 + 4 * i;
        own[i] = (p >= kLeftPx && p < kLeftPx + kOutPx) ? m : 0u;
        inb[i] = msb_to_bytes(m);
        interior_cols = interior_cols && (m == kHi) && (mr == kHi) && (ml == kHi);
    }

    B1Ctx ctx;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ctx.cin[i] = cin[i];
        ctx.vE[i] = vE[i];
        ctx.vSW[i] = vSW[i];
        ctx.own[i] = own[i];
        ctx.inb[i] = inb[i];
    }
    ctx.interior_cols = interior_cols;
    ctx.k7 = a.k7;
    ctx.k_thr = a.k_thr;
    ctx.one = one;
    ctx.height = a.height;
    ctx.gy0 = gy0;
    ctx.own_lo = HALO;
    ctx.own_hi = HALO + out_rows;
    ctx.lane = lane;
    ctx.list = list;
    ctx.cmap = cmap + lane;
    ctx.rcp = rcp;
    ctx.args = &a;
    ctx.x0 = x0;
    ctx.px0 = px0;

    uint32_t nfl[T], nrp[T];
#pragma unroll
    for (int t = 0; t < T; ++t) nfl[t] = nrp[t] = 0;

    __syncthreads();
    mbar_wait(&bar, 0);
    {
        const int zlo = a.width - x0, zhi = min((a.width + 15) / 16 * 16 - x0, kRP);
        if (zlo >= 0 && zlo < zhi) {
            const int nz = zhi - zlo;
            for (int i = threadIdx.x; i < sh * nz; i += kB1Threads) buf[0][(i / nz) * kRP + zlo + i % nz] = 0;
            __syncthreads();
        }
    }

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const uint8_t* src = buf[t & 1];
        uint8_t* dstb = buf[(t + 1) & 1];
        const int rlo = t + 1, rhi = sh - t - 1;
        const int blo = rlo + (rhi - rlo) * warp / kB1Warps;
        const int bhi = rlo + (rhi - rlo) * (warp + 1) / kB1Warps;
        uint32_t fl_acc = 0, rp_acc = 0;
        if (blo < bhi) {
            const uint8_t* colp = src + px0;
            ctx.dst = dstb + px0;
            // warm-up: pairs between rows blo-1 and blo
            B1State A, B;
            Row4 prev, first;
            load_row4(colp + (blo - 1) * kRP, prev);
            load_row4(colp + blo * kRP, first);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                A.c[i] = first.c[i];
                A.r[i] = first.r[i];
                A.l[i] = first.l[i];
            }
            {
                const int g = gy0 + blo;
                const uint32_t rv = (g - 1 >= 0 && g < a.height) ? 0xffffffffu : 0u;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    A.pS[i] = sim4<ALE>(prev.c[i], A.c[i], a.k7, one, cin[i] & rv);
                    A.pSE[i] = sim4<ALE>(prev.c[i], A.r[i], a.k7, one, vE[i] & rv);
                    A.pSW[i] = sim4<ALE>(prev.c[i], A.l[i], a.k7, one, vSW[i] & rv);
                }
            }
            // rows whose whole 3-row window lies inside the image
            const int ya = min(max(blo, 1 - gy0), bhi);
            const int yb = max(min(bhi, a.height - 1 - gy0), ya);
            ctx.src_tile = src;
            ctx.dst_tile = dstb;
            b1_sweep<ALE, false>(colp, blo, ya, A, B, ctx, fl_acc, rp_acc);
            b1_sweep<ALE, true>(colp, ya, yb, A, B, ctx, fl_acc, rp_acc);
            b1_sweep<ALE, false>(colp, yb, bhi, A, B, ctx, fl_acc, rp_acc);
        }
        nfl[t] += __dp4a(fl_acc, 0x01010101u, 0u);
        nrp[t] += __dp4a(rp_acc, 0x01010101u, 0u);
        __syncthreads();
        // replacement pass: one warp per row; the row's candidates are
        // compacted with one ballot prefix (<= 16 per lane) into the warp's
        // u16 list (px | interior << 15) and processed 32 at a time.
        for (int y = rlo + warp; y < rhi; y += kB1Warps) {
            const uint32_t e = cmap[y * 32 + lane];
            uint32_t m = e & 0xffffu;
            const uint32_t intr = (e >> 16) & 0x8000u;
            const int n = __popc(m);
            const unsigned lt = (1u << lane) - 1u;
            int excl = 0, total = 0;
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const unsigned b = __ballot_sync(0xffffffffu, (n >> k) & 1);
                excl += __popc(b & lt) << k;
                total += __popc(b) << k;
            }
            if (total == 0) continue;
            int pos = excl;
            while (m) {
                const int b = 31 - __clz(m);
                m ^= 1u << b;
                list[pos++] = static_cast<uint16_t>(intr | (px0 + b));
            }
            __syncwarp();
            for (int i = lane; i < total; i += 32) {
                const uint32_t it = list[i];
                nrp[t] += process_b1<ALE>(y, it & 0x7fff, it >> 15, src, dstb, x0, gy0, HALO, HALO + out_rows, a, one,
                                          rcp);
            }
            __syncwarp();
        }
        __syncthreads();
    }

    {
        const uint8_t* fin = buf[T & 1];
        constexpr int kOutChunks = kOutPx / 16;
        uint8_t* gbase = a.dst + img * a.image_stride + static_cast<int64_t>(y0) * a.pitch + (x0 + kLeftPx);
        for (int i = threadIdx.x; i < out_rows * kOutChunks; i += kB1Threads) {
            const int r = i / kOutChunks, ch = i - r * kOutChunks;
            if (x0 + kLeftPx + 16 * ch >= a.width) continue;
            const int y = HALO + r;
            const uint4 v = *reinterpret_cast<const uint4*>(fin + y * kRP + kLeftPx + 16 * ch);
            *reinterpret_cast<uint4*>(gbase + static_cast<int64_t>(y) * a.pitch + 16 * ch) = v;
        }
    }
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

}  // namespace phg
