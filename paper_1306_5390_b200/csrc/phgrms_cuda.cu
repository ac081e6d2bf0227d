// phgrms_cuda.cu -- host side of the B200-native P-HGRMS path: the C ABI of
// include/phgrms_b200.h over the kernels in kernels.cuh.
//
// Reference interfaces replaced (paths relative to /root/reference/proj):
//   compute_cardinality  include/phgrms/denoise.hpp:227-241 -> phg_cardinality
//   denoise_pass         include/phgrms/denoise.hpp:243-283 -> phg_denoise_pass
//   denoise              include/phgrms/denoise.hpp:292-311 -> phg_denoise
//   Parallel engine      include/phgrms/denoise.hpp:97-135  -> phg_denoise(bands)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/phgrms_b200.h"
#include "bp_launch.h"
#include "kernel_card.cuh"
#include "kernel_gen.cuh"
#include "kernel_h2.cuh"
#include "kernel_h2b2.cuh"
#include "kernels.cuh"

namespace {
thread_local std::string g_error;
}

// phg_last_error() for the entry points of the other translation units (pgm_io.cu)
namespace phg_internal {
void set_error(const std::string& msg) { g_error = msg; }
}  // namespace phg_internal

// phg_debug_rms: the fused kernels' RMS replacement for every S < n.
// (rcp_f as the kernels derive it, phg::rms_rcp; the host's 1/f must agree)
__global__ void rms_probe_kernel(uint32_t f, float rcp_f, uint32_t n, uint32_t* out) {
    const uint32_t S = blockIdx.x * blockDim.x + threadIdx.x;
    const float rk = f < 16 ? phg::rms_rcp<7>(f) : phg::rms_rcp<23>(f);
    if (S < n) out[S] = rk == rcp_f ? phg::h2_rms(S, f, rk) : 0xffffffffu;
}

namespace {

thread_local int64_t g_launches = 0;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

#define PHG_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? PHG_ENOMEM                        \
                        : (e_ == cudaErrorNoDevice || e_ == cudaErrorInsufficientDriver ||  \
                           e_ == cudaErrorNoKernelImageForDevice)                           \
                            ? PHG_ENODEV                                                    \
                            : PHG_ECUDA,                                                    \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                \
    } while (0)

#define PHG_TRY(expr)              \
    do {                           \
        int rc_ = (expr);          \
        if (rc_ != PHG_OK) return rc_; \
    } while (0)

// Exact messages of DenoiseParams::validate (denoise.hpp:41-49).
int validate(const phg_params* p) {
    if (!p) return fail(PHG_EINVAL, "null params");
    if (p->alpha < 1 || p->alpha > 255) return fail(PHG_EINVAL, "alpha must be in [1, 255]");
    if (p->beta < 1) return fail(PHG_EINVAL, "beta must be >= 1");
    if (p->max_iterations < 1) return fail(PHG_EINVAL, "iterations must be >= 1");
    if (p->card_threshold < 1) return fail(PHG_EINVAL, "card_threshold must be >= 1");
    if (p->border != PHG_BORDER_FAITHFUL && p->border != PHG_BORDER_INBOUNDS)
        return fail(PHG_EINVAL, "border must be Faithful or InBounds");
    return PHG_OK;
}

// A band step's buffers must hold its owned rows plus the halo that lies
// inside the image, and dst must have src's geometry (phg_dev_fused_step).
int check_band(const phg_dev_image& src, const phg_dev_image& dst, int row_base, int height, int own_lo,
               int own_hi, int halo) {
    if (dst.width != src.width || dst.pitch != src.pitch || dst.n_images != src.n_images ||
        dst.rows != src.rows || (src.n_images > 1 && dst.image_stride != src.image_stride))
        return fail(PHG_EINVAL, "dst geometry differs from src");
    const int need_lo = std::max(0, own_lo - halo), need_hi = std::min(height, own_hi + halo);
    if (row_base > need_lo || static_cast<int64_t>(row_base) + src.rows < need_hi)
        return fail(PHG_EINVAL, "band buffer does not hold the owned rows and their halo");
    return PHG_OK;
}

int check_dims(int w, int h) {
    // GrayImage ctor (image.hpp:24-34)
    if (w < 1 || h < 1) return fail(PHG_EINVAL, "image dimensions must be >= 1");
    return PHG_OK;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------- TMA encoding
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

// The image is viewed as [images][rows][chunks][16 px] so that one 4-D box
// {16, 33, SH, 1} lands as a dense [SH][528] shared tile (kernels.cuh).
int encode_map(CUtensorMap* map, const phg_dev_image& im, int box_rows, int box_chunks = phg::kChunks) {
    std::call_once(g_encode_once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!g_encode) return fail(PHG_ENODEV, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(im.data) & 15) || (im.pitch & 15) || (im.image_stride & 15))
        return fail(PHG_EINVAL, "device image must be 16-byte aligned with 16-byte pitches");
    if (im.pitch < round_up(im.width, 16)) return fail(PHG_EINVAL, "pitch must be >= width rounded up to 16");
    const int64_t chunks = round_up(im.width, 16) / 16;
    cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(chunks), static_cast<cuuint64_t>(im.rows),
                          static_cast<cuuint64_t>(im.n_images)};
    cuuint64_t strides[3] = {16, static_cast<cuuint64_t>(im.pitch),
                             static_cast<cuuint64_t>(im.n_images > 1 ? im.image_stride
                                                                     : im.pitch * im.rows)};
    cuuint32_t box[4] = {16, static_cast<cuuint32_t>(box_chunks), static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, im.data, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PHG_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return PHG_OK;
}

// ------------------------------------------------------ kernel dispatch
using FusedFn = void (*)(const CUtensorMap, const phg::TileArgs);

template <int B, int T, bool A>
FusedFn fused_ptr() {
    return phg::fused_tb_kernel<B, T, A>;
}

FusedFn select_fused(int beta, int T, bool ale) {
#define PHG_CASE(B, TT)                                                                 \
    if (beta == B && T == TT) return ale ? fused_ptr<B, TT, true>() : fused_ptr<B, TT, false>();
    PHG_CASE(1, 1) PHG_CASE(1, 2) PHG_CASE(1, 3) PHG_CASE(1, 4) PHG_CASE(1, 5) PHG_CASE(1, 6)
    PHG_CASE(1, 7) PHG_CASE(1, 8) PHG_CASE(2, 1) PHG_CASE(2, 2) PHG_CASE(2, 3) PHG_CASE(2, 4)
    PHG_CASE(3, 1) PHG_CASE(3, 2)
#undef PHG_CASE
    return nullptr;
}

// beta = 3: halo 3T <= kMaxHaloPx and load_row's +-3-byte funnel shifts
int max_fused(int beta) { return beta == 1 ? 5 : beta == 2 ? 4 : beta == 3 ? 2 : 0; }

// staged rows per tile for the generic kernel (tunable: PHG_ROWS)
int generic_rows_target() {
    static const int v = [] {
        const char* e = getenv("PHG_ROWS");
        return e ? std::max(16, std::min(200, atoi(e))) : 56;
    }();
    return v;
}

struct Launch {
    int th;
    int tiles_y;
};

// Output rows per tile: keep the staged region near 64 rows while not
// wasting rows on a ragged last tile.
Launch plan_rows(int own_rows, int halo, int rows_target) {
    const int target = std::max(8, rows_target - 2 * halo);
    const int tiles = std::max(1, (own_rows + target - 1) / target);
    const int th = (own_rows + tiles - 1) / tiles;
    return {th, (own_rows + th - 1) / th};
}

// Output rows per tile for the two-tile kernel, wave-aware: the launch runs
// ceil(CTAs / resident CTAs) waves of near-equal CTAs, each sweeping
// T*sh - T(T+1) rows, so small grids (one 4K image = 240 CTAs of 36 rows on
// 296 slots) pick the tile height that minimises waves x rows per CTA.
Launch plan_rows_h2(int own_rows, int halo, int rows_target, int n_images, int tiles_x, int per_cta = 2) {
    static const int slots = [] {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return 2 * sms;  // two CTAs per SM (smem bound)
    }();
    const int th_max = std::max(1, rows_target - 2 * halo);
    Launch best = plan_rows(own_rows, halo, rows_target);
    double best_cost = 1e300;
    for (int th = std::min(th_max, own_rows); th >= std::max(1, std::min(4, own_rows)); --th) {
        const int64_t tiles_y = (own_rows + th - 1) / th;
        const int64_t ctas = (static_cast<int64_t>(n_images) * tiles_x * tiles_y + per_cta - 1) / per_cta;
        const int64_t waves = (ctas + slots - 1) / slots;
        const int sh = th + 2 * halo;
        const double cost = static_cast<double>(waves) * (halo * sh - halo * (halo + 1) + 8);
        if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = {th, static_cast<int>(tiles_y)};
        }
    }
    // even out the row tiles at the chosen count
    const int th = (own_rows + best.tiles_y - 1) / best.tiles_y;
    return {th, (own_rows + th - 1) / th};
}

using H2Fn = void (*)(const CUtensorMap, const phg::H2Args);

template <int T, bool A>
H2Fn h2_ptr() {
    return phg::fused_h2_kernel<T, A>;
}

H2Fn select_h2(int T, bool ale) {
#define PHG_CASE(TT) \
    if (T == TT) return ale ? h2_ptr<TT, true>() : h2_ptr<TT, false>();
    PHG_CASE(1) PHG_CASE(2) PHG_CASE(3) PHG_CASE(4) PHG_CASE(5)
#undef PHG_CASE
    return nullptr;
}

template <int T, bool A>
H2Fn h2b2_ptr() {
    return phg::fused_h2b2_kernel<T, A>;
}

H2Fn select_h2b2(int T, bool ale) {
#define PHG_CASE(TT) \
    if (T == TT) return ale ? h2b2_ptr<TT, true>() : h2b2_ptr<TT, false>();
    PHG_CASE(1) PHG_CASE(2) PHG_CASE(3) PHG_CASE(4)
#undef PHG_CASE
    return nullptr;
}

// staged rows per tile for the two-tile fp16 kernel (tunable: PHG_H2_ROWS);
// 51 rows keep two CTAs (2 x 112.5 KB) resident per SM
int h2_rows_target() {
    static const int v = [] {
        const char* e = getenv("PHG_H2_ROWS");
        return e ? std::max(8, std::min(62, atoi(e))) : 46;
    }();
    return v;
}

// The fp16 two-tile kernel covers the reference defaults: beta = 1, Faithful
// borders, card_threshold <= 3 (PHG_NO_H2=1 forces fused_tb_kernel).
bool use_h2(const phg_params& p, int iters) {
    static const bool off = getenv("PHG_NO_H2") != nullptr;
    return !off && p.beta == 1 && p.border == PHG_BORDER_FAITHFUL && p.card_threshold <= 3 && iters <= 5;
}

// beta = 2 on both pipes (kernel_h2b2.cuh): Faithful, card_threshold <= 3
// (PHG_NO_H2B2=1 forces fused_tb_kernel<2>).
bool use_h2b2(const phg_params& p, int iters) {
    static const bool off = getenv("PHG_NO_H2B2") != nullptr;
    return !off && p.beta == 2 && p.border == PHG_BORDER_FAITHFUL && p.card_threshold <= 3 && iters <= 4;
}

uint16_t half_bits(float f) {
    // exact for the small integers and halves used here
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t sign = (u >> 16) & 0x8000u;
    const int e = static_cast<int>((u >> 23) & 0xff) - 127 + 15;
    const uint32_t m = (u >> 13) & 0x3ffu;
    if (f == 0.0f) return static_cast<uint16_t>(sign);
    return static_cast<uint16_t>(sign | (static_cast<uint32_t>(e) << 10) | m);
}

const phg::HaloPeers kNoPeers{};

int launch_h2(const phg_dev_image& src, const phg_dev_image& dst, int row_base, int height, int own_lo,
              int own_hi, const phg_params& p, int it0, int iters, uint64_t* counters, int kcap,
              cudaStream_t stream, const phg::HaloPeers& peers = kNoPeers, bool b2 = false) {
    H2Fn fn = b2 ? select_h2b2(iters, p.alpha <= 128) : select_h2(iters, p.alpha <= 128);
    if (!fn) return fail(PHG_EINVAL, "no two-tile kernel for this iteration count");
    const int halo = b2 ? 2 * iters : iters;
    const Launch L = plan_rows_h2(own_hi - own_lo, halo, h2_rows_target(), src.n_images,
                                  (src.width + phg::kOutPx - 1) / phg::kOutPx);
    const int sh = L.th + 2 * halo;
    if (sh > phg::kH2MaxRows) return fail(PHG_EINVAL, "tile too tall");
    const size_t smem = phg::h2_smem_bytes(sh);
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh));
    PHG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    phg::H2Args a;
    a.dst = dst.data;
    a.pitch = dst.pitch;
    a.image_stride = dst.image_stride;
    a.width = src.width;
    a.height = height;
    a.row_base = row_base;
    a.own_lo = own_lo;
    a.own_hi = own_hi;
    a.th = L.th;
    a.tiles_x = (src.width + phg::kOutPx - 1) / phg::kOutPx;
    a.tiles_y = L.tiles_y;
    const int64_t n_tiles = static_cast<int64_t>(src.n_images) * a.tiles_x * a.tiles_y;
    if (n_tiles > (int64_t(1) << 31) - 2) return fail(PHG_EINVAL, "too many tiles for one launch");
    a.n_tiles = static_cast<int>(n_tiles);
    const uint32_t ah = half_bits(static_cast<float>(p.alpha));
    a.alpha2 = ah | (ah << 16);
    a.k7 = ((256u - static_cast<uint32_t>(p.alpha)) & 0x7fu) * 0x01010101u;
    a.m = std::min(p.card_threshold - 2, 1);
    a.thr = p.card_threshold;
    a.alpha = p.alpha;
    a.it0 = it0;
    a.kcap = kcap;
    a.counters = reinterpret_cast<unsigned long long*>(counters);
    a.peers = peers;
    const unsigned grid = static_cast<unsigned>((n_tiles + 1) / 2);
    fn<<<grid, phg::kH2Threads, smem, stream>>>(map, a);
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// The packed-bit kernel (kernel_bp.cuh) runs beta = 1, Faithful borders,
// card_threshold <= 3 -- the reference defaults (PHG_NO_BP=1 falls back to
// the fp16 two-tile kernel).
bool use_bp(const phg_params& p, int iters) {
    static const bool off = getenv("PHG_NO_BP") != nullptr;
    return !off && p.beta == 1 && p.border == PHG_BORDER_FAITHFUL && p.card_threshold <= 3 && iters <= 5;
}

// staged rows per tile (tunable: PHG_BP_ROWS); 46 keeps two CTAs per SM
int bp_rows_target() {
    static const int v = [] {
        const char* e = getenv("PHG_BP_ROWS");
        return e ? std::max(8, std::min(phg::kBpMaxRows, atoi(e))) : phg::kBpMaxRows;
    }();
    return v;
}

// Column tiling of the packed-bit kernel: images up to 512 px wide put two
// full-width tiles in one CTA; up to 1024 px one full-width tile; wider ones
// 992 output columns per tile with 16-px aprons.
struct BpCols {
    bool wide;
    int tiles_x, x_step, x_apron;
};
BpCols bp_cols(int width) {
    if (width <= 512) return {false, 1, 512, 0};
    if (width <= 1024) return {true, 1, 1024, 0};
    return {true, (width + 991) / 992, 992, 16};
}

// beta = 2, Faithful, card_threshold <= 3: the packed-bit beta = 2 kernel
// (kernel_bp2.cuh; PHG_NO_BP2=1 falls back to fused_h2b2_kernel)
bool use_bp2(const phg_params& p, int iters) {
    static const bool off = getenv("PHG_NO_BP2") != nullptr;
    return !off && p.beta == 2 && p.border == PHG_BORDER_FAITHFUL && p.card_threshold <= 3 && iters <= 4;
}

int launch_bp(const phg_dev_image& src, const phg_dev_image& dst, int row_base, int height, int own_lo,
              int own_hi, const phg_params& p, int it0, int iters, uint64_t* counters, int kcap,
              cudaStream_t stream, const phg::HaloPeers& peers, bool early) {
    const bool b2 = p.beta == 2;
    const int halo = p.beta * iters;
    const BpCols cols = bp_cols(src.width);
    // one iteration on wide regions: the single-buffer form (direct HBM
    // stores) unless the band engine mirrors rows to peers.  (Storing the
    // last iteration of a T = 5 launch straight to HBM instead of through the
    // output loop measured slower: C4 918 vs 994 K, C5 1069 vs 1124 K.)
    static const bool no_direct = getenv("PHG_NO_DIRECT") != nullptr;
    const bool direct = iters == 1 && cols.wide && !no_direct && peers.ptr[0] == nullptr && peers.ptr[1] == nullptr;
    const int max_rows = direct ? (b2 ? phg::kBp2DirectMaxRows : phg::kBpDirectMaxRows)
                                : (b2 ? phg::kBp2MaxRows : phg::kBpMaxRows);
    const int target = direct ? max_rows : std::min(bp_rows_target(), max_rows);
    const Launch L = plan_rows_h2(own_hi - own_lo, halo, target, src.n_images, cols.tiles_x, cols.wide ? 1 : 2);
    const int sh = L.th + 2 * halo;
    if (sh > max_rows) return fail(PHG_EINVAL, "tile too tall");
    const size_t smem = b2 ? phg::bp2_smem(sh, direct) : phg::bp_smem(sh, direct);
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh, cols.wide ? 64 : 32));
    phg::BpArgs a{};
    a.dst = dst.data;
    a.pitch = dst.pitch;
    a.image_stride = dst.image_stride;
    a.width = src.width;
    a.height = height;
    a.row_base = row_base;
    a.own_lo = own_lo;
    a.own_hi = own_hi;
    a.th = L.th;
    a.tiles_x = cols.tiles_x;
    a.tiles_y = L.tiles_y;
    const int64_t n_tiles = static_cast<int64_t>(src.n_images) * a.tiles_x * a.tiles_y;
    if (n_tiles > (int64_t(1) << 31) - 2) return fail(PHG_EINVAL, "too many tiles for one launch");
    a.n_tiles = static_cast<int>(n_tiles);
    a.x_step = cols.x_step;
    a.x_apron = cols.x_apron;
    a.k7 = ((256u - static_cast<uint32_t>(p.alpha)) & 0x7fu) * 0x01010101u;
    a.one = 1u;
    a.sel2 = p.card_threshold == 2 ? ~0u : 0u;
    a.enable = p.card_threshold >= 2 ? ~0u : 0u;
    a.it0 = it0;
    a.kcap = kcap;
    a.early = early ? 1 : 0;
    a.counters = reinterpret_cast<unsigned long long*>(counters);
    a.peers = peers;
    const unsigned grid = static_cast<unsigned>(cols.wide ? n_tiles : (n_tiles + 1) / 2);
    if (b2)
        PHG_CUDA(phg::launch_bp2_kernel(iters, p.alpha <= 128, cols.wide, direct, map, a, grid, smem, stream));
    else
        PHG_CUDA(phg::launch_bp_kernel(iters, p.alpha <= 128, cols.wide, direct, map, a, grid, smem, stream));
    ++g_launches;
    return PHG_OK;
}

// residual_noise_count for beta = 1, card_threshold <= 3 (metrics.hpp:52-59):
// the packed-bit sweep alone (fused_bp_kernel's COUNT form, single buffer,
// up to 92-row tiles) -- C < thr is exactly its "flagged" decision.
int launch_bp_count(const phg_dev_image& src, int alpha, int thr, uint64_t* counts, cudaStream_t stream) {
    const BpCols cols = bp_cols(src.width);
    const Launch L = plan_rows_h2(src.rows, 1, phg::kBpDirectMaxRows, src.n_images, cols.tiles_x, cols.wide ? 1 : 2);
    const int sh = L.th + 2;
    if (sh > phg::kBpDirectMaxRows) return fail(PHG_EINVAL, "tile too tall");
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh, cols.wide ? 64 : 32));
    phg::BpArgs a{};
    a.pitch = src.pitch;
    a.image_stride = src.image_stride;
    a.width = src.width;
    a.height = src.rows;
    a.own_hi = src.rows;
    a.th = L.th;
    a.tiles_x = cols.tiles_x;
    a.tiles_y = L.tiles_y;
    const int64_t n_tiles = static_cast<int64_t>(src.n_images) * a.tiles_x * a.tiles_y;
    if (n_tiles > (int64_t(1) << 31) - 2) return fail(PHG_EINVAL, "too many tiles for one launch");
    a.n_tiles = static_cast<int>(n_tiles);
    a.x_step = cols.x_step;
    a.x_apron = cols.x_apron;
    a.k7 = ((256u - static_cast<uint32_t>(alpha)) & 0x7fu) * 0x01010101u;
    a.one = 1u;
    a.sel2 = thr == 2 ? ~0u : 0u;
    a.enable = thr >= 2 ? ~0u : 0u;
    a.kcap = 1;
    a.counters = reinterpret_cast<unsigned long long*>(counts);
    a.peers = kNoPeers;
    const unsigned grid = static_cast<unsigned>(cols.wide ? n_tiles : (n_tiles + 1) / 2);
    PHG_CUDA(phg::launch_bp_count_kernel(alpha <= 128, cols.wide, map, a, grid, phg::bp_smem(sh, true), stream));
    ++g_launches;
    return PHG_OK;
}

// beta = 1 cardinality map (kCardMap) or C < thr count (kCardCount) over
// whole images (rows = src.rows), fp16 two-tile sweep (kernel_card.cuh).
int launch_card_h2(const phg_dev_image& src, int alpha, int mode, int thr, int32_t* card, int64_t card_pitch,
                   uint64_t* counts, cudaStream_t stream) {
    const Launch L = plan_rows_h2(src.rows, 1, 42, src.n_images, (src.width + phg::kOutPx - 1) / phg::kOutPx);
    const int sh = L.th + 2;
    const size_t smem = phg::card_smem_bytes(sh);
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh));
    const void* fn = mode == phg::kCardMap ? reinterpret_cast<const void*>(phg::card_h2_kernel<phg::kCardMap>)
                                           : reinterpret_cast<const void*>(phg::card_h2_kernel<phg::kCardCount>);
    PHG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    phg::CardArgs a;
    a.card = card;
    a.card_pitch = card_pitch;
    a.card_stride = card_pitch * src.rows;
    a.width = src.width;
    a.height = src.rows;
    a.row_base = 0;
    a.own_lo = 0;
    a.own_hi = src.rows;
    a.th = L.th;
    a.tiles_x = (src.width + phg::kOutPx - 1) / phg::kOutPx;
    a.tiles_y = L.tiles_y;
    const int64_t n_tiles = static_cast<int64_t>(src.n_images) * a.tiles_x * a.tiles_y;
    if (n_tiles > (int64_t(1) << 31) - 2) return fail(PHG_EINVAL, "too many tiles for one launch");
    a.n_tiles = static_cast<int>(n_tiles);
    const uint32_t ah = half_bits(static_cast<float>(alpha));
    a.alpha2 = ah | (ah << 16);
    const uint32_t th = half_bits(static_cast<float>(std::min(thr, 1025) - 1));
    a.thr_h2 = th | (th << 16);
    a.counts = reinterpret_cast<unsigned long long*>(counts);
    const unsigned grid = static_cast<unsigned>((n_tiles + 1) / 2);
    if (mode == phg::kCardMap)
        phg::card_h2_kernel<phg::kCardMap><<<grid, 256, smem, stream>>>(map, a);
    else
        phg::card_h2_kernel<phg::kCardCount><<<grid, 256, smem, stream>>>(map, a);
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// compute_cardinality for beta >= 2 (and beta = 1 under PHG_NO_H2) on the
// byte-SIMD kernel in CARD mode: one staged sweep, int32 C per pixel.
int launch_card_tb(const phg_dev_image& src, int alpha, int beta, int32_t* card, int64_t card_pitch,
                   cudaStream_t stream) {
    const bool ale = alpha <= 128;
    FusedFn fn = nullptr;
    if (beta == 1) fn = ale ? phg::fused_tb_kernel<1, 1, true, true> : phg::fused_tb_kernel<1, 1, false, true>;
    if (beta == 2) fn = ale ? phg::fused_tb_kernel<2, 1, true, true> : phg::fused_tb_kernel<2, 1, false, true>;
    if (!fn) return fail(PHG_EINVAL, "no staged cardinality kernel for this beta");
    const Launch L = plan_rows(src.rows, beta, generic_rows_target());
    const int sh = L.th + 2 * beta;
    if (sh > 64) return fail(PHG_EINVAL, "tile too tall");
    const size_t smem = phg::smem_bytes(sh);
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh));
    PHG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    phg::TileArgs a{};
    a.dst = nullptr;
    a.pitch = src.pitch;
    a.image_stride = src.image_stride;
    a.width = src.width;
    a.height = src.rows;
    a.row_base = 0;
    a.own_lo = 0;
    a.own_hi = src.rows;
    a.th = L.th;
    a.k7 = ((256u - static_cast<uint32_t>(alpha)) & 0x7fu) * 0x01010101u;
    a.k_thr = (128u - 3u) * 0x01010101u;
    a.alpha = alpha;
    a.thr = 3;
    a.faithful = 1;
    a.it0 = 0;
    a.kcap = 1;
    a.counters = nullptr;
    a.one = 1u;
    a.card_out = card;
    a.card_pitch = card_pitch;
    a.card_stride = card_pitch * src.rows;
    const int tiles_x = (src.width + phg::kOutPx - 1) / phg::kOutPx;
    for (int z0 = 0; z0 < src.n_images; z0 += 65535) {
        const int nz = std::min(65535, src.n_images - z0);
        CUtensorMap m2 = map;
        phg::TileArgs a2 = a;
        if (z0) {
            phg_dev_image s2 = src;
            s2.data += z0 * src.image_stride;
            s2.n_images = nz;
            PHG_TRY(encode_map(&m2, s2, sh));
            a2.card_out += static_cast<int64_t>(z0) * a.card_stride;
        }
        // grid.y is capped at 65535: tall images run in pieces of tile rows,
        // each starting its owned rows ty0 tiles further down
        for (int ty0 = 0; ty0 < L.tiles_y; ty0 += 65535) {
            phg::TileArgs a3 = a2;
            a3.own_lo = a2.own_lo + ty0 * L.th;
            dim3 grid(tiles_x, std::min(65535, L.tiles_y - ty0), nz);
            fn<<<grid, phg::kThreads, smem, stream>>>(m2, a3);
            ++g_launches;
            PHG_CUDA(cudaGetLastError());
        }
    }
    return PHG_OK;
}

int launch_fused(const phg_dev_image& src, const phg_dev_image& dst, int row_base, int height,
                 int own_lo, int own_hi, const phg_params& p, int it0, int iters,
                 uint64_t* counters, int kcap, cudaStream_t stream, const phg::HaloPeers& peers = kNoPeers,
                 bool early = false) {
    if (use_bp(p, iters) || use_bp2(p, iters))
        return launch_bp(src, dst, row_base, height, own_lo, own_hi, p, it0, iters, counters, kcap, stream, peers,
                         early);
    if (use_h2(p, iters))
        return launch_h2(src, dst, row_base, height, own_lo, own_hi, p, it0, iters, counters, kcap, stream,
                         peers);
    if (use_h2b2(p, iters))
        return launch_h2(src, dst, row_base, height, own_lo, own_hi, p, it0, iters, counters, kcap, stream,
                         peers, true);
    FusedFn fn = select_fused(p.beta, iters, p.alpha <= 128);
    if (!fn) return fail(PHG_EINVAL, "no fused kernel for this beta / iteration count");
    const int halo = p.beta * iters;
    const Launch L = plan_rows(own_hi - own_lo, halo, generic_rows_target());
    const int sh = L.th + 2 * halo;
    const size_t smem = phg::smem_bytes(sh);
    if (sh > 64) return fail(PHG_EINVAL, "tile too tall");
    CUtensorMap map;
    PHG_TRY(encode_map(&map, src, sh));
    PHG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    phg::TileArgs a{};
    a.dst = dst.data;
    a.pitch = dst.pitch;
    a.image_stride = dst.image_stride;
    a.width = src.width;
    a.height = height;
    a.row_base = row_base;
    a.own_lo = own_lo;
    a.own_hi = own_hi;
    a.th = L.th;
    a.k7 = ((256u - static_cast<uint32_t>(p.alpha)) & 0x7fu) * 0x01010101u;
    a.k_thr = (128u - static_cast<uint32_t>(std::min(p.card_threshold, 127))) * 0x01010101u;
    a.alpha = p.alpha;
    a.thr = p.card_threshold;
    a.faithful = p.border == PHG_BORDER_FAITHFUL;
    a.it0 = it0;
    a.kcap = kcap;
    a.counters = reinterpret_cast<unsigned long long*>(counters);
    a.one = 1u;
    a.peers = peers;
    const int tiles_x = (src.width + phg::kOutPx - 1) / phg::kOutPx;
    for (int z0 = 0; z0 < src.n_images; z0 += 65535) {
        const int nz = std::min(65535, src.n_images - z0);
        // images beyond the first chunk: offset the tensor map and pointers
        CUtensorMap m2 = map;
        phg::TileArgs a2 = a;
        if (z0) {
            phg_dev_image s2 = src;
            s2.data += z0 * src.image_stride;
            s2.n_images = nz;
            PHG_TRY(encode_map(&m2, s2, sh));
            a2.dst += z0 * dst.image_stride;
            a2.counters += static_cast<int64_t>(z0) * kcap * 2;
        }
        for (int ty0 = 0; ty0 < L.tiles_y; ty0 += 65535) {
            phg::TileArgs a3 = a2;
            a3.own_lo = a2.own_lo + ty0 * L.th;
            dim3 grid(tiles_x, std::min(65535, L.tiles_y - ty0), nz);
            fn<<<grid, phg::kThreads, smem, stream>>>(m2, a3);
            ++g_launches;
            PHG_CUDA(cudaGetLastError());
        }
    }
    return PHG_OK;
}

int launch_scalar(int mode, const phg_dev_image& src, const phg_dev_image* dst,
                  const int32_t* card_in, int32_t* card_out, int64_t card_pitch, int row_base,
                  int height, int own_lo, int own_hi, const phg_params& p, int it0,
                  uint64_t* counters, int kcap, cudaStream_t stream,
                  const phg::HaloPeers& peers = kNoPeers) {
    phg::ScalarArgs a;
    a.src = src.data;
    a.dst = dst ? dst->data : nullptr;
    a.card_in = card_in;
    a.card_out = card_out;
    a.card_pitch = card_pitch;
    a.pitch = src.pitch;
    a.image_stride = src.image_stride;
    a.width = src.width;
    a.height = height;
    a.row_base = row_base;
    a.own_lo = own_lo;
    a.own_hi = own_hi;
    a.alpha = p.alpha;
    a.beta = p.beta;
    a.thr = p.card_threshold;
    a.faithful = p.border == PHG_BORDER_FAITHFUL;
    a.it0 = it0;
    a.kcap = kcap;
    a.counters = reinterpret_cast<unsigned long long*>(counters);
    a.peers = peers;
    const int rows = own_hi - own_lo;
    for (int z0 = 0; z0 < src.n_images; z0 += 65535) {
        const int nz = std::min(65535, src.n_images - z0);
        phg::ScalarArgs a2 = a;
        a2.src += z0 * src.image_stride;
        if (a2.dst) a2.dst += z0 * src.image_stride;
        if (a2.counters) a2.counters += static_cast<int64_t>(z0) * kcap * 2;
        if (a2.card_in) a2.card_in += static_cast<int64_t>(z0) * height * card_pitch;
        if (a2.card_out) a2.card_out += static_cast<int64_t>(z0) * height * card_pitch;
        for (int r0 = 0; r0 < rows; r0 += 65535) {
            phg::ScalarArgs a3 = a2;
            a3.own_lo = own_lo + r0;
            a3.own_hi = std::min(own_hi, a3.own_lo + 65535);
            dim3 grid((src.width + 255) / 256, a3.own_hi - a3.own_lo, nz);
            if (mode == phg::kModeCard)
                phg::scalar_kernel<phg::kModeCard><<<grid, 256, 0, stream>>>(a3);
            else if (mode == phg::kModeRemoval)
                phg::scalar_kernel<phg::kModeRemoval><<<grid, 256, 0, stream>>>(a3);
            else
                phg::scalar_kernel<phg::kModeFused><<<grid, 256, 0, stream>>>(a3);
            ++g_launches;
            PHG_CUDA(cudaGetLastError());
        }
    }
    return PHG_OK;
}

// One chunk of `iters` iterations on a (band) buffer: fused TB kernel when
// available, else one scalar fused launch per iteration (iters must be 1).
int step(const phg_dev_image& src, const phg_dev_image& dst, int row_base, int height, int own_lo,
         int own_hi, const phg_params& p, int it0, int iters, uint64_t* counters, int kcap,
         cudaStream_t stream, const phg::HaloPeers& peers = kNoPeers, bool early = false) {
    if (max_fused(p.beta) > 0)
        return launch_fused(src, dst, row_base, height, own_lo, own_hi, p, it0, iters, counters,
                            kcap, stream, peers, early);
    if (iters != 1) return fail(PHG_EINVAL, "beta >= 3 runs one iteration per launch");
    return launch_scalar(phg::kModeFused, src, &dst, nullptr, nullptr, 0, row_base, height, own_lo,
                         own_hi, p, it0, counters, kcap, stream, peers);
}

// Iterations per launch: the kernel's maximum, except for the beta = 2
// packed-bit kernel, whose temporal blocking costs more in halo rows (2 per
// side and iteration) than it saves in HBM traffic -- C3, k = 5: T3+T2
// 676 K, T2+T2+T1 700 K, five T1 launches 714 K Mpix-it/s (measured).
// `deep`: paths that pay per launch (the row-pipelined host path, whose
// wavefront grows with the launch count -- C3 e2e 181 K with T3+T2, 150 K
// with five T1 -- and the band engines, which exchange halos per launch)
// keep the deepest blocking.
int launch_depth(const phg_params& p, bool deep) {
    static const int cap = [] {
        const char* e = getenv("PHG_TMAX");  // temporal-blocking depth cap (tuning)
        return e ? std::max(1, atoi(e)) : 1 << 20;
    }();
    const int pref = (!deep && use_bp2(p, 1)) ? 1 : max_fused(p.beta);
    return std::max(1, std::min(cap, pref));
}

// Split k iterations into launches of at most launch_depth(p, deep), evenly.
std::vector<int> chunk_plan(int k, const phg_params& p, bool deep = false) {
    const int tmax = launch_depth(p, deep);
    const int n = (k + tmax - 1) / tmax;
    std::vector<int> c(n, k / n);
    for (int i = 0; i < k % n; ++i) ++c[i];
    return c;
}

// The resident path's plan for images of these dimensions.  beta = 1 on wide
// regions: large launches run T = 1 in the single-buffer DIRECT form (92-row
// tiles, 2% halo against 11% for T = 5 at 46 rows); below ~128 Mpx per launch
// its per-launch tail costs more than that saves.  Measured (k = 5, 30% s&p,
// tools/tmax_probe.py, T=5 vs T=1 Mpix-it/s): 8192^2 1059 vs 1006 K, 10240^2
// 1097 vs 1085 K, 12288^2 1119 vs 1133 K, 16384^2 1156 vs 1197 K, 32768^2
// 1169 vs 1227 K.
std::vector<int> resident_plan(const phg_params& p, int width, int64_t pixels) {
    if (max_fused(p.beta) <= 0) return std::vector<int>(p.max_iterations, 1);
    static const bool keep = getenv("PHG_TMAX") != nullptr;  // explicit depth cap: tuning runs
    if (!keep && use_bp(p, 1) && width > 512 && pixels >= (int64_t(128) << 20))
        return std::vector<int>(p.max_iterations, 1);
    return chunk_plan(p.max_iterations, p);
}

// ------------------------------------------------- layout conversion kernels
// Host images are unpadded ([n][h][w]); the fused kernel needs 16-byte
// pitched rows (TMA).  Copying through the copy engine with cudaMemcpy2D and
// w-byte rows is slow for narrow images (481 B rows), so the public API
// moves contiguous bytes over PCIe and re-pitches on the device.
__global__ void __launch_bounds__(256) pitch_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                    int w, int64_t pitch, int64_t rows, int to_pitched) {
    const int words = (w + 3) >> 2;
    const int64_t total = rows * words;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / words;
        const int c = static_cast<int>(i - r * words) * 4;
        const uint8_t* s = to_pitched ? src + r * w + c : src + r * pitch + c;
        uint8_t* d = to_pitched ? dst + r * pitch + c : dst + r * w + c;
        const int nb = min(4, w - c);
        if (to_pitched && nb == 4) {
            const uint32_t v = s[0] | (s[1] << 8) | (s[2] << 16) | (static_cast<uint32_t>(s[3]) << 24);
            *reinterpret_cast<uint32_t*>(d) = v;
        } else {
            for (int k = 0; k < nb; ++k) d[k] = s[k];
        }
    }
}

int launch_pitch(const uint8_t* src, uint8_t* dst, int w, int64_t pitch, int64_t rows, bool to_pitched,
                 cudaStream_t st) {
    const int64_t words = rows * ((w + 3) / 4);
    const int blocks = static_cast<int>(std::min<int64_t>((words + 255) / 256, 148 * 16));
    pitch_kernel<<<std::max(1, blocks), 256, 0, st>>>(src, dst, w, pitch, rows, to_pitched ? 1 : 0);
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// ------------------------------------------------------- per-device state
constexpr int kMaxRowChunks = 16;

// One state per (calling thread, device): streams, events and grow-only
// scratch buffers.  Per thread, so that concurrent callers never share a
// buffer or a stream -- the reference's functions are pure and "safe for
// concurrent callers" -- and concurrent calls on one device
// overlap on the GPU.  Freed when the thread exits.
struct DeviceState {
    int dev = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // chunked host<->device pipeline
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t pev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t rin[kMaxRowChunks] = {}, rcomp[kMaxRowChunks] = {};  // single-image row pipeline
    std::vector<std::pair<void*, size_t>> bufs;  // grow-only scratch slots

    DeviceState() = default;
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;
    ~DeviceState() {
        if (dev < 0) return;
        int prev = -1;
        if (cudaGetDevice(&prev) != cudaSuccess) return;  // runtime already torn down
        cudaSetDevice(dev);
        if (stream) cudaStreamSynchronize(stream);
        for (auto* p : pipe)
            if (p) cudaStreamSynchronize(p);
        for (auto& b : bufs)
            if (b.first) cudaFree(b.first);
        for (auto* e : {ev0, ev1}) if (e) cudaEventDestroy(e);
        for (auto* e : pev) if (e) cudaEventDestroy(e);
        for (int i = 0; i < kMaxRowChunks; ++i) {
            if (rin[i]) cudaEventDestroy(rin[i]);
            if (rcomp[i]) cudaEventDestroy(rcomp[i]);
        }
        for (auto* p : pipe) if (p) cudaStreamDestroy(p);
        if (stream) cudaStreamDestroy(stream);
        cudaSetDevice(prev);
    }
};

thread_local std::vector<std::unique_ptr<DeviceState>> g_dev;

int current_state(DeviceState** out, int* dev_out = nullptr) {
    int dev = 0;
    PHG_CUDA(cudaGetDevice(&dev));
    if (static_cast<int>(g_dev.size()) <= dev) g_dev.resize(dev + 1);
    if (!g_dev[dev]) g_dev[dev] = std::make_unique<DeviceState>();
    DeviceState& s = *g_dev[dev];
    if (!s.stream) {
        s.dev = dev;
        PHG_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        PHG_CUDA(cudaEventCreate(&s.ev0));
        PHG_CUDA(cudaEventCreate(&s.ev1));
        for (int i = 0; i < 3; ++i) {
            PHG_CUDA(cudaStreamCreateWithFlags(&s.pipe[i], cudaStreamNonBlocking));
            PHG_CUDA(cudaEventCreateWithFlags(&s.pev[i], cudaEventDisableTiming));
        }
        for (int i = 0; i < kMaxRowChunks; ++i) {
            PHG_CUDA(cudaEventCreateWithFlags(&s.rin[i], cudaEventDisableTiming));
            PHG_CUDA(cudaEventCreateWithFlags(&s.rcomp[i], cudaEventDisableTiming));
        }
    }
    *out = &s;
    if (dev_out) *dev_out = dev;
    return PHG_OK;
}

int scratch(DeviceState* s, int slot, size_t bytes, void** out) {
    if (static_cast<int>(s->bufs.size()) <= slot) s->bufs.resize(slot + 1, {nullptr, 0});
    auto& b = s->bufs[slot];
    if (b.second < bytes) {
        if (b.first) PHG_CUDA(cudaFree(b.first));
        b.first = nullptr;
        b.second = 0;
        PHG_CUDA(cudaMalloc(&b.first, bytes));
        b.second = bytes;
    }
    *out = b.first;
    return PHG_OK;
}

phg_dev_image make_image(void* data, int w, int rows, int n) {
    phg_dev_image im;
    im.data = static_cast<uint8_t*>(data);
    im.pitch = round_up(w, 16);
    im.image_stride = im.pitch * rows;
    im.width = w;
    im.rows = rows;
    im.n_images = n;
    im._pad = 0;
    return im;
}

int upload(const phg_dev_image& im, const uint8_t* host, cudaStream_t st) {
    PHG_CUDA(cudaMemcpy2DAsync(im.data, im.pitch, host, im.width, im.width,
                               static_cast<size_t>(im.rows) * im.n_images, cudaMemcpyHostToDevice, st));
    return PHG_OK;
}

int download(uint8_t* host, const phg_dev_image& im, cudaStream_t st) {
    PHG_CUDA(cudaMemcpy2DAsync(host, im.width, im.data, im.pitch, im.width,
                               static_cast<size_t>(im.rows) * im.n_images, cudaMemcpyDeviceToHost, st));
    return PHG_OK;
}

int finalize(const std::vector<uint64_t>& ctr, int n, int kcap, float ms, phg_pass_stats* stats,
             int* iters) {
    return phg_finalize_stats(ctr.data(), n, kcap, stats, iters) == PHG_OK
               ? [&] {
                     for (int i = 0; i < n; ++i) {
                         const int it = iters[i];
                         for (int j = 0; j < it; ++j)
                             stats[static_cast<int64_t>(i) * kcap + j].elapsed_ms = ms / std::max(1, it);
                     }
                     return PHG_OK;
                 }()
               : PHG_EINVAL;
}

// ------------------------------------------------- band-sharded engine
// The reference's Parallel engine splits rows with row_blocks
// (denoise.hpp:97-107) and joins after every pass.  Here each band is a
// separate device buffer holding its owned rows plus a beta*Tmax halo; after
// every fused launch the halo rows are refreshed from the bands that own
// them (the single-device stand-in for the NVLink / NCCL exchange of the
// multi-GPU path in paper_1306_5390_b200/dist.py).
struct Band {
    int lo, hi;         // owned global rows
    int blo, bhi;       // rows held in the buffer
    phg_dev_image a, b; // ping-pong buffers
};

int denoise_bands(DeviceState* s, const phg_dev_image& in, int w, int h, const phg_params& p,
                  int nbands, const phg_dev_image& out, uint64_t* counters) {
    std::vector<Band> bands;
    for (int k = 0; k < nbands; ++k) {
        const int lo = static_cast<int>(static_cast<int64_t>(h) * k / nbands);
        const int hi = static_cast<int>(static_cast<int64_t>(h) * (k + 1) / nbands);
        if (hi > lo) bands.push_back({lo, hi, 0, 0, {}, {}});
    }
    const std::vector<int> plan = chunk_plan(p.max_iterations, p, true);
    const int tmax = *std::max_element(plan.begin(), plan.end());
    const int halo = p.beta * tmax;
    int slot = 8;
    for (auto& b : bands) {
        b.blo = std::max(0, b.lo - halo);
        b.bhi = std::min(h, b.hi + halo);
        void *pa, *pb;
        const size_t bytes = static_cast<size_t>(round_up(w, 16)) * (b.bhi - b.blo);
        PHG_TRY(scratch(s, slot++, bytes, &pa));
        PHG_TRY(scratch(s, slot++, bytes, &pb));
        b.a = make_image(pa, w, b.bhi - b.blo, 1);
        b.b = make_image(pb, w, b.bhi - b.blo, 1);
        // scatter the input (owned + halo rows) into the band's first buffer
        PHG_CUDA(cudaMemcpy2DAsync(b.a.data, b.a.pitch, in.data + static_cast<int64_t>(b.blo) * in.pitch,
                                   in.pitch, w, b.bhi - b.blo, cudaMemcpyDeviceToDevice, s->stream));
    }
    int it0 = 0;
    for (size_t c = 0; c < plan.size(); ++c) {
        for (auto& b : bands)
            PHG_TRY(step(b.a, b.b, b.blo, h, b.lo, b.hi, p, it0, plan[c], counters,
                         p.max_iterations, s->stream));
        // halo exchange: every halo row of band i comes from its owner band
        for (auto& b : bands) {
            for (auto& o : bands) {
                if (&o == &b) continue;
                const int r0 = std::max(b.blo, o.lo), r1 = std::min(b.bhi, o.hi);
                if (r1 <= r0) continue;
                PHG_CUDA(cudaMemcpy2DAsync(b.b.data + static_cast<int64_t>(r0 - b.blo) * b.b.pitch,
                                           b.b.pitch,
                                           o.b.data + static_cast<int64_t>(r0 - o.blo) * o.b.pitch,
                                           o.b.pitch, w, r1 - r0, cudaMemcpyDeviceToDevice, s->stream));
            }
        }
        for (auto& b : bands) std::swap(b.a, b.b);
        it0 += plan[c];
    }
    for (auto& b : bands)
        PHG_CUDA(cudaMemcpy2DAsync(out.data + static_cast<int64_t>(b.lo) * out.pitch, out.pitch,
                                   b.a.data + static_cast<int64_t>(b.lo - b.blo) * b.a.pitch, b.a.pitch, w,
                                   b.hi - b.lo, cudaMemcpyDeviceToDevice, s->stream));
    return PHG_OK;
}

// -------------------------------------------- host generators (restated)
// synth_image (image.hpp:53-106): std::mt19937's sequence is fixed by the
// C++ standard, so this reproduces the reference bit for bit.
void synth(int w, int h, uint32_t seed, int kind, uint8_t* out) {
    const size_t n = static_cast<size_t>(w) * h;
    if (kind == 0) {
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c)
                out[static_cast<size_t>(r) * w + c] =
                    static_cast<uint8_t>(w == 1 ? 0 : static_cast<int>(255LL * c / (w - 1)));
        return;
    }
    if (kind == 1) {
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) out[static_cast<size_t>(r) * w + c] = ((r / 8 + c / 8) & 1) ? 192 : 64;
        return;
    }
    std::mt19937 gen(seed);
    std::vector<uint8_t> raw(n);
    for (auto& v : raw) v = static_cast<uint8_t>(gen() & 0xffu);
    for (int r = 0; r < h; ++r) {
        const int ra = std::max(0, r - 1), rb = std::min(h - 1, r + 1);
        for (int c = 0; c < w; ++c) {
            const int ca = std::max(0, c - 1), cb = std::min(w - 1, c + 1);
            int sum = 0;
            const int cnt = (rb - ra + 1) * (cb - ca + 1);
            for (int i = ra; i <= rb; ++i)
                for (int j = ca; j <= cb; ++j) sum += raw[static_cast<size_t>(i) * w + j];
            out[static_cast<size_t>(r) * w + c] = static_cast<uint8_t>(std::min(255, (sum + cnt / 2) / cnt));
        }
    }
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int phg_abi_version(void) { return PHG_ABI_VERSION; }
const char* phg_last_error(void) { return g_error.c_str(); }
int phg_validate_params(const phg_params* p) { return validate(p); }
int64_t phg_launch_count(void) { return g_launches; }
void phg_reset_launch_count(void) { g_launches = 0; }

int phg_device_count(int* count) {
    PHG_CUDA(cudaGetDeviceCount(count));
    return PHG_OK;
}

int phg_set_device(int device) {
    PHG_CUDA(cudaSetDevice(device));
    return PHG_OK;
}

int phg_max_fused_iterations(int beta) { return max_fused(beta); }

int phg_launch_plan(const phg_params* p, int width, int rows, int n_images, int* iters_per_launch, int cap) {
    PHG_TRY(validate(p));
    if (width < 1 || rows < 1 || n_images < 1) return fail(PHG_EINVAL, "bad image dimensions");
    const std::vector<int> plan = resident_plan(*p, width, static_cast<int64_t>(width) * rows * n_images);
    if (iters_per_launch) {
        if (cap < static_cast<int>(plan.size())) return fail(PHG_EINVAL, "launch plan capacity too small");
        std::copy(plan.begin(), plan.end(), iters_per_launch);
    }
    return static_cast<int>(plan.size());
}

const char* phg_fused_kernel_name(const phg_params* p, int iters) {
    static const char* const h2[] = {"", "fused_h2_kernel<T=1>", "fused_h2_kernel<T=2>", "fused_h2_kernel<T=3>",
                                     "fused_h2_kernel<T=4>", "fused_h2_kernel<T=5>"};
    static const char* const b1[] = {"", "fused_tb_kernel<beta=1,T=1>", "fused_tb_kernel<beta=1,T=2>",
                                     "fused_tb_kernel<beta=1,T=3>", "fused_tb_kernel<beta=1,T=4>",
                                     "fused_tb_kernel<beta=1,T=5>"};
    static const char* const b2[] = {"", "fused_tb_kernel<beta=2,T=1>", "fused_tb_kernel<beta=2,T=2>",
                                     "fused_tb_kernel<beta=2,T=3>", "fused_tb_kernel<beta=2,T=4>"};
    static const char* const b3[] = {"", "fused_tb_kernel<beta=3,T=1>", "fused_tb_kernel<beta=3,T=2>"};
    if (!p || iters < 1) return "";
    if (max_fused(p->beta) == 0) return iters == 1 ? "scalar_kernel<fused>" : "";
    if (iters > max_fused(p->beta)) return "";
    static const char* const h2b2[] = {"", "fused_h2b2_kernel<T=1>", "fused_h2b2_kernel<T=2>",
                                       "fused_h2b2_kernel<T=3>", "fused_h2b2_kernel<T=4>"};
    static const char* const bp[] = {"", "fused_bp_kernel<T=1>", "fused_bp_kernel<T=2>", "fused_bp_kernel<T=3>",
                                     "fused_bp_kernel<T=4>", "fused_bp_kernel<T=5>"};
    static const char* const bp2[] = {"", "fused_bp2_kernel<T=1>", "fused_bp2_kernel<T=2>",
                                      "fused_bp2_kernel<T=3>", "fused_bp2_kernel<T=4>"};
    if (use_bp(*p, iters)) return bp[iters];
    if (use_bp2(*p, iters)) return bp2[iters];
    if (use_h2(*p, iters)) return h2[iters];
    if (use_h2b2(*p, iters)) return h2b2[iters];
    return p->beta == 1 ? b1[iters] : p->beta == 2 ? b2[iters] : b3[iters];
}

int phg_finalize_stats(const uint64_t* ctr, int n, int kcap, phg_pass_stats* stats, int* iterations_run) {
    if (!ctr || !stats || !iterations_run || n < 0 || kcap < 1) return fail(PHG_EINVAL, "bad arguments");
    for (int i = 0; i < n; ++i) {
        int it = 0;
        for (int j = 0; j < kcap; ++j) {
            phg_pass_stats& s = stats[static_cast<int64_t>(i) * kcap + j];
            s.iteration = j + 1;
            s._pad = 0;
            s.flagged = static_cast<int64_t>(ctr[(static_cast<int64_t>(i) * kcap + j) * 2]);
            s.replaced = static_cast<int64_t>(ctr[(static_cast<int64_t>(i) * kcap + j) * 2 + 1]);
            s.elapsed_ms = 0.0;
            it = j + 1;
            if (s.replaced == 0) break;  // denoise.hpp:308
        }
        iterations_run[i] = it;
    }
    return PHG_OK;
}

int phg_dev_fused_step(const phg_dev_image* src, const phg_dev_image* dst, int row_base, int height,
                       int own_lo, int own_hi, const phg_params* p, int it0, int iters,
                       uint64_t* counters, int kcap, void* stream) {
    PHG_TRY(validate(p));
    if (!src || !dst || own_lo < 0 || own_hi > height || own_lo >= own_hi || iters < 1 ||
        it0 < 0 || it0 + iters > kcap)
        return fail(PHG_EINVAL, "bad band geometry");
    PHG_TRY(check_band(*src, *dst, row_base, height, own_lo, own_hi, p->beta * iters));
    if (max_fused(p->beta) > 0 && iters > max_fused(p->beta))
        return fail(PHG_EINVAL, "iters exceeds phg_max_fused_iterations(beta)");
    return step(*src, *dst, row_base, height, own_lo, own_hi, *p, it0, iters, counters, kcap,
                static_cast<cudaStream_t>(stream));
}

int phg_dev_fused_step_mirrored(const phg_dev_image* src, const phg_dev_image* dst, int row_base, int height,
                                int own_lo, int own_hi, const phg_params* p, int it0, int iters,
                                uint64_t* counters, int kcap, const phg_halo_peer* peers, int npeers,
                                void* stream) {
    PHG_TRY(validate(p));
    if (!src || !dst || own_lo < 0 || own_hi > height || own_lo >= own_hi || iters < 1 || it0 < 0 ||
        it0 + iters > kcap)
        return fail(PHG_EINVAL, "bad band geometry");
    PHG_TRY(check_band(*src, *dst, row_base, height, own_lo, own_hi, p->beta * iters));
    if (max_fused(p->beta) > 0 && iters > max_fused(p->beta))
        return fail(PHG_EINVAL, "iters exceeds phg_max_fused_iterations(beta)");
    if (npeers < 0 || npeers > 2 || (npeers > 0 && !peers)) return fail(PHG_EINVAL, "at most two halo peers");
    if (dst->n_images != 1) return fail(PHG_EINVAL, "halo peers need single-image bands");
    phg::HaloPeers hp{};
    for (int i = 0; i < npeers; ++i) {
        if (!peers[i].ptr || peers[i].lo < own_lo || peers[i].hi > own_hi)
            return fail(PHG_EINVAL, "halo peer rows must be owned rows");
        hp.ptr[i] = peers[i].ptr;
        hp.row0[i] = peers[i].row0;
        hp.lo[i] = peers[i].lo;
        hp.hi[i] = peers[i].hi;
    }
    return step(*src, *dst, row_base, height, own_lo, own_hi, *p, it0, iters, counters, kcap,
                static_cast<cudaStream_t>(stream), hp);
}

// CUDA IPC: a band buffer allocated by one process mapped into another (one
// process per GPU on an NVSwitch node).  Handles name whole allocations, so
// the pointer's offset inside its allocation travels with the handle.
int phg_ipc_get_handle(const void* dev_ptr, uint8_t* handle, uint64_t* offset) {
    if (!dev_ptr || !handle || !offset) return fail(PHG_EINVAL, "null argument");
    static PFN_cuMemGetAddressRange_v3020 range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                       q == cudaDriverEntryPointSuccess
                   ? reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn)
                   : nullptr;
    }();
    if (!range) return fail(PHG_ENODEV, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return fail(PHG_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t h;
    PHG_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle, &h, sizeof(h));
    *offset = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
    return PHG_OK;
}

int phg_ipc_open_handle(const uint8_t* handle, uint64_t offset, void** dev_ptr) {
    if (!handle || !dev_ptr) return fail(PHG_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    PHG_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<uint8_t*>(base) + offset;
    return PHG_OK;
}

int phg_ipc_close(void* dev_ptr, uint64_t offset) {
    if (!dev_ptr) return fail(PHG_EINVAL, "null argument");
    PHG_CUDA(cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset));
    return PHG_OK;
}

int phg_dev_denoise(const phg_dev_image* src, const phg_dev_image* dst, const phg_dev_image* tmp,
                    const phg_params* p, uint64_t* counters, void* stream) {
    PHG_TRY(validate(p));
    if (!src || !dst || !tmp) return fail(PHG_EINVAL, "null image");
    PHG_TRY(check_dims(src->width, src->rows));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int k = p->max_iterations;
    PHG_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint64_t) * 2 * k * src->n_images, st));
    const std::vector<int> plan =
        resident_plan(*p, src->width, static_cast<int64_t>(src->width) * src->rows * src->n_images);
    const int nl = static_cast<int>(plan.size());
    const phg_dev_image* cur = src;
    int it0 = 0;
    for (int i = 0; i < nl; ++i) {
        const phg_dev_image* out = ((nl - 1 - i) % 2 == 0) ? dst : tmp;
        // whole images: the counters of the previous launch are complete, so
        // converged images skip their iterations (early exit, kernel_bp.cuh)
        PHG_TRY(step(*cur, *out, 0, src->rows, 0, src->rows, *p, it0, plan[i], counters, k, st, kNoPeers, true));
        cur = out;
        it0 += plan[i];
    }
    return PHG_OK;
}

int phg_dev_cardinality(const phg_dev_image* src, int alpha, int beta, int32_t* card, int64_t card_pitch,
                        void* stream) {
    phg_params p{alpha, beta, 1, 1, 0};
    if (alpha < 1 || alpha > 255) return fail(PHG_EINVAL, "alpha must be in [1, 255]");
    if (beta < 1) return fail(PHG_EINVAL, "beta must be >= 1");
    if (beta == 1 && !getenv("PHG_NO_H2"))
        return launch_card_h2(*src, alpha, phg::kCardMap, 1, card, card_pitch, nullptr,
                              static_cast<cudaStream_t>(stream));
    if (beta <= 2) return launch_card_tb(*src, alpha, beta, card, card_pitch, static_cast<cudaStream_t>(stream));
    return launch_scalar(phg::kModeCard, *src, nullptr, nullptr, card, card_pitch, 0, src->rows, 0,
                         src->rows, p, 0, nullptr, 1, static_cast<cudaStream_t>(stream));
}

int phg_dev_residual_count(const phg_dev_image* src, int alpha, int beta, int card_threshold, uint64_t* counts,
                           void* stream) {
    if (alpha < 1 || alpha > 255) return fail(PHG_EINVAL, "alpha must be in [1, 255]");
    if (beta < 1) return fail(PHG_EINVAL, "beta must be >= 1");
    if (card_threshold < 1) return fail(PHG_EINVAL, "card_threshold must be >= 1");
    if (!src || !counts) return fail(PHG_EINVAL, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static const bool no_bp = getenv("PHG_NO_BP") != nullptr;
    if (beta == 1 && card_threshold <= 3 && !no_bp) return launch_bp_count(*src, alpha, card_threshold, counts, st);
    if (beta == 1 && !getenv("PHG_NO_H2"))
        return launch_card_h2(*src, alpha, phg::kCardCount, card_threshold, nullptr, 0, counts, st);
    // wider windows: scalar map into a stream-ordered temporary, then count
    void* pc = nullptr;
    const int64_t cpitch = round_up(src->width, 4);
    PHG_CUDA(cudaMallocAsync(&pc, sizeof(int32_t) * cpitch * src->rows * src->n_images, st));
    const int rc = phg_dev_cardinality(src, alpha, beta, static_cast<int32_t*>(pc), cpitch, stream);
    if (rc == PHG_OK) {
        dim3 grid(std::max(1, std::min(1184, static_cast<int>((static_cast<int64_t>(src->width) * src->rows + 255) / 256))),
                  src->n_images);
        phg::count_lt_kernel<<<grid, 256, 0, st>>>(static_cast<int32_t*>(pc), cpitch, src->width, src->rows,
                                                   src->n_images, card_threshold,
                                                   reinterpret_cast<unsigned long long*>(counts));
        ++g_launches;
    }
    const cudaError_t le = cudaGetLastError();
    PHG_CUDA(cudaFreeAsync(pc, st));
    if (rc != PHG_OK) return rc;
    PHG_CUDA(le);
    return PHG_OK;
}

int phg_dev_sse(const phg_dev_image* a, const phg_dev_image* b, uint64_t* sse, void* stream) {
    if (!a || !b || !sse) return fail(PHG_EINVAL, "null argument");
    if (a->width != b->width || a->rows != b->rows || a->n_images != b->n_images || a->pitch != b->pitch ||
        a->image_stride != b->image_stride)
        return fail(PHG_EINVAL, "mse: image dimensions differ");
    if ((reinterpret_cast<uintptr_t>(a->data) | reinterpret_cast<uintptr_t>(b->data) | a->pitch | a->image_stride) & 15)
        return fail(PHG_EINVAL, "device images must be 16-byte aligned with 16-byte pitches");
    const int64_t chunks = static_cast<int64_t>(a->n_images) * a->rows * ((a->width + 15) / 16);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8, (chunks + 255) / 256)));
    phg::sse_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        a->data, b->data, a->pitch, a->image_stride, a->width, a->rows, a->n_images,
        reinterpret_cast<unsigned long long*>(sse));
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

int phg_dev_removal(const phg_dev_image* src, const int32_t* card, int64_t card_pitch, const phg_params* p,
                    const phg_dev_image* dst, uint64_t* counters, void* stream) {
    PHG_TRY(validate(p));
    if (p->beta <= 2 && !getenv("PHG_NO_TILED_REMOVAL")) {
        // tiled byte-SIMD pass (kernel_card.cuh removal_tile_kernel)
        if ((reinterpret_cast<uintptr_t>(src->data) | reinterpret_cast<uintptr_t>(dst->data) | src->pitch |
             src->image_stride) & 15 || src->pitch != dst->pitch || src->image_stride != dst->image_stride)
            return fail(PHG_EINVAL, "device images must be 16-byte aligned with 16-byte pitches");
        phg::RemovalArgs a;
        a.src = src->data;
        a.dst = dst->data;
        a.card = card;
        a.card_pitch = card_pitch;
        a.card_stride = card_pitch * src->rows;
        a.pitch = src->pitch;
        a.image_stride = src->image_stride;
        a.width = src->width;
        a.height = src->rows;
        a.alpha = p->alpha;
        a.thr = p->card_threshold;
        a.faithful = p->border == PHG_BORDER_FAITHFUL;
        a.k7 = ((256u - static_cast<uint32_t>(p->alpha)) & 0x7fu) * 0x01010101u;
        a.counters = reinterpret_cast<unsigned long long*>(counters);
        const bool vec = (card_pitch & 3) == 0 && (reinterpret_cast<uintptr_t>(card) & 15) == 0;
        const bool ale = p->alpha <= 128;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (int z0 = 0; z0 < src->n_images; z0 += 65535) {
            phg::RemovalArgs a2 = a;
            a2.src += z0 * src->image_stride;
            a2.dst += z0 * src->image_stride;
            a2.card += z0 * a.card_stride;
            if (a2.counters) a2.counters += static_cast<int64_t>(z0) * 2;
            // grid.y is capped at 65535: tall images run in pieces of tile rows
            const int tiles_y = (src->rows + phg::kRmTH - 1) / phg::kRmTH;
            for (int ty0 = 0; ty0 < tiles_y; ty0 += 65535) {
                a2.row0 = ty0 * phg::kRmTH;
                dim3 grid((src->width + phg::kRmTW - 1) / phg::kRmTW, std::min(65535, tiles_y - ty0),
                          std::min(65535, src->n_images - z0));
                if (p->beta == 1) {
                    if (ale && vec) phg::removal_tile_kernel<true, true, 1><<<grid, 256, 0, st>>>(a2);
                    else if (ale) phg::removal_tile_kernel<true, false, 1><<<grid, 256, 0, st>>>(a2);
                    else if (vec) phg::removal_tile_kernel<false, true, 1><<<grid, 256, 0, st>>>(a2);
                    else phg::removal_tile_kernel<false, false, 1><<<grid, 256, 0, st>>>(a2);
                } else {
                    if (ale && vec) phg::removal_tile_kernel<true, true, 2><<<grid, 256, 0, st>>>(a2);
                    else if (ale) phg::removal_tile_kernel<true, false, 2><<<grid, 256, 0, st>>>(a2);
                    else if (vec) phg::removal_tile_kernel<false, true, 2><<<grid, 256, 0, st>>>(a2);
                    else phg::removal_tile_kernel<false, false, 2><<<grid, 256, 0, st>>>(a2);
                }
                ++g_launches;
                PHG_CUDA(cudaGetLastError());
            }
        }
        return PHG_OK;
    }
    return launch_scalar(phg::kModeRemoval, *src, dst, card, nullptr, card_pitch, 0, src->rows, 0,
                         src->rows, *p, 0, counters, 1, static_cast<cudaStream_t>(stream));
}

int phg_cardinality(const uint8_t* img, int w, int h, int alpha, int beta, int32_t* counts) {
    if (alpha < 1 || alpha > 255) return fail(PHG_EINVAL, "alpha must be in [1, 255]");
    if (beta < 1) return fail(PHG_EINVAL, "beta must be >= 1");
    PHG_TRY(check_dims(w, h));
    DeviceState* s;
    PHG_TRY(current_state(&s));
    void *pi, *pc;
    const phg_dev_image in = make_image(nullptr, w, h, 1);
    const int64_t cpitch = round_up(w, 4);
    PHG_TRY(scratch(s, 0, in.image_stride, &pi));
    PHG_TRY(scratch(s, 3, sizeof(int32_t) * cpitch * h, &pc));
    phg_dev_image im = make_image(pi, w, h, 1);
    PHG_TRY(upload(im, img, s->stream));
    PHG_TRY(phg_dev_cardinality(&im, alpha, beta, static_cast<int32_t*>(pc), cpitch, s->stream));
    PHG_CUDA(cudaMemcpy2DAsync(counts, sizeof(int32_t) * w, pc, sizeof(int32_t) * cpitch,
                               sizeof(int32_t) * w, h, cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    return PHG_OK;
}

int phg_dev_synth_smooth(const phg_dev_image* out, int row_base, int height, uint64_t seed, void* stream) {
    if (!out || !out->data) return fail(PHG_EINVAL, "null argument");
    PHG_TRY(check_dims(out->width, out->rows));
    if (row_base < 0 || row_base + out->rows > height) return fail(PHG_EINVAL, "rows outside the image");
    if (out->n_images < 1 || out->n_images > 65535) return fail(PHG_EINVAL, "1..65535 images per call");
    phg::GenArgs a{};
    a.img = out->data;
    a.pitch = out->pitch;
    a.image_stride = out->image_stride;
    a.width = out->width;
    a.rows = out->rows;
    a.n = out->n_images;
    a.row_base = row_base;
    a.height = height;
    a.seed = seed;
    dim3 grid((out->width + 255) / 256, std::min(out->rows, 65535), out->n_images);
    phg::gen_smooth_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

int phg_dev_inject_noise(const phg_dev_image* img, int row_base, int height, double density, double salt_ratio,
                         uint64_t seed, uint64_t* count, void* stream) {
    if (!img || !img->data) return fail(PHG_EINVAL, "null argument");
    if (row_base < 0 || row_base + img->rows > height) return fail(PHG_EINVAL, "rows outside the image");
    if (!(density >= 0.0 && density <= 1.0)) return fail(PHG_EINVAL, "density must be in [0, 1]");
    if (!(salt_ratio >= 0.0 && salt_ratio <= 1.0)) return fail(PHG_EINVAL, "salt_ratio must be in [0, 1]");
    PHG_TRY(check_dims(img->width, img->rows));
    if (density == 0.0) return PHG_OK;
    phg::GenArgs a{};
    a.img = img->data;
    a.pitch = img->pitch;
    a.image_stride = img->image_stride;
    a.width = img->width;
    a.rows = img->rows;
    a.row_base = row_base;
    a.height = height;
    a.seed = seed;
    a.all = density >= 1.0;
    a.salt_all = salt_ratio >= 1.0;
    a.thresh = a.all ? ~0ull : static_cast<uint64_t>(std::ldexp(density, 64));
    a.salt_thresh = a.salt_all ? ~0ull : static_cast<uint64_t>(std::ldexp(salt_ratio, 64));
    a.count = reinterpret_cast<unsigned long long*>(count);
    if (img->n_images > 65535) return fail(PHG_EINVAL, "at most 65535 images per call");
    a.n = img->n_images;
    dim3 grid((img->width + 255) / 256, std::min(img->rows, 65535), img->n_images);
    phg::gen_noise_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

int phg_residual_noise_count(const uint8_t* img, int w, int h, int alpha, int beta, int card_threshold,
                             uint64_t* count) {
    if (alpha < 1 || alpha > 255) return fail(PHG_EINVAL, "alpha must be in [1, 255]");
    if (beta < 1) return fail(PHG_EINVAL, "beta must be >= 1");
    if (card_threshold < 1) return fail(PHG_EINVAL, "card_threshold must be >= 1");
    if (!img || !count) return fail(PHG_EINVAL, "null argument");
    PHG_TRY(check_dims(w, h));
    DeviceState* s;
    PHG_TRY(current_state(&s));
    void *pi, *pk;
    const phg_dev_image in = make_image(nullptr, w, h, 1);
    PHG_TRY(scratch(s, 0, in.image_stride, &pi));
    PHG_TRY(scratch(s, 4, sizeof(uint64_t), &pk));
    phg_dev_image im = make_image(pi, w, h, 1);
    PHG_TRY(upload(im, img, s->stream));
    PHG_CUDA(cudaMemsetAsync(pk, 0, sizeof(uint64_t), s->stream));
    PHG_TRY(phg_dev_residual_count(&im, alpha, beta, card_threshold, static_cast<uint64_t*>(pk), s->stream));
    PHG_CUDA(cudaMemcpyAsync(count, pk, sizeof(uint64_t), cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    return PHG_OK;
}

int phg_debug_rms(int f, uint32_t n, uint32_t* out) {
    if (!out) return fail(PHG_EINVAL, "null argument");
    if ((f != 7 && f != 8 && f != 23 && f != 24) || n > (1u << 21))
        return fail(PHG_EINVAL, "phg_debug_rms: f in {7, 8, 23, 24}, n <= 2^21");
    if (n == 0) return PHG_OK;
    DeviceState* s;
    PHG_TRY(current_state(&s));
    void* pd;
    PHG_TRY(scratch(s, 4, sizeof(uint32_t) * n, &pd));
    rms_probe_kernel<<<(n + 255) / 256, 256, 0, s->stream>>>(static_cast<uint32_t>(f), 1.0f / static_cast<float>(f),
                                                              n, static_cast<uint32_t*>(pd));
    ++g_launches;
    PHG_CUDA(cudaGetLastError());
    PHG_CUDA(cudaMemcpyAsync(out, pd, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    return PHG_OK;
}

int phg_sse(const uint8_t* a, const uint8_t* b, int w, int h, uint64_t* sse) {
    if (!a || !b || !sse) return fail(PHG_EINVAL, "null argument");
    PHG_TRY(check_dims(w, h));
    DeviceState* s;
    PHG_TRY(current_state(&s));
    void *pa, *pb, *pk;
    const phg_dev_image in = make_image(nullptr, w, h, 1);
    PHG_TRY(scratch(s, 0, in.image_stride, &pa));
    PHG_TRY(scratch(s, 1, in.image_stride, &pb));
    PHG_TRY(scratch(s, 4, sizeof(uint64_t), &pk));
    phg_dev_image ia = make_image(pa, w, h, 1), ib = make_image(pb, w, h, 1);
    PHG_TRY(upload(ia, a, s->stream));
    PHG_TRY(upload(ib, b, s->stream));
    PHG_CUDA(cudaMemsetAsync(pk, 0, sizeof(uint64_t), s->stream));
    PHG_TRY(phg_dev_sse(&ia, &ib, static_cast<uint64_t*>(pk), s->stream));
    PHG_CUDA(cudaMemcpyAsync(sse, pk, sizeof(uint64_t), cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    return PHG_OK;
}

int phg_denoise_pass(const uint8_t* img, int w, int h, const int32_t* card, int cw, int ch,
                     const phg_params* p, uint8_t* out, phg_pass_stats* stats) {
    PHG_TRY(validate(p));
    if (cw != w || ch != h) return fail(PHG_EINVAL, "cardinality map does not match image");
    PHG_TRY(check_dims(w, h));
    DeviceState* s;
    PHG_TRY(current_state(&s));
    void *pi, *po, *pc, *pk;
    const int64_t cpitch = round_up(w, 4);
    const phg_dev_image probe = make_image(nullptr, w, h, 1);
    PHG_TRY(scratch(s, 0, probe.image_stride, &pi));
    PHG_TRY(scratch(s, 1, probe.image_stride, &po));
    PHG_TRY(scratch(s, 3, sizeof(int32_t) * cpitch * h, &pc));
    PHG_TRY(scratch(s, 4, sizeof(uint64_t) * 2, &pk));
    phg_dev_image im = make_image(pi, w, h, 1), om = make_image(po, w, h, 1);
    PHG_TRY(upload(im, img, s->stream));
    PHG_CUDA(cudaMemcpy2DAsync(pc, sizeof(int32_t) * cpitch, card, sizeof(int32_t) * w, sizeof(int32_t) * w, h,
                               cudaMemcpyHostToDevice, s->stream));
    PHG_CUDA(cudaMemsetAsync(pk, 0, sizeof(uint64_t) * 2, s->stream));
    PHG_CUDA(cudaEventRecord(s->ev0, s->stream));
    PHG_TRY(phg_dev_removal(&im, static_cast<int32_t*>(pc), cpitch, p, &om, static_cast<uint64_t*>(pk),
                            s->stream));
    PHG_CUDA(cudaEventRecord(s->ev1, s->stream));
    PHG_TRY(download(out, om, s->stream));
    uint64_t ctr[2];
    PHG_CUDA(cudaMemcpyAsync(ctr, pk, sizeof(ctr), cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    float ms = 0;
    PHG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    stats->iteration = 1;
    stats->_pad = 0;
    stats->flagged = static_cast<int64_t>(ctr[0]);
    stats->replaced = static_cast<int64_t>(ctr[1]);
    stats->elapsed_ms = ms;
    return PHG_OK;
}

// One large image from host to host with its rows pipelined (the e2e path
// of C2/C3/C5): the image is copied in as `npieces` row pieces (pipe[0]);
// it is computed as `nchunks` row chunks (pipe[1]), each launch of the
// k-iteration plan owning only the chunk's rows (own_lo/own_hi), and each
// chunk is copied out (pipe[2]) as soon as its last launch is done.
//   - launch 0 of chunk c waits only for the pieces holding its rows and
//     beta*T0-row halo;
//   - launches run as a wavefront: step j issues launch l of chunk j - l for
//     l = 0..L-1, so launch l of chunk c follows launch l-1 of chunks
//     c-1..c+1 (its halo) and precedes the ping-pong overwrite of its input
//     rows (chunks are taller than any halo).
// Only the owned rows of each launch change, so the result is bit-identical.
int denoise_rows_pipelined(DeviceState* s, const uint8_t* img, int w, int h, const phg_params& p, uint8_t* out,
                           uint64_t* ctr, int nchunks, int npieces) {
    const int k = p.max_iterations;
    const std::vector<int> plan = chunk_plan(k, p, true);
    const int L = static_cast<int>(plan.size());
    const int64_t pitch = round_up(w, 16), img_bytes = static_cast<int64_t>(w) * h;
    void *pin, *pout, *pa, *pb, *pc;
    const phg_dev_image probe = make_image(nullptr, w, h, 1);
    PHG_TRY(scratch(s, 6, static_cast<size_t>(img_bytes), &pin));
    PHG_TRY(scratch(s, 7, static_cast<size_t>(img_bytes), &pout));
    PHG_TRY(scratch(s, 0, probe.image_stride, &pa));
    PHG_TRY(scratch(s, 1, probe.image_stride, &pb));
    PHG_TRY(scratch(s, 2, probe.image_stride, &pc));
    phg_dev_image bufs[3] = {make_image(pa, w, h, 1), make_image(pb, w, h, 1), make_image(pc, w, h, 1)};
    auto split = [&](int n) {
        std::vector<int> r(n + 1);
        for (int c = 0; c <= n; ++c) r[c] = static_cast<int>(static_cast<int64_t>(h) * c / n);
        return r;
    };
    const std::vector<int> rp = split(npieces), rc = split(nchunks);
    auto piece_of = [&](int row) {
        int c = 0;
        while (c + 1 < npieces && rp[c + 1] <= row) ++c;
        return c;
    };
    cudaStream_t sin = s->pipe[0], scomp = s->pipe[1], sout = s->pipe[2];
    PHG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint64_t) * 2 * k, s->stream));
    PHG_CUDA(cudaEventRecord(s->ev0, s->stream));
    for (int i = 0; i < 3; ++i) PHG_CUDA(cudaStreamWaitEvent(s->pipe[i], s->ev0, 0));
    uint8_t* stin = static_cast<uint8_t*>(pin);
    uint8_t* stout = static_cast<uint8_t*>(pout);
    const bool dense = pitch == w;  // rows already 16-byte pitched: copy straight in and out
    for (int q = 0; q < npieces; ++q) {
        const int64_t rows = rp[q + 1] - rp[q];
        if (dense) {
            PHG_CUDA(cudaMemcpyAsync(bufs[0].data + rp[q] * pitch, img + static_cast<int64_t>(rp[q]) * w, rows * w,
                                     cudaMemcpyHostToDevice, sin));
        } else {
            PHG_CUDA(cudaMemcpyAsync(stin + static_cast<int64_t>(rp[q]) * w, img + static_cast<int64_t>(rp[q]) * w,
                                     rows * w, cudaMemcpyHostToDevice, sin));
            PHG_TRY(launch_pitch(stin + static_cast<int64_t>(rp[q]) * w, bufs[0].data + rp[q] * pitch, w, pitch, rows,
                                 true, sin));
        }
        PHG_CUDA(cudaEventRecord(s->rin[q], sin));
    }
    // launch l reads bufs[in(l)] and writes bufs[outb(l)]: 0 -> 1 -> 2 -> 1 -> 2 ...
    auto inb = [](int l) { return l == 0 ? 0 : (l % 2 ? 1 : 2); };
    auto outb = [](int l) { return l % 2 ? 2 : 1; };
    std::vector<int> it0(L, 0);
    for (int l = 1; l < L; ++l) it0[l] = it0[l - 1] + plan[l - 1];
    cudaPointerAttributes pattr{};
    const bool out_pinned = cudaPointerGetAttributes(&pattr, out) == cudaSuccess && pattr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a failed query on an unregistered pointer
    auto copy_out = [&](int c) -> int {
        const phg_dev_image& fin = bufs[outb(L - 1)];
        PHG_CUDA(cudaStreamWaitEvent(sout, s->rcomp[c], 0));
        const int64_t rows = rc[c + 1] - rc[c];
        if (dense) {
            PHG_CUDA(cudaMemcpyAsync(out + static_cast<int64_t>(rc[c]) * w, fin.data + rc[c] * pitch, rows * w,
                                     cudaMemcpyDeviceToHost, sout));
        } else {
            uint8_t* st = stout + static_cast<int64_t>(rc[c]) * w;
            PHG_TRY(launch_pitch(fin.data + rc[c] * pitch, st, w, pitch, rows, false, sout));
            PHG_CUDA(cudaMemcpyAsync(out + static_cast<int64_t>(rc[c]) * w, st, rows * w, cudaMemcpyDeviceToHost,
                                     sout));
        }
        return PHG_OK;
    };
    for (int j = 0; j < nchunks + L - 1; ++j) {
        for (int l = 0; l < L; ++l) {
            const int c = j - l;
            if (c < 0 || c >= nchunks) continue;
            if (l == 0) {
                const int need = std::min(h - 1, rc[c + 1] - 1 + p.beta * plan[0]);
                PHG_CUDA(cudaStreamWaitEvent(scomp, s->rin[piece_of(need)], 0));
            }
            PHG_TRY(step(bufs[inb(l)], bufs[outb(l)], 0, h, rc[c], rc[c + 1], p, it0[l], plan[l], ctr, k, scomp));
            if (l == L - 1) {
                PHG_CUDA(cudaEventRecord(s->rcomp[c], scomp));
                if (out_pinned) PHG_TRY(copy_out(c));
            }
        }
    }
    // A D2H into pageable memory blocks the calling thread until it is done,
    // which would hold back the launches queued behind it: into
    // pageable memory the copy-outs are queued after every launch instead.
    // (Into pinned memory they stay interleaved with the launches: queued
    // last, they measured 1.5x slower on C3 -- the copies then wait behind
    // the compute work in the hardware queues.)
    if (!out_pinned)
        for (int c = 0; c < nchunks; ++c) PHG_TRY(copy_out(c));
    for (int i = 0; i < 3; ++i) {
        PHG_CUDA(cudaEventRecord(s->pev[i], s->pipe[i]));
        PHG_CUDA(cudaStreamWaitEvent(s->stream, s->pev[i], 0));
    }
    PHG_CUDA(cudaEventRecord(s->ev1, s->stream));
    return PHG_OK;
}

// Row pieces (copy-in) and chunks (compute + copy-out) for one image; 0
// chunks = not worth pipelining (below 4 MB).  4-32 MB: 3 chunks over 8
// pieces (C2 4K image e2e: 98 K plain, 118 K pipelined; 2-8 chunks x 4-16
// pieces measured 109-118 K).  Larger: pieces ~2 MB+ (<= 16), chunks ~8 MB+
// (<= 12: C3 e2e with 8 / 12 / 16 chunks 175 / 191 / 179-188 K, C5 206 / 212
// / 210-219 K), never shorter than 32 rows.  PHG_ROW_CHUNKS / PHG_ROW_PIECES
// override.  Rows already 16-byte pitched (width % 16 == 0) are copied
// straight into / out of the pitched buffers.
// `halo` = beta * (iterations of the deepest launch): every chunk must be at
// least that tall, or a launch would read rows two chunks away that the
// wavefront has not produced yet (and its ping-pong overwrite would race
// with their readers).
void row_plan_for(int w, int h, int halo, int& nchunks, int& npieces) {
    const char* ev = getenv("PHG_ROW_CHUNKS");  // read per call (tuning sweeps)
    const int env = ev ? std::max(0, std::min(kMaxRowChunks, atoi(ev))) : -1;
    const char* pv = getenv("PHG_ROW_PIECES");
    const int64_t bytes = static_cast<int64_t>(w) * h;
    nchunks = npieces = 0;
    if (env == 0 || h < 64) return;
    if (env < 0 && bytes < (int64_t(4) << 20)) return;
    if (env < 0 && bytes < (int64_t(32) << 20)) {  // 4K-class images: 3 chunks, 8 pieces (C2: 98 -> 118 K)
        nchunks = std::max(1, std::min(3, h / 32));
        npieces = std::max(nchunks, std::min(8, h / 32));
    } else {
        nchunks = env > 0 ? env : static_cast<int>(std::min<int64_t>(12, bytes >> 23));
        nchunks = std::max(1, std::min(nchunks, h / 32));
        npieces = static_cast<int>(std::max<int64_t>(nchunks, std::min<int64_t>(kMaxRowChunks, bytes >> 21)));
        if (pv) npieces = std::max(1, std::min(kMaxRowChunks, atoi(pv)));
        npieces = std::min(npieces, h / 32);
        npieces = std::max(npieces, nchunks);
    }
    const int min_rows = std::max(32, halo);
    if (nchunks > 1 && h / nchunks < min_rows) nchunks = std::max(1, h / min_rows);
    npieces = std::max(npieces, nchunks);
}

int pipeline_halo(const phg_params& p) {
    const std::vector<int> plan = chunk_plan(p.max_iterations, p, true);
    return p.beta * (max_fused(p.beta) > 0 ? *std::max_element(plan.begin(), plan.end()) : 1);
}

int phg_denoise(const uint8_t* img, int w, int h, const phg_params* p, int bands, uint8_t* out,
                phg_pass_stats* stats, int* iterations_run) {
    PHG_TRY(validate(p));
    PHG_TRY(check_dims(w, h));
    DeviceState* s;
    PHG_TRY(current_state(&s));
    const int k = p->max_iterations;
    void *pi, *pa, *pb, *pk;
    const phg_dev_image probe = make_image(nullptr, w, h, 1);
    PHG_TRY(scratch(s, 0, probe.image_stride, &pi));
    PHG_TRY(scratch(s, 1, probe.image_stride, &pa));
    PHG_TRY(scratch(s, 2, probe.image_stride, &pb));
    PHG_TRY(scratch(s, 4, sizeof(uint64_t) * 2 * k, &pk));
    phg_dev_image im = make_image(pi, w, h, 1), am = make_image(pa, w, h, 1), bm = make_image(pb, w, h, 1);
    uint64_t* ctr = static_cast<uint64_t*>(pk);
    // EngineSpec::parallel(W) on one device: the result does not depend on
    // the partition (denoise.hpp:97-135), so W row bands would only add
    // launches and halo copies -- the single-image pipeline runs instead.
    // PHG_BAND_ENGINE=1 keeps the W-band engine (test hook for the band and
    // halo logic that the multi-device paths share).
    if (bands > 1 && !getenv("PHG_BAND_ENGINE")) bands = 1;
    int rchunks = 0, rpieces = 0;
    if (bands <= 1) row_plan_for(w, h, pipeline_halo(*p), rchunks, rpieces);
    if (rchunks > 0) {
        PHG_TRY(denoise_rows_pipelined(s, img, w, h, *p, out, ctr, rchunks, rpieces));
        std::vector<uint64_t> hc(2 * k);
        PHG_CUDA(cudaMemcpyAsync(hc.data(), ctr, sizeof(uint64_t) * 2 * k, cudaMemcpyDeviceToHost, s->stream));
        PHG_CUDA(cudaStreamSynchronize(s->stream));
        float ms = 0;
        PHG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
        return finalize(hc, 1, k, ms, stats, iterations_run);
    }
    PHG_TRY(upload(im, img, s->stream));
    PHG_CUDA(cudaEventRecord(s->ev0, s->stream));
    if (bands <= 1) {
        PHG_TRY(phg_dev_denoise(&im, &am, &bm, p, ctr, s->stream));
    } else {
        PHG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint64_t) * 2 * k, s->stream));
        PHG_TRY(denoise_bands(s, im, w, h, *p, bands, am, ctr));
    }
    PHG_CUDA(cudaEventRecord(s->ev1, s->stream));
    PHG_TRY(download(out, am, s->stream));
    std::vector<uint64_t> hc(2 * k);
    PHG_CUDA(cudaMemcpyAsync(hc.data(), ctr, sizeof(uint64_t) * 2 * k, cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    float ms = 0;
    PHG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    return finalize(hc, 1, k, ms, stats, iterations_run);
}

int phg_denoise_batch(const uint8_t* imgs, int n, int w, int h, const phg_params* p, uint8_t* out,
                      phg_pass_stats* stats, int* iterations_run) {
    PHG_TRY(validate(p));
    PHG_TRY(check_dims(w, h));
    if (n < 1) return fail(PHG_EINVAL, "batch must hold at least one image");
    if (n == 1) {
        int rc = 0, rp = 0;
        row_plan_for(w, h, pipeline_halo(*p), rc, rp);
        if (rc > 0) return phg_denoise(imgs, w, h, p, 1, out, stats, iterations_run);
    }
    DeviceState* s;
    PHG_TRY(current_state(&s));
    const int k = p->max_iterations;
    // Chunked pipeline over three streams: contiguous H2D of chunk i+1 and
    // D2H of chunk i-1 overlap the kernels of chunk i (host buffers should
    // be pinned for the copies to be asynchronous).
    // 8 chunks; 16 from 1024 images (C4, 4096 x 481x321, e2e over 5
    // interleaved runs: 8 chunks 210.9 K, 16 chunks 216.1 K Mpix-it/s; 12, 20
    // and 24 measured lower, 32 no better)
    static const int chunks_env = [] {
        const char* e = getenv("PHG_BATCH_CHUNKS");
        return e ? std::max(1, std::min(256, atoi(e))) : 0;
    }();
    const int nchunks = std::min(n, n >= 64 ? (chunks_env ? chunks_env : (n >= 1024 ? 16 : 8)) : 1);
    const int per = (n + nchunks - 1) / nchunks;
    const int64_t pitch = round_up(w, 16);
    const int64_t img_bytes = static_cast<int64_t>(w) * h, img_pitched = pitch * h;
    void *pk, *slot_mem[3] = {nullptr, nullptr, nullptr};
    const size_t slot_bytes = static_cast<size_t>(per) * (img_bytes + 3 * img_pitched) + 1024;
    for (int i = 0; i < std::min(3, nchunks); ++i) PHG_TRY(scratch(s, 20 + i, slot_bytes, &slot_mem[i]));
    PHG_TRY(scratch(s, 4, sizeof(uint64_t) * 2 * k * n, &pk));
    uint64_t* ctr = static_cast<uint64_t*>(pk);
    PHG_CUDA(cudaEventRecord(s->ev0, s->stream));
    for (int i = 0; i < 3; ++i) PHG_CUDA(cudaStreamWaitEvent(s->pipe[i], s->ev0, 0));
    for (int c = 0; c < nchunks; ++c) {
        const int i0 = c * per, m = std::min(per, n - i0);
        if (m <= 0) break;
        cudaStream_t st = s->pipe[c % 3];
        uint8_t* base = static_cast<uint8_t*>(slot_mem[c % 3]);
        uint8_t* stage = base;  // contiguous [m][h][w]
        uint8_t* pin = base + ((static_cast<int64_t>(per) * img_bytes + 255) / 256 * 256);
        phg_dev_image im = make_image(pin, w, h, m);
        phg_dev_image am = make_image(pin + img_pitched * per, w, h, m);
        phg_dev_image bm = make_image(pin + 2 * img_pitched * per, w, h, m);
        PHG_CUDA(cudaMemcpyAsync(stage, imgs + img_bytes * i0, img_bytes * m, cudaMemcpyHostToDevice, st));
        PHG_TRY(launch_pitch(stage, im.data, w, pitch, static_cast<int64_t>(h) * m, true, st));
        PHG_TRY(phg_dev_denoise(&im, &am, &bm, p, ctr + static_cast<int64_t>(2) * k * i0, st));
        PHG_TRY(launch_pitch(am.data, stage, w, pitch, static_cast<int64_t>(h) * m, false, st));
        PHG_CUDA(cudaMemcpyAsync(out + img_bytes * i0, stage, img_bytes * m, cudaMemcpyDeviceToHost, st));
    }
    for (int i = 0; i < 3; ++i) {
        PHG_CUDA(cudaEventRecord(s->pev[i], s->pipe[i]));
        PHG_CUDA(cudaStreamWaitEvent(s->stream, s->pev[i], 0));
    }
    PHG_CUDA(cudaEventRecord(s->ev1, s->stream));
    std::vector<uint64_t> hc(static_cast<size_t>(2) * k * n);
    PHG_CUDA(cudaMemcpyAsync(hc.data(), ctr, sizeof(uint64_t) * hc.size(), cudaMemcpyDeviceToHost, s->stream));
    PHG_CUDA(cudaStreamSynchronize(s->stream));
    float ms = 0;
    PHG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    return finalize(hc, n, k, ms / n, stats, iterations_run);
}

int phg_synth_image(int w, int h, uint32_t seed, int kind, uint8_t* out) {
    PHG_TRY(check_dims(w, h));
    if (kind < 0 || kind > 2) return fail(PHG_EINVAL, "unknown synth kind");
    synth(w, h, seed, kind, out);
    return PHG_OK;
}

// inject_sp_noise (noise.hpp:62-89): exact-count salt & pepper, partial
// Fisher-Yates over uint32 indices driven by mt19937 with rejection draws.
int64_t phg_inject_sp_noise(const uint8_t* img, int w, int h, double density, double salt_ratio,
                            uint32_t seed, uint8_t* out, uint8_t* mask) {
    if (!(density >= 0.0 && density <= 1.0)) return fail(PHG_EINVAL, "density must be in [0, 1]");
    if (!(salt_ratio >= 0.0 && salt_ratio <= 1.0)) return fail(PHG_EINVAL, "salt_ratio must be in [0, 1]");
    PHG_TRY(check_dims(w, h));
    const uint64_t total = static_cast<uint64_t>(w) * h;
    if (total > 0xffffffffull) return fail(PHG_EINVAL, "inject_sp_noise: image exceeds 2^32 - 1 pixels");
    const uint64_t n = static_cast<uint64_t>(std::llround(density * static_cast<double>(total)));
    const uint64_t salt = static_cast<uint64_t>(std::llround(salt_ratio * static_cast<double>(n)));
    std::memcpy(out, img, total);
    if (mask) std::memset(mask, 0, total);
    if (n == 0) return 0;
    std::vector<uint32_t> idx(total);
    std::iota(idx.begin(), idx.end(), 0u);
    std::mt19937 gen(seed);
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t bound = static_cast<uint32_t>(total - i);
        const uint32_t reject_below = (0u - bound) % bound;
        uint32_t r;
        do r = gen(); while (r < reject_below);
        const uint64_t j = i + r % bound;
        std::swap(idx[i], idx[j]);
        out[idx[i]] = i < salt ? 255 : 0;
        if (mask) mask[idx[i]] = 1;
    }
    return static_cast<int64_t>(n);
}

}  // extern "C"

// ===================================================== multi-device shards
// phg_denoise_sharded: the reference's Parallel engine (row_blocks over
// workers, denoise.hpp:97-135) with GPUs as the workers, for a C/C++ caller
// that has no torch.distributed.  The process drives every listed device
// itself (the one-process-per-GPU form is paper_1306_5390_b200/dist.py).
//   - a batch (n > 1) splits the images with the row_blocks formula, one
//     shard per list entry; each device runs phg_denoise_batch on its shards
//     from its own host thread.  No exchange.
//   - one image splits into row bands, band g on devices[g], each held with
//     a beta*Tmax halo.  When every band is at least a halo tall (its halo
//     then belongs to its two neighbours alone) the fused kernels themselves
//     store the owned rows that lie in a neighbour's halo into that
//     neighbour's next buffer (HaloPeers, kernels.cuh): peer stores over
//     NVLink, overlapped with the launch, and no exchange step.  The only
//     synchronisation is event waits: launch c of a band follows launch c-1
//     of both neighbours.  Thinner bands (or devices without peer access)
//     copy halo rows from their owners after every launch
//     (cudaMemcpyPeerAsync).
// A device may be listed more than once; its shards then run in order on
// that device.  Results are bit-identical to phg_denoise for every list.
namespace {

struct DeviceGuard {
    int prev = -1;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int check_devices(const int* devices, int ndev) {
    if (!devices || ndev < 1) return fail(PHG_EINVAL, "devices must list at least one GPU");
    int count = 0;
    PHG_CUDA(cudaGetDeviceCount(&count));
    for (int g = 0; g < ndev; ++g)
        if (devices[g] < 0 || devices[g] >= count)
            return fail(PHG_EINVAL, "device " + std::to_string(devices[g]) + " does not exist");
    return PHG_OK;
}

struct ShardBand {
    int dev;
    DeviceState* s;
    int lo, hi, blo, bhi;
    phg_dev_image a, b;
    cudaEvent_t done[2] = {nullptr, nullptr};  // after fused launch c: done[c & 1]
    uint64_t* ctr;               // the device's counters [k][2]
};

int sharded_bands(const uint8_t* img, int w, int h, const phg_params& p, const int* devices, int ndev,
                  uint8_t* out, phg_pass_stats* stats, int* iterations_run) {
    const int k = p.max_iterations;
    const std::vector<int> plan = chunk_plan(k, p, true);
    const int halo = p.beta * *std::max_element(plan.begin(), plan.end());
    const int64_t pitch = round_up(w, 16);
    std::vector<ShardBand> bands;
    std::vector<int> devs;  // unique, in first-use order
    std::vector<uint64_t*> dev_ctr;
    struct Events {
        std::vector<ShardBand>* b;
        ~Events() {
            for (auto& x : *b)
                for (auto e : x.done)
                    if (e) cudaEventDestroy(e);
        }
    } cleanup{&bands};
    const auto t0 = std::chrono::steady_clock::now();
    for (int g = 0; g < ndev; ++g) {
        const int lo = static_cast<int>(static_cast<int64_t>(h) * g / ndev);
        const int hi = static_cast<int>(static_cast<int64_t>(h) * (g + 1) / ndev);
        if (hi <= lo) continue;  // row_blocks skips empty blocks (denoise.hpp:104)
        ShardBand b{};
        b.dev = devices[g];
        PHG_CUDA(cudaSetDevice(b.dev));
        PHG_TRY(current_state(&b.s));
        const size_t di = std::find(devs.begin(), devs.end(), b.dev) - devs.begin();
        if (di == devs.size()) {
            void* pk;
            PHG_TRY(scratch(b.s, 5, sizeof(uint64_t) * 2 * k, &pk));
            PHG_CUDA(cudaMemsetAsync(pk, 0, sizeof(uint64_t) * 2 * k, b.s->stream));
            devs.push_back(b.dev);
            dev_ctr.push_back(static_cast<uint64_t*>(pk));
        }
        b.ctr = dev_ctr[di];
        b.lo = lo;
        b.hi = hi;
        b.blo = std::max(0, lo - halo);
        b.bhi = std::min(h, hi + halo);
        const int slot = 40 + 2 * g;
        void *pa, *pb;
        PHG_TRY(scratch(b.s, slot, static_cast<size_t>(pitch) * (b.bhi - b.blo), &pa));
        PHG_TRY(scratch(b.s, slot + 1, static_cast<size_t>(pitch) * (b.bhi - b.blo), &pb));
        b.a = make_image(pa, w, b.bhi - b.blo, 1);
        b.b = make_image(pb, w, b.bhi - b.blo, 1);
        bands.push_back(b);
        for (auto& e : bands.back().done) PHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ShardBand& nb = bands.back();
        PHG_CUDA(cudaMemcpy2DAsync(nb.a.data, pitch, img + static_cast<int64_t>(nb.blo) * w, w, w,
                                   nb.bhi - nb.blo, cudaMemcpyHostToDevice, nb.s->stream));
    }
    const int nb = static_cast<int>(bands.size());
    bool peer = !getenv("PHG_SHARD_COPY");
    for (int g = 0; g < nb; ++g) peer = peer && (nb == 1 || bands[g].hi - bands[g].lo >= halo);
    for (int g = 0; peer && g + 1 < nb; ++g) {
        const int d0 = bands[g].dev, d1 = bands[g + 1].dev;
        if (d0 == d1) continue;
        int ok01 = 0, ok10 = 0;
        PHG_CUDA(cudaDeviceCanAccessPeer(&ok01, d0, d1));
        PHG_CUDA(cudaDeviceCanAccessPeer(&ok10, d1, d0));
        if (!ok01 || !ok10) {
            peer = false;
            break;
        }
        for (const auto& pr : {std::make_pair(d0, d1), std::make_pair(d1, d0)}) {
            PHG_CUDA(cudaSetDevice(pr.first));
            const cudaError_t e = cudaDeviceEnablePeerAccess(pr.second, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else {
                PHG_CUDA(e);
            }
        }
    }
    int it0 = 0;
    if (peer) {
        for (size_t c = 0; c < plan.size(); ++c) {
            for (int g = 0; g < nb; ++g) {
                ShardBand& b = bands[g];
                PHG_CUDA(cudaSetDevice(b.dev));
                phg::HaloPeers hp{};
                if (g > 0) {  // rows of b in the upper neighbour's lower halo
                    const ShardBand& u = bands[g - 1];
                    if (c > 0) PHG_CUDA(cudaStreamWaitEvent(b.s->stream, u.done[(c - 1) & 1], 0));
                    hp.ptr[0] = u.b.data;
                    hp.row0[0] = u.blo;
                    hp.lo[0] = b.lo;
                    hp.hi[0] = std::min(b.hi, u.bhi);
                }
                if (g + 1 < nb) {  // rows of b in the lower neighbour's upper halo
                    const ShardBand& d = bands[g + 1];
                    if (c > 0) PHG_CUDA(cudaStreamWaitEvent(b.s->stream, d.done[(c - 1) & 1], 0));
                    hp.ptr[1] = d.b.data;
                    hp.row0[1] = d.blo;
                    hp.lo[1] = std::max(b.lo, d.blo);
                    hp.hi[1] = b.hi;
                }
                PHG_TRY(step(b.a, b.b, b.blo, h, b.lo, b.hi, p, it0, plan[c], b.ctr, k, b.s->stream, hp));
                PHG_CUDA(cudaEventRecord(b.done[c & 1], b.s->stream));
            }
            for (auto& b : bands) std::swap(b.a, b.b);
            it0 += plan[c];
        }
    }
    for (size_t c = 0; !peer && c < plan.size(); ++c) {
        const int iters = plan[c];
        for (auto& b : bands) {
            PHG_CUDA(cudaSetDevice(b.dev));
            PHG_TRY(step(b.a, b.b, b.blo, h, b.lo, b.hi, p, it0, iters, b.ctr, k, b.s->stream));
            PHG_CUDA(cudaEventRecord(b.done[0], b.s->stream));
        }
        // halo rows of band b from their owners.  Every owner o of a halo row
        // of b also reads b's rows (the halo relation is symmetric), which
        // orders b's copy before o's launch two chunks on (the WAR on o.b).
        for (auto& b : bands) {
            PHG_CUDA(cudaSetDevice(b.dev));
            for (auto& o : bands) {
                if (&o == &b) continue;
                const int r0 = std::max(b.blo, o.lo), r1 = std::min(b.bhi, o.hi);
                if (r1 <= r0) continue;
                PHG_CUDA(cudaStreamWaitEvent(b.s->stream, o.done[0], 0));
                PHG_CUDA(cudaMemcpyPeerAsync(b.b.data + (r0 - b.blo) * pitch, b.dev,
                                             o.b.data + (r0 - o.blo) * pitch, o.dev, (r1 - r0) * pitch,
                                             b.s->stream));
            }
        }
        for (auto& b : bands) std::swap(b.a, b.b);
        it0 += iters;
    }
    for (auto& b : bands) {
        PHG_CUDA(cudaSetDevice(b.dev));
        PHG_CUDA(cudaMemcpy2DAsync(out + static_cast<int64_t>(b.lo) * w, w,
                                   b.a.data + static_cast<int64_t>(b.lo - b.blo) * pitch, pitch, w, b.hi - b.lo,
                                   cudaMemcpyDeviceToHost, b.s->stream));
    }
    std::vector<uint64_t> total(2 * k, 0), part(2 * k);
    for (size_t d = 0; d < devs.size(); ++d) {
        PHG_CUDA(cudaSetDevice(devs[d]));
        DeviceState* s;
        PHG_TRY(current_state(&s));
        PHG_CUDA(cudaMemcpyAsync(part.data(), dev_ctr[d], sizeof(uint64_t) * 2 * k, cudaMemcpyDeviceToHost,
                                 s->stream));
        PHG_CUDA(cudaStreamSynchronize(s->stream));
        for (int i = 0; i < 2 * k; ++i) total[i] += part[i];
    }
    const float ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return finalize(total, 1, k, ms, stats, iterations_run);
}

int sharded_batch(const uint8_t* imgs, int n, int w, int h, const phg_params* p, const int* devices, int ndev,
                  uint8_t* out, phg_pass_stats* stats, int* iterations_run) {
    const int k = p->max_iterations;
    const int64_t img_bytes = static_cast<int64_t>(w) * h;
    std::vector<int> devs;
    for (int g = 0; g < ndev; ++g)
        if (std::find(devs.begin(), devs.end(), devices[g]) == devs.end()) devs.push_back(devices[g]);
    struct Result {
        int rc = PHG_OK;
        std::string err;
        int64_t launches = 0;
    };
    std::vector<Result> res(devs.size());
    auto work = [&](size_t d) {
        Result& r = res[d];
        const cudaError_t e = cudaSetDevice(devs[d]);
        if (e != cudaSuccess) {
            r.rc = PHG_ECUDA;
            r.err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
            return;
        }
        g_launches = 0;
        for (int g = 0; g < ndev && r.rc == PHG_OK; ++g) {
            if (devices[g] != devs[d]) continue;
            const int i0 = static_cast<int>(static_cast<int64_t>(n) * g / ndev);
            const int i1 = static_cast<int>(static_cast<int64_t>(n) * (g + 1) / ndev);
            if (i1 <= i0) continue;
            r.rc = phg_denoise_batch(imgs + img_bytes * i0, i1 - i0, w, h, p, out + img_bytes * i0,
                                     stats + static_cast<int64_t>(k) * i0, iterations_run + i0);
            if (r.rc != PHG_OK) r.err = g_error;
        }
        r.launches = g_launches;
    };
    std::vector<std::thread> pool;
    for (size_t d = 1; d < devs.size(); ++d) pool.emplace_back(work, d);
    const int64_t mine = g_launches;
    work(0);
    const int64_t here = res[0].launches;
    for (auto& t : pool) t.join();
    g_launches = mine + here;
    for (size_t d = 1; d < devs.size(); ++d) g_launches += res[d].launches;
    for (auto& r : res)
        if (r.rc != PHG_OK) return fail(r.rc, r.err);
    return PHG_OK;
}

}  // namespace

extern "C" int phg_denoise_sharded(const uint8_t* imgs, int n, int w, int h, const phg_params* p,
                                   const int* devices, int ndev, uint8_t* out, phg_pass_stats* stats,
                                   int* iterations_run) {
    PHG_TRY(validate(p));
    PHG_TRY(check_dims(w, h));
    if (n < 1) return fail(PHG_EINVAL, "batch must hold at least one image");
    if (!devices || ndev < 1) return fail(PHG_EINVAL, "devices must list at least one GPU");
    PHG_TRY(check_devices(devices, ndev));
    DeviceGuard guard;
    if (n > 1) return sharded_batch(imgs, n, w, h, p, devices, ndev, out, stats, iterations_run);
    return sharded_bands(imgs, w, h, *p, devices, ndev, out, stats, iterations_run);
}
