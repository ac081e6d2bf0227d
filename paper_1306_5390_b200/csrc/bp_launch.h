// bp_launch.h -- host entry of the packed-bit beta = 1 kernel (bp.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "kernels.cuh"  // HaloPeers

namespace phg {

constexpr int kBpMaxRows = 46;   // staged rows: two CTAs per SM (beta = 1)
constexpr int kBp2MaxRows = 45;  // beta = 2 (larger band-edge handover)
constexpr int kBp2DirectMaxRows = 90;  // beta = 2, one iteration, one staged buffer
constexpr int kBpDirectMaxRows = 92;   // beta = 1, one iteration, one staged buffer

struct BpArgs {
    uint8_t* dst;
    int64_t pitch;
    int64_t image_stride;
    int width;
    int height;      // global image height
    int row_base;    // global row of buffer row 0
    int own_lo;      // first owned global row
    int own_hi;      // one past the last owned global row
    int th;          // output rows per tile
    int tiles_x;     // column tiles per image (wide)
    int tiles_y;     // row tiles per image
    int n_tiles;     // n_images * tiles_y * tiles_x
    int x_step;      // output columns per column tile
    int x_apron;     // region column of the first output column
    uint32_t k7;     // ((256-alpha) & 0x7f) in every byte
    uint32_t one;    // runtime 1 (keeps the carry-trick add on the FMA pipe)
    uint32_t sel2;   // ~0 when card_threshold == 2 (flag <=> no similar neighbour)
    uint32_t enable; // 0 when card_threshold == 1 (nothing is ever flagged)
    int it0;
    int kcap;
    int early;       // skip images whose iteration it0-1 replaced nothing (fixed point)
    unsigned long long* counters;  // [n_images][kcap][2]
    HaloPeers peers;               // single-image bands only (kernels.cuh)
};

// Launches fused_bp_kernel<T, alpha <= 128, wide[, direct]> with `grid` CTAs.
cudaError_t launch_bp_kernel(int T, bool ale, bool wide, bool direct, const CUtensorMap& map, const BpArgs& a,
                             unsigned grid, size_t smem, cudaStream_t stream);
// dynamic shared memory of one CTA staging sh rows
size_t bp_smem(int sh, bool direct = false);
// The count-only form (fused_bp_kernel<1, ale, wide, false, true>): pixels
// with C < card_threshold per image into a.counters[image]; one staged buffer.
cudaError_t launch_bp_count_kernel(bool ale, bool wide, const CUtensorMap& map, const BpArgs& a, unsigned grid,
                                   size_t smem, cudaStream_t stream);
// the beta = 2 kernel (kernel_bp2.cuh), T <= 4; `direct`: the single-buffer
// T = 1 form that stores straight to HBM (wide regions, no peer mirrors)
cudaError_t launch_bp2_kernel(int T, bool ale, bool wide, bool direct, const CUtensorMap& map, const BpArgs& a,
                              unsigned grid, size_t smem, cudaStream_t stream);
size_t bp2_smem(int sh, bool direct = false);

}  // namespace phg
