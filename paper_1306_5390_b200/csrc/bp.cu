// bp.cu -- instantiations of fused_bp_kernel (kernel_bp.cuh, beta = 1),
// compiled as their own translation unit so the library builds in parallel.
#include <cuda.h>
#include <cuda_runtime.h>

#include "bp_launch.h"
#include "kernel_bp.cuh"

namespace phg {

namespace {

using BpFn = void (*)(const CUtensorMap, const BpArgs);

template <int T>
BpFn pick(bool ale, bool wide) {
    if (wide) return ale ? fused_bp_kernel<T, true, true> : fused_bp_kernel<T, false, true>;
    return ale ? fused_bp_kernel<T, true, false> : fused_bp_kernel<T, false, false>;
}

BpFn select(int T, bool ale, bool wide, bool direct) {
    if (direct) {
        if (T != 1 || !wide) return nullptr;
        return ale ? fused_bp_kernel<1, true, true, true> : fused_bp_kernel<1, false, true, true>;
    }
    switch (T) {
        case 1: return pick<1>(ale, wide);
        case 2: return pick<2>(ale, wide);
        case 3: return pick<3>(ale, wide);
        case 4: return pick<4>(ale, wide);
        case 5: return pick<5>(ale, wide);
        default: return nullptr;
    }
}

}  // namespace


cudaError_t launch_bp_kernel(int T, bool ale, bool wide, bool direct, const CUtensorMap& map, const BpArgs& a,
                             unsigned grid, size_t smem, cudaStream_t stream) {
    BpFn fn = select(T, ale, wide, direct);
    if (!fn) return cudaErrorInvalidValue;
    // always the largest tile's size: concurrent callers with different tile
    // heights must never lower the limit under another caller's launch
    const size_t cap = direct ? bp_smem(kBpDirectMaxRows, true) : bp_smem(kBpMaxRows);
    if (smem > cap) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap));
    if (e != cudaSuccess) return e;
    fn<<<grid, kBpThreads, smem, stream>>>(map, a);
    return cudaGetLastError();
}

size_t bp_smem(int sh, bool direct) { return static_cast<size_t>(bp_smem_bytes(sh, direct)); }

cudaError_t launch_bp_count_kernel(bool ale, bool wide, const CUtensorMap& map, const BpArgs& a, unsigned grid,
                                   size_t smem, cudaStream_t stream) {
    BpFn fn = wide ? (ale ? fused_bp_kernel<1, true, true, false, true> : fused_bp_kernel<1, false, true, false, true>)
                   : (ale ? fused_bp_kernel<1, true, false, false, true> : fused_bp_kernel<1, false, false, false, true>);
    const size_t cap = bp_smem(kBpDirectMaxRows, true);
    if (smem > cap) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap));
    if (e != cudaSuccess) return e;
    fn<<<grid, kBpThreads, smem, stream>>>(map, a);
    return cudaGetLastError();
}

}  // namespace phg
