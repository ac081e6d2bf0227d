// bp2.cu -- instantiations of fused_bp2_kernel (kernel_bp2.cuh, beta = 2),
// compiled as their own translation unit so the library builds in parallel.
#include <cuda.h>
#include <cuda_runtime.h>

#include "bp_launch.h"
#include "kernel_bp2.cuh"

namespace phg {

namespace {

using BpFn = void (*)(const CUtensorMap, const BpArgs);

template <int T>
BpFn pick2(bool ale, bool wide) {
    if (wide) return ale ? fused_bp2_kernel<T, true, true> : fused_bp2_kernel<T, false, true>;
    return ale ? fused_bp2_kernel<T, true, false> : fused_bp2_kernel<T, false, false>;
}

BpFn select2(int T, bool ale, bool wide, bool direct) {
    if (direct) {
        if (T != 1 || !wide) return nullptr;
        return ale ? fused_bp2_kernel<1, true, true, true> : fused_bp2_kernel<1, false, true, true>;
    }
    switch (T) {
        case 1: return pick2<1>(ale, wide);
        case 2: return pick2<2>(ale, wide);
        case 3: return pick2<3>(ale, wide);
        case 4: return pick2<4>(ale, wide);
        default: return nullptr;
    }
}

}  // namespace

cudaError_t launch_bp2_kernel(int T, bool ale, bool wide, bool direct, const CUtensorMap& map, const BpArgs& a,
                              unsigned grid, size_t smem, cudaStream_t stream) {
    BpFn fn = select2(T, ale, wide, direct);
    if (!fn) return cudaErrorInvalidValue;
    const size_t cap = direct ? bp2_smem(kBp2DirectMaxRows, true) : bp2_smem(kBp2MaxRows);
    if (smem > cap) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap));
    if (e != cudaSuccess) return e;
    fn<<<grid, kBpThreads, smem, stream>>>(map, a);
    return cudaGetLastError();
}

size_t bp2_smem(int sh, bool direct) { return static_cast<size_t>(bp2_smem_bytes(sh, direct)); }

}  // namespace phg
