#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1306_5390_b200/csrc/kernels.cuh"
using namespace phg;
__global__ void k_param(const __grid_constant__ CUtensorMap m, uint8_t* out, int bytes, int x, int y) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_expect_tx(&bar, bytes); tma_load_3d(smem, &m, x, y, 0, &bar); }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}
__global__ void k_gmem(const CUtensorMap* m, uint8_t* out, int bytes, int x, int y) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_expect_tx(&bar, bytes); tma_load_3d(smem, m, x, y, 0, &bar); }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s -> %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  int W=7, H=7, pitch=16;
  uint8_t* d; CK(cudaMalloc(&d, 4096)); CK(cudaMemset(d, 7, 4096));
  uint8_t* o; CK(cudaMalloc(&o, 1<<20));
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t str[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch*H};
  int sh = 17;
  cuuint32_t box[3] = {256, (cuuint32_t)sh, 1}, es[3] = {1,1,1};
  if (mode & 1) { box[0] = 64; }
  if (mode & 2) { str[1] = 4096; }
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, (mode & 4) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = box[0]*box[1];
  printf("mode %d enc=%d bytes=%d\n", mode, (int)r, bytes);
  CK(cudaFuncSetAttribute(k_param, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  CK(cudaFuncSetAttribute(k_gmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  if (mode & 8) {
    CUtensorMap* dm; CK(cudaMalloc(&dm, sizeof(m))); CK(cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice));
    k_gmem<<<1, 128, 65536>>>(dm, o, bytes, (mode & 16) ? 0 : -8, (mode & 16) ? 0 : -5);
  } else {
    k_param<<<1, 128, 65536>>>(m, o, bytes, atoi(argv[2]), atoi(argv[3]));
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  uint8_t h[64]; CK(cudaMemcpy(h, o + 5*box[0], 64, cudaMemcpyDeviceToHost));
  for (int i = 0; i < 20; ++i) printf("%d ", h[i]); printf("\n");
  return 0;
}
