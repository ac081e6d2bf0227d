#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_IT 4096
__device__ __forceinline__ uint32_t op(int o, uint32_t a, uint32_t b, uint32_t one) {
  uint32_t r;
  switch (o) {
    case 0: return __vabsdiffu4(a, b);
    case 1: asm volatile("lop3.b32 %0, %1, %2, 0x7f7f7f7f, 0x6a;" : "=r"(r) : "r"(a), "r"(b)); return r;
    case 2: asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b)); return r;
    case 3: return __funnelshift_l(a, b, 8);
    case 4: asm volatile("prmt.b32 %0, %1, %2, 0xba98;" : "=r"(r) : "r"(a), "r"(b)); return r;
    case 5: return __dp4a(a, b, a);
    case 6: asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
  return a;
}
template <int O1, int O2>
__global__ void k(uint32_t* out, uint32_t a0, uint32_t b0, uint32_t one) {
  uint32_t a[8], b = b0 + threadIdx.x;
  #pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 ^ (i * 0x01010101u) ^ threadIdx.x;
  for (int it = 0; it < N_IT; ++it) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (i & 1) ? op(O2, a[i], b, one) : op(O1, a[i], b, one);
  }
  uint32_t s = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
const char* nm[] = {"VABS", "LOP3", "IMAD", "SHF", "PRMT", "IDP", "IADD"};
template <int O1, int O2> void run(uint32_t* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<O1, O2><<<148 * 8, 256>>>(d, 1, 2, 1);
  cudaEventRecord(e0);
  k<O1, O2><<<148 * 8, 256>>>(d, 1, 2, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * 8 * 256 * N_IT * 8;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s+%s: %.1f thread-ops/clk/SM\n", nm[O1], nm[O2], ops / (ms * 1e-3 * clk * 1e3) / 148);
}
int main() {
  uint32_t* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  run<0,1>(d); run<0,2>(d); run<1,2>(d); run<3,2>(d); run<4,2>(d); run<5,1>(d); run<5,2>(d); run<0,5>(d);
  run<0,3>(d); run<1,3>(d); run<0,4>(d); run<1,4>(d); run<6,1>(d); run<6,0>(d); run<6,2>(d); run<6,5>(d);
  return 0;
}
