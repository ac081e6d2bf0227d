// Throughput probe: which SM pipe executes the SWAR building blocks on sm_100a?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_IT 4096
template <int OP>
__global__ void k(uint32_t* out, uint32_t a0, uint32_t b0, uint32_t one) {
  uint32_t a[8], b = b0 + threadIdx.x;
  #pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 ^ (i * 0x01010101u) ^ threadIdx.x;
  for (int it = 0; it < N_IT; ++it) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = __vabsdiffu4(a[i], b);                                  // VABSDIFF4
      if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, 0x7f7f7f7f, 0x6a;" : "+r"(a[i]) : "r"(b)); // LOP3
      if (OP == 2) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));  // IMAD.HI
      if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(one), "r"(b)); // IMAD
      if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));         // IADD
      if (OP == 5) a[i] = __funnelshift_l(a[i], b, 8);                              // SHF
      if (OP == 6) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0xba98;" : "=r"(r) : "r"(a[i]), "r"(b)); a[i] = r; } // PRMT
      if (OP == 7) a[i] = __dp4a(a[i], b, a[i]);                                      // IDP.4A
      if (OP == 8) { a[i] = (a[i] >> 7) + b; }                                     // LEA.HI / SHF+ADD
      if (OP == 9) { a[i] = __popc(a[i]) + b; }                                    // POPC
    }
  }
  uint32_t s = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> float run(uint32_t* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<OP><<<148 * 8, 256>>>(d, 1, 2, 1);
  cudaEventRecord(e0);
  k<OP><<<148 * 8, 256>>>(d, 1, 2, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * 8 * 256 * N_IT * 8;  // thread-ops
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("op %d: %.3f ms  -> %.1f thread-ops/clk/SM\n", OP, ms, ops / cyc / 148);
  return ms;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  const char* names[] = {"VABSDIFF4","LOP3","IMAD.HI","IMAD","IADD","SHF","PRMT","IDP4A","shr+add","POPC+add"};
  run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d); run<5>(d); run<6>(d); run<7>(d); run<8>(d); run<9>(d);
  for (int i = 0; i < 10; ++i) printf("%d=%s ", i, names[i]); printf("\n");
  return 0;
}
