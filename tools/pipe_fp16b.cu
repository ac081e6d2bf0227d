// Pipe-throughput probe: packed fp16 (FMA pipe) vs byte-SIMD integer (ALU pipe)
// ops on sm_100a, alone and interleaved 1:1 / 2:1.  Reports warp-lane ops per
// clock per SM (128 = full issue rate of the 4 SM sub-partitions).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_IT 2048
template <int O>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) {
  uint32_t r;
  if (O == 0) asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 1) asm volatile("fma.rn.f16x2 %0, %1, %2, %1;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 2) asm volatile("{.reg .b32 t; abs.f16x2 t, %1; sub.sat.f16x2 %0, %2, t;}" : "=r"(r) : "r"(a), "r"(b));
  if (O == 3) asm volatile("lop3.b32 %0, %1, %2, 0x7f7f7f7f, 0x6a;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 4) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 5) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 6) asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 7) r = __vabsdiffu4(a, b);
  if (O == 8) asm volatile("add.f32 %0, %1, %2;" : "=f"(*(float*)&r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)));
  if (O == 9) asm volatile("set.lt.f16x2.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 10) asm volatile("add.u32 %0, %1, %2; add.u32 %0, %0, %1;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 11) asm volatile("mad.hi.u32 %0, %1, 33554432, %2;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 12) { asm volatile("{.reg .b32 t; shr.u32 t, %1, 7; add.u32 %0, t, %2;}" : "=r"(r) : "r"(a), "r"(b)); }
  if (O == 13) asm volatile("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 14) asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(a), "r"(b));
  if (O == 15) asm volatile("dp4a.u32.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// pattern: ops O1 (n1 of them) then O2 (n2) per round, 8 independent chains
template <int O1, int N1, int O2, int N2>
__global__ void k(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t a[8], b = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 ^ (i * 0x00010001u) ^ threadIdx.x;
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int j = 0; j < N1; ++j) a[i] = op<O1>(a[i], b);
#pragma unroll
      for (int j = 0; j < N2; ++j) a[i] = op<O2>(a[i], b);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
const char* nm[] = {"HADD2", "HFMA2", "HADD2.SAT|abs|", "LOP3", "IADD", "PRMT", "HMNMX2", "VABSDIFF4", "FADD", "HSET2", "IADD3x3", "IMAD.HI", "LEA.HI", "SHF", "IMAD", "IDP4A"};
template <int O1, int N1, int O2, int N2> void run(uint32_t* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<O1, N1, O2, N2><<<148 * 8, 256>>>(d, 0x3c003c00u, 0x3c013c01u);
  cudaEventRecord(e0);
  k<O1, N1, O2, N2><<<148 * 8, 256>>>(d, 0x3c003c00u, 0x3c013c01u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * 8 * 256 * N_IT * 8 * (N1 + N2);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-16s x%d + %-16s x%d : %6.1f lane-ops/clk/SM (at %d MHz nominal)\n", nm[O1], N1, nm[O2], N2,
         ops / (ms * 1e-3 * clk * 1e3) / 148, clk / 1000);
}
int main() {
  uint32_t* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  run<4,1,4,1>(d); run<4,1,3,1>(d); run<4,1,7,1>(d); run<4,2,3,1>(d); run<4,2,7,1>(d); run<4,1,2,1>(d);
  run<11,1,11,1>(d); run<11,1,3,1>(d); run<11,1,7,1>(d); run<12,1,12,1>(d); run<12,1,11,1>(d);
  run<13,1,13,1>(d); run<13,1,2,1>(d); run<14,1,14,1>(d); run<14,1,3,1>(d); run<15,1,15,1>(d); run<15,1,3,1>(d);
  run<6,1,7,1>(d); run<6,1,2,1>(d); run<3,1,7,1>(d); run<2,1,11,1>(d); run<4,1,11,1>(d);
  return 0;
}
