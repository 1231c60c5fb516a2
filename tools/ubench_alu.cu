// Micro-benchmark: per-SM throughput of the integer instructions the pair test uses.
// Each thread runs 8 independent dependency chains; result = lane-ops / clk / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
template <int OP>
__global__ void kern(uint32_t* out, uint32_t p, uint32_t q, int iters) {
  uint32_t v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 7 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) v[c] = __viaddmin_s16x2(v[c], p, q);
      if (OP == 1) v[c] = __vimin_s16x2_relu(v[c], p);
      if (OP == 2) v[c] = v[c] & p & q;          // LOP3
      if (OP == 3) v[c] = __umulhi(v[c], p) + q; // IMAD.HI with addend
      if (OP == 4) v[c] = v[c] * p + q;          // IMAD
      if (OP == 5) v[c] = min(v[c], p) ;         // IMNMX
      if (OP == 6) v[c] = v[c] + p + q;          // IADD3
      if (OP == 7) { v[c] = __viaddmin_s16x2(v[c], p, q); v[c] = v[c] * p + q; }  // alu+fma mix
      if (OP == 8) { v[c] = __viaddmin_s16x2(v[c], p, q); v[c] = __viaddmin_s16x2_relu(v[c], q, p); v[c] = __vimin_s16x2_relu(v[c], p); v[c] = v[c] * p + q; v[c] = __umulhi(v[c], q) + p; }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
void run(const char* name, int ops_per_iter, uint32_t* out, int sms, int clk_khz) {
  const int iters = 4096, threads = 256, blocks = sms * 8;
  kern<OP><<<blocks, threads>>>(out, 0x00050003u, 0x00070009u, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(out, 0x00050003u, 0x00070009u, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double lane_ops = (double)blocks * threads * iters * CHAINS * ops_per_iter;
  double cycles = ms * 1e-3 * clk_khz * 1e3;
  printf("%-28s %8.3f ms  %7.2f lane-ops/clk/SM (at %d MHz)\n", name, ms, lane_ops / cycles / sms, clk_khz / 1000);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; cudaMalloc(&out, (size_t)p.multiProcessorCount * 8 * 256 * 4);
  run<0>("VIADDMNMX.S16x2", 1, out, p.multiProcessorCount, clk);
  run<1>("VIMNMX.S16x2.RELU", 1, out, p.multiProcessorCount, clk);
  run<2>("LOP3", 1, out, p.multiProcessorCount, clk);
  run<3>("IMAD.HI(+addend)", 1, out, p.multiProcessorCount, clk);
  run<4>("IMAD", 1, out, p.multiProcessorCount, clk);
  run<5>("IMNMX", 1, out, p.multiProcessorCount, clk);
  run<6>("IADD3", 1, out, p.multiProcessorCount, clk);
  run<7>("VIADDMNMX+IMAD", 2, out, p.multiProcessorCount, clk);
  run<8>("3xVI + IMAD + IMAD.HI", 5, out, p.multiProcessorCount, clk);
  return 0;
}
