// Microbenchmark: warp-instruction throughput of FFMA (3-reg), FFMA2, FADD2, FMUL2, DFMA per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void kern(float* out, int iters, float s) {
  float2 a[8], b = make_float2(s, s * 1.0001f), c = make_float2(1.0f - s, 0.5f);
  float x[8];
  double d[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.1f); x[i] = a[i].x; d[i] = x[i]; }
  float xb = b.x, xc = c.x;
  double db = b.x, dc = c.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) x[i] = fmaf(x[i], xb, xc);
      if (KIND == 1) a[i] = __ffma2_rn(a[i], b, c);
      if (KIND == 2) a[i] = __fadd2_rn(a[i], b);
      if (KIND == 3) a[i] = __fmul2_rn(a[i], b);
      if (KIND == 4) d[i] = fma(d[i], db, dc);
      if (KIND == 5) { a[i] = __ffma2_rn(a[i], b, c); x[i] = fmaf(x[i], xb, xc); }
      if (KIND == 6) { a[i] = __ffma2_rn(a[i], b, c); d[i] = fma(d[i], db, dc); }
      if (KIND == 7) { a[i] = __ffma2_rn(a[i], b, c); if (i & 1) d[i] = fma(d[i], db, dc); }
      if (KIND == 8) { a[i] = __ffma2_rn(a[i], b, c); if ((i & 3) == 0) d[i] = fma(d[i], db, dc); }
    }
  }
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += a[i].x + a[i].y + x[i] + (float)d[i];
  if (acc == 123.456f) out[0] = acc;
}
template <int KIND>
void run(const char* name, int per_iter) {
  float* out; cudaMalloc(&out, 4);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  kern<KIND><<<blocks, threads>>>(out, 16, 0.999f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<KIND><<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = double(blocks) * threads / 32 * iters * per_iter;
  double per_smsp_per_s = warp_instr / (148 * 4) / (ms * 1e-3);
  printf("%-10s %8.3f ms  %.3e warp-instr/s/SMSP  (=%.3f /clk at 1.9GHz)\n", name, ms, per_smsp_per_s, per_smsp_per_s / 1.9e9);
  cudaFree(out);
}
int main() {
  run<0>("FFMA", 8); run<1>("FFMA2", 8); run<2>("FADD2", 8); run<3>("FMUL2", 8); run<4>("DFMA", 8); run<5>("FFMA2+FFMA", 16); run<6>("FFMA2+DFMA", 16); run<7>("2FFMA2+DFMA", 12); run<8>("4FFMA2+DFMA", 10);
  return 0;
}
