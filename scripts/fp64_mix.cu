// Microbenchmark: can DFMA (FP64 pipe) and DMMA (FP64 tensor pipe) run concurrently
// on one SM?  Warps split by role inside one kernel; also one warp interleaving both.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_body(double (&a)[8], double b, double c) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
}
__device__ __forceinline__ void dmma_body(double (&d)[8][2], double a, double b) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[i][0]), "+d"(d[i][1])
                 : "d"(a), "d"(b));
}

// mode 0: all DFMA; 1: all DMMA; 2: even warps DFMA, odd warps DMMA; 3: each warp both
__global__ void k_mix(double* out, int iters, int mode) {
  double a[8], b = 1.0000001, c = 0.9999999;
  double d[8][2];
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 1e-3 + i;
    d[i][0] = d[i][1] = i;
  }
  const int warp = threadIdx.x >> 5;
  const bool do_f = mode == 0 || mode == 3 || (mode == 2 && !(warp & 1));
  const bool do_m = mode == 1 || mode == 3 || (mode == 2 && (warp & 1));
  for (int it = 0; it < iters; ++it) {
    if (do_f) {  // 64 DFMA per lane = the flops of 8 DMMA m8n8k4 per warp
#pragma unroll
      for (int r = 0; r < 8; ++r) dfma_body(a, b, c);
    }
    if (do_m) dmma_body(d, a[0] * 1e-30 + 1e-3, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 4, threads = 512;
  const char* names[4] = {"DFMA only", "DMMA only", "split warps", "both per warp"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      float ms;
      cudaEventRecord(e0);
      k_mix<<<blocks, threads>>>(out, iters, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)blocks * threads / 32;
      double ff = 0, fm = 0;
      const double per_f = 2.0 * 64 * iters * 32, per_m = 2.0 * 256 * 8 * iters;
      if (mode == 0) ff = warps * per_f;
      if (mode == 1) fm = warps * per_m;
      if (mode == 2) ff = warps / 2 * per_f, fm = warps / 2 * per_m;
      if (mode == 3) ff = warps * per_f, fm = warps * per_m;
      printf("%-14s %8.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", names[mode], ms,
             ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9);
    }
  return 0;
}
