// Microbenchmark of the M2L inner loop shape (scripts/, not part of libtb):
// each thread keeps T targets x 16 accumulators, and per "pair" loads 16
// source moments (shared by the T targets) and T x 20 tensor values from
// shared memory, then does T x 70 FMAs. Reports DFMA/s against the 64/clk/SM
// peak for T = 1, 2 at 512 / 256 threads per CTA, and a register-only
// variant (no shared loads) to separate operand delivery from the FMA issue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_contract.cu -o probe_contract
#include <cstdio>
#include <cuda_runtime.h>

template <int T, bool SMEM>
__global__ void k(double *sink, int iters) {
  __shared__ double M[64 * 16];
  __shared__ double D[64 * 20];
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) M[i] = 1e-3 * i;
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) D[i] = 1e-4 * i;
  __syncthreads();
  double L[T][16];
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int k = 0; k < 16; ++k) L[t][k] = 0.0;
  const int lane = threadIdx.x & 31;
  double m[16], d[T][20];
#pragma unroll
  for (int k = 0; k < 16; ++k) m[k] = 1.0 + k * 1e-3;
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int k = 0; k < 20; ++k) d[t][k] = 1.0 + (k + t) * 1e-4;
  for (int it = 0; it < iters; ++it) {
    if (SMEM) {
      const int mo = ((it + (lane >> 3)) & 63) * 16, dof = ((it + lane) & 63) * 20;
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        const double2 a = *reinterpret_cast<const double2 *>(M + mo + k);
        m[k] = a.x;
        m[k + 1] = a.y;
      }
#pragma unroll
      for (int t = 0; t < T; ++t)
#pragma unroll
        for (int k = 0; k < 20; k += 2) {
          const double2 a = *reinterpret_cast<const double2 *>(D + ((dof + 20 * t) & 1279) + k);
          d[t][k] = a.x;
          d[t][k + 1] = a.y;
        }
    }
    // 70 FMAs per target: every accumulator gets ~4-5 terms (the M2L mix)
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int s = 0; s < 16; ++s)
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if ((s * 7 + q * 3) % 16 < 4 + (s < 6 ? 1 : 0) && (s + q) % 1 == 0)
            L[t][q] = fma(m[s], d[t][(s + q) % 20], L[t][q]);
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += L[t][k];
  if (acc == 12345.0) sink[threadIdx.x] = acc;
}

template <int T, bool SMEM>
void run(int threads, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<T, SMEM>, threads, 0);
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, k<T, SMEM>);
  double *sink;
  cudaMalloc(&sink, 8 * 1024);
  const int blocks = sms * occ;
  k<T, SMEM><<<blocks, threads>>>(sink, iters / 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<T, SMEM><<<blocks, threads>>>(sink, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  // count FMAs per iteration per thread (same predicate as the kernel)
  int per = 0;
  for (int s = 0; s < 16; ++s)
    for (int q = 0; q < 16; ++q)
      if ((s * 7 + q * 3) % 16 < 4 + (s < 6 ? 1 : 0)) ++per;
  const double fmas = (double)blocks * threads * iters * per * T;
  const double rate = fmas / (ms * 1e-3);
  printf("{\"T\": %d, \"smem\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"regs\": %d, "
         "\"fma_per_pair\": %d, \"dfma_per_s\": %.4g, \"frac_of_64_per_clk_at_1965\": %.3f}\n",
         T, (int)SMEM, threads, occ, at.numRegs, per, rate, rate / (64.0 * sms * 1.965e9));
  cudaFree(sink);
}

int main() {
  run<1, true>(512, 4000);
  run<1, true>(256, 4000);
  run<2, true>(256, 4000);
  run<2, true>(512, 4000);
  run<1, false>(512, 4000);
  run<2, false>(256, 4000);
  return 0;
}
