// FP64 tensor-core (DMMA) issue-rate probe (scripts/, not part of libtb):
// mma.sync.aligned.m8n8k4.row.col.f64 in a dependent-free loop, 8 independent
// accumulator tiles per warp, all operands in registers. Prints the achieved
// FP64 FMA rate against the DFMA peak measured by tb_fp64_probe, to decide
// whether FP64 tensor cores can help the FMM kernels on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int TILES>
__global__ void k(double *sink, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(c[t][0]), "+d"(c[t][1])
          : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

// The leaf-kernel shape: per K-chunk one B element and, for each of G row
// groups, one A element per lane read from shared memory, then G DMMAs.
template <int G>
__global__ void k_smem(double *sink, int iters) {
  __shared__ double A[4096], B[1024];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) A[i] = 1e-3 * i;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) B[i] = 1e-4 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double c[G][2];
#pragma unroll
  for (int g = 0; g < G; ++g) c[g][0] = c[g][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double b = B[((it & 31) * 32 + lane) & 1023];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double a = A[((it * 7 + g * 128 + w * 512) + (lane >> 2) + 24 * (lane & 3)) & 4095];
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(c[g][0]), "+d"(c[g][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < G; ++g) s += c[g][0] + c[g][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

// Pipe sharing: warps with MODE bit 0 run DMMA tiles, warps with bit 1 run
// 8 independent DFMA chains; MODE 3 = half the warps each (warp parity).
template <int MODE>
__global__ void k_mix(double *sink, int iters) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool do_mma = MODE == 1 || (MODE == 3 && (w & 1) == 0);
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 1e-3 * t;
  if (do_mma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
            : "+d"(c[t][0]), "+d"(c[t][1])
            : "d"(a), "d"(b));
    }
  } else {
    // 8 DFMAs per DMMA-equivalent step keep the instruction counts comparable
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int t = 0; t < 8; ++t) c[t][0] = fma(c[t][0], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *sink;
  cudaMalloc(&sink, 8 * 1024);
  const int iters = 20000;
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (1024 / threads);
    k<8><<<blocks, threads>>>(sink, iters / 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<8><<<blocks, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 256 FMAs per warp
    const double fmas = (double)blocks * (threads / 32) * iters * 8 * 256;
    printf("{\"threads\": %d, \"blocks\": %d, \"dmma_fma_per_s\": %.4g, \"err\": \"%s\"}\n",
           threads, blocks, fmas / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  }
  for (int threads : {256, 512}) {
    const int blocks = sms;   // one CTA per SM, like a 110 KB-staged leaf CTA
    k_smem<4><<<blocks, threads>>>(sink, iters / 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_smem<4><<<blocks, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)blocks * (threads / 32) * iters * 4 * 256;
    printf("{\"smem_operands\": 1, \"threads\": %d, \"dmma_fma_per_s\": %.4g}\n", threads,
           fmas / (ms * 1e-3));
  }
  // pipe sharing: DMMA-only, DFMA-only and mixed at the same warp count;
  // FMA rates per kind (a DMMA = 256 FMAs per warp, a DFMA = 32)
  {
    const int threads = 512, blocks = sms * 2, it = iters / 4;
    auto run = [&](void (*kern)(double *, int)) {
      kern<<<blocks, threads>>>(sink, it / 10);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(sink, it);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      return ms * 1e-3;
    };
    const double warps = (double)blocks * threads / 32;
    const double per_warp = (double)it * 8 * 256;   // FMAs per warp in either mode
    const double t1 = run(k_mix<1>), t2 = run(k_mix<2>), t3 = run(k_mix<3>);
    printf("{\"pipe_sharing\": 1, \"dmma_only_fma_per_s\": %.4g, \"dfma_only_fma_per_s\": %.4g, "
           "\"mixed_total_fma_per_s\": %.4g, \"mixed_s\": %.4g, \"dmma_only_s\": %.4g, "
           "\"dfma_only_s\": %.4g}\n",
           warps * per_warp / t1, warps * per_warp / t2, warps * per_warp / t3, t3, t1, t2);
  }
  return 0;
}
