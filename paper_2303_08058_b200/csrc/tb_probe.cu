// tb_probe.cu — FP64 issue-rate microbenchmark: the denominator of the FP64
// half of every roofline in DESIGN.md (MEASURED_PEAKS.json carries only HBM
// and bf16 numbers). Each thread runs 8 independent dependency chains of one
// FP64 instruction type so latency is hidden; the grid fills every SM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace {

constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(256) k_fp64_probe(double *sink, int64_t iters, double a,
                                                    double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = a + 1e-3 * (threadIdx.x + c);
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == TB_PROBE_DADD) {
        x[c] = __dadd_rn(x[c], b);
      } else if (OP == TB_PROBE_DMUL) {
        x[c] = __dmul_rn(x[c], a);
      } else if (OP == TB_PROBE_DFMA) {
        x[c] = __fma_rn(x[c], a, b);
      } else {  // DMUL then DADD, the K2 transform pair (2 instructions)
        x[c] = __dadd_rn(__dmul_rn(x[c], a), b);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) sink[threadIdx.x] = s;   // never true; keeps the chains live
}

// the fast paths with the intrinsic fallback where they flag, as K6 uses them
__global__ void k_divsqrt_fast(const double *a, const double *b, int64_t n, double *q_out,
                               double *r_out, unsigned long long *slow_count) {
  unsigned long long slow = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool okd = true, oks = true;
    double q = tb::div_rn_fast(a[i], b[i], okd);
    double r = tb::sqrt_rn_fast(a[i], oks);
    slow += !okd;
    slow += !oks;
    if (!okd) q = __ddiv_rn(a[i], b[i]);
    if (!oks) r = __dsqrt_rn(a[i]);
    q_out[i] = q;
    r_out[i] = r;
  }
  atomicAdd(slow_count, slow);
}

}  // namespace

extern "C" int tb_divsqrt_fast(tb_stream_t s, const double *a, const double *b, int64_t n,
                               double *q, double *r, unsigned long long *slow_count) {
  if (n < 0 || (n > 0 && (!a || !b || !q || !r)) || !slow_count) return TB_E_INVALID;
  if (n == 0) return TB_OK;
  k_divsqrt_fast<<<tb::sm_count() * 8, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      a, b, n, q, r, slow_count);
  return tb::last_error();
}

extern "C" int tb_fp64_probe(int op, int64_t iters, double *instr_per_s, double *sm_mhz) {
  if (!instr_per_s || iters <= 0 || op < TB_PROBE_DADD || op > TB_PROBE_DMUL_DADD)
    return TB_E_INVALID;
  int dev = 0, occ = 0;
  cudaGetDevice(&dev);
  const int sms = tb::sm_count();
  void (*kern)(double *, int64_t, double, double) =
      op == TB_PROBE_DADD   ? k_fp64_probe<TB_PROBE_DADD>
      : op == TB_PROBE_DMUL ? k_fp64_probe<TB_PROBE_DMUL>
      : op == TB_PROBE_DFMA ? k_fp64_probe<TB_PROBE_DFMA>
                            : k_fp64_probe<TB_PROBE_DMUL_DADD>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (occ < 1) occ = 1;
  const int blocks = sms * occ;
  double *sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess) return tb::last_error();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 256>>>(sink, iters / 8 + 1, 1.0000001, 1e-9);   // warm-up / clocks up
  cudaEventRecord(e0);
  kern<<<blocks, 256>>>(sink, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  int rc = tb::rc(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per_iter = (op == TB_PROBE_DMUL_DADD ? 2.0 : 1.0) * kChains;
  *instr_per_s = (double)blocks * 256.0 * (double)iters * per_iter / (ms * 1e-3);
  if (sm_mhz) {
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    *sm_mhz = khz / 1000.0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return rc;
}
