// tb_star.cu — the coupled rotating-star step (north_star "full rotating-star
// step"): hydro (K6) + FMM gravity (K7) + a second-order Runge-Kutta update,
// device-resident on a global lattice, dt from the CFL condition on device
// (no host round trip inside a step).
//
// PARITY UNPINNED (the reference has no physics); the spec is
// oracle/star_oracle.py. The update arithmetic below is restated operation by
// operation (no FMA), so the only difference from the oracle is the FMM's
// (<= 1e-10 relative, see tb_fmm.cu).
//
// State: U [5][N][N][N] (rho, sx, sy, sz, E; z,y,x, x fastest), periodic hydro
// boundary, isolated gravity.
//   k_star_pad    U -> Up [5][N+4]^3 (periodic 2-cell ghost layer) for the
//                 hydro kernel's 4-D TMA boxes.
//   k_star_cfl    dt = cfl * dx / max_s amax[s] (one CTA), written on device.
//   k_star_stage  L(U) = dU/dt_hydro + (0, rho g, s.g);
//                 stage 1: U1 = U + dt L(U);  stage 2: U' = 0.5 (U + (U1 + dt L(U1))).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace {

constexpr int NF = 5, NG = 2;

// U [5][nz][n][n] (a slab, or the whole lattice) -> Up [5][nz+4][n+4][n+4]:
// x, y wrap periodically inside the slab; z takes the 2 planes below / above
// from lo / hi ([5][2][n][n], the z-neighbours' planes) or, when they are
// null (one device), wraps inside the slab.
// One warp per padded row (f, z, y): the source row is resolved once, then
// the row is copied as 16-byte pairs — the shift by NG = 2 cells keeps both
// sides 16-byte aligned (n even, rows of n + 4 doubles): pair 0 is the left
// ghost pair (cells n-2, n-1), pairs 1..n/2 the row, pair n/2+1 the right
// ghost pair (cells 0, 1).
__global__ void __launch_bounds__(256) k_star_pad(const double *__restrict__ U,
                                                  const double *__restrict__ lo,
                                                  const double *__restrict__ hi,
                                                  double *__restrict__ Up, int n, int nz) {
  const int P = n + 2 * NG, Pz = nz + 2 * NG;
  const int64_t plane = (int64_t)n * n;
  const int64_t rows = (int64_t)NF * Pz * P;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int pairs = n / 2 + 2;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const int y = (int)(row % P), z = (int)((row / P) % Pz), f = (int)(row / ((int64_t)P * Pz));
    const int sy = (y - NG + n) % n, zl = z - NG;
    const double *src;
    if (zl >= 0 && zl < nz)
      src = U + ((int64_t)f * nz + zl) * plane;
    else if (!lo)
      src = U + ((int64_t)f * nz + (zl + nz) % nz) * plane;
    else if (zl < 0)
      src = lo + ((int64_t)f * NG + (zl + NG)) * plane;
    else
      src = hi + ((int64_t)f * NG + (zl - nz)) * plane;
    const double2 *s2 = reinterpret_cast<const double2 *>(src + (int64_t)sy * n);
    double2 *d2 = reinterpret_cast<double2 *>(Up + row * P);
    for (int j0 = 0; j0 < pairs; j0 += 4 * 32) {   // 4 loads in flight per lane
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * 32 + lane;
        const int k = j == 0 ? n / 2 - 1 : (j == pairs - 1 ? 0 : j - 1);
        if (j < pairs) v[u] = __ldg(s2 + k);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * 32 + lane;
        if (j < pairs) d2[j] = v[u];
      }
    }
  }
}

// max that propagates NaN (numpy's np.maximum / amax.max(), which the spec's
// dt follows): a sub-grid that blew up makes dt NaN instead of being skipped
__device__ __forceinline__ double max_nan(double a, double b) {
  return (a != a || a > b) ? a : b;
}

__global__ void __launch_bounds__(1024) k_star_cfl(const double *__restrict__ amax, int64_t nsub,
                                                   double dx, double cfl,
                                                   double *__restrict__ dt) {
  __shared__ double part[32];
  double m = -CUDART_INF;
  for (int64_t i = threadIdx.x; i < nsub; i += blockDim.x) m = max_nan(m, amax[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : -CUDART_INF;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *dt = __ddiv_rn(__dmul_rn(cfl, dx), m);
  }
}

// One RK stage per cell. dudt is in sub-grid layout [S][5][8][8][8]
// (the hydro kernel's output), g = the FMM output's force rows [3][N^3].
template <int STAGE>
__global__ void __launch_bounds__(256) k_star_stage(const double *__restrict__ U0,
                                                    const double *__restrict__ Uc,
                                                    const double *__restrict__ dudt,
                                                    const double *__restrict__ g,
                                                    const double *__restrict__ dtp, int n,
                                                    int nz, double *__restrict__ Unew) {
  const int64_t ncell = (int64_t)n * n * nz;   // this slab's cells
  const int nb = n / 8;
  const double dt = *dtp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % n), y = (int)((i / n) % n), z = (int)(i / ((int64_t)n * n));
    const int64_t sub = ((int64_t)(z >> 3) * nb + (y >> 3)) * nb + (x >> 3);
    const int64_t loc = ((z & 7) * 8 + (y & 7)) * 8 + (x & 7);
    const double *du = dudt + sub * (NF * 512) + loc;
    const double gx = g[i], gy = g[ncell + i], gz = g[2 * ncell + i];
    double u[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) u[f] = Uc[f * ncell + i];
    double L[NF];
    L[0] = du[0];
    L[1] = __dadd_rn(du[512], __dmul_rn(u[0], gx));
    L[2] = __dadd_rn(du[2 * 512], __dmul_rn(u[0], gy));
    L[3] = __dadd_rn(du[3 * 512], __dmul_rn(u[0], gz));
    L[4] = __dadd_rn(du[4 * 512],
                     __dadd_rn(__dadd_rn(__dmul_rn(u[1], gx), __dmul_rn(u[2], gy)),
                               __dmul_rn(u[3], gz)));
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const double v = __dadd_rn(u[f], __dmul_rn(dt, L[f]));
      Unew[f * ncell + i] = STAGE == 1 ? v : __dmul_rn(0.5, __dadd_rn(U0[f * ncell + i], v));
    }
  }
}

inline cudaStream_t strm(tb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t n, int threads) {
  const int64_t cap = (int64_t)tb::sm_count() * 8;
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < cap ? b : cap);
}

}  // namespace

extern "C" {

int tb_star_pad_slab(tb_stream_t s, const double *U, int64_t n, int64_t nz, const double *lo,
                     const double *hi, double *Up) {
  if (!U || !Up || n < 8 || n % 8 || nz < 8 || nz % 8 || (!lo != !hi)) return TB_E_INVALID;
  const int64_t P = n + 2 * NG, Pz = nz + 2 * NG;
  k_star_pad<<<grid_for(NF * P * Pz * 32, 256), 256, 0, strm(s)>>>(U, lo, hi, Up, (int)n,
                                                                   (int)nz);
  return tb::last_error();
}

int tb_star_pad(tb_stream_t s, const double *U, int64_t n, double *Up) {
  return tb_star_pad_slab(s, U, n, n, nullptr, nullptr, Up);
}

int tb_star_cfl(tb_stream_t s, const double *amax, int64_t nsub, double dx, double cfl,
                double *dt) {
  if (!amax || !dt || nsub <= 0 || !(dx > 0.0) || !(cfl > 0.0)) return TB_E_INVALID;
  k_star_cfl<<<1, 1024, 0, strm(s)>>>(amax, nsub, dx, cfl, dt);
  return tb::last_error();
}

int tb_star_stage(tb_stream_t s, int stage, const double *U0, const double *Uc,
                  const double *dudt, const double *g, const double *dt, int64_t n, int64_t nz,
                  double *Unew) {
  if (!Uc || !dudt || !g || !dt || !Unew || n < 8 || n % 8 || nz < 8 || nz % 8 ||
      (stage != 1 && stage != 2) || (stage == 2 && !U0))
    return TB_E_INVALID;
  const int64_t cells = n * n * nz;
  if (stage == 1)
    k_star_stage<1><<<grid_for(cells, 256), 256, 0, strm(s)>>>(U0, Uc, dudt, g, dt, (int)n,
                                                                (int)nz, Unew);
  else
    k_star_stage<2><<<grid_for(cells, 256), 256, 0, strm(s)>>>(U0, Uc, dudt, g, dt, (int)n,
                                                                (int)nz, Unew);
  return tb::last_error();
}

}  // extern "C"
