// tb_hydro.cu — K6: hydro reconstruct-and-flux over a batch of octree leaf
// sub-grids (8^3 interior cells + 2-cell ghost layers, 5 conserved FP64
// fields in SoA), the north_star's "hydro reconstruct+flux only" kernel.
//
// PARITY UNPINNED (no hydro in the reference): the
// arithmetic is the self-authored spec in oracle/hydro_oracle.py, restated
// operation by operation (no FMA) so the GPU is bit-identical to it.
//
// Per CTA and sub-grid: one bulk copy (TMA engine, mbarrier completion)
// stages the 69,120-byte ghosted sub-grid in shared memory; conserved ->
// primitive in place; for each direction the 576 face fluxes (minmod PLM +
// Kurganov-Tadmor/LLF) go to a shared flux buffer and every thread folds the
// flux differences of its interior cells into registers; dU/dt is written
// coalesced and the sub-grid's max signal speed is block-reduced.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <type_traits>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace {

constexpr int NG = 2, NI = 8, NT = 12, NF = 5;
constexpr int NCELL = NT * NT * NT;            // 1728
constexpr int NFACE = (NI + 1) * NI * NI;      // 576 faces per direction
// threads per CTA: 256, or 320 with TB_HYDRO_VARIANT bit 4
constexpr int threads_of(int v) { return (v & 16) ? 320 : 256; }
constexpr int kDefaultVariant = 1532;
constexpr int kSmem = (NF * NCELL + 2 * NF * NFACE) * 8;   // 115,200 B (2 CTAs/SM)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bit 9 (probe only): per-CTA %globaltimer stamps — entry, first sub-grid
// staged, last sub-grid's faces done, exit — for the launch's head and tail
// (tb_hydro_stamps; scripts/k6_stamps_probe.py)
constexpr int kStampCtas = 1024;
__device__ unsigned long long g_k6_stamps[kStampCtas][4];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// bit 10's work counters: [slot][next sub-grid, finished CTAs], zero at
// module load and reset by each launch's last CTA; a launch takes the next
// slot of the ring, so launches on concurrent streams (the machine's
// executors) do not share one
constexpr unsigned kWorkSlots = 4096;
__device__ unsigned int g_k6_work[kWorkSlots][2];
std::atomic<unsigned> g_work_next{0};

struct State {
  double u[NF], f[NF], a;
};

// Left/right state -> conserved vector, flux along d, signal speed |vn|+cs.
template <bool FAST>
__device__ __forceinline__ void face_state(double rho, double vx, double vy, double vz,
                                           double p, double gamma, double igm1, int d,
                                           State &s, bool &ok) {
  double cs;
  if constexpr (FAST)
    cs = tb::sqrt_rn_fast(tb::div_rn_fast(__dmul_rn(gamma, p), rho, ok), ok);
  else
    cs = __dsqrt_rn(__ddiv_rn(__dmul_rn(gamma, p), rho));
  const double vv = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)),
                              __dmul_rn(vz, vz));
  const double e = __dadd_rn(__dmul_rn(p, igm1), __dmul_rn(__dmul_rn(0.5, rho), vv));
  const double vn = d == 0 ? vx : (d == 1 ? vy : vz);
  const double mx = __dmul_rn(rho, vx), my = __dmul_rn(rho, vy), mz = __dmul_rn(rho, vz);
  s.u[0] = rho;
  s.u[1] = mx;
  s.u[2] = my;
  s.u[3] = mz;
  s.u[4] = e;
  double fmx = __dmul_rn(mx, vn), fmy = __dmul_rn(my, vn), fmz = __dmul_rn(mz, vn);
  if (d == 0)
    fmx = __dadd_rn(fmx, p);
  else if (d == 1)
    fmy = __dadd_rn(fmy, p);
  else
    fmz = __dadd_rn(fmz, p);
  s.f[0] = __dmul_rn(rho, vn);
  s.f[1] = fmx;
  s.f[2] = fmy;
  s.f[3] = fmz;
  s.f[4] = __dmul_rn(__dadd_rn(e, p), vn);
  s.a = __dadd_rn(fabs(vn), cs);
}

__device__ __forceinline__ double minmod(double dl, double dr) {
  const double pick = fabs(dl) < fabs(dr) ? dl : dr;
  return __dmul_rn(dl, dr) <= 0.0 ? 0.0 : pick;
}

// N consecutive faces c0 .. c0+N-1 of the line (ti, tj) along d: the N+3
// cells they read per field are loaded once and each interior slope is formed
// once for the two faces that use it. Face c lies between 12-grid cells c+1
// and c+2 along d; its flux goes to Fb at a fixed (slow transverse, fast
// transverse, face) layout per d.
template <int N, bool FAST>
__device__ __forceinline__ void face_segment_impl(const double *W, double *Fb, int d, int stride,
                                                  int ti, int tj, int c0, double gamma,
                                                  double igm1, double &amax, bool &ok) {
  int base;
  if (d == 0)
    base = ((NG + tj) * NT + (NG + ti)) * NT + c0;
  else if (d == 1)
    base = ((NG + tj) * NT + c0) * NT + (NG + ti);
  else
    base = (c0 * NT + (NG + tj)) * NT + (NG + ti);
  double qL[N][NF], qR[N][NF];
#pragma unroll
  for (int v = 0; v < NF; ++v) {
    const double *w = W + v * NCELL + base;
    double q[N + 3];
#pragma unroll
    for (int e = 0; e < N + 3; ++e) q[e] = w[e * stride];
    double sl[N + 1];
#pragma unroll
    for (int e = 0; e < N + 1; ++e)
      sl[e] = minmod(__dadd_rn(q[e + 1], -q[e]), __dadd_rn(q[e + 2], -q[e + 1]));
#pragma unroll
    for (int cc = 0; cc < N; ++cc) {
      qL[cc][v] = __dadd_rn(q[cc + 1], __dmul_rn(0.5, sl[cc]));
      qR[cc][v] = __dadd_rn(q[cc + 2], -__dmul_rn(0.5, sl[cc + 1]));
    }
  }
#pragma unroll
  for (int cc = 0; cc < N; ++cc) {
    const int c = c0 + cc;
    State L, R;
    face_state<FAST>(qL[cc][0], qL[cc][1], qL[cc][2], qL[cc][3], qL[cc][4], gamma, igm1, d, L,
                     ok);
    face_state<FAST>(qR[cc][0], qR[cc][1], qR[cc][2], qR[cc][3], qR[cc][4], gamma, igm1, d, R,
                     ok);
    const double a = fmax(L.a, R.a);
    amax = fmax(amax, a);
    const double ha = __dmul_rn(0.5, a);
    int idx;
    if (d == 0)
      idx = (tj * NI + ti) * 9 + c;          // (k, j, face i)
    else if (d == 1)
      idx = (tj * 9 + c) * NI + ti;          // (k, face j, i)
    else
      idx = (c * NI + tj) * NI + ti;         // (face k, j, i)
#pragma unroll
    for (int v = 0; v < NF; ++v)
      Fb[v * NFACE + idx] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(L.f[v], R.f[v])),
                                      -__dmul_rn(ha, __dadd_rn(R.u[v], -L.u[v])));
  }
}

// FAST: branch-free divide / square-root fast paths (tb_internal.h), so the
// independent chains of a thread's faces interleave; a thread where any of
// them flags (never for physical states) redoes its segment with the IEEE
// intrinsics. Either way the fluxes are the intrinsics' bit for bit.
// the rare IEEE-intrinsic redo, out of line (keeps the hot loop compact)
template <int N>
__device__ __noinline__ double face_segment_slow(const double *W, double *Fb, int d, int stride,
                                                 int ti, int tj, int c0, double gamma,
                                                 double igm1, double amax) {
  bool ok = true;
  face_segment_impl<N, false>(W, Fb, d, stride, ti, tj, c0, gamma, igm1, amax, ok);
  return amax;
}

template <int N, bool FAST, bool SLOW_OUT_OF_LINE = false>
__device__ __forceinline__ void face_segment(const double *W, double *Fb, int d, int stride,
                                             int ti, int tj, int c0, double gamma, double igm1,
                                             double &amax) {
  bool ok = true;
  if constexpr (FAST) {
    double am = amax;
    face_segment_impl<N, true>(W, Fb, d, stride, ti, tj, c0, gamma, igm1, am, ok);
    if (!ok) {
      if constexpr (SLOW_OUT_OF_LINE) {
        am = face_segment_slow<N>(W, Fb, d, stride, ti, tj, c0, gamma, igm1, amax);
      } else {
        am = amax;
        face_segment_impl<N, false>(W, Fb, d, stride, ti, tj, c0, gamma, igm1, am, ok);
      }
    }
    amax = am;
  } else {
    face_segment_impl<N, false>(W, Fb, d, stride, ti, tj, c0, gamma, igm1, amax, ok);
  }
}

// LATTICE = false: U is [nsub][5][12][12][12] (ghosted sub-grids), staged by
// one 1-D bulk copy. LATTICE = true: U is a ghost-padded global lattice
// [5][N+4][N+4][N+4] described by `map`; sub-grid s (x fastest, nb per edge)
// is staged by one 4-D TMA box {12,12,12,5} at (8 bx, 8 by, 8 bz, 0) — the
// same shared-memory layout, no per-sub-grid ghost copies in HBM.
template <bool LATTICE, int V>
__global__ void __launch_bounds__(threads_of(V), 2)
    k_hydro_flux(const double *__restrict__ U, const __grid_constant__ CUtensorMap map, int nb,
                 double *__restrict__ dudt, double *__restrict__ amax_out, int64_t nsub,
                 double dx, double gamma, unsigned int slot) {
  extern __shared__ __align__(128) double sm[];
  double *W = sm;                        // [5][1728] primitives (staged U)
  double *Fb0 = sm + NF * NCELL;         // [2][5][576] face fluxes, by direction parity
  __shared__ __align__(8) uint64_t bar;
  // bit 10: dynamic sub-grid assignment — after its first (blockIdx.x), a CTA
  // takes the next sub-grid from work[0] when it starts one (work[1] counts
  // finished CTAs; the last resets both for the slot's next launch). The
  // static stride left CTAs finishing up to 43 us apart at config 2 (SM
  // pairing, slow-path sub-grids; scripts/k6_stamps_probe.py).
  constexpr bool kDynamic = (V & 1024) != 0;
  __shared__ int64_t s_next[2];
  unsigned int *const work = g_k6_work[slot % kWorkSlots];
  constexpr int kThreads = threads_of(V);
  constexpr int kCellsPerThread = (NI * NI * NI + kThreads - 1) / kThreads;   // 2
  __shared__ double s_amax[kThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double gm1 = __dadd_rn(gamma, -1.0);
  const double igm1 = __ddiv_rn(1.0, gm1), idx = __ddiv_rn(1.0, dx);
  constexpr bool kStamps = (V & 512) != 0;
  if (kStamps && t == 0 && blockIdx.x < kStampCtas) g_k6_stamps[blockIdx.x][0] = gtimer();
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage sub-grid s (one bulk copy / TMA box of 69,120 B) into W
  auto issue = [&](int64_t s) {
    const uint32_t bytes = NF * NCELL * 8;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(bytes)
                 : "memory");
    if constexpr (LATTICE) {
      const int bx = (int)(s % nb), by = (int)((s / nb) % nb), bz = (int)(s / ((int64_t)nb * nb));
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(W)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(8 * bx), "r"(8 * by), "r"(8 * bz), "r"(0),
          "r"(smem_u32(&bar))
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
          "%2, [%3];" ::"r"(smem_u32(W)),
          "l"(U + s * (int64_t)(NF * NCELL)), "r"(bytes), "r"(smem_u32(&bar))
          : "memory");
    }
  };
  // bit 6: pull sub-grid s into L2 (no shared memory) when s - gridDim.x
  // starts, so the later bulk copy into W streams from L2
  auto prefetch_l2 = [&](int64_t s) {
    if constexpr (LATTICE) {
      const int bx = (int)(s % nb), by = (int)((s / nb) % nb), bz = (int)(s / ((int64_t)nb * nb));
      asm volatile(
          "cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(
              reinterpret_cast<uint64_t>(&map)),
          "r"(8 * bx), "r"(8 * by), "r"(8 * bz), "r"(0)
          : "memory");
    } else {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       U + s * (int64_t)(NF * NCELL)),
                   "r"((uint32_t)(NF * NCELL * 8))
                   : "memory");
    }
  };
  auto wait_bar = [&](uint64_t *b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\nHW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HW_%=;\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
  };
  if (t == 0 && blockIdx.x < nsub) issue(blockIdx.x);
  uint32_t phase = 0;
  int it = 0;
  for (int64_t s = blockIdx.x; s < nsub; phase ^= 1, ++it) {
    // the sub-grid this CTA stages next (issued after the last face pass)
    int64_t nxt = 0;
    if constexpr (kDynamic) {
      if (t == 0) {
        nxt = (int64_t)gridDim.x + (int64_t)atomicAdd(work, 1u);
        s_next[(it + 1) & 1] = nxt;
      }
    } else {
      nxt = s + gridDim.x;
    }
    if ((V & 64) && t == 0 && nxt < nsub) prefetch_l2(nxt);
    wait_bar(&bar, phase);
    if ((V & 256) && t == 0) amax_out[s] = 0.0;   // bit 8's atomic max starts at +0
    if (kStamps && t == 0 && s == blockIdx.x && blockIdx.x < kStampCtas)
      g_k6_stamps[blockIdx.x][1] = gtimer();
    // ---- conserved -> primitive, in place --------------------------------
    constexpr bool kFast = (V & 8) != 0;
    constexpr bool kSlowOut = (V & 32) != 0;
    auto to_primitive_ir = [&](int c, double ir) {
      const double sx = W[NCELL + c], sy = W[2 * NCELL + c], sz = W[3 * NCELL + c],
                   E = W[4 * NCELL + c];
      const double vx = __dmul_rn(sx, ir), vy = __dmul_rn(sy, ir), vz = __dmul_rn(sz, ir);
      const double ke = __dmul_rn(
          0.5, __dadd_rn(__dadd_rn(__dmul_rn(sx, vx), __dmul_rn(sy, vy)), __dmul_rn(sz, vz)));
      W[NCELL + c] = vx;
      W[2 * NCELL + c] = vy;
      W[3 * NCELL + c] = vz;
      W[4 * NCELL + c] = __dmul_rn(gm1, __dadd_rn(E, -ke));
    };
    auto to_primitive = [&](int c) { to_primitive_ir(c, __ddiv_rn(1.0, W[c])); };
    if constexpr (kFast) {
      // kG cells at a time: their fast reciprocals interleave; a flagged
      // group is redone with the intrinsic (bit 7: one group of 6 covers the
      // 5.4 cells per thread of a 320-thread CTA in a single pass)
      constexpr int kG = (V & 128) ? 6 : 4;
      // NU cells c0 + u * kThreads (u < NU): fast reciprocals interleaved, the
      // group redone with the intrinsic if any flags, then converted
      auto group = [&](int c0, auto nu) {
        constexpr int NU = decltype(nu)::value;
        double ir[NU];
        bool ok = true;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const int c = c0 + u * kThreads;
          ir[u] = tb::div_rn_fast(1.0, c < NCELL ? W[c] : 1.0, ok);
        }
        if (!ok) {
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int c = c0 + u * kThreads;
            ir[u] = __ddiv_rn(1.0, c < NCELL ? W[c] : 1.0);
          }
        }
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const int c = c0 + u * kThreads;
          if (c < NCELL) to_primitive_ir(c, ir[u]);
        }
      };
#pragma unroll 1
      for (int c0 = t; c0 < NCELL; c0 += kG * kThreads) group(c0, std::integral_constant<int, kG>());
    } else {
#pragma unroll 4
      for (int c = t; c < NCELL; c += kThreads) to_primitive(c);
    }
    __syncthreads();
    double du[NF][kCellsPerThread];
    double amax = -CUDART_INF;
    // bit 2: the direction loop unrolled (d compile-time in each copy)
    constexpr int kUnrollD = (V & 4) ? 3 : 1;
#pragma unroll kUnrollD
    for (int d = 0; d < 3; ++d) {
      const int stride = d == 0 ? 1 : (d == 1 ? NT : NT * NT);
      // two flux buffers by direction parity: the fold of d and the faces of
      // d + 1 need no barrier between them
      double *Fb = Fb0 + (d & 1) * (NF * NFACE);
      // ---- face fluxes along d ------------------------------------------
      // 192 threads, three consecutive faces of one line each: the 6 cells
      // they read per field are loaded once and each interior slope (cells
      // c0+1 .. c0+4) is formed once for the two faces that use it
      if constexpr (V & 16) {
        // 10 warps: warps 0-7 take two consecutive faces of a line (segments
        // 0-1, 2-3, 4-5, 6-7), warps 8-9 the last face (8)
        if (t < 4 * NI * NI) {
          int g, ti, tj;
          if (d == 0) {
            g = t % 4;
            ti = (t / 4) % NI;
            tj = t / (4 * NI);
          } else {
            ti = t % NI;
            g = (t / NI) % 4;
            tj = t / (4 * NI);
          }
          face_segment<2, kFast, kSlowOut>(W, Fb, d, stride, ti, tj, 2 * g, gamma, igm1, amax);
        } else {
          const int u = t - 4 * NI * NI;
          face_segment<1, kFast, kSlowOut>(W, Fb, d, stride, u % NI, u / NI, 8, gamma, igm1, amax);
        }
      } else if constexpr (V & 1) {
        // all 8 warps: warps 0-5 take two consecutive faces of a line
        // (segments 0-1, 2-3, 4-5), warps 6-7 the last three (6-8)
        if (t < 3 * NI * NI) {
          int g, ti, tj;
          if (d == 0) {
            g = t % 3;
            ti = (t / 3) % NI;
            tj = t / (3 * NI);
          } else {
            ti = t % NI;
            g = (t / NI) % 3;
            tj = t / (3 * NI);
          }
          face_segment<2, kFast, kSlowOut>(W, Fb, d, stride, ti, tj, 2 * g, gamma, igm1, amax);
        } else {
          const int u = t - 3 * NI * NI;
          face_segment<3, kFast, kSlowOut>(W, Fb, d, stride, u % NI, u / NI, 6, gamma, igm1, amax);
        }
      } else if (t < 3 * NI * NI) {
        // 192 threads, three consecutive faces of one line each
        int g, ti, tj;
        if (d == 0) {
          g = t % 3;
          ti = (t / 3) % NI;
          tj = t / (3 * NI);
        } else {
          ti = t % NI;
          g = (t / NI) % 3;
          tj = t / (3 * NI);
        }
        face_segment<3, kFast, kSlowOut>(W, Fb, d, stride, ti, tj, 3 * g, gamma, igm1, amax);
      }
      __syncthreads();
      // every face of this sub-grid is done with W: stream the next one in
      // under the last fold, the output and the signal-speed reduction
      if (d == 2 && t == 0 && nxt < nsub) issue(nxt);
      if (kStamps && d == 2 && t == 0 && nxt >= nsub && blockIdx.x < kStampCtas)
        g_k6_stamps[blockIdx.x][2] = gtimer();
      // ---- fold this direction's flux differences into the cells ----------
#pragma unroll
      for (int m = 0; m < kCellsPerThread; ++m) {
        const int cell = t + kThreads * m;          // interior index (k, j, i)
        if ((NI * NI * NI) % kThreads != 0 && cell >= NI * NI * NI) break;
        const int ci = cell % NI, cj = (cell / NI) % NI, ck = cell / (NI * NI);
        int lo, hi;
        if (d == 0) {
          lo = (ck * NI + cj) * 9 + ci;
          hi = lo + 1;
        } else if (d == 1) {
          lo = (ck * 9 + cj) * NI + ci;
          hi = lo + NI;
        } else {
          lo = (ck * NI + cj) * NI + ci;
          hi = lo + NI * NI;
        }
#pragma unroll
        for (int v = 0; v < NF; ++v) {
          const double diff = __dadd_rn(Fb[v * NFACE + hi], -Fb[v * NFACE + lo]);
          du[v][m] = d == 0 ? diff : __dadd_rn(du[v][m], diff);
        }
      }
    }
    // ---- dU/dt = -(du / dx), coalesced ------------------------------------
    double *out = dudt + s * (int64_t)(NF * NI * NI * NI);
#pragma unroll
    for (int m = 0; m < kCellsPerThread; ++m) {
      if ((NI * NI * NI) % kThreads != 0 && t + kThreads * m >= NI * NI * NI) break;
#pragma unroll
      for (int v = 0; v < NF; ++v)
        out[v * (NI * NI * NI) + t + kThreads * m] = -__dmul_rn(du[v][m], idx);
    }
    // ---- max signal speed of the sub-grid ---------------------------------
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if constexpr (V & 256) {
      // bit 8: no end-of-sub-grid barrier — each warp folds its maximum into
      // amax_out[s] with a global atomic on the value's bits (a signal speed
      // is >= 0, and non-negative doubles order like their int64 bits);
      // amax_out[s] was zeroed by thread 0 before the conversion barrier. The
      // next sub-grid's conversion barrier still separates this fold of Fb
      // from its face pass.
      if (lane == 0)
        atomicMax(reinterpret_cast<long long *>(amax_out + s), __double_as_longlong(amax));
    } else {
      if (lane == 0) s_amax[warp] = amax;
      __syncthreads();
      if (t == 0) {
        double m = s_amax[0];
        for (int w = 1; w < kThreads / 32; ++w) m = fmax(m, s_amax[w]);
        amax_out[s] = m;
      }
    }
    // s_next[(it + 1) & 1] was written before this sub-grid's conversion
    // barrier; thread 0 rewrites that slot only after the next sub-grid's
    // barriers, which every thread must pass first
    if constexpr (kDynamic)
      s = s_next[(it + 1) & 1];
    else
      s = nxt;
  }
  if constexpr (kDynamic) {
    if (t == 0) {
      __threadfence();
      if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {   // last CTA out: reset the slot
        work[0] = 0;
        work[1] = 0;
        __threadfence();
      }
    }
  }
  if (kStamps && blockIdx.x < kStampCtas) {
    __syncthreads();
    if (t == 0) g_k6_stamps[blockIdx.x][3] = gtimer();
  }
}

template <bool LATTICE, int V>
int launch_v(tb_stream_t s, const double *U, const CUtensorMap &map, int nb, double *dudt,
             double *amax, int64_t nsub, double dx, double gamma) {
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_hydro_flux<LATTICE, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hydro_flux<LATTICE, V>, threads_of(V),
                                                      kSmem) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  int64_t blocks = (int64_t)tb::sm_count() * occ;
  if (blocks > nsub) blocks = nsub;
  const unsigned slot = (V & 1024) ? g_work_next.fetch_add(1) % kWorkSlots : 0u;
  k_hydro_flux<LATTICE, V><<<(int)blocks, threads_of(V), kSmem, reinterpret_cast<cudaStream_t>(s)>>>(
      U, map, nb, dudt, amax, nsub, dx, gamma, slot);
  return tb::last_error();
}

// TB_HYDRO_VARIANT selects the schedule (all bit-identical; K6 has
// the A/B numbers): bit 0 = all warps on faces, bit 2 = direction loop
// unrolled, bit 3 = branch-free divide / square-root fast paths, bit 4 = 320
// threads (2-face segments + one single face per line), bit 5 = the fast
// paths' fallback out of line, bit 6 = the next sub-grid prefetched into L2
// when this one starts, bit 7 = the conversion's reciprocals in one group of
// 6 per thread, bit 8 = the sub-grid's max signal speed folded by per-warp
// global atomics instead of a closing CTA barrier, bit 9 = per-CTA timer
// stamps (probe only), bit 10 = dynamic sub-grid assignment from a work
// counter. Built: 0 (round 1's first schedule), 1, 9, 13, 28, 60, 124, 252,
// 508, 1532 (default: 508 + dynamic; config 2 0.149 -> 0.143 ms, 32768
// sub-grids 1.073 -> 1.010 ms), 1020 / 2044 (508 / 1532 with stamps); the
// other measured variants were removed (round 2: 288 threads with two faces
// each everywhere, 0.167 ms vs 0.148 — still 96 registers, fewer warps; the
// first sub-grid staged in two parts so its conversion starts on the first,
// 0.1438 vs 0.1432 ms — no gain).
int hydro_variant() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("TB_HYDRO_VARIANT");
    v = e ? (atoi(e) & 2047) : kDefaultVariant;
  }
  return v;
}

template <bool LATTICE>
int launch(tb_stream_t s, const double *U, const CUtensorMap &map, int nb, double *dudt,
           double *amax, int64_t nsub, double dx, double gamma) {
  switch (hydro_variant()) {
    case 1: return launch_v<LATTICE, 1>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 9: return launch_v<LATTICE, 9>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 13: return launch_v<LATTICE, 13>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 28: return launch_v<LATTICE, 28>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 0: return launch_v<LATTICE, 0>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 124: return launch_v<LATTICE, 124>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 252: return launch_v<LATTICE, 252>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 508: return launch_v<LATTICE, 508>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 1020: return launch_v<LATTICE, 1020>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 1532: return launch_v<LATTICE, 1532>(s, U, map, nb, dudt, amax, nsub, dx, gamma);
    case 2044: return launch_v<LATTICE, 2044>(s, U, map, nb, dudt, amax, nsub, dx, gamma);

    default: return launch_v<LATTICE, kDefaultVariant>(s, U, map, nb, dudt, amax, nsub, dx,
                                                       gamma);
  }
}

}  // namespace

// Probe: the bit-9 variant's per-CTA stamps (ns) of the last launch,
// [ctas][entry, first staged, last faces done, exit]; n <= 1024 CTAs.
extern "C" int tb_hydro_stamps(unsigned long long *out, int n) {
  if (!out || n < 0 || n > kStampCtas) return TB_E_INVALID;
  return tb::rc(cudaMemcpyFromSymbol(out, g_k6_stamps, sizeof(unsigned long long) * 4 * n));
}

extern "C" int tb_hydro_flux(tb_stream_t s, const double *U, double *dudt, double *amax,
                             int64_t nsub, double dx, double gamma) {
  if (nsub < 0 || (nsub > 0 && (!U || !dudt || !amax)) || !(dx > 0.0) || !(gamma > 1.0))
    return TB_E_INVALID;
  if (nsub == 0) return TB_OK;
  if (reinterpret_cast<uintptr_t>(U) & 15) return TB_E_INVALID;
  CUtensorMap unused{};
  return launch<false>(s, U, unused, 0, dudt, amax, nsub, dx, gamma);
}

extern "C" int tb_hydro_flux_lattice(tb_stream_t s, const double *Up, int64_t n, int64_t nz,
                                     double *dudt, double *amax, double dx, double gamma) {
  if (!Up || !dudt || !amax || n < 8 || n % 8 || nz < 8 || nz % 8 || !(dx > 0.0) ||
      !(gamma > 1.0))
    return TB_E_INVALID;
  if (reinterpret_cast<uintptr_t>(Up) & 15) return TB_E_INVALID;
  const uint64_t P = (uint64_t)n + 2 * NG, Pz = (uint64_t)nz + 2 * NG;
  const uint64_t dims[4] = {P, P, Pz, (uint64_t)NF};
  const uint64_t strides[3] = {P * 8, P * P * 8, P * P * Pz * 8};
  const uint32_t box[4] = {NT, NT, NT, NF};
  CUtensorMap map;
  const int r = tb::encode_tiled(&map, 4, const_cast<double *>(Up), dims, strides, box);
  if (r != TB_OK) return r;
  const int nb = (int)(n / NI);
  return launch<true>(s, Up, map, nb, dudt, amax, (int64_t)nb * nb * (nz / NI), dx, gamma);
}
