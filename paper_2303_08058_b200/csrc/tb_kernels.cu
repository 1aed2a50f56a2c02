// tb_kernels.cu — sm_100a kernels for the sub-grid step path.
//
// K1  k_launch       : kernel_transform(kind) / registered affine kinds on a
//                      fused staging buffer (src/miniapp.py:40-53,
//                      src/executors.py:257-284). HBM-bound, 16 B per cell.
// K2  k_step[_bulk]  : one fused time step over many sub-grids, one warp per
//                      sub-grid (src/miniapp.py:116-133 == src/reference.py:31-47),
//                      the step's exact sum and min folded into a
//                      superaccumulator (src/miniapp.py:138-171); optionally the
//                      last CTA closes the step (K4 fused).
//                      k_step      : direct ld.global.nc into registers
//                                    (optionally with a register prefetch);
//                      k_step_bulk : per-warp ring of shared-memory slots fed by
//                                    the bulk-copy (TMA) engine + mbarriers.
// K4  k_acc_finalize : correctly rounded sum (== math.fsum) + dt + checksum,
//                      one warp.
//
// Bit-exactness (SURVEY.md §7 hard part 1): every transform is
// __dmul_rn followed by __dadd_rn — never an FMA; the per-sub-grid sum is
// numpy's pairwise order, mapped onto one warp: lane j owns block j/8 and
// accumulator j%8 of the 4x128 pairwise tree and holds
// a[128*(j/8) + (j%8) + 8*i], i = 0..15, in registers.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace {

__constant__ double kC1[TB_KINDS] = {1.0000003, 0.9999998, 1.0000001, 0.9999997,
                                     1.0000002};
__constant__ double kC2[TB_KINDS] = {1e-07, -1e-07, 2e-07, 5e-08, -2e-07};

__device__ __forceinline__ double xform(double x, double c1, double c2) {
  return __dadd_rn(__dmul_rn(x, c1), c2);
}

// Streaming 8-byte load that does not allocate in L1 (each old-state value is
// read once by its owner warp; neighbour faces are L2 hits).
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ long long ld_cg_s64(const int64_t *p) {
  long long v;
  asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ K1 --
template <int OP>
__global__ void __launch_bounds__(256) k_launch(double *__restrict__ d, int64_t n,
                                                double c1, double c2) {
  if (OP == TB_OP_NONE) return;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // cudaMalloc'd staging is 256-B aligned; sub-views may not be 16-B aligned.
  const int64_t head = (reinterpret_cast<uintptr_t>(d) & 15) ? 1 : 0;
  if (head && tid == 0 && n > 0) d[0] = xform(d[0], c1, c2);
  double2 *v = reinterpret_cast<double2 *>(d + head);
  const int64_t nv = (n - head) / 2;
  for (int64_t i = tid; i < nv; i += stride) {
    double2 x = v[i];
    x.x = xform(x.x, c1, c2);
    x.y = xform(x.y, c1, c2);
    v[i] = x;
  }
  const int64_t tail = head + 2 * nv;
  if (tail < n && tid == 0) d[tail] = xform(d[tail], c1, c2);
}

__global__ void k_empty() {}
__global__ void k_trap() { __trap(); }

// K1g: one aggregated batch whose members are read and written where they
// live (mapped pinned host rows of the machine's task arena): member =
// blockIdx.y, 16-byte vector accesses, the same two roundings as K1.
// Completion word (tb_done): the launch's last CTA stores seq into a mapped
// pinned host word once every CTA's writes are visible system-wide, so the
// host sees the batch complete by reading memory — no event record, no
// driver query. The CTA counter lives in device memory, is zero before the
// launch and is reset by the last CTA (launches on one stream are ordered).
struct DoneArgs {
  unsigned long long *word;
  unsigned long long seq;
  unsigned *ctas;
};

static bool done_args(const tb_done *done, DoneArgs *d) {
  *d = DoneArgs{nullptr, 0, nullptr};
  if (!done) return true;
  if (!done->word || !done->ctas || (reinterpret_cast<uintptr_t>(done->word) & 7)) return false;
  *d = DoneArgs{reinterpret_cast<unsigned long long *>(done->word),
                (unsigned long long)done->seq, done->ctas};
  return true;
}

__device__ __forceinline__ void signal_done(const DoneArgs &d) {
  if (!d.word) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y;
    if (atomicAdd(d.ctas, 1u) == total - 1) {
      *d.ctas = 0;
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long *>(d.word) = d.seq;
    }
  }
}

struct GatherArgs {
  const double *src[TB_GATHER_MAX];
  double *dst[TB_GATHER_MAX];
  int64_t n[TB_GATHER_MAX];
  double c1, c2;
  DoneArgs done;
};

__global__ void __launch_bounds__(256) k_launch_gather(const __grid_constant__ GatherArgs a) {
  const int m = blockIdx.y;
  const double2 *s = reinterpret_cast<const double2 *>(a.src[m]);
  double2 *d = reinterpret_cast<double2 *>(a.dst[m]);
  const int64_t n2 = a.n[m] / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = s[i];
    x.x = xform(x.x, a.c1, a.c2);
    x.y = xform(x.y, a.c1, a.c2);
    d[i] = x;
  }
  signal_done(a.done);
}

// K1e: a gather batch whose members may be a task's FIRST round (flag bit 0:
// the input rows are the sub-grids' cells, folded with the previous
// generation's neighbour faces before the transform — src/miniapp.py:119-126)
// and/or its LAST round (bit 1: per sub-grid, the min and numpy's pairwise sum
// of the 512 transformed values — src/miniapp.py:133). One CTA of 256 threads
// per (sub-grid, member); each thread owns cells 2t, 2t+1.
struct GatherEdgeArgs {
  const double *src[TB_GATHER_MAX];
  double *dst[TB_GATHER_MAX];
  int64_t g0[TB_GATHER_MAX];      // the member's first sub-grid (ring index)
  int32_t nsub[TB_GATHER_MAX];    // sub-grids in the member
  uint8_t flags[TB_GATHER_MAX];
  const double *faces;            // [S][2][8]: (left face, right face) snapshot
  double *mins, *sums;            // [S]
  int64_t S;
  double c1, c2;
  DoneArgs done;
};

__global__ void __launch_bounds__(256) k_launch_gather_edge(const __grid_constant__ GatherEdgeArgs a) {
  const int m = blockIdx.y, k = blockIdx.x, t = threadIdx.x;
  if (k >= a.nsub[m]) {   // no sub-grid here (a shorter member): only count in
    signal_done(a.done);
    return;
  }
  const int flags = a.flags[m];
  const int64_t g = a.g0[m] + k;
  const double2 *src = reinterpret_cast<const double2 *>(a.src[m] + (int64_t)k * TB_CELLS);
  double2 *dst = reinterpret_cast<double2 *>(a.dst[m] + (int64_t)k * TB_CELLS);
  double2 x = src[t];
  if ((flags & 1) && (t < TB_FACE / 2 || t >= (TB_CELLS - TB_FACE) / 2)) {
    // ghost fold against the neighbours' previous-generation faces
    const bool left = t < TB_FACE / 2;
    const int64_t nb = left ? (g - 1 + a.S) % a.S : (g + 1) % a.S;
    const double *f = a.faces + nb * 2 * TB_FACE + (left ? TB_FACE : 0);
    const int i = left ? 2 * t : 2 * t - (TB_CELLS - TB_FACE);
    x.x = __dmul_rn(0.5, __dadd_rn(x.x, f[i]));
    x.y = __dmul_rn(0.5, __dadd_rn(x.y, f[i + 1]));
  }
  x.x = xform(x.x, a.c1, a.c2);
  x.y = xform(x.y, a.c1, a.c2);
  dst[t] = x;
  if (!(flags & 2)) {
    signal_done(a.done);
    return;
  }
  // per-sub-grid min (exact) and pairwise sum in numpy's order: four blocks
  // of 128, each summed by 8 strided accumulators r[j] = p[j] + p[j+8] + ...
  // (in that order), combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then
  // (b0+b1)+(b2+b3) — the host's pairwise512 (oracle/tb_oracle.c)
  __shared__ double v[TB_CELLS];
  __shared__ double wmin[8];
  v[2 * t] = x.x;
  v[2 * t + 1] = x.y;
  double mn = fmin(x.x, x.y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((t & 31) == 0) wmin[t >> 5] = mn;
  __syncthreads();
  if (t < 32) {
    const int blk = t >> 3, j = t & 7;
    const double *p = v + 128 * blk + j;
    double r = p[0];
#pragma unroll
    for (int i = 8; i < 128; i += 8) r = __dadd_rn(r, p[i]);
    // lanes 8*blk .. 8*blk+7 hold r[0..7] of block blk
    const double r01 = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));        // j even
    const double r0123 = __dadd_rn(r01, __shfl_down_sync(0xffffffffu, r01, 2));  // j % 4 == 0
    const double b = __dadd_rn(r0123, __shfl_down_sync(0xffffffffu, r0123, 4));  // j == 0
    const double b01 = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 8));        // blk even
    const double tot = __dadd_rn(b01, __shfl_down_sync(0xffffffffu, b01, 16));   // lane 0
    double wm = t < 8 ? wmin[t] : CUDART_INF;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) wm = fmin(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (t == 0) {
      a.sums[g] = tot;
      a.mins[g] = wm;
    }
  }
  signal_done(a.done);
}

__global__ void k_spin(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((int64_t)(t - t0) < ns);
}

__global__ void k_init_cells(double *__restrict__ cells, int64_t subgrids,
                             int64_t lo, int64_t n) {
  const double scale = (double)(subgrids * 1000 + TB_CELLS);
  const int64_t total = n * TB_CELLS;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = k / TB_CELLS;
    const int i = (int)(k % TB_CELLS);
    // (g*1000.0 + i) is an exact integer in double; the division rounds once.
    cells[k] = __ddiv_rn(__dadd_rn(__dmul_rn((double)(lo + g), 1000.0), (double)i),
                         scale);
  }
}

// ---------------------------------------------------- superaccumulator --
// Order-preserving int64 key of a double (non-NaN): min over keys == min
// over values, so the min can be combined with atomicMin / ncclMin(int64).
__device__ __forceinline__ long long min_key(double x) {
  long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double key_to_double(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffLL));
}

constexpr long long kKeyInf = 0x7ff0000000000000LL;   // min_key(+inf)

// Add x exactly into 32-bit-digit int64 limbs (digit i weighs 2^(32i-1074)).
// x = mant * 2^(p - 1074) with p = biased exponent - 1 (0 for subnormals).
__device__ __forceinline__ void acc_add_digits(unsigned long long *limbs, double x) {
  if (x == 0.0) return;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int ex = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & ((1ULL << 52) - 1);
  int p = 0;
  if (ex != 0) {
    mant |= 1ULL << 52;
    p = ex - 1;
  }
  const int limb = p >> 5, off = p & 31;
  const unsigned long long lo = mant << off;
  const unsigned long long hi = off ? (mant >> (64 - off)) : 0ULL;
  const bool neg = (long long)bits < 0;
  const unsigned long long d0 = lo & 0xffffffffULL, d1 = lo >> 32, d2 = hi;
  atomicAdd(limbs + limb, neg ? (0ULL - d0) : d0);
  if (d1) atomicAdd(limbs + limb + 1, neg ? (0ULL - d1) : d1);
  if (d2) atomicAdd(limbs + limb + 2, neg ? (0ULL - d2) : d2);
}

// Flush a block's shared limbs + min key into the global accumulator.
__device__ __forceinline__ void acc_flush(const unsigned long long *s_limbs,
                                          long long block_min_key, int64_t *acc) {
  for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) {
    const unsigned long long v = s_limbs[i];
    if (v) atomicAdd(reinterpret_cast<unsigned long long *>(acc) + i, v);
  }
  if (threadIdx.x == 0)
    atomicMin(reinterpret_cast<long long *>(acc) + TB_ACC_MIN_WORD, block_min_key);
}

// Exact sum of an arbitrary vector into acc (the reduction half of K2).
__global__ void __launch_bounds__(256) k_acc_add(const double *__restrict__ x,
                                                 int64_t n, int64_t *acc) {
  __shared__ unsigned long long s_limbs[TB_ACC_LIMBS];
  __shared__ long long s_min[8];
  for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) s_limbs[i] = 0ULL;
  __syncthreads();
  double m = CUDART_INF;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    acc_add_digits(s_limbs, v);
    m = fmin(m, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = min_key(m);
  __syncthreads();
  long long bm = s_min[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) bm = min(bm, s_min[w]);
  acc_flush(s_limbs, bm, acc);
}

__global__ void k_acc_reset(int64_t *acc) {
  for (int i = threadIdx.x; i < TB_ACC_WORDS; i += blockDim.x)
    acc[i] = (i == TB_ACC_MIN_WORD) ? kKeyInf : 0;
}

// ------------------------------------------------------ step finalize --
// Correctly rounded (half-even) value of the exact sum in the limbs, plus dt
// and the running checksum, computed by ONE full warp. Only the carry chain
// over the occupied limbs [lo, hi] is sequential (a few limbs for real data);
// sign, leading-digit search, window and sticky bit are warp-parallel.
constexpr int kDigits = 96;   // >= TB_ACC_LIMBS + carry growth; 3 per lane

__device__ void warp_finalize(int64_t *acc, double *piece, double *dt,
                              double *checksum, int reset) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const long long a0 = ld_cg_s64(acc + lane);
  const long long a1 = ld_cg_s64(acc + lane + 32);
  const long long a2 = (lane + 64 < TB_ACC_LIMBS) ? ld_cg_s64(acc + lane + 64) : 0;
  const unsigned n0 = __ballot_sync(full, a0 != 0), n1 = __ballot_sync(full, a1 != 0),
                 n2 = __ballot_sync(full, a2 != 0);
  double p = 0.0;
  if (n0 | n1 | n2) {
    const int lo = n0 ? __ffs(n0) - 1 : (n1 ? 31 + __ffs(n1) : 63 + __ffs(n2));
    const int hi = n2 ? 95 - __clz(n2) : (n1 ? 63 - __clz(n1) : 31 - __clz(n0));
    // Warp-uniform carry chain over the occupied limbs; limb i comes from its
    // owner lane by shuffle, digit i is kept by that lane (m0/m1/m2).
    uint32_t m0 = 0u, m1 = 0u, m2 = 0u;
    long long carry = 0;
    int i = lo;
    for (; i < kDigits; ++i) {
      const long long x0 = __shfl_sync(full, a0, i & 31);
      const long long x1 = __shfl_sync(full, a1, i & 31);
      const long long x2 = __shfl_sync(full, a2, i & 31);
      const long long li = i > hi ? 0LL : (i < 32 ? x0 : (i < 64 ? x1 : x2));
      const long long v = li + carry;
      if (lane == (i & 31)) {
        const uint32_t d = (uint32_t)(v & 0xffffffffLL);
        if (i < 32) m0 = d; else if (i < 64) m1 = d; else m2 = d;
      }
      carry = v >> 32;   // arithmetic shift
      if (i >= hi && (carry == 0 || carry == -1)) break;
    }
    const bool neg = carry < 0;
    if (neg) {   // sign-extend above the last written digit
      if (lane > i) m0 = 0xffffffffu;
      if (lane + 32 > i) m1 = 0xffffffffu;
      if (lane + 64 > i) m2 = 0xffffffffu;
    }

    if (neg) {  // magnitude = two's complement negation, digit-parallel
      const unsigned z0 = __ballot_sync(full, m0 != 0), z1 = __ballot_sync(full, m1 != 0),
                     z2 = __ballot_sync(full, m2 != 0);
      const int z = z0 ? __ffs(z0) - 1 : (z1 ? 31 + __ffs(z1) : 63 + __ffs(z2));
      auto negd = [&](uint32_t d, int idx) -> uint32_t {
        return idx < z ? 0u : (idx == z ? (uint32_t)(0u - d) : ~d);
      };
      m0 = negd(m0, lane);
      m1 = negd(m1, lane + 32);
      m2 = negd(m2, lane + 64);
    }
    const unsigned t0 = __ballot_sync(full, m0 != 0), t1 = __ballot_sync(full, m1 != 0),
                   t2 = __ballot_sync(full, m2 != 0);
    const int top = t2 ? 95 - __clz(t2) : (t1 ? 63 - __clz(t1) : 31 - __clz(t0));
    auto digit = [&](int k) -> uint32_t {   // warp-collective fetch of digit k
      const int kk = k < 0 ? 0 : k;
      const uint32_t a = __shfl_sync(full, m0, kk & 31), b = __shfl_sync(full, m1, kk & 31),
                     c = __shfl_sync(full, m2, kk & 31);
      const uint32_t v = kk < 32 ? a : (kk < 64 ? b : c);
      return k < 0 ? 0u : v;
    };
    const uint32_t wt = digit(top), wm = digit(top - 1), wl = digit(top - 2);
    const bool below = (lane < top - 2 && m0 != 0) || (lane + 32 < top - 2 && m1 != 0) ||
                       (lane + 64 < top - 2 && m2 != 0);
    const bool sticky_low = __ballot_sync(full, below) != 0;
    if (lane == 0) {
      const unsigned __int128 W = ((unsigned __int128)wt << 64) |
                                  ((unsigned __int128)wm << 32) | (unsigned __int128)wl;
      const int base = 32 * (top - 2);
      const int nbits = 32 * top + (32 - __clz((int)wt));
      unsigned long long mant;
      int e2;
      if (nbits <= 53) {
        mant = (unsigned long long)(W >> (-base));   // only when top <= 1: base < 0
        e2 = -TB_ACC_BIAS;
      } else {
        const int rel = nbits - 53 - base;           // in [12, 43]
        mant = (unsigned long long)(W >> rel);
        const bool guard = (W >> (rel - 1)) & 1;
        const bool sticky =
            sticky_low || (W & ((((unsigned __int128)1) << (rel - 1)) - 1)) != 0;
        if (guard && (sticky || (mant & 1ULL))) mant += 1;
        e2 = (nbits - 53) - TB_ACC_BIAS;
      }
      p = scalbn((double)mant, e2);
      if (neg) p = -p;
    }
  }
  if (lane == 0) {
    if (piece) *piece = p;
    if (dt) *dt = key_to_double(ld_cg_s64(acc + TB_ACC_MIN_WORD));
    if (checksum) *checksum = __dadd_rn(*checksum, p);   // src/miniapp.py:227
  }
  __syncwarp();
  if (reset)
    for (int i = lane; i < TB_ACC_WORDS; i += 32)
      acc[i] = (i == TB_ACC_MIN_WORD) ? kKeyInf : 0;
}

__global__ void k_acc_finalize(int64_t *acc, double *piece, double *dt,
                               double *checksum, int reset) {
  if (threadIdx.x < 32) warp_finalize(acc, piece, dt, checksum, reset);
}

__device__ void warp_acc_flush_strided(const double *sums, int64_t first, int64_t stride,
                                       int64_t n, unsigned long long *limbs);

// Close a step from its per-sub-grid (sum, min) in one standalone launch
// (tb_step_close: the last step of a deferred run): every CTA folds a slice
// (exact digits, warp-merged windows; min of the mins) into acc, and the last
// CTA to finish rounds — == math.fsum of the sums and the min-tree dt
// (src/miniapp.py:138-171). acc must be reset (it is reset again after).
__global__ void __launch_bounds__(256) k_step_close(const double *sums, const double *mins,
                                                    int64_t n, int64_t *acc, double *piece,
                                                    double *dt, double *checksum) {
  __shared__ unsigned long long c_limbs[TB_ACC_LIMBS];
  __shared__ long long c_min;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < TB_ACC_LIMBS; i += blockDim.x) c_limbs[i] = 0ULL;
  if (t == 0) c_min = kKeyInf;
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  warp_acc_flush_strided(sums, gw, nw, n, c_limbs);
  double m = CUDART_INF;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + t; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmin(m, __ldcg(mins + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMin(&c_min, min_key(m));
  __syncthreads();
  if (warp != 0) return;
  for (int i = lane; i < TB_ACC_LIMBS; i += 32) {
    const unsigned long long v = c_limbs[i];
    if (v) atomicAdd(reinterpret_cast<unsigned long long *>(acc) + i, v);
  }
  if (lane == 0) atomicMin(reinterpret_cast<long long *>(acc) + TB_ACC_MIN_WORD, c_min);
  __threadfence();
  __syncwarp();
  unsigned long long tk = 0;
  if (lane == 0)
    tk = atomicAdd(reinterpret_cast<unsigned long long *>(acc) + TB_ACC_COUNT_WORD, 1ULL);
  tk = __shfl_sync(0xffffffffu, tk, 0);
  if (tk == (unsigned long long)gridDim.x - 1) {
    __threadfence();
    warp_finalize(acc, piece, dt, checksum, 1);
  }
}

// ------------------------------------------------------------------ K2 --
constexpr int kStepThreads = 256;
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStages = 2;   // default bulk-copy ring depth per warp
// Slot layout: the four 128-cell blocks of a sub-grid at a 1088-B pitch
// (1 KiB + 64 B pad) so lanes (b, r) and (b+1, r) sit in opposite bank halves:
// each 8-byte LDS of the warp is exactly 2 wavefronts (conflict-free).
constexpr int kBlkPitch = 136;                    // doubles per padded block
constexpr int kSlot = 4 * kBlkPitch;              // doubles per slot (4352 B)
constexpr int bulk_smem(int stages) { return kStepWarps * stages * kSlot * 8; }
// 2 stages: 68 KiB/CTA -> 3 CTAs (24 warps)/SM; 1 stage: 34 KiB -> 4 CTAs
// (32 warps, register-limited) with one sub-grid in flight per warp.

struct StepArgs {
  const double *old;
  double *out;
  int64_t n;
  const double *left_face;
  const double *right_face;
  int chains, kpc;
  double *mins, *sums;
  int64_t *acc;
  double *piece, *dt, *checksum;   // fused finalize outputs (single device)
  int finalize;
  // deferred close: this launch writes only per-sub-grid (sum, min); every
  // streaming warp folds its share of the PREVIOUS step's (prev_sums,
  // prev_mins) exactly into prev_acc early in the launch, and the grid's
  // extra last CTA waits for all shares and rounds them into prev_piece /
  // prev_dt, checksum += piece
  int64_t *prev_acc;
  const double *prev_sums, *prev_mins;
  double *prev_piece, *prev_dt;
  int finalizer;
};

__device__ void warp_finalize(int64_t *acc, double *piece, double *dt,
                              double *checksum, int reset);
__device__ __forceinline__ long long ld_acquire_s64(const int64_t *p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The deferred close's extra CTA (returns true if this CTA is it): waits for
// every streaming CTA's share of the previous step (the count word), then
// rounds. The shares arrive early in the launch, so this is off the step's
// critical path.
__device__ __forceinline__ bool finalizer_cta(const StepArgs &a) {
  if (!a.finalizer || blockIdx.x != gridDim.x - 1) return false;
  if (threadIdx.x < 32) {
    const long long want = (long long)gridDim.x - 1;
    while (ld_acquire_s64(a.prev_acc + TB_ACC_COUNT_WORD) < want) __nanosleep(256);
    warp_finalize(a.prev_acc, a.prev_piece, a.prev_dt, a.checksum, 1);
  }
  return true;
}

template <int CHAINS, int KPC>
__device__ __forceinline__ void run_chains(double (&v)[16], int chains, int kpc) {
  if (CHAINS > 0) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
#pragma unroll
      for (int k = 0; k < KPC; ++k) {
        const double c1 = kC1[k], c2 = kC2[k];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = xform(v[i], c1, c2);
      }
  } else {
    for (int c = 0; c < chains; ++c)
      for (int k = 0; k < kpc; ++k) {
        const double c1 = kC1[k], c2 = kC2[k];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = xform(v[i], c1, c2);
      }
  }
}

// Everything once this lane's 16 cells are in registers: ghost fold,
// transforms, store, pairwise sum + min (src/miniapp.py:119-133).
// The ghost-face value this lane folds in (lanes 0..7: the left neighbour's
// right face; lanes 24..31: the right neighbour's left face; others 0). Issued
// together with the sub-grid's own loads so its latency overlaps theirs.
__device__ __forceinline__ double load_face(const StepArgs &a, int64_t g, int lane) {
  const int r = lane & 7;
  if (lane < 8) {
    const double *lf =
        g == 0 ? a.left_face : a.old + (g - 1) * TB_CELLS + (TB_CELLS - TB_FACE);
    return ld_stream(lf + r);
  }
  if (lane >= 24) {
    const double *rf = g == a.n - 1 ? a.right_face : a.old + (g + 1) * TB_CELLS;
    return ld_stream(rf + r);
  }
  return 0.0;
}

// Exact accumulation off the per-sub-grid path: lane 0 parks each sub-grid's
// sum in its warp's shared buffer (one store); every kSumBuf sub-grids and at
// the end the warp converts 32 sums at a time in parallel and, when they share
// their 3-digit window (the common case), warp-reduces the digits so lane 0
// issues just 3 shared atomics.
constexpr int kSumBuf = 64;

struct SumBuf {
  int cnt = 0;
};

// min over the warp's 16x32 values on the integer pipe: order-preserving
// int64 keys (min_key), a per-lane 64-bit min, then two 32-bit warp
// reductions (high word; low word among the lanes holding the minimal high
// word). The FP64 pipe — K2's co-limit with HBM — keeps only the transforms
// and the pairwise sum (20 fewer FP64 instructions per lane and sub-grid).
// Same result as the fmin tree for every non-NaN input.
__device__ __forceinline__ double warp_min_alu(const double (&v)[16]) {
  long long k = min_key(v[0]);
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    const long long x = min_key(v[i]);
    k = x < k ? x : k;
  }
  const int hi = (int)(k >> 32);
  const unsigned lo = (unsigned)(k & 0xffffffffLL);
  const int hmin = __reduce_min_sync(0xffffffffu, hi);
  const unsigned lmin = __reduce_min_sync(0xffffffffu, hi == hmin ? lo : 0xffffffffu);
  return key_to_double((long long)(((unsigned long long)(unsigned)hmin << 32) | lmin));
}

__device__ __forceinline__ long long shfl_sum_s64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ void warp_acc_flush(const double *sums, int cnt, unsigned long long *limbs) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < cnt; base += 32) {
    const double x = base + lane < cnt ? sums[base + lane] : 0.0;
    int l = -1;
    long long d0 = 0, d1 = 0, d2 = 0;
    if (x != 0.0) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
      const int ex = (int)((bits >> 52) & 0x7ff);
      unsigned long long mant = bits & ((1ULL << 52) - 1);
      int p = 0;
      if (ex != 0) {
        mant |= 1ULL << 52;
        p = ex - 1;
      }
      l = p >> 5;
      const int off = p & 31;
      const unsigned long long lo = mant << off;
      const unsigned long long hi = off ? (mant >> (64 - off)) : 0ULL;
      d0 = (long long)(lo & 0xffffffffULL);
      d1 = (long long)(lo >> 32);
      d2 = (long long)hi;
      if ((long long)bits < 0) {
        d0 = -d0;
        d1 = -d1;
        d2 = -d2;
      }
    }
    const int lmax = __reduce_max_sync(0xffffffffu, l);
    const bool same = __all_sync(0xffffffffu, l < 0 || l == lmax);
    if (same) {
      if (lmax < 0) continue;
      d0 = shfl_sum_s64(d0);
      d1 = shfl_sum_s64(d1);
      d2 = shfl_sum_s64(d2);
      if (lane == 0) {
        if (d0) atomicAdd(limbs + lmax, (unsigned long long)d0);
        if (d1) atomicAdd(limbs + lmax + 1, (unsigned long long)d1);
        if (d2) atomicAdd(limbs + lmax + 2, (unsigned long long)d2);
      }
    } else if (l >= 0) {
      if (d0) atomicAdd(limbs + l, (unsigned long long)d0);
      if (d1) atomicAdd(limbs + l + 1, (unsigned long long)d1);
      if (d2) atomicAdd(limbs + l + 2, (unsigned long long)d2);
    }
  }
}

// warp_acc_flush over sums[first + k*stride], k = 0.. while < n
__device__ void warp_acc_flush_strided(const double *sums, int64_t first, int64_t stride,
                                       int64_t n, unsigned long long *limbs) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = first; base < n; base += 32 * stride) {
    const int64_t i = base + lane * stride;
    const double x = i < n ? __ldcg(sums + i) : 0.0;
    int l = -1;
    long long d0 = 0, d1 = 0, d2 = 0;
    if (x != 0.0) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
      const int ex = (int)((bits >> 52) & 0x7ff);
      unsigned long long mant = bits & ((1ULL << 52) - 1);
      int p = 0;
      if (ex != 0) {
        mant |= 1ULL << 52;
        p = ex - 1;
      }
      l = p >> 5;
      const int off = p & 31;
      const unsigned long long lo = mant << off;
      const unsigned long long hi = off ? (mant >> (64 - off)) : 0ULL;
      d0 = (long long)(lo & 0xffffffffULL);
      d1 = (long long)(lo >> 32);
      d2 = (long long)hi;
      if ((long long)bits < 0) {
        d0 = -d0;
        d1 = -d1;
        d2 = -d2;
      }
    }
    const int lmax = __reduce_max_sync(0xffffffffu, l);
    if (__all_sync(0xffffffffu, l < 0 || l == lmax)) {
      if (lmax < 0) continue;
      d0 = shfl_sum_s64(d0);
      d1 = shfl_sum_s64(d1);
      d2 = shfl_sum_s64(d2);
      if (lane == 0) {
        if (d0) atomicAdd(limbs + lmax, (unsigned long long)d0);
        if (d1) atomicAdd(limbs + lmax + 1, (unsigned long long)d1);
        if (d2) atomicAdd(limbs + lmax + 2, (unsigned long long)d2);
      }
    } else if (l >= 0) {
      if (d0) atomicAdd(limbs + l, (unsigned long long)d0);
      if (d1) atomicAdd(limbs + l + 1, (unsigned long long)d1);
      if (d2) atomicAdd(limbs + l + 2, (unsigned long long)d2);
    }
  }
}

// A streaming warp's share of the previous step's close: the (sum, min) of
// the sub-grids it also streams this step (same grid stride, a handful),
// folded once its own pipeline runs. No CTA barrier (a warp may have no
// sub-grids): the CTA's last warp to fold (s_min[1] = ticket, s_min[0] = min
// key, both set at kernel start) adds the CTA's digits to prev_acc and
// counts the CTA in for the waiting close CTA.
__device__ __forceinline__ void fold_previous(const StepArgs &a, int64_t g0, int64_t gstride,
                                              unsigned long long *s_limbs, long long *s_min) {
  const int lane = threadIdx.x & 31;
  warp_acc_flush_strided(a.prev_sums, g0, gstride, a.n, s_limbs);
  double m = CUDART_INF;
  for (int64_t g = g0 + lane * gstride; g < a.n; g += 32 * gstride)
    m = fmin(m, __ldcg(a.prev_mins + g));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMin(&s_min[0], min_key(m));
  __threadfence_block();
  __syncwarp();
  unsigned long long tk = 0;
  if (lane == 0) tk = atomicAdd(reinterpret_cast<unsigned long long *>(&s_min[1]), 1ULL);
  tk = __shfl_sync(0xffffffffu, tk, 0);
  if (tk != (unsigned long long)(blockDim.x >> 5) - 1) return;
  __threadfence_block();
  for (int i = lane; i < TB_ACC_LIMBS; i += 32) {
    const unsigned long long v = *reinterpret_cast<volatile unsigned long long *>(s_limbs + i);
    if (v) atomicAdd(reinterpret_cast<unsigned long long *>(a.prev_acc) + i, v);
  }
  if (lane == 0) {
    atomicMin(reinterpret_cast<long long *>(a.prev_acc) + TB_ACC_MIN_WORD,
              *reinterpret_cast<volatile long long *>(&s_min[0]));
    __threadfence();
    atomicAdd(reinterpret_cast<unsigned long long *>(a.prev_acc) + TB_ACC_COUNT_WORD, 1ULL);
  }
}

template <int CHAINS, int KPC, bool ALUMIN = false>
__device__ __forceinline__ void subgrid_body(const StepArgs &a, int64_t g, int lane,
                                             double (&v)[16], double face,
                                             unsigned long long *s_limbs, double &wmin,
                                             double *wsums, SumBuf &sb) {
  const int r = lane & 7;
  // Ghost fold against the previous generation: cells 0..7 are lanes 0..7 at
  // i = 0; cells 504..511 are lanes 24..31 at i = 15. Add rounds; *0.5 exact.
  if (lane < 8)
    v[0] = __dmul_rn(0.5, __dadd_rn(v[0], face));
  else if (lane >= 24)
    v[15] = __dmul_rn(0.5, __dadd_rn(v[15], face));
  run_chains<CHAINS, KPC>(v, a.chains, a.kpc);
  double *dst = a.out + g * TB_CELLS + 128 * (lane >> 3) + r;
#pragma unroll
  for (int i = 0; i < 16; ++i) dst[8 * i] = v[i];
  // numpy pairwise: r_j = a[j] + a[j+8] + ... sequentially, then
  // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) per block and (B0+B1)+(B2+B3).
  double s = v[0], m = v[0];
  if (ALUMIN) {
#pragma unroll
    for (int i = 1; i < 16; ++i) s = __dadd_rn(s, v[i]);
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, x));
    m = warp_min_alu(v);
  } else {
#pragma unroll
    for (int i = 1; i < 16; ++i) {
      s = __dadd_rn(s, v[i]);
      m = fmin(m, v[i]);
    }
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, x));
      m = fmin(m, __shfl_xor_sync(0xffffffffu, m, x));
    }
  }
  if (lane == 0) {
    if (a.sums) a.sums[g] = s;
    if (a.mins) a.mins[g] = m;
  }
  if (a.acc) {
    if (lane == 0) wsums[sb.cnt] = s;
    if (++sb.cnt == kSumBuf) {
      __syncwarp();
      warp_acc_flush(wsums, kSumBuf, s_limbs);
      __syncwarp();
      sb.cnt = 0;
    }
  }
  wmin = fmin(wmin, m);
}

// Block epilogue: flush shared limbs + block min into acc; with finalize, the
// last CTA to finish (threadfence + ticket) closes the step with one warp.
__device__ __forceinline__ void step_epilogue(const StepArgs &a,
                                              unsigned long long *s_limbs,
                                              long long *s_min, double wmin,
                                              double *wsums = nullptr, int nsums = 0) {
  if (!a.acc) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (wsums) {
    __syncwarp();
    warp_acc_flush(wsums, nsums, s_limbs);
  }
  if (lane == 0) s_min[warp] = min_key(wmin);
  __syncthreads();                    // the CTA's limbs and warp minima are in smem
  if (warp != 0) return;              // warp 0 publishes; the rest retire now
  long long bm = s_min[0];
#pragma unroll
  for (int w = 1; w < kStepWarps; ++w) bm = min(bm, s_min[w]);
  int64_t *acc = a.acc;
  for (int i = lane; i < TB_ACC_LIMBS; i += 32) {
    const unsigned long long v = s_limbs[i];
    if (v) atomicAdd(reinterpret_cast<unsigned long long *>(acc) + i, v);
  }
  if (lane == 0)
    atomicMin(reinterpret_cast<long long *>(acc) + TB_ACC_MIN_WORD, bm);
  if (!a.finalize) return;
  // Last-CTA ticket: each publishing lane fences its own atomics, then lane 0
  // takes a ticket; the CTA that draws gridDim.x-1 closes the step.
  __threadfence();
  __syncwarp();
  unsigned long long t = 0;
  if (lane == 0)
    t = atomicAdd(reinterpret_cast<unsigned long long *>(a.acc) + TB_ACC_COUNT_WORD, 1ULL);
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t == (unsigned long long)gridDim.x - 1) {
    __threadfence();
    warp_finalize(a.acc, a.piece, a.dt, a.checksum, 1);
  }
}

// K2a: direct loads into registers (ld.global.nc, no L1 allocate). With PF,
// the next sub-grid's 16 values per lane are loaded before this one is
// transformed (register double buffer: more MLP, fewer resident warps).
template <int CHAINS, int KPC, bool PF, int MINB = 4>
__global__ void __launch_bounds__(kStepThreads, MINB) k_step(StepArgs a) {
  __shared__ unsigned long long s_limbs[TB_ACC_LIMBS];
  __shared__ long long s_min[kStepWarps];
  __shared__ double s_sums[kStepWarps][kSumBuf];
  if (finalizer_cta(a)) return;
  if (a.acc) {
    for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) s_limbs[i] = 0ULL;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int lane_off = 128 * (lane >> 3) + (lane & 7);
  const int64_t gstride = (int64_t)(gridDim.x - a.finalizer) * kStepWarps;
  double wmin = CUDART_INF;
  SumBuf sb;
  int64_t g = (int64_t)blockIdx.x * kStepWarps + warp;
  if (PF) {
    double nxt[16], nface = 0.0;
    if (g < a.n) {
      const double *src = a.old + g * TB_CELLS + lane_off;
#pragma unroll
      for (int i = 0; i < 16; ++i) nxt[i] = ld_stream(src + 8 * i);
      nface = load_face(a, g, lane);
    }
    for (; g < a.n; g += gstride) {
      double v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = nxt[i];
      const double face = nface;
      const int64_t gn = g + gstride;
      if (gn < a.n) {
        const double *src = a.old + gn * TB_CELLS + lane_off;
#pragma unroll
        for (int i = 0; i < 16; ++i) nxt[i] = ld_stream(src + 8 * i);
        nface = load_face(a, gn, lane);
      }
      subgrid_body<CHAINS, KPC>(a, g, lane, v, face, s_limbs, wmin, s_sums[warp], sb);
    }
  } else {
    for (; g < a.n; g += gstride) {
      const double *src = a.old + g * TB_CELLS + lane_off;
      double v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = ld_stream(src + 8 * i);
      const double face = load_face(a, g, lane);
      subgrid_body<CHAINS, KPC>(a, g, lane, v, face, s_limbs, wmin, s_sums[warp], sb);
    }
  }
  step_epilogue(a, s_limbs, s_min, wmin, s_sums[warp], sb.cnt);
}

// K2c: a warp PAIR per sub-grid, 8 cells per lane (half the registers of
// K2a, so twice the resident warps). Warp q of the pair holds blocks 2q and
// 2q+1; lane (h, bb, r) holds a[128(2q+bb) + r + 8(8h + i')], i' = 0..7. The
// pairwise order is kept exactly: the h=0 lane's sequential partial of r_j is
// handed to its h=1 partner (shuffle) which continues the same sequence;
// butterflies give B_{2q}+B_{2q+1} per warp; (B0+B1)+(B2+B3) is formed across
// the pair through shared memory behind a 64-thread named barrier.
template <int CHAINS, int KPC>
__device__ __forceinline__ void run_chains8(double (&v)[8], int chains, int kpc) {
  if (CHAINS > 0) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
#pragma unroll
      for (int k = 0; k < KPC; ++k) {
        const double c1 = kC1[k], c2 = kC2[k];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = xform(v[i], c1, c2);
      }
  } else {
    for (int c = 0; c < chains; ++c)
      for (int k = 0; k < kpc; ++k) {
        const double c1 = kC1[k], c2 = kC2[k];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = xform(v[i], c1, c2);
      }
  }
}

template <int CHAINS, int KPC>
__global__ void __launch_bounds__(kStepThreads, 6) k_step_pair(StepArgs a) {
  __shared__ unsigned long long s_limbs[TB_ACC_LIMBS];
  __shared__ long long s_min[kStepWarps];
  __shared__ double s_pair[2][kStepWarps / 2][2][2];   // [parity][pair][q][sum,min]
  if (finalizer_cta(a)) return;
  if (a.acc) {
    for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) s_limbs[i] = 0ULL;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int pair = warp >> 1, q = warp & 1;
  const int h = lane >> 4, bb = (lane >> 3) & 1, r = lane & 7;
  const int blk = 2 * q + bb;
  const int lane_off = 128 * blk + r + 64 * h;
  constexpr int kPairs = kStepWarps / 2;
  double wmin = CUDART_INF;
  int it = 0;
  for (int64_t g = (int64_t)blockIdx.x * kPairs + pair; g < a.n;
       g += (int64_t)(gridDim.x - a.finalizer) * kPairs, ++it) {
    const double *src = a.old + g * TB_CELLS + lane_off;
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ld_stream(src + 8 * i);
    if (q == 0 && lane < 8) {            // cells 0..7: block 0, i = 0
      const double *lf =
          g == 0 ? a.left_face : a.old + (g - 1) * TB_CELLS + (TB_CELLS - TB_FACE);
      v[0] = __dmul_rn(0.5, __dadd_rn(v[0], lf[r]));
    } else if (q == 1 && lane >= 24) {   // cells 504..511: block 3, i = 15
      const double *rf = g == a.n - 1 ? a.right_face : a.old + (g + 1) * TB_CELLS;
      v[7] = __dmul_rn(0.5, __dadd_rn(v[7], rf[r]));
    }
    run_chains8<CHAINS, KPC>(v, a.chains, a.kpc);
    double *dst = a.out + g * TB_CELLS + lane_off;
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[8 * i] = v[i];
    double part = v[0], m = v[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) m = fmin(m, v[i]);
    if (h == 0) {
#pragma unroll
      for (int i = 1; i < 8; ++i) part = __dadd_rn(part, v[i]);
    }
    const double from_h0 = __shfl_xor_sync(0xffffffffu, part, 16);
    double sacc = from_h0;   // h=1: continue the sequence a[j+64], a[j+72], ...
#pragma unroll
    for (int i = 0; i < 8; ++i) sacc = __dadd_rn(sacc, v[i]);
    // r-butterfly (xor 1, 2, 4) then the bb pair (xor 8); meaningful in h=1
#pragma unroll
    for (int x = 1; x < 16; x <<= 1) sacc = __dadd_rn(sacc, __shfl_xor_sync(0xffffffffu, sacc, x));
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, x));
    double(*slot)[2] = s_pair[it & 1][pair];
    if (lane == 16) {
      slot[q][0] = sacc;
      slot[q][1] = m;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
    if (q == 0 && lane == 0) {
      const double s = __dadd_rn(slot[0][0], slot[1][0]);
      const double mm = fmin(slot[0][1], slot[1][1]);
      if (a.sums) a.sums[g] = s;
      if (a.mins) a.mins[g] = mm;
      if (a.acc) acc_add_digits(s_limbs, s);
    }
    wmin = fmin(wmin, m);
  }
  step_epilogue(a, s_limbs, s_min, wmin);
}

// K2b: each warp streams its sub-grids through a kStages-deep ring of 4 KiB
// shared-memory slots filled by the bulk-copy (TMA) engine
// (cp.async.bulk ... mbarrier::complete_tx), so the next sub-grids are in
// flight while this one is transformed — no registers spent on prefetch.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// One sub-grid = four 1 KiB bulk copies into the padded slot, one barrier.
__device__ __forceinline__ void bulk_load_subgrid(double *slot, const double *src,
                                                  uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(TB_CELLS * 8)
               : "memory");
#pragma unroll
  for (int b = 0; b < 4; ++b)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(slot + b * kBlkPitch)),
        "l"(src + 128 * b), "r"(1024), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int CHAINS, int KPC, int STAGES, bool ALUMIN = false>
// 4 CTAs per SM (64 registers)
__global__ void __launch_bounds__(kStepThreads, 4) k_step_bulk(StepArgs a) {
  constexpr int kStages = STAGES;
  extern __shared__ __align__(128) double ring[];   // [warps][stages][padded 512]
  __shared__ __align__(8) uint64_t bars[kStepWarps][kStages];
  __shared__ unsigned long long s_limbs[TB_ACC_LIMBS];
  __shared__ long long s_min[kStepWarps];
  __shared__ double s_sums[kStepWarps][kSumBuf];
  // Programmatic dependent launch: the next step's grid is released now (all
  // CTAs of this one-wave grid are resident), so its CTAs take the SM slots
  // ours free and wait here — everything below reads the previous step's
  // output, so nothing runs before the previous grid has completed and
  // flushed. A no-op when launched without the attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (finalizer_cta(a)) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) s_limbs[i] = 0ULL;
  if (threadIdx.x == 0) {   // the deferred fold's min key and warp ticket
    s_min[0] = kKeyInf;
    s_min[1] = 0;
  }
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double *slots = ring + (size_t)warp * kStages * kSlot;
  const int64_t gstride = (int64_t)(gridDim.x - a.finalizer) * kStepWarps;
  const int64_t g0 = (int64_t)blockIdx.x * kStepWarps + warp;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      const int64_t g = g0 + s * gstride;
      if (g < a.n) bulk_load_subgrid(slots + s * kSlot, a.old + g * TB_CELLS, &bars[warp][s]);
    }
  }
  // deferred close: fold the previous step's share under the first bulk
  // copy's latency
  if (a.finalizer) fold_previous(a, g0, gstride, s_limbs, s_min);
  double wmin = CUDART_INF;
  SumBuf sb;
  int it = 0;
  for (int64_t g = g0; g < a.n; g += gstride, ++it) {
    const int s = it % kStages;
    // this sub-grid's ghost faces: issued before waiting for its bulk copy so
    // the two latencies overlap (neighbour warps are loading those lines now)
    const double face = load_face(a, g, lane);
    mbar_wait(&bars[warp][s], (uint32_t)((it / kStages) & 1));
    const double *src = slots + s * kSlot + kBlkPitch * (lane >> 3) + (lane & 7);
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = src[8 * i];
    __syncwarp();
    const int64_t gn = g + kStages * gstride;
    if (lane == 0 && gn < a.n) {
      // generic-proxy reads of the slot must be ordered before the
      // async-proxy write that refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load_subgrid(slots + s * kSlot, a.old + gn * TB_CELLS, &bars[warp][s]);
    }
    subgrid_body<CHAINS, KPC, ALUMIN>(a, g, lane, v, face, s_limbs, wmin, s_sums[warp], sb);
  }
  step_epilogue(a, s_limbs, s_min, wmin, s_sums[warp], sb.cnt);
}

int g_step_impl = TB_STEP_AUTO;
// programmatic dependent launch of consecutive steps (TB_STEP_PDL=0 disables)
const bool g_step_pdl = [] {
  const char *e = getenv("TB_STEP_PDL");
  return !(e && e[0] == '0');
}();
int g_step_spw = 0;   // sub-grids per warp per CTA; 0 = persistent (one wave)

// CTAs for n sub-grids: one resident wave (occ CTAs per SM) by default, or
// ceil(n / (warps * spw)) CTAs so the hardware scheduler balances the tail.
inline int step_grid_streaming(int64_t n, int occ);
// + the finalizer CTA when it is used (kept co-resident: at most occ*SMs CTAs)
inline int step_grid(int64_t n, int occ, int finalizer = 0) {
  int b = step_grid_streaming(n, occ);
  if (finalizer) {
    const int cap = tb::sm_count() * occ;
    if (b >= cap && cap > 1) b = cap - 1;
    b += 1;
  }
  return b;
}

inline int step_grid_streaming(int64_t n, int occ) {
  if (g_step_spw > 0) {
    int64_t b = (n + (int64_t)kStepWarps * g_step_spw - 1) / ((int64_t)kStepWarps * g_step_spw);
    return (int)(b < 1 ? 1 : (b > (1LL << 30) ? (1LL << 30) : b));
  }
  int64_t b = (n + kStepWarps - 1) / kStepWarps;
  const int64_t cap = (int64_t)tb::sm_count() * occ;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

inline int grid_for(int64_t work, int per_block, int max_blocks) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

template <typename K>
int occupancy(K kernel, int smem) {
  int o = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, kStepThreads, smem) !=
          cudaSuccess ||
      o < 1)
    o = 1;
  return o;
}

// the per-sub-grid min on the integer pipe (warp_min_alu); TB_STEP_ALUMIN=0
// keeps the FP64 fmin tree (A/B)
const bool g_step_alumin = [] {
  const char *e = getenv("TB_STEP_ALUMIN");
  return !(e && e[0] == '0');
}();

template <int CHAINS, int KPC, int STAGES, bool ALUMIN>
void launch_bulk_impl(cudaStream_t st, const StepArgs &a) {
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(k_step_bulk<CHAINS, KPC, STAGES, ALUMIN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, bulk_smem(STAGES));
    occ = occupancy(k_step_bulk<CHAINS, KPC, STAGES, ALUMIN>, bulk_smem(STAGES));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)step_grid(a.n, occ, a.finalizer));
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = bulk_smem(STAGES);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_step_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_step_bulk<CHAINS, KPC, STAGES, ALUMIN>, a);
}

template <int CHAINS, int KPC, int STAGES>
void launch_bulk(cudaStream_t st, const StepArgs &a) {
  if (g_step_alumin)
    launch_bulk_impl<CHAINS, KPC, STAGES, true>(st, a);
  else
    launch_bulk_impl<CHAINS, KPC, STAGES, false>(st, a);
}

int launch_step(cudaStream_t st, StepArgs a) {
  const bool fixed = a.chains == 3 && a.kpc == 5;
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.old) & 15) == 0);
  // AUTO = the single-slot bulk-copy ring (measured, % of HBM roofline at
  // 32768 / 262144 sub-grids: bulk1 70.4 / 87.5, reg 70.2 / 84.5,
  // bulk (2 slots) 65.2 / 86.2); registers when the state is not 16-B aligned.
  const bool bulk = aligned && g_step_impl == TB_STEP_BULK;
  if (g_step_impl == TB_STEP_AUTO && aligned && fixed) {
    launch_bulk<3, 5, 1>(st, a);
    return tb::last_error();
  }
  if (bulk) {
    if (fixed)
      launch_bulk<3, 5, kStages>(st, a);
    else
      launch_bulk<0, 0, kStages>(st, a);
  } else if (g_step_impl == TB_STEP_BULK1 && aligned) {
    if (fixed)
      launch_bulk<3, 5, 1>(st, a);
    else
      launch_bulk<0, 0, 1>(st, a);
  } else if (g_step_impl == TB_STEP_REGPF) {
    static int occ_f = 0, occ_g = 0;
    if (fixed) {
      if (!occ_f) occ_f = occupancy(k_step<3, 5, true>, 0);
      const int blocks = step_grid(a.n, occ_f, a.finalizer);
      k_step<3, 5, true><<<blocks, kStepThreads, 0, st>>>(a);
    } else {
      if (!occ_g) occ_g = occupancy(k_step<0, 0, true>, 0);
      const int blocks = step_grid(a.n, occ_g, a.finalizer);
      k_step<0, 0, true><<<blocks, kStepThreads, 0, st>>>(a);
    }
  } else if (g_step_impl == TB_STEP_LEAN && fixed) {
    // registers capped at 48 (5 CTAs = 40 warps per SM; a few spill slots)
    static int occ = 0;
    if (!occ) occ = occupancy(k_step<3, 5, false, 5>, 0);
    k_step<3, 5, false, 5><<<step_grid(a.n, occ, a.finalizer), kStepThreads, 0, st>>>(a);
  } else if (g_step_impl == TB_STEP_PAIR) {
    // a warp pair per sub-grid: the grid helper counts pairs as "warps"
    static int occ_f = 0, occ_g = 0;
    int &occ = fixed ? occ_f : occ_g;
    if (!occ) occ = fixed ? occupancy(k_step_pair<3, 5>, 0) : occupancy(k_step_pair<0, 0>, 0);
    const int blocks = step_grid(2 * a.n, occ, a.finalizer);
    if (fixed)
      k_step_pair<3, 5><<<blocks, kStepThreads, 0, st>>>(a);
    else
      k_step_pair<0, 0><<<blocks, kStepThreads, 0, st>>>(a);
  } else {
    static int occ_f = 0, occ_g = 0;
    if (fixed) {
      if (!occ_f) occ_f = occupancy(k_step<3, 5, false>, 0);
      const int blocks = step_grid(a.n, occ_f, a.finalizer);
      k_step<3, 5, false><<<blocks, kStepThreads, 0, st>>>(a);
    } else {
      if (!occ_g) occ_g = occupancy(k_step<0, 0, false>, 0);
      const int blocks = step_grid(a.n, occ_g, a.finalizer);
      k_step<0, 0, false><<<blocks, kStepThreads, 0, st>>>(a);
    }
  }
  return tb::last_error();
}


// ------------------------------------------- peer-memory accumulator reduce --
// The step's cross-rank reduction without a collective library: every rank
// adds its local limbs into EVERY rank's accumulator with system-scope
// atomics over NVLink (a handful of non-zero limbs), bumps each rank's
// arrival counter, then spins until its own counter reaches nranks and
// finalises locally — all ranks round the identical exact sum. The arrival
// wait is also the cross-rank step barrier the peer-memory halo relies on.
// peer_accs[p] points at rank p's accumulator for this step's parity (mapped
// with CUDA IPC; the own entry is local). Accumulators alternate parity each
// step, so a fast rank's next contributions never meet a slow rank's reset.
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct P2pWatch {          // the arrival wait's watchdog (tb_acc_allreduce_p2p_ex)
  int64_t timeout_ns;      // 0: wait forever
  int64_t rank, step;
  volatile int64_t *diag;  // mapped pinned host words, readable after a trap
};

__global__ void k_acc_allreduce_p2p(int64_t *local_acc, int64_t *const *peer_accs,
                                    int nranks, int64_t *my_acc, double *piece, double *dt,
                                    double *checksum, P2pWatch w) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  // 1. publish this rank's contribution to every rank (including itself)
  for (int p = 0; p < nranks; ++p) {
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(peer_accs[p]);
    for (int i = lane; i < TB_ACC_LIMBS; i += 32) {
      const long long v = ld_cg_s64(local_acc + i);
      if (v) atomicAdd_system(dst + i, (unsigned long long)v);
    }
    if (lane == 0)
      atomicMin_system(reinterpret_cast<long long *>(dst) + TB_ACC_MIN_WORD,
                       ld_cg_s64(local_acc + TB_ACC_MIN_WORD));
  }
  __threadfence_system();
  __syncwarp();
  if (lane == 0)
    for (int p = 0; p < nranks; ++p)
      atomicAdd_system(reinterpret_cast<unsigned long long *>(peer_accs[p]) + TB_ACC_COUNT_WORD,
                       1ULL);
  // 2. local accumulator is free again
  for (int i = lane; i < TB_ACC_WORDS; i += 32)
    local_acc[i] = (i == TB_ACC_MIN_WORD) ? kKeyInf : 0;
  // 3. wait for every rank's contribution, then round it (and reset)
  if (lane == 0) {
    const unsigned long long *cnt =
        reinterpret_cast<const unsigned long long *>(my_acc) + TB_ACC_COUNT_WORD;
    // a rank that never arrives (died, or launched a different step count)
    // must not hang the job: after the watchdog's timeout the kernel leaves
    // (rank, step, arrivals seen) in host memory and traps, and the host
    // reports which rank waited for whom (timeout 0 = wait forever, e.g.
    // under a debugger or a profiler's kernel replay on another rank)
    unsigned long long t0, t, seen;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((seen = ld_acquire_sys_u64(cnt)) < (unsigned long long)nranks) {
      __nanosleep(200);
      if (w.timeout_ns <= 0) continue;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((int64_t)(t - t0) > w.timeout_ns) {
        if (w.diag) {
          w.diag[1] = w.rank;
          w.diag[2] = w.step;
          w.diag[3] = (int64_t)seen;
          __threadfence_system();
          w.diag[0] = 0x7470325774696d65LL;   // "tp2Wtime": the words are valid
          __threadfence_system();
        }
        __trap();
      }
    }
  }
  __syncwarp();
  __threadfence_system();
  warp_finalize(my_acc, piece, dt, checksum, 1);
}

}  // namespace

// ------------------------------------------------------------ launchers --
extern "C" {

int tb_set_option(int key, int value) {
  if (key == TB_OPT_STEP_IMPL) {
    if (value < TB_STEP_AUTO || value > TB_STEP_BULK1) return TB_E_INVALID;
    g_step_impl = value;
    return TB_OK;
  }
  if (key == TB_OPT_STEP_SPW) {
    if (value < 0) return TB_E_INVALID;
    g_step_spw = value;
    return TB_OK;
  }
  return TB_E_INVALID;
}

int tb_launch(tb_stream_t s, int op, int kind, double c1, double c2, double *d,
              int64_t n) {
  if (n < 0 || (n > 0 && d == nullptr)) return TB_E_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  if (op == TB_OP_KIND) {
    if (kind < 0 || kind >= TB_KINDS) return TB_E_INVALID;
    static const double h1[TB_KINDS] = {1.0000003, 0.9999998, 1.0000001, 0.9999997,
                                        1.0000002};
    static const double h2[TB_KINDS] = {1e-07, -1e-07, 2e-07, 5e-08, -2e-07};
    c1 = h1[kind];
    c2 = h2[kind];
    op = TB_OP_AFFINE;
  }
  if (op == TB_OP_TRAP) {   // fault injection: a device-side trap
    k_trap<<<1, 32, 0, st>>>();
    return tb::last_error();
  }
  if (op == TB_OP_NONE || n == 0) {
    k_empty<<<1, 32, 0, st>>>();
    return tb::last_error();
  }
  if (op != TB_OP_AFFINE) return TB_E_INVALID;
  const int blocks = grid_for((n + 1) / 2, 256, tb::sm_count() * 8);
  k_launch<TB_OP_AFFINE><<<blocks, 256, 0, st>>>(d, n, c1, c2);
  return tb::last_error();
}

int tb_launch_gather_done(tb_stream_t s, int op, int kind, double c1, double c2,
                          const double *const *src, double *const *dst, const int64_t *n,
                          int members, const tb_done *done) {
  if (members < 1 || members > TB_GATHER_MAX || !src || !dst || !n) return TB_E_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  if (op == TB_OP_TRAP) {
    k_trap<<<1, 32, 0, st>>>();
    return tb::last_error();
  }
  if (op == TB_OP_KIND) {
    if (kind < 0 || kind >= TB_KINDS) return TB_E_INVALID;
    static const double h1[TB_KINDS] = {1.0000003, 0.9999998, 1.0000001, 0.9999997,
                                        1.0000002};
    static const double h2[TB_KINDS] = {1e-07, -1e-07, 2e-07, 5e-08, -2e-07};
    c1 = h1[kind];
    c2 = h2[kind];
  } else if (op == TB_OP_NONE) {
    if (done) return TB_E_INVALID;   // nothing would signal the word
    k_empty<<<1, 32, 0, st>>>();
    return tb::last_error();
  } else if (op != TB_OP_AFFINE) {
    return TB_E_INVALID;
  }
  GatherArgs a;
  int64_t nmax = 0;
  for (int i = 0; i < members; ++i) {
    if (!src[i] || !dst[i] || n[i] < 0 || (n[i] & 1) ||
        ((reinterpret_cast<uintptr_t>(src[i]) | reinterpret_cast<uintptr_t>(dst[i])) & 15))
      return TB_E_INVALID;
    a.src[i] = src[i];
    a.dst[i] = dst[i];
    a.n[i] = n[i];
    nmax = n[i] > nmax ? n[i] : nmax;
  }
  a.c1 = c1;
  a.c2 = c2;
  if (!done_args(done, &a.done)) return TB_E_INVALID;
  const int bx = grid_for(nmax / 2 > 0 ? nmax / 2 : 1, 256, 64);
  k_launch_gather<<<dim3((unsigned)bx, (unsigned)members), 256, 0, st>>>(a);
  return tb::last_error();
}

int tb_launch_gather(tb_stream_t s, int op, int kind, double c1, double c2,
                     const double *const *src, double *const *dst, const int64_t *n,
                     int members) {
  return tb_launch_gather_done(s, op, kind, c1, c2, src, dst, n, members, nullptr);
}

int tb_launch_gather_edge(tb_stream_t s, int kind, const double *const *src,
                          double *const *dst, const int64_t *g0, const int32_t *nsub,
                          const uint8_t *flags, int members, const double *faces,
                          double *mins, double *sums, int64_t S, const tb_done *done) {
  if (members < 1 || members > TB_GATHER_MAX || !src || !dst || !g0 || !nsub || !flags ||
      kind < 0 || kind >= TB_KINDS || S < 1)
    return TB_E_INVALID;
  static const double h1[TB_KINDS] = {1.0000003, 0.9999998, 1.0000001, 0.9999997, 1.0000002};
  static const double h2[TB_KINDS] = {1e-07, -1e-07, 2e-07, 5e-08, -2e-07};
  GatherEdgeArgs a;
  int nmax = 1;
  bool fold = false, reduce = false;
  for (int i = 0; i < members; ++i) {
    if (!src[i] || !dst[i] || nsub[i] < 1 || g0[i] < 0 || g0[i] + nsub[i] > S ||
        ((reinterpret_cast<uintptr_t>(src[i]) | reinterpret_cast<uintptr_t>(dst[i])) & 15))
      return TB_E_INVALID;
    a.src[i] = src[i];
    a.dst[i] = dst[i];
    a.g0[i] = g0[i];
    a.nsub[i] = nsub[i];
    a.flags[i] = flags[i];
    fold |= (flags[i] & 1) != 0;
    reduce |= (flags[i] & 2) != 0;
    nmax = nsub[i] > nmax ? nsub[i] : nmax;
  }
  if ((fold && !faces) || (reduce && (!mins || !sums))) return TB_E_INVALID;
  a.faces = faces;
  a.mins = mins;
  a.sums = sums;
  a.S = S;
  a.c1 = h1[kind];
  a.c2 = h2[kind];
  if (!done_args(done, &a.done)) return TB_E_INVALID;
  k_launch_gather_edge<<<dim3((unsigned)nmax, (unsigned)members), TB_CELLS / 2, 0,
                         reinterpret_cast<cudaStream_t>(s)>>>(a);
  return tb::last_error();
}

int tb_transform(tb_stream_t s, int kind, double *d, int64_t n) {
  return tb_launch(s, TB_OP_KIND, kind, 0.0, 0.0, d, n);
}

int tb_barrier(tb_stream_t s) {
  k_empty<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>();
  return tb::last_error();
}

int tb_spin(tb_stream_t s, int64_t ns) {
  if (ns < 0) return TB_E_INVALID;
  k_spin<<<1, 1, 0, reinterpret_cast<cudaStream_t>(s)>>>(ns);
  return tb::last_error();
}

int tb_init_cells(tb_stream_t s, double *cells, int64_t subgrids, int64_t lo,
                  int64_t n) {
  if (!cells || subgrids < 1 || lo < 0 || n < 0 || lo + n > subgrids)
    return TB_E_INVALID;
  if (n == 0) return TB_OK;
  const int blocks = grid_for(n * TB_CELLS, 256, tb::sm_count() * 8);
  k_init_cells<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(cells, subgrids,
                                                                      lo, n);
  return tb::last_error();
}

static int step_args(StepArgs *a, const double *old, double *out, int64_t n,
                     const double *left_face, const double *right_face, int chains,
                     int kpc, double *mins, double *sums, int64_t *acc) {
  if (n < 0 || chains < 0 || kpc < 0 || kpc > TB_KINDS) return TB_E_INVALID;
  if (n > 0 && (!old || !out || old == out || !left_face || !right_face))
    return TB_E_INVALID;
  *a = StepArgs{old, out, n, left_face, right_face, chains, kpc, mins, sums, acc,
                nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return TB_OK;
}

int tb_step(tb_stream_t s, const double *old, double *out, int64_t n,
            const double *left_face, const double *right_face, int chains,
            int kernels_per_chain, double *mins, double *sums, int64_t *acc) {
  StepArgs a;
  const int r = step_args(&a, old, out, n, left_face, right_face, chains,
                          kernels_per_chain, mins, sums, acc);
  if (r != TB_OK) return r;
  if (n == 0) return TB_OK;
  return launch_step(reinterpret_cast<cudaStream_t>(s), a);
}

int tb_step_final(tb_stream_t s, const double *old, double *out, int64_t n,
                  const double *left_face, const double *right_face, int chains,
                  int kernels_per_chain, double *mins, double *sums, int64_t *acc,
                  double *piece, double *dt, double *checksum) {
  StepArgs a;
  int r = step_args(&a, old, out, n, left_face, right_face, chains, kernels_per_chain,
                    mins, sums, acc);
  if (r != TB_OK) return r;
  if (!acc) return TB_E_INVALID;
  if (n == 0) return tb_acc_finalize(s, acc, piece, dt, checksum, 1);
  a.piece = piece;
  a.dt = dt;
  a.checksum = checksum;
  a.finalize = 1;
  return launch_step(reinterpret_cast<cudaStream_t>(s), a);
}

int tb_step_close(tb_stream_t s, const double *sums, const double *mins, int64_t n,
                  int64_t *acc, double *piece, double *dt, double *checksum) {
  if (!acc || n < 0 || (n > 0 && (!sums || !mins))) return TB_E_INVALID;
  int64_t blocks = (n + 2047) / 2048;   // >= 8 values per thread
  const int64_t cap = (int64_t)tb::sm_count() * 2;
  if (blocks < 1) blocks = 1;
  if (blocks > cap) blocks = cap;
  k_step_close<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      sums, mins, n, acc, piece, dt, checksum);
  return tb::last_error();
}

int tb_step_deferred(tb_stream_t s, const double *old, double *out, int64_t n,
                     const double *left_face, const double *right_face, int chains,
                     int kernels_per_chain, double *sums, double *mins,
                     const double *prev_sums, const double *prev_mins, int64_t *acc,
                     double *prev_piece, double *prev_dt, double *checksum) {
  StepArgs a;
  int r = step_args(&a, old, out, n, left_face, right_face, chains, kernels_per_chain,
                    mins, sums, nullptr);
  if (r != TB_OK) return r;
  if (n > 0 && (!sums || !mins)) return TB_E_INVALID;
  if (prev_sums && (!prev_mins || !acc || prev_sums == sums)) return TB_E_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  if (n == 0)
    return prev_sums ? tb_step_close(s, prev_sums, prev_mins, 0, acc, prev_piece, prev_dt,
                                     checksum)
                     : TB_OK;
  if (!prev_sums) return launch_step(st, a);
  if ((reinterpret_cast<uintptr_t>(old) & 15) != 0) {
    // the in-launch close lives in the bulk-copy kernel only
    r = launch_step(st, a);
    return r == TB_OK ? tb_step_close(s, prev_sums, prev_mins, n, acc, prev_piece, prev_dt,
                                      checksum)
                      : r;
  }
  a.prev_acc = acc;
  a.prev_sums = prev_sums;
  a.prev_mins = prev_mins;
  a.prev_piece = prev_piece;
  a.prev_dt = prev_dt;
  a.checksum = checksum;
  a.finalizer = 1;
  if (chains == 3 && kernels_per_chain == 5)
    launch_bulk<3, 5, 1>(st, a);
  else
    launch_bulk<0, 0, 1>(st, a);
  return tb::last_error();
}

int tb_acc_reset(tb_stream_t s, int64_t *acc) {
  if (!acc) return TB_E_INVALID;
  k_acc_reset<<<1, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(acc);
  return tb::last_error();
}

int tb_acc_add(tb_stream_t s, const double *x, int64_t n, int64_t *acc) {
  if (!acc || n < 0 || (n > 0 && !x)) return TB_E_INVALID;
  if (n == 0) return TB_OK;
  const int blocks = grid_for(n, 256, tb::sm_count() * 4);
  k_acc_add<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(x, n, acc);
  return tb::last_error();
}

int tb_acc_finalize(tb_stream_t s, int64_t *acc, double *piece, double *dt,
                    double *checksum, int reset) {
  if (!acc) return TB_E_INVALID;
  k_acc_finalize<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(acc, piece, dt,
                                                                   checksum, reset);
  return tb::last_error();
}

int tb_acc_allreduce_p2p_ex(tb_stream_t s, int64_t *local_acc, int64_t *const *peer_accs,
                            int nranks, int64_t *my_acc, double *piece, double *dt,
                            double *checksum, int64_t timeout_ns, int64_t rank, int64_t step,
                            int64_t *diag) {
  if (!local_acc || !peer_accs || !my_acc || nranks < 1 || timeout_ns < 0) return TB_E_INVALID;
  P2pWatch w{timeout_ns, rank, step, diag};
  k_acc_allreduce_p2p<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      local_acc, peer_accs, nranks, my_acc, piece, dt, checksum, w);
  return tb::last_error();
}

int tb_acc_allreduce_p2p(tb_stream_t s, int64_t *local_acc, int64_t *const *peer_accs,
                         int nranks, int64_t *my_acc, double *piece, double *dt,
                         double *checksum) {
  // default watchdog: TB_P2P_TIMEOUT_S seconds (default 30; 0 disables)
  static const int64_t timeout_ns = [] {
    const char *e = getenv("TB_P2P_TIMEOUT_S");
    const double sec = e ? atof(e) : 30.0;
    return (int64_t)(sec > 0 ? sec * 1e9 : 0);
  }();
  return tb_acc_allreduce_p2p_ex(s, local_acc, peer_accs, nranks, my_acc, piece, dt, checksum,
                                 timeout_ns, -1, -1, nullptr);
}

}  // extern "C"
