// tb_kernels.cu — sm_100a kernels for the sub-grid step path.
//
// K1  k_launch      : kernel_transform(kind) / registered affine kinds on a
//                     fused staging buffer (src/miniapp.py:40-53,
//                     src/executors.py:257-284). HBM-bound, 16 B per cell.
// K2  k_step        : one fused time step over many sub-grids, one warp per
//                     sub-grid (src/miniapp.py:116-133 == src/reference.py:31-47),
//                     with the step's exact sum and min folded into a
//                     superaccumulator (src/miniapp.py:138-171).
// K4  k_acc_finalize: correctly rounded sum (== math.fsum) + dt + checksum.
//
// Bit-exactness (SURVEY.md §7 hard part 1): every transform is
// __dmul_rn followed by __dadd_rn — never an FMA; the per-sub-grid sum is
// numpy's pairwise order, mapped onto one warp: lane j owns block j/8 and
// accumulator j%8 of the 4x128 pairwise tree and holds
// a[128*(j/8) + (j%8) + 8*i], i = 0..15, in registers.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

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
                                          long long block_min_key,
                                          int64_t *acc) {
  for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) {
    const unsigned long long v = s_limbs[i];
    if (v) atomicAdd(reinterpret_cast<unsigned long long *>(acc) + i, v);
  }
  if (threadIdx.x == 0)
    atomicMin(reinterpret_cast<long long *>(acc) + TB_ACC_MIN_WORD, block_min_key);
}

// ------------------------------------------------------------------ K2 --
constexpr int kStepThreads = 256;
constexpr int kStepWarps = kStepThreads / 32;

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

template <int CHAINS, int KPC>
__global__ void __launch_bounds__(kStepThreads)
    k_step(const double *__restrict__ old, double *__restrict__ out, int64_t n,
           const double *__restrict__ left_face, const double *__restrict__ right_face,
           int chains, int kpc, double *__restrict__ mins, double *__restrict__ sums,
           int64_t *__restrict__ acc) {
  __shared__ unsigned long long s_limbs[TB_ACC_LIMBS];
  __shared__ long long s_min[kStepWarps];
  if (acc) {
    for (int i = threadIdx.x; i < TB_ACC_LIMBS; i += blockDim.x) s_limbs[i] = 0ULL;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int r = lane & 7;                 // accumulator within a 128-block
  const int lane_off = 128 * (lane >> 3) + r;
  double wmin = CUDART_INF;

  for (int64_t g = (int64_t)blockIdx.x * kStepWarps + warp; g < n;
       g += (int64_t)gridDim.x * kStepWarps) {
    const double *src = old + g * TB_CELLS + lane_off;
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = ld_stream(src + 8 * i);
    // Ghost fold against the previous generation (src/miniapp.py:119-126):
    // cells 0..7 are lanes 0..7 at i = 0; cells 504..511 are lanes 24..31 at
    // i = 15. The add rounds; the *0.5 is exact.
    if (lane < 8) {
      const double *lf =
          g == 0 ? left_face : old + (g - 1) * TB_CELLS + (TB_CELLS - TB_FACE);
      v[0] = __dmul_rn(0.5, __dadd_rn(v[0], lf[r]));
    } else if (lane >= 24) {
      const double *rf = g == n - 1 ? right_face : old + (g + 1) * TB_CELLS;
      v[15] = __dmul_rn(0.5, __dadd_rn(v[15], rf[r]));
    }
    run_chains<CHAINS, KPC>(v, chains, kpc);
    double *dst = out + g * TB_CELLS + lane_off;
#pragma unroll
    for (int i = 0; i < 16; ++i) dst[8 * i] = v[i];

    // numpy pairwise sum: r_j = a[j] + a[j+8] + ... (sequential), then
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) per block, (B0+B1)+(B2+B3).
    double s = v[0];
    double m = v[0];
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
    if (lane == 0) {
      if (sums) sums[g] = s;
      if (mins) mins[g] = m;
      if (acc) acc_add_digits(s_limbs, s);
    }
    wmin = fmin(wmin, m);
  }
  if (acc) {
    if (lane == 0) s_min[warp] = min_key(wmin);
    __syncthreads();
    long long bm = s_min[0];
#pragma unroll
    for (int w = 1; w < kStepWarps; ++w) bm = min(bm, s_min[w]);
    acc_flush(s_limbs, bm, acc);
  }
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
    acc[i] = (i == TB_ACC_MIN_WORD) ? 0x7ff0000000000000LL /* key(+inf) */ : 0;
}

// Correctly rounded (half-even) value of the exact sum held in the limbs.
__device__ double acc_round(const int64_t *acc) {
  constexpr int ND = TB_ACC_LIMBS + 2;
  uint32_t d[ND];
  long long carry = 0;
  for (int i = 0; i < TB_ACC_LIMBS; ++i) {
    const long long v = acc[i] + carry;      // |acc[i]| < 2^62 by construction
    d[i] = (uint32_t)(v & 0xffffffffLL);
    carry = v >> 32;                         // arithmetic shift
  }
  d[TB_ACC_LIMBS] = (uint32_t)(carry & 0xffffffffLL);
  d[TB_ACC_LIMBS + 1] = (uint32_t)((carry >> 32) & 0xffffffffLL);
  const bool neg = (d[ND - 1] >> 31) & 1u;
  if (neg) {
    unsigned long long c = 1;
    for (int i = 0; i < ND; ++i) {
      const unsigned long long v = (unsigned long long)(uint32_t)~d[i] + c;
      d[i] = (uint32_t)v;
      c = v >> 32;
    }
  }
  int top = -1;
  for (int i = ND - 1; i >= 0; --i)
    if (d[i]) {
      top = i;
      break;
    }
  if (top < 0) return 0.0;
  const int nbits = top * 32 + (32 - __clz((int)d[top]));
  const int shift = nbits > 53 ? nbits - 53 : 0;
  // Gather bits [shift, nbits) into mant; guard = bit shift-1; sticky below.
  auto bit = [&](int k) -> unsigned { return (d[k >> 5] >> (k & 31)) & 1u; };
  unsigned long long mant = 0;
  for (int k = nbits - 1; k >= shift; --k) mant = (mant << 1) | bit(k);
  if (shift > 0) {
    const unsigned guard = bit(shift - 1);
    bool sticky = false;
    const int gk = shift - 1;                  // bits strictly below guard
    for (int w = 0; w < (gk >> 5) && !sticky; ++w) sticky = d[w] != 0;
    if (!sticky && (gk & 31)) sticky = (d[gk >> 5] & ((1u << (gk & 31)) - 1u)) != 0;
    if (guard && (sticky || (mant & 1ULL))) mant += 1;
  }
  const double r = scalbn((double)mant, shift - TB_ACC_BIAS);
  return neg ? -r : r;
}

__global__ void k_acc_finalize(int64_t *acc, double *piece, double *dt,
                               double *checksum, int reset) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double p = acc_round(acc);
  if (piece) *piece = p;
  if (dt) *dt = key_to_double(acc[TB_ACC_MIN_WORD]);
  if (checksum) *checksum = __dadd_rn(*checksum, p);   // src/miniapp.py:227
  if (reset)
    for (int i = 0; i < TB_ACC_WORDS; ++i)
      acc[i] = (i == TB_ACC_MIN_WORD) ? 0x7ff0000000000000LL : 0;
}

inline int grid_for(int64_t work, int threads, int max_blocks) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

}  // namespace

// ------------------------------------------------------------ launchers --
extern "C" {

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
  if (op == TB_OP_NONE || n == 0) {
    k_empty<<<1, 32, 0, st>>>();
    return tb::last_error();
  }
  if (op != TB_OP_AFFINE) return TB_E_INVALID;
  const int blocks = grid_for((n + 1) / 2, 256, tb::sm_count() * 8);
  k_launch<TB_OP_AFFINE><<<blocks, 256, 0, st>>>(d, n, c1, c2);
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

int tb_step(tb_stream_t s, const double *old, double *out, int64_t n,
            const double *left_face, const double *right_face, int chains,
            int kernels_per_chain, double *mins, double *sums, int64_t *acc) {
  if (n < 0 || chains < 0 || kernels_per_chain < 0 ||
      kernels_per_chain > TB_KINDS)
    return TB_E_INVALID;
  if (n == 0) return TB_OK;
  if (!old || !out || old == out || !left_face || !right_face) return TB_E_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  // Persistent grid: exactly the resident CTAs of one wave (occupancy-derived,
  // x148 SMs); each warp walks sub-grids with a grid stride.
  const bool fixed = chains == 3 && kernels_per_chain == 5;
  static int occ_fixed = 0, occ_generic = 0;
  int &occ = fixed ? occ_fixed : occ_generic;
  if (occ == 0) {
    int o = 0;
    cudaError_t e = fixed ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                &o, k_step<3, 5>, kStepThreads, 0)
                          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                &o, k_step<0, 0>, kStepThreads, 0);
    occ = (e == cudaSuccess && o > 0) ? o : 4;
  }
  const int blocks = grid_for(n, kStepWarps, tb::sm_count() * occ);
  if (fixed)
    k_step<3, 5><<<blocks, kStepThreads, 0, st>>>(old, out, n, left_face, right_face,
                                                  chains, kernels_per_chain, mins,
                                                  sums, acc);
  else
    k_step<0, 0><<<blocks, kStepThreads, 0, st>>>(old, out, n, left_face, right_face,
                                                  chains, kernels_per_chain, mins,
                                                  sums, acc);
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

}  // extern "C"
