// tb_fmm.cu — K7: FMM gravity over a uniform octree of 8^3-cell sub-grids
// (the north_star's "FMM monopole/multipole stencil-interaction kernels",
// BASELINE.json config 3).
//
// PARITY UNPINNED (the reference has no gravity solver): the
// spec is the self-authored oracle/fmm_oracle.py; results agree with it per
// cell within the north_star's FP64 tolerance (1e-10 relative), not bit for
// bit — FMAs and rsqrt are used freely here.
//
// Layout (one device workspace, tb_fmm_workspace_bytes):
//   for level l in [0, L): Mhat_l [N_l^3][20], Mred_l [N_l^3][18], Loc_l
//   [N_l^3][20] (N_l = 8*2^l, cells z,y,x with x fastest, one record per cell),
//   Dtab_l [33][912] (l >= 1); L0part [8][512][20].
//   Mhat holds the raw Cartesian moments pre-multiplied by the M2L source
//   coefficient -(-1)^m mult(B)/m! (M2M input); Mred their traceless
//   reduction to 16 moments + 2 zero pads (M2L input), so the interaction is
//   a pure FMA chain; Dtab_l holds, per stencil stage, the derivative tensors
//   of the 27 distinct child offsets (zero for near pairs).
//
// Kernels
//   k_fmm_up    P2M+M2M, one level per launch, one thread per parent: child
//               offsets are +-h/2 per axis, so the multipole sums are signed
//               sums of the children (compile-time signs), no shuffles.
//   k_fmm_m2l   multipole interactions of ALL levels in ONE launch (a CTA per
//               level-l sub-grid, heaviest level first; level 0 split over 8
//               CTAs). The interaction stencil is walked as 33 parent-near
//               offsets P: for each, the 8^3 x 18 source block at 2P is staged
//               by one 4-D TMA load (OOB = zero mass: the isolated boundary)
//               plus a bulk copy of that stage's 27 derivative tensors,
//               double-buffered on mbarriers; each thread (one target cell)
//               takes the 8 children of its parent's neighbour P and contracts
//               their moments with the tensor of its offset (LDS.128 pairs,
//               70 FMAs on the traceless reduction, no branch: near pairs
//               have D = 0).
//   k_fmm_down  L2L, one level per launch (level 0: sums the 8 partials).
//   k_fmm_leaf_mma  monopole interactions at the leaves on the FP64 tensor
//               cores (default): a 264-point stencil whose weights 1/|q|,
//               q/|q|^3 depend only on the integer offset q is, for the two
//               octants of a parent that differ in x, a GEMM (rows = parents,
//               K = source offsets, N = 4 components x 2 octants) done with
//               mma.sync.m8n8k4.f64 on leaf densities staged parity-split in
//               shared memory; then the parent's local expansion is evaluated
//               at the leaf (L2P).
//   k_fmm_leaf  the same on the DFMA pipe (TB_LEAF_MMA=0): a warp owns one
//               octant so q is warp-uniform and the weights come from
//               constant memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <cmath>
#include <utility>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace {

constexpr int NC = 20;
constexpr int kMaxLevel = 7;

// ------------------------------------------------------- compile-time tables
struct Comp {
  int n, a[3];
};
constexpr Comp kComps[NC] = {
    {0, {0, 0, 0}}, {1, {0, 0, 0}}, {1, {1, 0, 0}}, {1, {2, 0, 0}}, {2, {0, 0, 0}},
    {2, {0, 1, 0}}, {2, {0, 2, 0}}, {2, {1, 1, 0}}, {2, {1, 2, 0}}, {2, {2, 2, 0}},
    {3, {0, 0, 0}}, {3, {0, 0, 1}}, {3, {0, 0, 2}}, {3, {0, 1, 1}}, {3, {0, 1, 2}},
    {3, {0, 2, 2}}, {3, {1, 1, 1}}, {3, {1, 1, 2}}, {3, {1, 2, 2}}, {3, {2, 2, 2}}};

constexpr int find_comp(int n, const int *a) {
  for (int k = 0; k < NC; ++k) {
    if (kComps[k].n != n) continue;
    bool eq = true;
    for (int q = 0; q < n; ++q)
      if (kComps[k].a[q] != a[q]) eq = false;
    if (eq) return k;
  }
  return -1;
}

// Index of the sorted concatenation of two components (or -1 beyond order 3).
constexpr int merge(int t, int s) {
  int a[6] = {0, 0, 0, 0, 0, 0};
  int n = 0;
  for (int q = 0; q < kComps[t].n; ++q) a[n++] = kComps[t].a[q];
  for (int q = 0; q < kComps[s].n; ++q) a[n++] = kComps[s].a[q];
  if (n > 3) return -1;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (a[j] < a[i]) {
        const int x = a[i];
        a[i] = a[j];
        a[j] = x;
      }
  return find_comp(n, a);
}

constexpr int fact(int n) { return n <= 1 ? 1 : n * fact(n - 1); }

constexpr int mult(int s) {
  int c[3] = {0, 0, 0};
  for (int q = 0; q < kComps[s].n; ++q) c[kComps[s].a[q]]++;
  return fact(kComps[s].n) / (fact(c[0]) * fact(c[1]) * fact(c[2]));
}

// M2L source coefficient: L^(n)_A = sum_s [-(-1)^m mult(s)/m!] M_s D_{A+s}.
constexpr double m2l_scale(int s) {
  return (kComps[s].n % 2 ? 1.0 : -1.0) * mult(s) / fact(kComps[s].n);
}
// L2L monomial coefficient mult(B)/k!.
constexpr double l2l_scale(int b) { return double(mult(b)) / fact(kComps[b].n); }

struct Term {
  int t, s, b, c;
};
template <int CAP>
struct Table {
  Term v[CAP];
  int n;
};

// M2L: L[t] += Mhat[s] * D[merge(t,s)]   (t, s, b = D index). Source-major
// order: consecutive FMAs update different accumulators (ILP).
constexpr Table<84> make_m2l() {
  Table<84> T{};
  int k = 0;
  for (int s = 0; s < NC; ++s)
    for (int t = 0; t < NC; ++t)
      if (kComps[t].n + kComps[s].n <= 3) T.v[k++] = Term{t, s, merge(t, s), 1};
  T.n = k;
  return T;
}
// L2L / L2P: Lchild[t] += Lparent[merge(t,b)] * mono_hat[b]   (t, s = parent, b)
constexpr Table<84> make_l2l() {
  Table<84> T{};
  int k = 0;
  for (int t = 0; t < NC; ++t)
    for (int b = 0; b < NC; ++b)
      if (kComps[t].n + kComps[b].n <= 3) T.v[k++] = Term{t, merge(t, b), b, 1};
  T.n = k;
  return T;
}
// M2M: Mparent[t] += c * Mchild[s] * d^b, from prod_a (s_a + d_a) over the
// subsets of t's index positions.
constexpr Table<84> make_m2m() {
  Table<84> T{};
  int k = 0;
  for (int t = 0; t < NC; ++t) {
    const int n = kComps[t].n;
    for (int mask = 0; mask < (1 << n); ++mask) {
      int sa[3] = {0, 0, 0}, ra[3] = {0, 0, 0};
      int ns = 0, nr = 0;
      for (int q = 0; q < n; ++q) {
        if (mask >> q & 1)
          sa[ns++] = kComps[t].a[q];
        else
          ra[nr++] = kComps[t].a[q];
      }
      const int b = find_comp(ns, sa), s = find_comp(nr, ra);   // already sorted
      bool found = false;
      for (int e = 0; e < k; ++e)
        if (T.v[e].t == t && T.v[e].s == s && T.v[e].b == b) {
          T.v[e].c += 1;
          found = true;
        }
      if (!found) T.v[k++] = Term{t, s, b, 1};
    }
  }
  T.n = k;
  return T;
}

constexpr auto kM2L = make_m2l();
constexpr auto kL2L = make_l2l();
constexpr auto kM2M = make_m2m();
static_assert(kM2L.n == 84 && kL2L.n == 84 && kM2M.n == 84, "term tables");

// Traceless reduction. The derivative tensors of 1/r are traceless
// (D_{..zz} = -D_{..xx} - D_{..yy}), so (i) a source's zz-containing moments
// fold into reduced moments (M'xx = Mxx - Mzz, M'xxx = Mxxx - Mxzz, ...), 16
// instead of 20, and (ii) the local expansions are traceless too, so only
// their 16 independent components (no zz index pair) are accumulated and the
// other 4 are rebuilt at the end: 70 FMAs per pair instead of 84.
constexpr int kRed[16] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 11, 12, 13, 14, 16, 17};
constexpr Table<84> make_m2l_red() {
  Table<84> T{};
  int k = 0;
  for (int r = 0; r < 16; ++r)
    for (int q = 0; q < 16; ++q) {
      const int t = kRed[q], s = kRed[r];
      if (kComps[t].n + kComps[s].n <= 3) T.v[k++] = Term{t, r, merge(t, s), 1};
    }
  T.n = k;
  return T;
}
constexpr auto kM2LRed = make_m2l_red();
static_assert(kM2LRed.n == 70, "reduced M2L table");

template <typename F, int... K>
__device__ __forceinline__ void unroll_impl(F &&f, std::integer_sequence<int, K...>) {
  (f(std::integral_constant<int, K>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void unroll(F &&f) {
  unroll_impl(f, std::make_integer_sequence<int, N>{});
}

// d^b for every component b (times a per-component constant from SCALE).
template <bool L2L_SCALED>
__device__ __forceinline__ void monomials(double dx, double dy, double dz, double (&m)[NC]) {
  const double d[3] = {dx, dy, dz};
  unroll<NC>([&](auto K) {
    constexpr Comp C = kComps[K];
    double v = 1.0;
    if (C.n > 0) v = d[C.a[0]];
    if (C.n > 1) v = v * d[C.a[1]];
    if (C.n > 2) v = v * d[C.a[2]];
    constexpr double sc = l2l_scale(K);
    if (L2L_SCALED) v = v * sc;
    m[K] = v;
  });
}

// Derivative tensor of 1/r at R up to order 3 (symmetric storage).
__device__ __forceinline__ void d_tensor(double x, double y, double z, double (&D)[NC]) {
  const double r2 = fma(z, z, fma(y, y, x * x));
  const double r1 = rsqrt(r2);
  const double i2 = r1 * r1;
  const double r3 = r1 * i2;
  const double f5 = 3.0 * r3 * i2;          // 3 / r^5
  const double f7 = 5.0 * f5 * i2;          // 15 / r^7
  const double R[3] = {x, y, z};
  D[0] = r1;
  D[1] = -x * r3;
  D[2] = -y * r3;
  D[3] = -z * r3;
  unroll<NC>([&](auto K) {
    constexpr Comp C = kComps[K];
    if constexpr (C.n == 2) {
      const double v = R[C.a[0]] * R[C.a[1]] * f5;
      D[K] = C.a[0] == C.a[1] ? v - r3 : v;
    } else if constexpr (C.n == 3) {
      constexpr int a = C.a[0], b = C.a[1], c = C.a[2];
      const double p = R[a] * R[b] * R[c];
      double t = 0.0;
      if (b == c) t += R[a];
      if (a == c) t += R[b];
      if (a == b) t += R[c];
      D[K] = (a == b || b == c || a == c) ? fma(f5, t, -p * f7) : -p * f7;
    }
  });
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\nFW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FW_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// The 33 parent-near offsets (|P|^2 <= 4), x fastest — same order as
// oracle/fmm_oracle.py PNEAR.
struct PTab {
  int8_t p[33][3];
};
constexpr PTab make_ptab() {
  PTab T{};
  int k = 0;
  for (int z = -2; z <= 2; ++z)
    for (int y = -2; y <= 2; ++y)
      for (int x = -2; x <= 2; ++x)
        if (x * x + y * y + z * z <= 4) {
          T.p[k][0] = (int8_t)x;
          T.p[k][1] = (int8_t)y;
          T.p[k][2] = (int8_t)z;
          ++k;
        }
  return T;
}
__constant__ PTab c_pnear = make_ptab();
// P = (0,0,0): every child pair of it is near (|o - c|^2 <= 3), so its M2L
// stage is all zero tensors — the M2L walks the other 32 stages only.
constexpr int self_stage() {
  const PTab T = make_ptab();
  for (int k = 0; k < 33; ++k)
    if (T.p[k][0] == 0 && T.p[k][1] == 0 && T.p[k][2] == 0) return k;
  return -1;
}
constexpr int kSelfStage = self_stage();
static_assert(kSelfStage == 16, "PNEAR order");
constexpr int kM2LStages = 32;
__host__ __device__ constexpr int m2l_stage(int s) { return s + (s >= kSelfStage); }

// Leaf stencil weights by integer offset q = i - j in [-5,5]^3:
// (1/|q|, qx/|q|^3, qy/|q|^3, qz/|q|^3); q = 0 -> 0 (the self term).
__constant__ double c_w[11 * 11 * 11][4];
// The same table in global memory for lane-divergent gathers (L1-resident).
__device__ double g_w[11 * 11 * 11][4];


// Reduced moment records (the M2L's source) hold 16 moments padded to 18
// doubles (144 B): the 4 cells a warp reads per LDS.128 (stride 2 cells = 18
// chunks) land on distinct bank groups. Raw records ([N^3][20]) feed M2M.
constexpr int MS = 18;
// Per-stage D table: the 27 offsets e = o - c + 1 in {0,1,2}^3 at 16-byte
// chunk strides 17 / 50 / 156 (distinct mod 8 for the 8 octants of a warp).
constexpr int kDX = 17, kDY = 50, kDZ = 156;
constexpr int kDChunks = 2 * kDZ + 2 * kDY + 2 * kDX + NC / 2;   // 456
constexpr int kDStage = 2 * kDChunks;                            // 912 doubles
constexpr int kMStage = 512 * MS;                                // 9216 doubles
constexpr int kStage = kMStage + kDStage;                        // 81,024 B
constexpr uint32_t kMBytes = kMStage * 8, kDBytes = kDStage * 8;

struct Params {
  CUtensorMap maps[kMaxLevel];     // level l reduced records, 4-D {18, N, N, nz + 2 halo}
  double *Loc[kMaxLevel];          // [nz][N][N][20] (this rank's planes)
  const double *Dtab[kMaxLevel];   // [33][912], levels >= 1
  double *L0part;                  // [8][512][20]
  int nbz[kMaxLevel];              // this rank's sub-grid planes (N/8 when replicated)
  int zoff[kMaxLevel];             // halo planes below plane 0 in the reduced records
  int L;                           // max_level (leaves); multipole levels 0..L-1
};

// ---------------------------------------------------------------- upward
// One thread per parent cell. Child c sits at d = (s_x, s_y, s_z) h/2 from
// the parent's centre (s_a = 2 c_a - 1), so every monomial d^b is a
// compile-time sign times (h/2)^|b|: for leaf children (monopoles) each
// moment is a signed sum of the 8 child masses; for finer-level children the
// exact M2M shift is 84 FMAs per child with folded signs. The thread writes
// its parent's raw (pre-scaled) record and the traceless-reduced record.
template <int C>
constexpr double child_sign(int b) {
  double v = 1.0;
  for (int q = 0; q < kComps[b].n; ++q) v *= ((C >> kComps[b].a[q]) & 1) ? 1.0 : -1.0;
  return v;
}

__global__ void __launch_bounds__(256) k_fmm_up(const double *__restrict__ rho,
                                                const double *__restrict__ child,
                                                double *__restrict__ parent,
                                                double *__restrict__ parent_red, int Np,
                                                int Npz, double hc) {
  // parents: Np x Np x Npz (this rank's planes); all pointers at local plane 0
  __shared__ __align__(16) double stage[256 * NC];   // the block's records
  const int64_t npar = (int64_t)Np * Np * Npz;
  const int64_t first = (int64_t)blockIdx.x * blockDim.x;
  // a thread past the end recomputes the last parent (its record is not
  // copied out) so every thread reaches the block's barriers
  const int64_t pidx = min(first + threadIdx.x, npar - 1);
  const int nrec = (int)min((int64_t)blockDim.x, npar - first);
  const int px = (int)(pidx % Np), py = (int)((pidx / Np) % Np),
            pz = (int)(pidx / ((int64_t)Np * Np));
  const int Nc = 2 * Np;
  const double h2 = 0.5 * hc;
  const double hp[4] = {1.0, h2, h2 * h2, h2 * h2 * h2};
  double M[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) M[k] = 0.0;
  if (rho) {
    const double vol = hc * hc * hc;
    double m[8];
#pragma unroll
    for (int r = 0; r < 4; ++r) {      // r = (cz, cy); x pair by one 16-B load
      const int cy = r & 1, cz = r >> 1;
      const double2 v = __ldg(reinterpret_cast<const double2 *>(
          rho + ((int64_t)(2 * pz + cz) * Nc + (2 * py + cy)) * Nc + 2 * px));
      m[2 * r] = v.x * vol;
      m[2 * r + 1] = v.y * vol;
    }
    unroll<8>([&](auto C) {
      unroll<NC>([&](auto K) {
        constexpr double sg = child_sign<decltype(C)::value>(K);
        M[K] = sg > 0 ? M[K] + m[C] : M[K] - m[C];
      });
    });
    unroll<NC>([&](auto K) { M[K] = M[K] * hp[kComps[K].n]; });
  } else {
    unroll<8>([&](auto C) {
      constexpr int Cv = decltype(C)::value;
      constexpr int cx = Cv & 1, cy = (Cv >> 1) & 1, cz = Cv >> 2;
      const double2 *rec = reinterpret_cast<const double2 *>(
          child + (((int64_t)(2 * pz + cz) * Nc + (2 * py + cy)) * Nc + (2 * px + cx)) * NC);
      double Mc[NC];
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) {
        const double2 a = __ldg(rec + k);
        Mc[2 * k] = a.x;
        Mc[2 * k + 1] = a.y;
      }
      unroll<kM2M.n>([&](auto E) {
        constexpr Term T = kM2M.v[E];
        // child raw records are pre-scaled: undo the source scale here
        constexpr double coef = T.c * child_sign<decltype(C)::value>(T.b) / m2l_scale(T.s);
        M[T.t] = fma(coef * Mc[T.s], hp[kComps[T.b].n], M[T.t]);
      });
    });
  }
  unroll<NC>([&](auto K) {
    constexpr double sc = m2l_scale(K);
    M[K] = M[K] * sc;
  });
  // records leave through shared memory so each warp store instruction
  // writes 512 contiguous bytes (a record per thread would be a 160-B stride)
  const int t = threadIdx.x;
  double2 *st2 = reinterpret_cast<double2 *>(stage);
#pragma unroll
  for (int k = 0; k < NC / 2; ++k) st2[t * (NC / 2) + k] = make_double2(M[2 * k], M[2 * k + 1]);
  __syncthreads();
  double2 *raw = reinterpret_cast<double2 *>(parent + first * NC);
  for (int i = t; i < nrec * (NC / 2); i += blockDim.x) raw[i] = st2[i];
  __syncthreads();
  // traceless reduction (see kRed): fold the zz-containing moments
  const double red[MS] = {M[0],          M[1],          M[2],          M[3],
                          M[4] - M[9],   M[5],          M[6],          M[7] - M[9],
                          M[8],          M[10] - M[15], M[11] - M[18], M[12] - M[19],
                          M[13] - M[15], M[14],         M[16] - M[18], M[17] - M[19],
                          0.0,           0.0};
#pragma unroll
  for (int k = 0; k < MS / 2; ++k) st2[t * (MS / 2) + k] = make_double2(red[2 * k], red[2 * k + 1]);
  __syncthreads();
  double2 *rd = reinterpret_cast<double2 *>(parent_red + first * MS);
  for (int i = t; i < nrec * (MS / 2); i += blockDim.x) rd[i] = st2[i];
}

// --------------------------------------------------------- M2L D tables
// Dtab[level][stage k][entry e] = D(q h) with q = (e - 1) - 2 P_k, or 0 where
// the pair is near (|q|^2 <= 4): those children then contribute nothing and
// the interaction loop needs no branch.
struct TabPtrs {
  double *p[kMaxLevel];
};
__global__ void __launch_bounds__(32) k_fmm_dtab(const TabPtrs T) {
  const int k = blockIdx.x, lev = blockIdx.y + 1, e = threadIdx.x;
  double *tab = T.p[lev] + (size_t)k * kDStage;
  for (int i = e; i < kDStage; i += 32) tab[i] = 0.0;
  __syncwarp();
  if (e >= 27) return;
  const int ex = e % 3, ey = (e / 3) % 3, ez = e / 9;
  const int qx = ex - 1 - 2 * c_pnear.p[k][0], qy = ey - 1 - 2 * c_pnear.p[k][1],
            qz = ez - 1 - 2 * c_pnear.p[k][2];
  if (qx * qx + qy * qy + qz * qz <= 4) return;
  const double h = 1.0 / double(8 << lev);
  double D[NC];
  d_tensor(qx * h, qy * h, qz * h, D);
  double *dst = tab + 2 * (ex * kDX + ey * kDY + ez * kDZ);
#pragma unroll
  for (int i = 0; i < NC; ++i) dst[i] = D[i];
}

// ------------------------------------------------------------------- M2L
constexpr int kT = 2;                             // targets per thread
constexpr int kM2LThreads = 512 / kT;
constexpr int kM2LSmem = 2 * kStage * 8;          // 162,048 B

__device__ __forceinline__ void load20(const double *p, double (&v)[NC]) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
  for (int k = 0; k < NC / 2; ++k) {
    const double2 a = q[k];
    v[2 * k] = a.x;
    v[2 * k + 1] = a.y;
  }
}

__device__ __forceinline__ void load16(const double *p, double (&v)[16]) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 a = q[k];
    v[2 * k] = a.x;
    v[2 * k + 1] = a.y;
  }
}

// L (independent components) += reduced source moments x D: 70 FMAs.
__device__ __forceinline__ void contract(double (&L)[NC], const double (&M)[16],
                                         const double (&D)[NC]) {
  unroll<kM2LRed.n>([&](auto E) {
    constexpr Term T = kM2LRed.v[E];
    L[T.t] = fma(M[T.s], D[T.b], L[T.t]);
  });
}

// Rebuild the 4 dependent components of a traceless local expansion.
__device__ __forceinline__ void untrace(double (&L)[NC]) {
  L[9] = -(L[4] + L[7]);
  L[15] = -(L[10] + L[13]);
  L[18] = -(L[11] + L[16]);
  L[19] = -(L[12] + L[17]);
}

__device__ __forceinline__ void issue_stage(const Params &P, int lev, double *dst,
                                            uint64_t *bar, int k, int X0, int Y0, int Z0) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(kMBytes + kDBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(&P.maps[lev])), "r"(0), "r"(X0 + 2 * c_pnear.p[k][0]),
      "r"(Y0 + 2 * c_pnear.p[k][1]), "r"(Z0 + 2 * c_pnear.p[k][2]), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst + kMStage)),
      "l"(P.Dtab[lev] + (size_t)k * kDStage), "r"(kDBytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kM2LThreads, 1) k_fmm_m2l(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  // thread = (octant, parent x) x two parents 2 planes apart in z: both
  // targets share the octant, hence every derivative tensor D (one load
  // feeds 2 x 70 FMAs); the source records differ
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int ox = lane & 1, oy = (lane >> 1) & 1, oz = (lane >> 2) & 1;
  const int px = lane >> 3, py = w & 3, pzb = w >> 2;
  const int lx = 2 * px + ox, ly = 2 * py + oy;
  int lz[kT];
#pragma unroll
  for (int r = 0; r < kT; ++r) lz[r] = 2 * (pzb + 2 * r) + oz;
  // decode the job: levels L-1 .. 1 (8^l sub-grids each), then 8 level-0 slabs
  int job = blockIdx.x, lev = 0, sub = 0;
  for (int l = P.L - 1; l >= 1; --l) {
    const int cnt = (1 << (2 * l)) * P.nbz[l];
    if (job < cnt) {
      lev = l;
      sub = job;
      break;
    }
    job -= cnt;
  }
  if (t == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double L[kT][NC];
#pragma unroll
  for (int r = 0; r < kT; ++r)
#pragma unroll
    for (int k = 0; k < NC; ++k) L[r][k] = 0.0;

  if (lev == 0) {
    // level-0 slab `job`: all 512 targets against the sources with z == job
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_u32(&bar[0])),
                   "r"(kMBytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(sm)),
          "l"(reinterpret_cast<uint64_t>(&P.maps[0])), "r"(0), "r"(0), "r"(0), "r"(0),
          "r"(smem_u32(&bar[0]))
          : "memory");
    }
    mbar_wait(&bar[0], 0);
    const double h = 1.0 / 8.0;
    const int jz = job;
#pragma unroll
    for (int r = 0; r < kT; ++r) {
#pragma unroll 1
      for (int jy = 0; jy < 8; ++jy)
#pragma unroll 1
        for (int jx = 0; jx < 8; ++jx) {
          const int qx = lx - jx, qy = ly - jy, qz = lz[r] - jz;
          if (qx * qx + qy * qy + qz * qz > 4) {
            double D[NC], M[16];
            d_tensor(qx * h, qy * h, qz * h, D);
            load16(sm + ((jz * 8 + jy) * 8 + jx) * MS, M);
            contract(L[r], M, D);
          }
        }
      untrace(L[r]);
      double2 *dst = reinterpret_cast<double2 *>(
          P.L0part + ((size_t)job * 512 + (lz[r] * 8 + ly) * 8 + lx) * NC);
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) dst[k] = make_double2(L[r][2 * k], L[r][2 * k + 1]);
    }
    return;
  }

  const int nb = 1 << lev;
  const int X0 = 8 * (sub % nb), Y0 = 8 * ((sub / nb) % nb), Z0 = 8 * (sub / (nb * nb));
  const int ZT = Z0 + P.zoff[lev];     // TMA z of the sub-grid in the halo'd records
  if (t == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_stage(P, lev, sm, &bar[0], m2l_stage(0), X0, Y0, ZT);
    issue_stage(P, lev, sm + kStage, &bar[1], m2l_stage(1), X0, Y0, ZT);
  }
  // lane-dependent parts of the source cell and of the D-table entry
  const int cbase = ((2 * pzb) * 8 + 2 * py) * 8 + 2 * px;   // target 0; target 1 is +256
  const int dbase = (ox + 1) * kDX + (oy + 1) * kDY + (oz + 1) * kDZ;
#pragma unroll 1
  for (int k = 0; k < kM2LStages; ++k) {
    const int buf = k & 1;
    mbar_wait(&bar[buf], (k >> 1) & 1);
    const double *Ms = sm + buf * kStage;
    const double *Ds = Ms + kMStage;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
      double D[NC];
      load20(Ds + 2 * (dbase - cx * kDX - cy * kDY - cz * kDZ), D);
#pragma unroll
      for (int r = 0; r < kT; ++r) {
        double M[16];
        load16(Ms + (cbase + 256 * r + (cz * 8 + cy) * 8 + cx) * MS, M);
        contract(L[r], M, D);
      }
    }
    __syncthreads();            // every thread is done with this buffer
    if (t == 0 && k + 2 < kM2LStages) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_stage(P, lev, sm + buf * kStage, &bar[buf], m2l_stage(k + 2), X0, Y0, ZT);
    }
  }
  const int N = 8 << lev;
#pragma unroll
  for (int r = 0; r < kT; ++r) {
    untrace(L[r]);
    double2 *dst = reinterpret_cast<double2 *>(
        P.Loc[lev] + (((size_t)(Z0 + lz[r]) * N + (Y0 + ly)) * N + (X0 + lx)) * NC);
#pragma unroll
    for (int k = 0; k < NC / 2; ++k) dst[k] = make_double2(L[r][2 * k], L[r][2 * k + 1]);
  }
}

// ------------------------------------------------------------------ L2L
// Child cells: N x N x nzc (this rank's planes, global plane z0c + local);
// the parent array's local plane 0 is global plane z0p (0 when replicated).
__global__ void __launch_bounds__(256) k_fmm_down(const double *__restrict__ Lp,
                                                  double *__restrict__ Lc,
                                                  const double *__restrict__ L0part, int N,
                                                  int nzc, int z0c, int z0p, double h) {
  const int64_t n = (int64_t)N * N * nzc;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double out[NC];
  if (L0part) {   // level 0: sum the 8 slab partials in a fixed order
#pragma unroll
    for (int k = 0; k < NC; ++k) out[k] = 0.0;
    for (int s = 0; s < 8; ++s) {
      double v[NC];
      load20(L0part + ((size_t)s * 512 + i) * NC, v);
#pragma unroll
      for (int k = 0; k < NC; ++k) out[k] += v[k];
    }
  } else {
    const int x = (int)(i % N), y = (int)((i / N) % N), z = (int)(i / ((int64_t)N * N));
    const int Nq = N / 2;
    const int pz = ((z0c + z) >> 1) - z0p;
    const int64_t pi = ((int64_t)pz * Nq + (y >> 1)) * Nq + (x >> 1);
    double mono[NC], Lpar[NC];
    monomials<true>(((x & 1) - 0.5) * h, ((y & 1) - 0.5) * h, ((z & 1) - 0.5) * h, mono);
    load20(Lp + pi * NC, Lpar);
    load20(Lc + i * NC, out);
    unroll<kL2L.n>([&](auto E) {
      constexpr Term T = kL2L.v[E];
      out[T.t] = fma(Lpar[T.s], mono[T.b], out[T.t]);
    });
  }
  double2 *dst = reinterpret_cast<double2 *>(Lc + i * NC);
#pragma unroll
  for (int k = 0; k < NC / 2; ++k) dst[k] = make_double2(out[2 * k], out[2 * k + 1]);
}

// ------------------------------------------------------------ leaf (P2P)
constexpr int kLeafThreads = 256;
// Each thread: one octant, 2 parent rows in y x 4 parent planes in z = 8
// targets sharing every stencil weight (4 constant loads per 32 FMAs).
constexpr int kRY = 2, kRZ = 4;
constexpr int kTX = 8, kTY = 8 * kRY, kTZ = 16;          // targets per CTA tile
constexpr int kSX = 12, kSY = (kTY + 8) / 2, kSZ = (kTZ + 8) / 2;   // per-parity extents
constexpr int kPar = kSX * kSY * kSZ;                    // x' padded 8 -> 12 (banks)
constexpr int kLeafSmem = 8 * kPar * 8;                  // 110,592 B

// Leaves: N x N x nz (this rank's planes). rho points at local plane 0 and
// its planes [zmin, zmax) are readable (a halo of exchanged planes, or just
// [0, N) on one device); the rest reads as zero (isolated boundary).
__global__ void __launch_bounds__(kLeafThreads, 2)
    k_fmm_leaf(const double *__restrict__ rho, int zmin, int zmax,
               const double *__restrict__ Lpar, double *__restrict__ out, int N, int nz,
               double h) {
  extern __shared__ __align__(128) double S[];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int ntx = N / kTX, nty = N / kTY;
  const int tile = blockIdx.x;
  const int X0 = (tile % ntx) * kTX, Y0 = ((tile / ntx) % nty) * kTY,
            Z0 = (tile / (ntx * nty)) * kTZ;
  // ---- stage rho over [X0-4, X0+kTX+4) x [Y0-4, Y0+kTY+4) x [Z0-4, Z0+kTZ+4),
  //      split by parity: S[c][z'][y'][x'] with coordinate = 2*primed + c;
  //      8-byte cp.async (all in flight at once), zero-filled outside the domain
  constexpr int kEx = kTX + 8, kEy = kTY + 8, kEz = kTZ + 8;
  for (int e = t; e < kEx * kEy * kEz; e += kLeafThreads) {
    const int rx = e % kEx, ry = (e / kEx) % kEy, rz = e / (kEx * kEy);
    const int gx = X0 - 4 + rx, gy = Y0 - 4 + ry, gz = Z0 - 4 + rz;
    const bool in = gx >= 0 && gx < N && gy >= 0 && gy < N && gz >= zmin && gz < zmax;
    const double *src = in ? rho + ((int64_t)gz * N + gy) * N + gx : rho;
    const int c = (rx & 1) | ((ry & 1) << 1) | ((rz & 1) << 2);
    double *dst = S + c * kPar + ((rz >> 1) * kSY + (ry >> 1)) * kSX + (rx >> 1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(in ? 8 : 0)
                 : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // ---- warp = child octant o; lane = (px, py, pz low bit); targets over
  //      (ry: py + 4 ry) x (r: pz = pzl + 2 r)
  const int ox = w & 1, oy = (w >> 1) & 1, oz = w >> 2;
  const int px = lane & 3, py = (lane >> 2) & 3, pzl = lane >> 4;
  double acc[kRY * kRZ][4];
#pragma unroll
  for (int r = 0; r < kRY * kRZ; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[r][k] = 0.0;
#pragma unroll 1
  for (int k = 0; k < 33; ++k) {
    const int Px = c_pnear.p[k][0], Py = c_pnear.p[k][1], Pz = c_pnear.p[k][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
      const int qx = ox - 2 * Px - cx, qy = oy - 2 * Py - cy, qz = oz - 2 * Pz - cz;
      const int wi = ((qz + 5) * 11 + (qy + 5)) * 11 + (qx + 5);
      const double w0 = c_w[wi][0], w1 = c_w[wi][1], w2 = c_w[wi][2], w3 = c_w[wi][3];
      const double *base = S + c * kPar + ((py + Py + 2) * kSX) + (px + Px + 2);
#pragma unroll
      for (int ry = 0; ry < kRY; ++ry)
#pragma unroll
        for (int r = 0; r < kRZ; ++r) {
          const double m = base[(pzl + 2 * r + Pz + 2) * (kSX * kSY) + 4 * ry * kSX];
          double(&a)[4] = acc[ry * kRZ + r];
          a[0] = fma(m, w0, a[0]);
          a[1] = fma(m, w1, a[1]);
          a[2] = fma(m, w2, a[2]);
          a[3] = fma(m, w3, a[3]);
        }
    }
  }
  // ---- L2P from the parent's expansion (level L-1) and the output --------
  double mono[NC];
  monomials<true>((ox - 0.5) * h, (oy - 0.5) * h, (oz - 0.5) * h, mono);
  const int Nq = N / 2;
  const size_t n = (size_t)N * N * nz;
  const double h2 = h * h;
#pragma unroll
  for (int rr = 0; rr < kRY * kRZ; ++rr) {
    const int ry = rr / kRZ, r = rr % kRZ;
    const int x = X0 + 2 * px + ox, y = Y0 + 2 * (py + 4 * ry) + oy,
              z = Z0 + 2 * (pzl + 2 * r) + oz;
    double phi = -h2 * acc[rr][0];
    double gr[3] = {h * acc[rr][1], h * acc[rr][2], h * acc[rr][3]};
    if (Lpar) {
      const size_t pi = ((size_t)(z >> 1) * Nq + (y >> 1)) * Nq + (x >> 1);
      double Lp[NC];
      const double2 *rec = reinterpret_cast<const double2 *>(Lpar + pi * NC);
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) {
        const double2 a = __ldg(rec + k);
        Lp[2 * k] = a.x;
        Lp[2 * k + 1] = a.y;
      }
      unroll<kL2L.n>([&](auto E) {
        constexpr Term T = kL2L.v[E];
        if constexpr (T.t == 0) phi = fma(Lp[T.s], mono[T.b], phi);
        if constexpr (T.t >= 1 && T.t <= 3) gr[T.t - 1] = fma(Lp[T.s], mono[T.b], gr[T.t - 1]);
      });
    }
    const size_t i = ((size_t)z * N + y) * N + x;
    out[i] = phi;
    out[n + i] = -gr[0];
    out[2 * n + i] = -gr[1];
    out[3 * n + i] = -gr[2];
  }
}

// ----------------------------------------------- leaf on FP64 tensor cores
// The leaf sum out[i][k] = sum_j m_j W(i - j)[k] is a GEMM per pair of
// targets that share a parent p: rows = parents, K = the 264 source offsets
// (P in PNEAR, child c), N = 4 components x 2 octants (o, o + e_x). Both
// octants of a parent read the same sources j = 2(p + P) + c (one A
// operand) and differ only in the weights W(o - 2P - c) (B), so every tensor
// FMA is useful (the self term's weights are zero). One mma.sync.m8n8k4.f64
// takes 8 x-consecutive parents as rows and 4 children (one z-half) of one
// offset P as K: 33 x 2 = 66 K-chunks. A CTA (8 warps) covers 16 x 8 x 4
// leaves: warp = (octant pair: oy, oz) x (parent plane in z); its 4 row
// groups are the 4 parent rows in y.
constexpr int kMX = 16, kMY = 8, kMZ = 4;                  // leaves per CTA tile
constexpr int kMSX = 12, kMSY = 8, kMSZ = 6;               // per-parity staged extents
constexpr int kMPar = kMSX * kMSY * kMSZ + 4;              // 580: planes 4 apart mod 16
constexpr int kMAcc = kMX * kMY * kMZ * 4;                 // tile results [z][y][x][4]
constexpr int kLeafMmaSmem = (8 * kMPar + kMAcc) * 8;      // 53,504 B

__global__ void __launch_bounds__(256) k_fmm_leaf_mma(const double *__restrict__ rho, int zmin,
                                                      int zmax, const double *__restrict__ Lpar,
                                                      double *__restrict__ out, int N, int nz,
                                                      double h) {
  extern __shared__ __align__(128) double S[];
  double *acc = S + 8 * kMPar;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int ntx = N / kMX, nty = N / kMY;
  const int tile = blockIdx.x;
  const int X0 = (tile % ntx) * kMX, Y0 = ((tile / ntx) % nty) * kMY,
            Z0 = (tile / (ntx * nty)) * kMZ;
  // ---- stage rho over [X0-4, X0+20) x [Y0-4, Y0+12) x [Z0-4, Z0+8), split by
  //      parity as in k_fmm_leaf (zero outside the readable planes)
  constexpr int kEx = 2 * kMSX, kEy = 2 * kMSY, kEz = 2 * kMSZ;
  for (int e = t; e < kEx * kEy * kEz; e += 256) {
    const int rx = e % kEx, ry = (e / kEx) % kEy, rz = e / (kEx * kEy);
    const int gx = X0 - 4 + rx, gy = Y0 - 4 + ry, gz = Z0 - 4 + rz;
    const bool in = gx >= 0 && gx < N && gy >= 0 && gy < N && gz >= zmin && gz < zmax;
    const double *src = in ? rho + ((int64_t)gz * N + gy) * N + gx : rho;
    const int c = (rx & 1) | ((ry & 1) << 1) | ((rz & 1) << 2);
    double *dst = S + c * kMPar + ((rz >> 1) * kMSY + (ry >> 1)) * kMSX + (rx >> 1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(in ? 8 : 0)
                 : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int oy = w & 1, oz = (w >> 1) & 1, zsel = w >> 2;
  const int kk = lane & 3, nn = lane >> 2;    // B fragment B[kk][nn]; A fragment A[nn][kk]
  const int ox = nn >> 2, comp = nn & 3;      // B column nn: octant (ox, oy, oz), component
  const int cx = kk & 1, cy = kk >> 1;
  // per-lane bases; an offset P then adds -2 (121 Pz + 11 Py + Px) to the
  // weight index and (Pz kMSY + Py) kMSX + Px to the source address
  int wbase[2], abase[2];
#pragma unroll
  for (int hz = 0; hz < 2; ++hz) {
    wbase[hz] = (((oz - hz + 5) * 11 + (oy - cy + 5)) * 11 + (ox - cx + 5)) * 4 + comp;
    abase[hz] = (kk | (hz << 2)) * kMPar + ((zsel + 2) * kMSY + 2) * kMSX + (nn + 2);
  }
  const double *gw = &g_w[0][0];
  double C[4][2];
#pragma unroll
  for (int g = 0; g < 4; ++g) C[g][0] = C[g][1] = 0.0;
#pragma unroll 1
  for (int k = 0; k < 33; ++k) {
    const int Px = c_pnear.p[k][0], Py = c_pnear.p[k][1], Pz = c_pnear.p[k][2];
    const int woff = -8 * ((Pz * 11 + Py) * 11 + Px);
    const int aoff = (Pz * kMSY + Py) * kMSX + Px;
#pragma unroll
    for (int hz = 0; hz < 2; ++hz) {
      const double b = __ldg(gw + wbase[hz] + woff);
      const double *a0 = S + abase[hz] + aoff;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double a = a0[g * kMSX];
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
            : "+d"(C[g][0]), "+d"(C[g][1])
            : "d"(a), "d"(b));
      }
    }
  }
  // ---- C[g]: lane holds (row nn, columns 2kk, 2kk+1) -> tile results
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = 2 * kk + e, cox = col >> 2, k = col & 3;
      const int x = 2 * nn + cox, y = 2 * g + oy, z = 2 * zsel + oz;
      acc[((z * kMY + y) * kMX + x) * 4 + k] = C[g][e];
    }
  __syncthreads();
  // ---- L2P from the parent's expansion and the output, x-fastest -------
  const int Nq = N / 2;
  const size_t n = (size_t)N * N * nz;
  const double h2 = h * h;
  for (int e = t; e < kMX * kMY * kMZ; e += 256) {
    const int lx = e % kMX, ly = (e / kMX) % kMY, lz = e / (kMX * kMY);
    const int x = X0 + lx, y = Y0 + ly, z = Z0 + lz;
    const double *a = acc + e * 4;
    double phi = -h2 * a[0];
    double gr[3] = {h * a[1], h * a[2], h * a[3]};
    if (Lpar) {
      double mono[NC];
      monomials<true>(((lx & 1) - 0.5) * h, ((ly & 1) - 0.5) * h, ((lz & 1) - 0.5) * h, mono);
      const size_t pi = ((size_t)(z >> 1) * Nq + (y >> 1)) * Nq + (x >> 1);
      double Lp[NC];
      const double2 *rec = reinterpret_cast<const double2 *>(Lpar + pi * NC);
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) {
        const double2 v = __ldg(rec + k);
        Lp[2 * k] = v.x;
        Lp[2 * k + 1] = v.y;
      }
      unroll<kL2L.n>([&](auto E) {
        constexpr Term T = kL2L.v[E];
        if constexpr (T.t == 0) phi = fma(Lp[T.s], mono[T.b], phi);
        if constexpr (T.t >= 1 && T.t <= 3) gr[T.t - 1] = fma(Lp[T.s], mono[T.b], gr[T.t - 1]);
      });
    }
    const size_t i = ((size_t)z * N + y) * N + x;
    out[i] = phi;
    out[n + i] = -gr[0];
    out[2 * n + i] = -gr[1];
    out[3 * n + i] = -gr[2];
  }
}

// ------------------------------------------------------------------ host
// Slab geometry for `ranks` devices, each owning N/ranks leaf planes in z.
// Levels l >= lp are partitioned: this rank keeps its nz_l = N_l/ranks planes
// (z0_l = rank * nz_l) and the reduced records carry 4 halo planes on each
// side (zero, or the neighbours' planes after an exchange). Levels < lp are
// replicated: full lattices on every rank; level lp-1 is assembled by an
// all-gather of the ranks' slabs (each computes its own from level lp), the
// coarser ones are then computed redundantly. One rank: lp = 1, nothing to
// exchange, the halos stay zero (= the isolated boundary).
struct Geom {
  int L, R, r, lp;
  int n[kMaxLevel + 1], nz[kMaxLevel + 1], z0[kMaxLevel + 1], halo[kMaxLevel + 1];
};

constexpr int kHalo = 4;

bool make_geom(int L, int R, int r, Geom *g) {
  if (L < 1 || L > kMaxLevel || R < 1 || (R & (R - 1)) || r < 0 || r >= R) return false;
  const int N = 8 << L;
  if (N / R < 16 || N % (16 * R)) return false;   // leaf tiles are 16 planes deep
  g->L = L;
  g->R = R;
  g->r = r;
  g->lp = 1;
  while (g->lp < L && (8 << g->lp) / R < 8) ++g->lp;
  for (int l = 0; l <= L; ++l) {
    g->n[l] = 8 << l;
    const bool part = l >= g->lp;
    g->nz[l] = part ? g->n[l] / R : g->n[l];
    g->z0[l] = part ? r * g->nz[l] : 0;
    g->halo[l] = part && l < L ? kHalo : 0;
  }
  return true;
}

struct Layout {
  size_t M[kMaxLevel], Mred[kMaxLevel], Loc[kMaxLevel], Dtab[kMaxLevel], L0part,
      total;   // byte offsets
};

Layout layout(const Geom &g) {
  Layout lo{};
  size_t off = 0;
  for (int l = 0; l < g.L; ++l) {
    const size_t plane = (size_t)g.n[l] * g.n[l];
    // the gathered level keeps full raw/reduced records (its slab is computed
    // locally, the rest arrives by all-gather)
    const size_t nzr = (l == g.lp - 1) ? (size_t)g.n[l] : (size_t)g.nz[l];
    lo.M[l] = off;
    off += plane * nzr * NC * 8;
    lo.Mred[l] = off;
    off += plane * (nzr + 2 * g.halo[l]) * MS * 8;
    lo.Loc[l] = off;
    off += plane * g.nz[l] * NC * 8;
    lo.Dtab[l] = off;
    if (l) off += (size_t)33 * kDStage * 8;
  }
  lo.L0part = off;
  off += (size_t)8 * 512 * NC * 8;
  lo.total = off;
  return lo;
}

int ensure_weights() {
  static int done_mask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 31 && (done_mask >> dev & 1)) return TB_OK;
  static double w[11 * 11 * 11][4];
  for (int z = -5; z <= 5; ++z)
    for (int y = -5; y <= 5; ++y)
      for (int x = -5; x <= 5; ++x) {
        double *e = w[((z + 5) * 11 + (y + 5)) * 11 + (x + 5)];
        const double r2 = double(x * x + y * y + z * z);
        if (r2 == 0.0) {
          e[0] = e[1] = e[2] = e[3] = 0.0;
          continue;
        }
        const double r1 = 1.0 / std::sqrt(r2);
        const double r3 = r1 / r2;
        e[0] = r1;
        e[1] = x * r3;
        e[2] = y * r3;
        e[3] = z * r3;
      }
  int r = tb::rc(cudaMemcpyToSymbol(c_w, w, sizeof w));
  if (r == TB_OK) r = tb::rc(cudaMemcpyToSymbol(g_w, w, sizeof w));
  if (r == TB_OK && dev < 31) done_mask |= 1 << dev;
  return r;
}

int make_params(const Geom &g, double *work, Params *P) {
  const Layout lo = layout(g);
  char *base = reinterpret_cast<char *>(work);
  *P = Params{};
  P->L = g.L;
  P->L0part = reinterpret_cast<double *>(base + lo.L0part);
  for (int l = 0; l < g.L; ++l) {
    double *M = reinterpret_cast<double *>(base + lo.Mred[l]);
    P->Loc[l] = reinterpret_cast<double *>(base + lo.Loc[l]);
    P->Dtab[l] = reinterpret_cast<const double *>(base + lo.Dtab[l]);
    P->nbz[l] = g.nz[l] / 8;
    P->zoff[l] = g.halo[l];
    const uint64_t N = (uint64_t)g.n[l];
    const uint64_t planes = (uint64_t)((l == g.lp - 1) ? g.n[l] : g.nz[l]) + 2 * g.halo[l];
    const uint64_t dims[4] = {(uint64_t)MS, N, N, planes};
    const uint64_t strides[3] = {MS * 8, MS * 8 * N, MS * 8 * N * N};
    const uint32_t box[4] = {(uint32_t)MS, 8, 8, 8};
    const int r = tb::encode_tiled(&P->maps[l], 4, M, dims, strides, box);
    if (r != TB_OK) return r;
  }
  return TB_OK;
}

inline cudaStream_t strm(tb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// parents of level l from level l+1 (or from the leaves when l == L-1)
void launch_up(tb_stream_t s, const Geom &g, const Layout &lo, char *base, const double *rho,
               int l) {
  const int Np = g.n[l];
  // parent planes computed here: this rank's slab (the gathered level too)
  const int npz = (l >= g.lp - 1 && g.R > 1) ? g.nz[l + 1] / 2 : g.nz[l];
  const int pz0 = (l == g.lp - 1) ? g.z0[l + 1] / 2 : 0;   // local plane in the array
  const size_t plane = (size_t)Np * Np;
  double *raw = reinterpret_cast<double *>(base + lo.M[l]) + plane * pz0 * NC;
  double *red = reinterpret_cast<double *>(base + lo.Mred[l]) + plane * (pz0 + g.halo[l]) * MS;
  const double *child =
      l == g.L - 1 ? nullptr : reinterpret_cast<const double *>(base + lo.M[l + 1]);
  const int64_t npar = (int64_t)plane * npz;
  k_fmm_up<<<(unsigned)((npar + 255) / 256), 256, 0, strm(s)>>>(
      l == g.L - 1 ? rho : nullptr, child, raw, red, Np, npz, 1.0 / double(2 * Np));
}

// leaf variant: FP64 tensor cores (k_fmm_leaf_mma, default) or the DFMA
// stencil (k_fmm_leaf, TB_LEAF_MMA=0)
const bool g_leaf_mma = [] {
  const char *e = getenv("TB_LEAF_MMA");
  return !(e && e[0] == '0');
}();

}  // namespace

extern "C" {

int tb_fmm_slab_workspace_bytes(int max_level, int ranks, uint64_t *bytes) {
  Geom g;
  if (!bytes || !make_geom(max_level, ranks, 0, &g)) return TB_E_INVALID;
  *bytes = layout(g).total;
  return TB_OK;
}

int tb_fmm_slab_layout(int max_level, int ranks, int rank, int level, uint64_t *info) {
  Geom g;
  if (!info || !make_geom(max_level, ranks, rank, &g) || level < 0 || level > max_level)
    return TB_E_INVALID;
  const Layout lo = layout(g);
  const bool multipole = level < max_level;
  info[0] = multipole ? lo.M[level] : 0;
  info[1] = multipole ? lo.Mred[level] : 0;
  info[2] = multipole ? lo.Loc[level] : 0;
  info[3] = (uint64_t)g.n[level];
  info[4] = (uint64_t)g.nz[level];
  info[5] = (uint64_t)g.z0[level];
  info[6] = (uint64_t)g.halo[level];
  info[7] = (uint64_t)g.lp;
  return TB_OK;
}

int tb_fmm_slab_upward(tb_stream_t s, int max_level, int ranks, int rank, const double *rho,
                       double *work) {
  Geom g;
  if (!rho || !work || !make_geom(max_level, ranks, rank, &g)) return TB_E_INVALID;
  const Layout lo = layout(g);
  char *base = reinterpret_cast<char *>(work);
  // one rank: every level; several: the partitioned levels and this rank's
  // slab of the gathered level lp-1 (tb_fmm_slab_coarse does the rest)
  const int stop = ranks == 1 ? 0 : g.lp - 1;
  for (int l = max_level - 1; l >= stop; --l) launch_up(s, g, lo, base, rho, l);
  return tb::last_error();
}

int tb_fmm_slab_coarse(tb_stream_t s, int max_level, int ranks, int rank, double *work) {
  Geom g;
  if (!work || !make_geom(max_level, ranks, rank, &g)) return TB_E_INVALID;
  if (ranks == 1) return TB_OK;
  const Layout lo = layout(g);
  char *base = reinterpret_cast<char *>(work);
  for (int l = g.lp - 2; l >= 0; --l) launch_up(s, g, lo, base, nullptr, l);
  return tb::last_error();
}

int tb_fmm_slab_m2l(tb_stream_t s, int max_level, int ranks, int rank, double *work) {
  Geom g;
  if (!work || !make_geom(max_level, ranks, rank, &g)) return TB_E_INVALID;
  Params P;
  int r = make_params(g, work, &P);
  if (r != TB_OK) return r;
  static bool attr = false;
  if (!attr) {
    r = tb::rc(cudaFuncSetAttribute(k_fmm_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kM2LSmem));
    if (r != TB_OK) return r;
    attr = true;
  }
  if (max_level > 1) {
    TabPtrs T{};
    for (int l = 1; l < max_level; ++l) T.p[l] = const_cast<double *>(P.Dtab[l]);
    k_fmm_dtab<<<dim3(33, max_level - 1), 32, 0, strm(s)>>>(T);
  }
  int jobs = 8;
  for (int l = 1; l < max_level; ++l) jobs += (1 << (2 * l)) * P.nbz[l];
  k_fmm_m2l<<<jobs, kM2LThreads, kM2LSmem, strm(s)>>>(P);
  return tb::last_error();
}

int tb_fmm_slab_downward(tb_stream_t s, int max_level, int ranks, int rank, double *work) {
  Geom g;
  if (!work || !make_geom(max_level, ranks, rank, &g)) return TB_E_INVALID;
  const Layout lo = layout(g);
  char *base = reinterpret_cast<char *>(work);
  for (int l = 0; l < max_level; ++l) {
    const int N = g.n[l];
    const int64_t n = (int64_t)N * N * g.nz[l];
    double *Lc = reinterpret_cast<double *>(base + lo.Loc[l]);
    const double *Lp = l ? reinterpret_cast<const double *>(base + lo.Loc[l - 1]) : nullptr;
    const double *part = l ? nullptr : reinterpret_cast<const double *>(base + lo.L0part);
    k_fmm_down<<<(unsigned)((n + 255) / 256), 256, 0, strm(s)>>>(
        Lp, Lc, part, N, g.nz[l], g.z0[l], l ? g.z0[l - 1] : 0, 1.0 / N);
  }
  return tb::last_error();
}

int tb_fmm_slab_leaf(tb_stream_t s, int max_level, int ranks, int rank, const double *rho,
                     int zmin, int zmax, const double *work, double *out) {
  Geom g;
  if (!rho || !out || !work || !make_geom(max_level, ranks, rank, &g) || zmin > 0 ||
      zmax < g.nz[max_level])
    return TB_E_INVALID;
  int r = ensure_weights();
  if (r != TB_OK) return r;
  static bool attr = false;
  if (!attr) {
    r = tb::rc(cudaFuncSetAttribute(k_fmm_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kLeafSmem));
    if (r != TB_OK) return r;
    attr = true;
  }
  const Layout lo = layout(g);
  const double *Lpar = reinterpret_cast<const double *>(reinterpret_cast<const char *>(work) +
                                                        lo.Loc[max_level - 1]);
  const int N = g.n[max_level], nz = g.nz[max_level];
  if (g_leaf_mma) {
    static bool attr_mma = false;
    if (!attr_mma) {
      r = tb::rc(cudaFuncSetAttribute(k_fmm_leaf_mma,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kLeafMmaSmem));
      if (r != TB_OK) return r;
      attr_mma = true;
    }
    const int tiles = (N / kMX) * (N / kMY) * (nz / kMZ);
    k_fmm_leaf_mma<<<tiles, 256, kLeafMmaSmem, strm(s)>>>(rho, zmin, zmax, Lpar, out, N, nz,
                                                          1.0 / N);
    return tb::last_error();
  }
  const int tiles = (N / kTX) * (N / kTY) * (nz / kTZ);
  k_fmm_leaf<<<tiles, kLeafThreads, kLeafSmem, strm(s)>>>(rho, zmin, zmax, Lpar, out, N, nz,
                                                          1.0 / N);
  return tb::last_error();
}

// ---- one device (the slab API with one rank) -----------------------------
int tb_fmm_workspace_bytes(int max_level, uint64_t *bytes) {
  return tb_fmm_slab_workspace_bytes(max_level, 1, bytes);
}

int tb_fmm_upward(tb_stream_t s, int max_level, const double *rho, double *work) {
  return tb_fmm_slab_upward(s, max_level, 1, 0, rho, work);
}

int tb_fmm_m2l(tb_stream_t s, int max_level, double *work) {
  return tb_fmm_slab_m2l(s, max_level, 1, 0, work);
}

int tb_fmm_downward(tb_stream_t s, int max_level, double *work) {
  return tb_fmm_slab_downward(s, max_level, 1, 0, work);
}

int tb_fmm_leaf(tb_stream_t s, int max_level, const double *rho, const double *work,
                double *out) {
  return tb_fmm_slab_leaf(s, max_level, 1, 0, rho, 0, 8 << max_level, work, out);
}

int tb_fmm_solve(tb_stream_t s, int max_level, const double *rho, double *work, double *out) {
  int r = tb_fmm_upward(s, max_level, rho, work);
  if (r == TB_OK) r = tb_fmm_m2l(s, max_level, work);
  if (r == TB_OK) r = tb_fmm_downward(s, max_level, work);
  if (r == TB_OK) r = tb_fmm_leaf(s, max_level, rho, work, out);
  return r;
}

}  // extern "C"
