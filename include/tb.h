/*
 * tb.h — C ABI of libtb, the B200-native replacement for the reference's
 * simulated device + per-kind compute closures + poll registry.
 *
 * Reference: /root/reference/pkg/src/taskbridge/ (cited below as src/...).
 * The reference is pure Python; its "device" is a discrete-event simulator
 * (src/device.py) whose ops carry numpy closures. Each entry point below
 * replaces one reference interface; the Python host package
 * (paper_2303_08058_b200/) binds them with ctypes and keeps the reference's
 * duck types (DeviceQueue / DeviceEvent / VirtualDevice / PollRegistry).
 *
 * Conventions
 *  - extern "C", plain pointers and sizes; no C++ exceptions cross the ABI.
 *  - Return codes: TB_OK (0); TB_NOT_READY (1) for queries that would block
 *    or a busy single-entrant guard; negative values are errors:
 *    -(int)cudaError_t for CUDA failures, TB_E_* for ABI misuse.
 *  - Device pointers are plain `void*`/`double*` in device memory; host
 *    staging pointers passed to the async copies should be pinned
 *    (tb_host_alloc) for true async DMA.
 *  - Streams are cudaStream_t values carried as uint64 (tb_stream_t); 0 is
 *    the legacy default stream. Events are pooled cudaEvent_t
 *    (cudaEventDisableTiming) carried as tb_event_t.
 *  - Every kernel is hand-written for sm_100a (csrc/tb_kernels.cu).
 */
#ifndef TB_H_
#define TB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_ABI_VERSION 1

#define TB_OK 0
#define TB_NOT_READY 1
#define TB_E_INVALID (-10000)   /* bad argument (null pointer, n < 0, ...) */
#define TB_E_NOMEM (-10001)     /* host-side allocation failed             */
#define TB_E_CLOSED (-10002)    /* object already destroyed/closed         */

/* Workload geometry (src/miniapp.py:30-37). */
#define TB_CELLS 512            /* 8x8x8 cells per sub-grid                */
#define TB_FACE 8               /* flat ring face: first/last 8 cells      */
#define TB_KINDS 5              /* kernel kinds with fixed (C1, C2)        */

/* Exact step accumulator (replaces math.fsum, src/miniapp.py:168-169, and the
 * min-tree, src/miniapp.py:138-149). Layout in int64 words:
 *   [0, TB_ACC_LIMBS)  signed 32-bit digits of sum(x) * 2^1074, carry-save
 *   TB_ACC_MIN_WORD    order-preserving int64 key of min(x)
 *   TB_ACC_COUNT_WORD  finished-CTA ticket used by tb_step_final
 * Multi-GPU: all-reduce words [0, TB_ACC_LIMBS) with SUM and word
 * TB_ACC_MIN_WORD with MIN (int64); the result is partition-independent. */
#define TB_ACC_LIMBS 68
#define TB_ACC_BIAS 1074
#define TB_ACC_MIN_WORD 68
#define TB_ACC_COUNT_WORD 70    /* CTA ticket for the fused finalize        */
#define TB_ACC_WORDS 72         /* padded to a 64-byte multiple            */

/* Kernel descriptor ops for tb_launch / tb_agg_launch (what a registered
 * kind's transform does; src/executors.py:171-172, src/miniapp.py:40-53). */
#define TB_OP_NONE 0            /* launch an empty kernel (timing-only op) */
#define TB_OP_KIND 1            /* x = x*C1[kind] + C2[kind], two roundings */
#define TB_OP_AFFINE 2          /* x = x*c1 + c2, two roundings             */
#define TB_OP_TRAP 3            /* fault injection: the kernel traps (tests) */

/* tb_set_option keys/values. */
#define TB_OPT_STEP_IMPL 1      /* which K2 variant tb_step launches        */
#define TB_STEP_AUTO 0          /* 1-slot bulk ring (aligned, 3x5 chain)    */
#define TB_STEP_REG 1           /* direct ld.global.nc into registers       */
#define TB_STEP_BULK 2          /* cp.async.bulk smem ring + mbarriers      */
#define TB_STEP_REGPF 3         /* registers + next-sub-grid prefetch       */
#define TB_STEP_LEAN 4          /* registers capped at 48 (more warps/SM)   */
#define TB_STEP_PAIR 5          /* a warp pair per sub-grid, 8 cells/lane   */
#define TB_STEP_BULK1 6         /* bulk-copy ring, 1 slot per warp          */
#define TB_OPT_STEP_SPW 2       /* K2 sub-grids per warp per CTA; 0 = one
                                   persistent wave (default)                 */

typedef uint64_t tb_stream_t;
typedef uint64_t tb_event_t;
typedef uint64_t tb_poll_t;     /* native poll registry handle             */
typedef uint64_t tb_htq_t;      /* host-task queue handle                  */

/* ------------------------------------------------------------ device -- */
int tb_abi_version(void);
const char *tb_error_string(int rc);
/* VirtualDevice.__init__ (src/device.py:205-257): bind the calling thread to
 * `device` (cudaSetDevice) and warm the event pool. */
int tb_init(int device);
int tb_device_count(int *n);
int tb_sm_count(int device, int *n);
int tb_device_sync(void);
/* Process-wide tuning switches (ablations), e.g. TB_OPT_STEP_IMPL. */
int tb_set_option(int key, int value);

/* ------------------------------------------------------------ queues -- */
/* VirtualDevice.queue() (src/device.py:259-264): one in-order queue. */
int tb_stream_create(tb_stream_t *s);
int tb_stream_destroy(tb_stream_t s);
/* DeviceQueue.incomplete_count() > 0 (src/device.py:179-180): TB_OK when
 * idle, TB_NOT_READY while work is outstanding. */
int tb_stream_query(tb_stream_t s);
int tb_stream_sync(tb_stream_t s);

/* ------------------------------------------------------------ events -- */
/* DeviceQueue.submit(op) -> DeviceEvent (src/device.py:176-177, 116): record a
 * pooled event after everything queued so far. Also the DUMMY queue marker of
 * Integration.get_future_queue (src/bridge.py:92-101). */
int tb_event_record(tb_stream_t s, tb_event_t *ev);
/* DeviceEvent.is_complete() (src/device.py:102-103): TB_OK when complete,
 * TB_NOT_READY otherwise. Never blocks. */
int tb_event_query(tb_event_t ev);
/* VirtualDevice.event_wait (src/device.py:281-309): block until complete
 * (the FENCE baseline). */
int tb_event_wait(tb_event_t ev);
int tb_event_release(tb_event_t ev);
/* VirtualDevice(record_timeline=True) (src/device.py:223-224,512-514): a
 * timing-enabled event (not pooled) recorded on s; tb_tevent_elapsed gives
 * the ms from a to b once both completed (TB_NOT_READY before). */
int tb_tevent_record(tb_stream_t s, tb_event_t *ev);
int tb_tevent_elapsed(tb_event_t a, tb_event_t b, double *ms);
int tb_tevent_release(tb_event_t ev);
int tb_stream_wait_event(tb_stream_t s, tb_event_t ev);
/* VirtualDevice(event_pool=...) (src/device.py:221,410-411): 1 = recycle
 * events through the pool, 0 = create/destroy per record (ablation). */
int tb_event_pool_set(int enabled);
int tb_event_pool_stats(int64_t *created, int64_t *reused, int64_t *live);

/* ------------------------------------------------------------ memory -- */
int tb_malloc(void **p, size_t n);
int tb_free(void *p);
int tb_host_alloc(void **p, size_t n);       /* pinned host memory         */
int tb_host_free(void *p);
/* make_h2d / make_d2h compute closures (src/executors.py:278-279, 283-284). */
int tb_memcpy_h2d(tb_stream_t s, void *dst, const void *src, size_t n);
int tb_memcpy_d2h(tb_stream_t s, void *dst, const void *src, size_t n);
int tb_memcpy_d2d(tb_stream_t s, void *dst, const void *src, size_t n);
int tb_memset(tb_stream_t s, void *p, int value, size_t n);

/* ----------------------------------------------------------- kernels -- */
/* K1: kernel_transform(kind)(view) (src/miniapp.py:40-53) on n doubles in
 * place: x = __dadd_rn(__dmul_rn(x, C1[kind]), C2[kind]). */
int tb_transform(tb_stream_t s, int kind, double *d, int64_t n);
/* A registered kind's transform (src/executors.py:171-172) as a descriptor:
 * op = TB_OP_NONE | TB_OP_KIND | TB_OP_AFFINE. */
int tb_launch(tb_stream_t s, int op, int kind, double c1, double c2, double *d,
              int64_t n);
/* make_barrier() (src/device.py:136-137): an empty ordering kernel. */
int tb_barrier(tb_stream_t s);
/* Keep a queue busy for `ns` nanoseconds (stands in for the reference tests'
 * long make_kernel(100_000) gate ops, pkg/tests/test_executors.py:129). */
int tb_spin(tb_stream_t s, int64_t ns);
/* SubGrid.__init__ (src/miniapp.py:72-77) for sub-grids [lo, lo+n) of S:
 * cells[g][i] = ((lo+g)*1000 + i) / (S*1000 + 512), correctly rounded. */
int tb_init_cells(tb_stream_t s, double *cells, int64_t subgrids, int64_t lo,
                  int64_t n);

/* One AggregationExecutor batch (src/executors.py:257-284) as one call:
 * H2D(dbuf <- hbuf) ; kernel(op, kind, c1, c2) over nbytes/8 doubles ;
 * [barrier if barrier != 0] ; D2H(hbuf <- dbuf) ; record *done.
 * hbuf holds the marshalled members on entry and the landing on completion. */
int tb_agg_launch(tb_stream_t s, int op, int kind, double c1, double c2,
                  double *dbuf, double *hbuf, size_t nbytes, int barrier,
                  tb_event_t *done);

/* K2: one fused time step over n consecutive sub-grids (src/miniapp.py:116-133
 * per sub-grid == src/reference.py:31-47): ghost fold against the previous
 * generation, chains x kernels_per_chain transforms, per-sub-grid min and
 * numpy-order pairwise sum. old/out: [n][512] doubles (out != old).
 * left_face: 8 doubles, right face of the sub-grid before old[0];
 * right_face: 8 doubles, left face of the sub-grid after old[n-1] (pass
 * old+(n-1)*512+504 and old for a full single-device ring).
 * mins/sums: optional [n] outputs (NULL to skip).
 * acc: optional TB_ACC_WORDS accumulator; the step's exact sum and min are
 * added into it (NULL to skip). */
int tb_step(tb_stream_t s, const double *old, double *out, int64_t n,
            const double *left_face, const double *right_face, int chains,
            int kernels_per_chain, double *mins, double *sums, int64_t *acc);
/* tb_step with the step closed in the same launch (single device): the last
 * CTA to finish rounds the accumulator exactly as tb_acc_finalize(..., reset=1)
 * would and writes piece / dt / checksum (device pointers, may be NULL).
 * acc is required and must be reset (tb_acc_reset) before the first use. */
int tb_step_final(tb_stream_t s, const double *old, double *out, int64_t n,
                  const double *left_face, const double *right_face, int chains,
                  int kernels_per_chain, double *mins, double *sums, int64_t *acc,
                  double *piece, double *dt, double *checksum);
/* Back-to-back single-device steps with the exact close off the critical
 * path: this launch only writes each sub-grid's pairwise sum and min (sums,
 * mins: [n], required — the reference's per-sub-grid outputs,
 * src/miniapp.py:133), and one extra CTA reduces the PREVIOUS step's
 * (prev_sums, prev_mins) — exact sum == math.fsum, min — through the scratch
 * accumulator acc into prev_piece / prev_dt and *checksum += prev_piece while
 * the other CTAs stream. prev_sums = NULL on the first step; sums/mins must
 * alternate between two buffers; tb_step_close closes the last step (acc
 * reset on entry, as after every close). */
int tb_step_deferred(tb_stream_t s, const double *old, double *out, int64_t n,
                     const double *left_face, const double *right_face, int chains,
                     int kernels_per_chain, double *sums, double *mins,
                     const double *prev_sums, const double *prev_mins, int64_t *acc,
                     double *prev_piece, double *prev_dt, double *checksum);
int tb_step_close(tb_stream_t s, const double *sums, const double *mins, int64_t n,
                  int64_t *acc, double *piece, double *dt, double *checksum);
/* Zero an accumulator (limbs = 0, min = +inf). */
int tb_acc_reset(tb_stream_t s, int64_t *acc);
/* Exact sum of n doubles into acc (the reduction half of tb_step). */
int tb_acc_add(tb_stream_t s, const double *x, int64_t n, int64_t *acc);
/* Close a step (src/miniapp.py:164-171 + :227): piece = correctly rounded
 * sum (== math.fsum), dt = min; if checksum != NULL: *checksum += piece.
 * Outputs are device pointers (any may be NULL). reset != 0 re-zeroes acc. */
int tb_acc_finalize(tb_stream_t s, int64_t *acc, double *piece, double *dt,
                    double *checksum, int reset);

/* ---------------------------------------------------- peer memory -- */
/* CUDA IPC for the multi-GPU ring: export the allocation containing dptr
 * (handle = TB_IPC_HANDLE_BYTES bytes; *offset = dptr - allocation base, so
 * sub-allocated buffers work), map a peer's export (returns the base), unmap. With the
 * neighbours' state buffers mapped, tb_step's left_face/right_face may point
 * into peer HBM: the ring halo exchange (src/miniapp.py:119-121 across a
 * partition boundary) is then two 64-byte NVLink loads inside K2. */
#define TB_IPC_HANDLE_BYTES 64
int tb_ipc_get_handle(void *dptr, uint8_t *handle, uint64_t *offset);
int tb_ipc_open_handle(const uint8_t *handle, void **dptr);
int tb_ipc_close(void *dptr);

/* The step's cross-rank reduction over peer memory (replaces the two
 * all-reduces of the multi-GPU step, and is its step barrier): adds
 * local_acc into every rank's accumulator for this step's parity
 * (peer_accs: DEVICE array of nranks pointers, IPC-mapped, own entry local)
 * with system-scope atomics, bumps each rank's TB_ACC_COUNT_WORD, resets
 * local_acc, waits until my_acc has nranks arrivals, then finalises my_acc
 * exactly as tb_acc_finalize(..., reset=1). Accumulators must alternate
 * between two parities step to step. The arrival wait traps after
 * TB_P2P_TIMEOUT_S seconds (environment; default 30, 0 = never). */
int tb_acc_allreduce_p2p(tb_stream_t s, int64_t *local_acc, int64_t *const *peer_accs,
                         int nranks, int64_t *my_acc, double *piece, double *dt,
                         double *checksum);
/* The same with an explicit watchdog: timeout_ns (0 = wait forever) and a
 * diagnostic record — diag: 4 int64 in mapped pinned host memory
 * (tb_host_alloc), written before the trap as {0x7470325774696d65, rank,
 * step, arrivals seen} so the host can say which rank waited for whom even
 * after the context is lost. */
int tb_acc_allreduce_p2p_ex(tb_stream_t s, int64_t *local_acc, int64_t *const *peer_accs,
                            int nranks, int64_t *my_acc, double *piece, double *dt,
                            double *checksum, int64_t timeout_ns, int64_t rank, int64_t step,
                            int64_t *diag);

/* K6 (north_star "hydro reconstruct+flux only", BASELINE config 2; PARITY
 * UNPINNED — no hydro exists in the reference, SPEC.md:17,490 — the spec is
 * oracle/hydro_oracle.py): dU/dt of a batch of nsub sub-grids.
 * U: [nsub][5][12][12][12] float64 (rho, sx, sy, sz, E; 8^3 interior cells
 * with 2-cell ghost layers, i fastest, 16-B aligned); dudt: [nsub][5][8][8][8];
 * amax: [nsub] max signal speed (CFL). Minmod PLM on primitives + Kurganov-
 * Tadmor/LLF flux, ideal gas with adiabatic index gamma, cell size dx. */
int tb_hydro_flux(tb_stream_t s, const double *U, double *dudt, double *amax,
                  int64_t nsub, double dx, double gamma);

/* K6 on a ghost-padded global lattice (the coupled step's layout):
 * Up [5][n+4][n+4][n+4] (2-cell ghost layer already filled, e.g. by
 * tb_star_pad); sub-grid s = (bz*nb + by)*nb + bx (nb = n/8) is staged by one
 * 4-D TMA box; dudt [nb^3][5][8][8][8], amax [nb^3] as tb_hydro_flux. A z-slab
 * of nz planes (Up [5][nz+4][n+4][n+4]) gives nb*nb*nz/8 sub-grids. */
int tb_hydro_flux_lattice(tb_stream_t s, const double *Up, int64_t n, int64_t nz,
                          double *dudt, double *amax, double dx, double gamma);
/* Profiling probe (not on the product path): the per-CTA %globaltimer
 * stamps, ns, of the last K6 launch made with TB_HYDRO_VARIANT=1020 —
 * out[n][4] = entry, first sub-grid staged, last faces done, exit; n <= 1024. */
int tb_hydro_stamps(unsigned long long *out, int n);

/* The coupled rotating-star step (PARITY UNPINNED; spec oracle/star_oracle.py):
 * U [5][n][n][n] lattice (rho, sx, sy, sz, E), periodic hydro, isolated FMM
 * gravity. tb_star_pad fills Up with the periodic ghost layer; tb_star_cfl
 * writes dt = cfl*dx/max(amax) to device memory; tb_star_stage applies
 * L(U) = dU/dt + (0, rho g, s.g) with g = rows 1..3 of the FMM output:
 * stage 1: Unew = Uc + dt L(Uc); stage 2: Unew = 0.5 (U0 + (Uc + dt L(Uc)))
 * (Unew may alias U0). No FMA: matches the oracle's rounding. */
int tb_star_pad(tb_stream_t s, const double *U, int64_t n, double *Up);
/* Slab of nz planes: lo/hi = the 2 planes below/above from the z-neighbours
 * ([5][2][n][n]; both null = wrap inside the slab). */
int tb_star_pad_slab(tb_stream_t s, const double *U, int64_t n, int64_t nz, const double *lo,
                     const double *hi, double *Up);
int tb_star_cfl(tb_stream_t s, const double *amax, int64_t nsub, double dx, double cfl,
                double *dt);
int tb_star_stage(tb_stream_t s, int stage, const double *U0, const double *Uc,
                  const double *dudt, const double *g, const double *dt, int64_t n, int64_t nz,
                  double *Unew);

/* K7 (north_star "FMM monopole/multipole stencil-interaction kernels",
 * BASELINE config 3; PARITY UNPINNED — no gravity exists in the reference,
 * the spec is oracle/fmm_oracle.py, matched to 1e-10
 * relative): gravity of a uniform octree of depth max_level (1..7) whose
 * leaves are the N^3 cells of rho (N = 8 * 2^max_level, lattice z,y,x with
 * x fastest, unit cube, isolated boundary). work: device workspace of
 * tb_fmm_workspace_bytes (per-level moments and local expansions);
 * out: [4][N^3] = phi, gx, gy, gz (g = -grad phi, G = 1).
 * tb_fmm_solve = upward (P2M + M2M) ; m2l (all multipole levels, one launch) ;
 * downward (L2L) ; leaf (monopole stencil + L2P), all on stream s. */
int tb_fmm_workspace_bytes(int max_level, uint64_t *bytes);
int tb_fmm_upward(tb_stream_t s, int max_level, const double *rho, double *work);
int tb_fmm_m2l(tb_stream_t s, int max_level, double *work);
int tb_fmm_downward(tb_stream_t s, int max_level, double *work);
int tb_fmm_leaf(tb_stream_t s, int max_level, const double *rho, const double *work,
                double *out);
int tb_fmm_solve(tb_stream_t s, int max_level, const double *rho, double *work, double *out);

/* The same solve split over `ranks` devices by z-slabs of the leaf lattice
 * (ranks a power of two, N/ranks a multiple of 16; the single-device calls
 * above are ranks = 1). Levels >= lp are partitioned (this rank keeps
 * N_l/ranks planes; reduced moment records carry 4 halo planes per side that
 * the caller fills from the z-neighbours — zero at the domain boundary —
 * between upward and m2l); levels < lp are replicated: the caller all-gathers
 * the raw and reduced records of level lp-1 (each rank computes its own
 * slab of it in tb_fmm_slab_upward), then tb_fmm_slab_coarse builds the
 * coarser levels. The workspace must be zeroed once (halo planes).
 * info (tb_fmm_slab_layout, 8 words): byte offsets of the level's raw
 * records [nzr][N][N][20], reduced records [nzr+2 halo][N][N][18] and local
 * expansions [nz][N][N][20]; N; nz (planes kept); z0 (global plane of local
 * plane 0); halo; lp. Leaves: rho points at this rank's first leaf plane,
 * planes [zmin, zmax) relative to it are readable; out [4][nz][N][N]. */
int tb_fmm_slab_workspace_bytes(int max_level, int ranks, uint64_t *bytes);
int tb_fmm_slab_layout(int max_level, int ranks, int rank, int level, uint64_t *info);
int tb_fmm_slab_upward(tb_stream_t s, int max_level, int ranks, int rank, const double *rho,
                       double *work);
int tb_fmm_slab_coarse(tb_stream_t s, int max_level, int ranks, int rank, double *work);
int tb_fmm_slab_m2l(tb_stream_t s, int max_level, int ranks, int rank, double *work);
int tb_fmm_slab_downward(tb_stream_t s, int max_level, int ranks, int rank, double *work);
int tb_fmm_slab_leaf(tb_stream_t s, int max_level, int ranks, int rank, const double *rho,
                     int zmin, int zmax, const double *work, double *out);

/* FP64 issue-rate probe (roofline denominator; no reference counterpart):
 * runs one FP64 instruction type on 8 independent chains per thread over a
 * full grid on the current device and returns thread-instructions/s and the
 * nominal SM clock (MHz). op = TB_PROBE_*. Blocking. */
#define TB_PROBE_DADD 0
#define TB_PROBE_DMUL 1
#define TB_PROBE_DFMA 2
#define TB_PROBE_DMUL_DADD 3
int tb_fp64_probe(int op, int64_t iters, double *instr_per_s, double *sm_mhz);

/* The branch-free division / square-root fast paths the hydro kernel uses
 * (no reference counterpart), exposed for testing: for i < n, q[i] = a[i] /
 * b[i] and r[i] = sqrt(a[i]) through the fast path (the IEEE intrinsic where
 * it flags); *slow_count += the flagged cases. The tests compare q and r
 * bitwise with IEEE division and square root. Device pointers; enqueued on s. */
int tb_divsqrt_fast(tb_stream_t s, const double *a, const double *b, int64_t n, double *q,
                    double *r, unsigned long long *slow_count);

/* -------------------------------------------------- poll registry -- */
/* PollRegistry (src/runtime/polling.py:17-147): a lock-free MPSC inbox of
 * (event, token) and a poll-owned pending vector, drained by a single-entrant
 * poll body that queries events with cudaEventQuery. */
int tb_poll_create(tb_poll_t *reg);
int tb_poll_destroy(tb_poll_t reg);
/* PollRegistry.add (polling.py:53-55): any thread, lock-free. `chain`: 0, or
 * an id of the in-order queue the event was recorded on — entries of one chain
 * complete in registration order, so poll only queries each chain's head. */
int tb_poll_add(tb_poll_t reg, tb_event_t ev, uint64_t chain, uint64_t token);
/* tb_poll_add with the event's record order on its chain (seq > 0, increasing
 * in record order, assigned under the queue's lock): the entry is placed in
 * record order even when it is registered after a later-recorded event of the
 * same queue (registration runs outside the queue lock, as in the reference's
 * Integration.get_future, src/bridge.py:54-70). */
int tb_poll_add_seq(tb_poll_t reg, tb_event_t ev, uint64_t chain, uint64_t seq,
                    uint64_t token);
/* PollRegistry.poll (polling.py:80-120): drain inbox, re-check pending,
 * write up to cap fired tokens (FIFO within a chain). TB_NOT_READY (and
 * *nfired = 0) when another thread holds the guard. Complete entries beyond
 * cap stay pending. Never blocks (cudaEventQuery only). status (optional,
 * parallel to fired): 0, or -cudaError when the event's query reported a
 * device fault — the caller faults that entry's future instead of running
 * its callback (errors surface as Faulted futures, src/executors.py:50-55,
 * src/runtime/polling.py:71-75). */
int tb_poll(tb_poll_t reg, uint64_t *fired, int32_t *status, int cap, int *nfired);
int tb_poll_pending(tb_poll_t reg, int64_t *n);
/* abandon_all (polling.py:122-147): remove every entry; complete[i] says
 * whether token i's event had completed (1: run callback), not (0: abandon)
 * or faulted (2: fault the future). */
int tb_poll_drain(tb_poll_t reg, uint64_t *tokens, uint8_t *complete, int cap,
                  int *n);
int tb_poll_entry_high_water(tb_poll_t reg, int *hw);

/* ---------------------------------------------------- host tasks -- */
/* VirtualDevice.register_host_task (src/device.py:311-321) and its
 * dispatcher threads (src/device.py:541-567): after `ev` completes on the
 * device, `token` becomes available to tb_htq_next. Implemented with
 * cudaStreamWaitEvent + a stream callback on side streams owned by the queue;
 * the CUDA callback only enqueues (no CUDA calls, no Python). */
int tb_htq_create(int side_streams, tb_htq_t *q);
int tb_host_task(tb_htq_t q, tb_event_t ev, uint64_t token);
/* Block up to timeout_us for the next ready token: TB_OK / TB_NOT_READY
 * (timeout) / TB_E_CLOSED (closed and empty). *status (optional): 0, or
 * -cudaError when the device faulted before the event (fault the future). */
int tb_htq_next(tb_htq_t q, uint64_t *token, int *status, int64_t timeout_us);
int tb_htq_close(tb_htq_t q);
int tb_htq_destroy(tb_htq_t q);

/* ------------------------------------------------- native machine -- */
/* The reference machine (src/cli.py:199-232 run_single: Runtime + device +
 * Integration + executors + run_scenario) as one native call: a C++
 * work-stealing pool whose workers run the mini-app's per-sub-grid tasks, an
 * aggregation executor per CUDA stream, and completion surfaced by event
 * POLLING in the workers' idle loop, by HOSTTASK threads, or by FENCE. */
#define TB_MODE_POLLING 0
#define TB_MODE_HOSTTASK 1
#define TB_MODE_FENCE 2

typedef struct {
  int64_t subgrids;          /* ScenarioConfig.subgrids                     */
  int64_t steps;
  int64_t chains;            /* 3 */
  int64_t kernels_per_chain; /* 5 */
  int64_t workers;           /* RunConfig.workers                            */
  int64_t executors;         /* RunConfig.executors (CUDA streams)           */
  int64_t max_agg;           /* RunConfig.max_agg                            */
  int64_t mode;              /* TB_MODE_*                                    */
  int64_t inject_barriers;   /* barrier op between kernel and D2H            */
  int64_t barrier_elision;   /* drop those barriers                          */
  int64_t task_subgrids;     /* sub-grids per task (1 = reference structure) */
  int64_t hosttask_threads;  /* 2 */
  int64_t zero_copy;         /* 0: the reference op sequence (H2D ; kernel ;
                                D2H per batch). 1: the batch kernel runs in
                                place on the pinned staging buffer (mapped
                                host memory over PCIe): one launch + one event
                                per batch, no copy ops (mini-app only).
                                2: no staging at all — the tasks' work
                                buffers live in one pinned arena and the
                                batch kernel reads each member's rows and
                                writes its output rows there directly
                                (tb_launch_gather): no marshal/scatter
                                memcpy, one launch + one event per batch.
                                3: gather, with each task's rounds resident
                                in HBM — round 1 reads the host-folded rows
                                from pinned memory, the last round writes
                                them back there, the rounds between ping-pong
                                in device memory (two PCIe crossings per
                                sub-grid and step instead of 30).           */
  int64_t fault_at_launch;   /* fault injection (tests): the k-th batch launch
                                of the run (k >= 1) runs a trapping kernel;
                                the device fault must surface as this call's
                                error, in every mode. 0 = off.               */
  int64_t completion;        /* how batch completion reaches the scheduler:
                                TB_COMPLETION_EVENTS (0): a CUDA event per
                                batch and idleness probe, queried by the poll
                                body / synchronized by FENCE / stream
                                callbacks for HOSTTASK. TB_COMPLETION_WORDS
                                (1, zero_copy >= 2, POLLING or FENCE): the
                                batch kernel's last CTA stores the batch's
                                sequence number in its executor's mapped
                                word (tb_done); the poll body / FENCE read
                                memory, a probe waits for the executor's
                                last issued number — no event records, no
                                driver queries.                              */
} tb_machine_config;

#define TB_COMPLETION_EVENTS 0
#define TB_COMPLETION_WORDS 1

typedef struct {             /* StepMetrics (src/miniapp.py:103-113)         */
  double wall_ms, dt, piece;
  int64_t launches, transfers, event_waits, full, idle, members;
} tb_machine_step;

/* Runs cfg->steps steps; *checksum = sum of pieces (src/miniapp.py:227);
 * steps_out[cfg->steps] (optional); cells_out[subgrids*512] (optional). */
int tb_machine_run(const tb_machine_config *cfg, double *checksum,
                   tb_machine_step *steps_out, double *cells_out);
/* tb_machine_run on the caller's cells (run_scenario on an existing
 * Scenario, src/miniapp.py:185-229): cells [subgrids][512] hold the initial
 * state on entry and are advanced in place (each task writes its sub-grids
 * back, src/miniapp.py:132), so they hold the final state on success and the
 * state the tasks reached on a device fault. The task arenas of zero_copy
 * 2/3 are cached in the library between runs. exec_stats (optional):
 * [steps][executors][max_agg + 3] int64 — per step and executor, batches by
 * member count (index = count) then full- and idle-triggered launches (the
 * AggregationExecutor's batch_sizes / reasons, src/executors.py:166-169). */
int tb_machine_run_cells(const tb_machine_config *cfg, double *cells, double *checksum,
                         tb_machine_step *steps_out, int64_t *exec_stats);
/* One aggregated batch whose members stay where they are (zero_copy = 2):
 * dst[i][0..n[i]) = transform(src[i][0..n[i])) for i < members, the pointers
 * being device-accessible (device or mapped pinned host memory, 16-B
 * aligned, n[i] even). op/kind/c1/c2 as tb_launch. Up to
 * TB_GATHER_MAX members per launch. */
#define TB_GATHER_MAX 256
int tb_launch_gather(tb_stream_t s, int op, int kind, double c1, double c2,
                     const double *const *src, double *const *dst, const int64_t *n,
                     int members);
/* A batch's completion word: the launch's last CTA stores seq into *word
 * (mapped pinned host memory, 8-B aligned) after every CTA's writes are
 * visible system-wide; ctas is a device counter that is 0 before the launch
 * and reset to 0 by the last CTA (one per stream: launches on a stream are
 * ordered). The host then sees completion by reading memory — no event
 * record, no driver query (the machine's completion = words). */
typedef struct {
  uint64_t *word;
  uint64_t seq;
  unsigned *ctas;
} tb_done;
/* tb_launch_gather that also signals *done (NULL = none; op must be
 * TB_OP_KIND / TB_OP_AFFINE, or TB_OP_TRAP for fault injection, which never
 * signals). */
int tb_launch_gather_done(tb_stream_t s, int op, int kind, double c1, double c2,
                          const double *const *src, double *const *dst, const int64_t *n,
                          int members, const tb_done *done);
/* A gather batch of kind `kind` whose members are whole sub-grids and may be
 * a task's first and/or last round (the machine's direct mode, zero_copy =
 * 4): member i = sub-grids [g0[i], g0[i] + nsub[i]) of the S-ring, read from
 * src[i] and written to dst[i] ([nsub[i]][512], device-accessible, 16-B
 * aligned). flags[i] bit 0: fold the first and last 8 cells of each input
 * sub-grid with the neighbours' faces (faces [S][2][8] = (left, right) of the
 * previous generation; src/miniapp.py:119-126) before the transform; bit 1:
 * mins[g] / sums[g] = min and numpy-order pairwise sum of each output
 * sub-grid (src/miniapp.py:133). Same two roundings as tb_launch. done:
 * as tb_launch_gather_done (NULL = none). */
int tb_launch_gather_edge(tb_stream_t s, int kind, const double *const *src,
                          double *const *dst, const int64_t *g0, const int32_t *nsub,
                          const uint8_t *flags, int members, const double *faces,
                          double *mins, double *sums, int64_t S, const tb_done *done);

/* One aggregated hydro batch (the Octo-Tiger use of src/executors.py:257-284,
 * PAPER.md:762-773): H2D(din <- hin: nsub ghosted sub-grids [5][12^3]) ;
 * K6 ; D2H(hout <- dout: dU/dt [nsub][5][512] then amax [nsub]) ; record
 * *done. din/dout device, hin/hout pinned host. */
int tb_agg_launch_hydro(tb_stream_t s, double *din, const double *hin, int64_t nsub,
                        double *dout, double *hout, double dx, double gamma,
                        tb_event_t *done);

/* The same machine on the north_star's hydro kernel (PARITY UNPINNED; spec
 * oracle/hydro_oracle.py euler_step): per step, one task per task_subgrids
 * sub-grids builds their periodic ghost layers on the host and schedules a
 * K6 request on its executor (aggregated up to max_agg per launch, completed
 * by cfg->mode); then dt = cfl*dx/max(amax) and U += dt*dU/dt (host tasks).
 * subgrids must be a cube n^3 (sub-grid order x fastest); chains,
 * kernels_per_chain, inject_barriers, barrier_elision are ignored.
 * U_in/U_out: [subgrids][5][8][8][8]; piece = exact sum of all rho. */
int tb_machine_run_hydro(const tb_machine_config *cfg, const double *U_in, double *U_out,
                         double cfl, double gamma, tb_machine_step *steps_out);

#ifdef __cplusplus
}
#endif
#endif /* TB_H_ */
