// tb_runtime.cu — the device layer of libtb: queues (CUDA streams), pooled
// completion events, memory, the fused aggregation launch, the native poll
// registry and the host-task dispatcher.
//
// Replaces the reference's simulated accelerator (src/device.py) and the
// Python poll body (src/runtime/polling.py). Design notes:
//  * Queues are non-blocking CUDA streams: in-order like DeviceQueue
//    (src/device.py:157-180), ordered on the device, no host lock.
//  * Events come from a pool of cudaEventDisableTiming events, so recording
//    costs no allocation (the reference's event_pool toggle,
//    src/device.py:221,410-411).
//  * The poll registry keeps the reference contract — lock-free producers,
//    single-entrant poll body that never blocks — but queries events in
//    native code and hands back fired tokens in one call, so the Python side
//    takes the GIL once per poll rather than once per event.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace tb {
namespace {

std::atomic<int> g_device{-1};
thread_local int t_device = -1;

// Bind the calling thread to the device chosen by tb_init (once per thread).
inline int ensure_device() {
  const int d = g_device.load(std::memory_order_relaxed);
  if (d < 0 || t_device == d) return TB_OK;
  const int r = rc(cudaSetDevice(d));
  if (r == TB_OK) t_device = d;
  return r;
}

// ------------------------------------------------------------ event pool --
struct EventPool {
  std::mutex mu;
  std::vector<cudaEvent_t> free_list;
  bool enabled = true;
  int64_t created = 0, reused = 0, live = 0;
};
EventPool &pool() {
  static EventPool *p = new EventPool();  // leaked on purpose: no exit-order issues
  return *p;
}

int event_acquire(cudaEvent_t *out) {
  EventPool &p = pool();
  {
    std::lock_guard<std::mutex> g(p.mu);
    if (p.enabled && !p.free_list.empty()) {
      *out = p.free_list.back();
      p.free_list.pop_back();
      ++p.reused;
      ++p.live;
      return TB_OK;
    }
  }
  const int r = rc(cudaEventCreateWithFlags(out, cudaEventDisableTiming));
  if (r == TB_OK) {
    std::lock_guard<std::mutex> g(p.mu);
    ++p.created;
    ++p.live;
  }
  return r;
}

int event_release(cudaEvent_t e) {
  EventPool &p = pool();
  {
    std::lock_guard<std::mutex> g(p.mu);
    --p.live;
    if (p.enabled) {
      p.free_list.push_back(e);
      return TB_OK;
    }
  }
  return rc(cudaEventDestroy(e));
}

inline cudaStream_t S(tb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline cudaEvent_t E(tb_event_t e) { return reinterpret_cast<cudaEvent_t>(e); }

// ---------------------------------------------------------- poll registry --
struct PollNode {
  cudaEvent_t ev;
  uint64_t chain;
  uint64_t token;
  uint64_t seq;     // record order on the chain (0: append in registration order)
  PollNode *next;
};

// Entries on the same non-zero chain (an in-order queue) complete in
// registration order, so the poll body only queries each chain's head.
struct Registry {
  std::atomic<PollNode *> inbox{nullptr};
  std::vector<PollNode *> unchained;                              // guard holder
  std::unordered_map<uint64_t, std::deque<PollNode *>> chains;    // guard holder
  std::atomic<bool> guard{false};
  std::atomic<int> entries{0};
  std::atomic<int> high_water{0};
  std::atomic<int64_t> pending_n{0};

  void drain_inbox() {
    PollNode *list = inbox.exchange(nullptr, std::memory_order_acquire);
    PollNode *fifo = nullptr;
    while (list) {  // reverse the LIFO stack
      PollNode *nx = list->next;
      list->next = fifo;
      fifo = list;
      list = nx;
    }
    while (fifo) {
      PollNode *nx = fifo->next;
      if (fifo->chain) {
        // keep each chain in record order: a producer may register after a
        // later-recorded event of the same stream (registration happens
        // outside the queue lock), and the poll body queries only the head
        std::deque<PollNode *> &dq = chains[fifo->chain];
        auto pos = dq.end();
        if (fifo->seq)
          while (pos != dq.begin() && (*(pos - 1))->seq > fifo->seq) --pos;
        dq.insert(pos, fifo);
      } else {
        unchained.push_back(fifo);
      }
      fifo = nx;
    }
  }
};

// --------------------------------------------------------- host-task queue --
struct Htq;
struct HtItem {
  Htq *q;
  uint64_t token;
};
struct Htq {
  std::vector<cudaStream_t> side;
  std::atomic<unsigned> rr{0};
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::pair<uint64_t, int>> ready;   // (token, 0 or -cudaError)
  bool closed = false;
};

// A stream callback (not cudaLaunchHostFunc, which is never called once the
// context has faulted): it receives the stream's status, so a device fault
// reaches the waiting future as an error instead of leaving it pending.
void CUDART_CB ht_trampoline(cudaStream_t, cudaError_t status, void *p) {
  // Runs on a CUDA driver thread: no CUDA calls, no Python — only enqueue.
  HtItem *it = static_cast<HtItem *>(p);
  Htq *q = it->q;
  {
    std::lock_guard<std::mutex> g(q->mu);
    q->ready.emplace_back(it->token, status == cudaSuccess ? 0 : -(int)status);
  }
  q->cv.notify_one();
  delete it;
}

}  // namespace

int sm_count() {
  static std::atomic<int> cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cached[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      v <= 0)
    v = 148;
  cached[dev].store(v, std::memory_order_relaxed);
  return v;
}

int encode_tiled(CUtensorMap *map, int rank, void *base, const uint64_t *dims,
                 const uint64_t *strides_bytes, const uint32_t *box) {
  using Fn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                          const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                          const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn enc = nullptr;
  if (!enc) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    const int r = rc(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (r != TB_OK) return r;
    if (!p || q != cudaDriverEntryPointSuccess) return TB_E_INVALID;
    enc = reinterpret_cast<Fn>(p);
  }
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, base, d, st, b, e,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? TB_OK
             : TB_E_INVALID;
}

}  // namespace tb

using namespace tb;

extern "C" {

int tb_abi_version(void) { return TB_ABI_VERSION; }

const char *tb_error_string(int r) {
  if (r == TB_OK) return "ok";
  if (r == TB_NOT_READY) return "not ready";
  if (r == TB_E_INVALID) return "invalid argument";
  if (r == TB_E_NOMEM) return "out of host memory";
  if (r == TB_E_CLOSED) return "closed";
  if (r < 0) return cudaGetErrorString(static_cast<cudaError_t>(-r));
  return "unknown";
}

int tb_init(int device) {
  int n = 0;
  int r = rc(cudaGetDeviceCount(&n));
  if (r != TB_OK) return r;
  if (device < 0 || device >= n) return TB_E_INVALID;
  g_device.store(device);
  t_device = -1;
  r = ensure_device();
  if (r != TB_OK) return r;
  r = rc(cudaFree(nullptr));  // create/attach the primary context
  if (r != TB_OK) return r;
  // Warm the event pool so steady-state records never allocate.
  std::vector<cudaEvent_t> warm(64);
  for (auto &e : warm)
    if ((r = event_acquire(&e)) != TB_OK) return r;
  for (auto &e : warm) event_release(e);
  return TB_OK;
}

int tb_device_count(int *n) {
  if (!n) return TB_E_INVALID;
  return rc(cudaGetDeviceCount(n));
}

int tb_sm_count(int device, int *n) {
  if (!n) return TB_E_INVALID;
  return rc(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, device));
}

int tb_device_sync(void) {
  ensure_device();
  return rc(cudaDeviceSynchronize());
}

// ----------------------------------------------------------------- queues
int tb_stream_create(tb_stream_t *s) {
  if (!s) return TB_E_INVALID;
  ensure_device();
  cudaStream_t st;
  const int r = rc(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  if (r == TB_OK) *s = reinterpret_cast<tb_stream_t>(st);
  return r;
}

int tb_stream_destroy(tb_stream_t s) {
  ensure_device();
  return rc(cudaStreamDestroy(S(s)));
}

int tb_stream_query(tb_stream_t s) {
  ensure_device();
  const cudaError_t e = cudaStreamQuery(S(s));
  if (e == cudaErrorNotReady) return TB_NOT_READY;
  return rc(e);
}

int tb_stream_sync(tb_stream_t s) {
  ensure_device();
  return rc(cudaStreamSynchronize(S(s)));
}

// ----------------------------------------------------------------- events
int tb_event_record(tb_stream_t s, tb_event_t *ev) {
  if (!ev) return TB_E_INVALID;
  ensure_device();
  cudaEvent_t e;
  int r = event_acquire(&e);
  if (r != TB_OK) return r;
  r = rc(cudaEventRecord(e, S(s)));
  if (r != TB_OK) {
    event_release(e);
    return r;
  }
  *ev = reinterpret_cast<tb_event_t>(e);
  return TB_OK;
}

// Timing events for CudaDevice(record_timeline=True): created per record
// (not pooled — a diagnostic mode), destroyed on release.
int tb_tevent_record(tb_stream_t s, tb_event_t *ev) {
  if (!ev) return TB_E_INVALID;
  ensure_device();
  cudaEvent_t e;
  int r = rc(cudaEventCreate(&e));
  if (r != TB_OK) return r;
  r = rc(cudaEventRecord(e, S(s)));
  if (r != TB_OK) {
    cudaEventDestroy(e);
    return r;
  }
  *ev = reinterpret_cast<tb_event_t>(e);
  return TB_OK;
}

int tb_tevent_elapsed(tb_event_t a, tb_event_t b, double *ms) {
  if (!a || !b || !ms) return TB_E_INVALID;
  const cudaError_t qa = cudaEventQuery(E(a)), qb = cudaEventQuery(E(b));
  if (qa == cudaErrorNotReady || qb == cudaErrorNotReady) return TB_NOT_READY;
  float f = 0.f;
  const int r = rc(cudaEventElapsedTime(&f, E(a), E(b)));
  if (r == TB_OK) *ms = (double)f;
  return r;
}

int tb_tevent_release(tb_event_t ev) {
  if (!ev) return TB_E_INVALID;
  return rc(cudaEventDestroy(E(ev)));
}

int tb_event_query(tb_event_t ev) {
  const cudaError_t e = cudaEventQuery(E(ev));
  if (e == cudaErrorNotReady) return TB_NOT_READY;
  return rc(e);
}

int tb_event_wait(tb_event_t ev) { return rc(cudaEventSynchronize(E(ev))); }

int tb_event_release(tb_event_t ev) {
  if (!ev) return TB_E_INVALID;
  return event_release(E(ev));
}

int tb_stream_wait_event(tb_stream_t s, tb_event_t ev) {
  ensure_device();
  return rc(cudaStreamWaitEvent(S(s), E(ev), 0));
}

int tb_event_pool_set(int enabled) {
  EventPool &p = pool();
  std::vector<cudaEvent_t> drop;
  {
    std::lock_guard<std::mutex> g(p.mu);
    p.enabled = enabled != 0;
    if (!p.enabled) drop.swap(p.free_list);
  }
  for (auto e : drop) cudaEventDestroy(e);
  return TB_OK;
}

int tb_event_pool_stats(int64_t *created, int64_t *reused, int64_t *live) {
  EventPool &p = pool();
  std::lock_guard<std::mutex> g(p.mu);
  if (created) *created = p.created;
  if (reused) *reused = p.reused;
  if (live) *live = p.live;
  return TB_OK;
}

// ----------------------------------------------------------------- memory
int tb_malloc(void **p, size_t n) {
  if (!p) return TB_E_INVALID;
  ensure_device();
  return rc(cudaMalloc(p, n ? n : 1));
}
int tb_free(void *p) {
  ensure_device();
  return rc(cudaFree(p));
}
int tb_host_alloc(void **p, size_t n) {
  if (!p) return TB_E_INVALID;
  ensure_device();
  return rc(cudaHostAlloc(p, n ? n : 1, cudaHostAllocPortable));
}
int tb_host_free(void *p) { return rc(cudaFreeHost(p)); }

int tb_memcpy_h2d(tb_stream_t s, void *dst, const void *src, size_t n) {
  if (n && (!dst || !src)) return TB_E_INVALID;
  ensure_device();
  return n ? rc(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, S(s))) : TB_OK;
}
int tb_memcpy_d2h(tb_stream_t s, void *dst, const void *src, size_t n) {
  if (n && (!dst || !src)) return TB_E_INVALID;
  ensure_device();
  return n ? rc(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, S(s))) : TB_OK;
}
int tb_memcpy_d2d(tb_stream_t s, void *dst, const void *src, size_t n) {
  if (n && (!dst || !src)) return TB_E_INVALID;
  ensure_device();
  return n ? rc(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, S(s))) : TB_OK;
}
int tb_memset(tb_stream_t s, void *p, int value, size_t n) {
  if (n && !p) return TB_E_INVALID;
  ensure_device();
  return n ? rc(cudaMemsetAsync(p, value, n, S(s))) : TB_OK;
}

// ------------------------------------------------------------ peer memory
// CUDA IPC: a rank exports its state buffers, ring neighbours map them and
// K2 reads the two ghost faces straight out of the neighbour's HBM (NVLink
// P2P on a multi-GPU node) — the halo exchange becomes two 64-byte loads.
int tb_ipc_get_handle(void *dptr, uint8_t *handle, uint64_t *offset) {
  if (!dptr || !handle || !offset) return TB_E_INVALID;
  ensure_device();
  // IPC exports whole allocations; sub-allocators (e.g. a caching allocator)
  // hand out interior pointers, so find the allocation base first.
  using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    int r = rc(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (r != TB_OK) return r;
    if (!fn || q != cudaDriverEntryPointSuccess) return TB_E_INVALID;
    get_range = reinterpret_cast<GetRange>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0)
    return TB_E_INVALID;
  cudaIpcMemHandle_t h;
  const int r = rc(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
  if (r == TB_OK) {
    memcpy(handle, &h, sizeof h);
    *offset = reinterpret_cast<unsigned long long>(dptr) - base;
  }
  return r;
}

int tb_ipc_open_handle(const uint8_t *handle, void **dptr) {
  if (!handle || !dptr) return TB_E_INVALID;
  ensure_device();
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return rc(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int tb_ipc_close(void *dptr) {
  if (!dptr) return TB_E_INVALID;
  ensure_device();
  return rc(cudaIpcCloseMemHandle(dptr));
}

// ------------------------------------------------------- aggregation batch
int tb_agg_launch(tb_stream_t s, int op, int kind, double c1, double c2,
                  double *dbuf, double *hbuf, size_t nbytes, int barrier,
                  tb_event_t *done) {
  if (!dbuf || !hbuf || !done || (nbytes % sizeof(double)) != 0) return TB_E_INVALID;
  ensure_device();
  nvtxRangePushA("tb_agg_launch");
  int r = tb_memcpy_h2d(s, dbuf, hbuf, nbytes);
  if (r == TB_OK) r = tb_launch(s, op, kind, c1, c2, dbuf, (int64_t)(nbytes / 8));
  if (r == TB_OK && barrier) r = tb_barrier(s);
  if (r == TB_OK) r = tb_memcpy_d2h(s, hbuf, dbuf, nbytes);
  if (r == TB_OK) r = tb_event_record(s, done);
  nvtxRangePop();
  return r;
}

int tb_agg_launch_hydro(tb_stream_t s, double *din, const double *hin, int64_t nsub,
                        double *dout, double *hout, double dx, double gamma,
                        tb_event_t *done) {
  if (!din || !hin || !dout || !hout || !done || nsub < 1) return TB_E_INVALID;
  ensure_device();
  const size_t in_bytes = (size_t)nsub * 5 * 1728 * 8, out_bytes = (size_t)nsub * (5 * 512 + 1) * 8;
  int r = tb_memcpy_h2d(s, din, hin, in_bytes);
  if (r == TB_OK) r = tb_hydro_flux(s, din, dout, dout + nsub * 5 * 512, nsub, dx, gamma);
  if (r == TB_OK) r = tb_memcpy_d2h(s, hout, dout, out_bytes);
  if (r == TB_OK) r = tb_event_record(s, done);
  return r;
}

// ---------------------------------------------------------- poll registry
int tb_poll_create(tb_poll_t *reg) {
  if (!reg) return TB_E_INVALID;
  Registry *r = new (std::nothrow) Registry();
  if (!r) return TB_E_NOMEM;
  *reg = reinterpret_cast<tb_poll_t>(r);
  return TB_OK;
}

int tb_poll_destroy(tb_poll_t reg) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r) return TB_E_INVALID;
  r->drain_inbox();
  for (PollNode *p : r->unchained) delete p;
  for (auto &kv : r->chains)
    for (PollNode *p : kv.second) delete p;
  delete r;
  return TB_OK;
}

int tb_poll_add(tb_poll_t reg, tb_event_t ev, uint64_t chain, uint64_t token) {
  return tb_poll_add_seq(reg, ev, chain, 0, token);
}

int tb_poll_add_seq(tb_poll_t reg, tb_event_t ev, uint64_t chain, uint64_t seq,
                    uint64_t token) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r || !ev) return TB_E_INVALID;
  PollNode *n = new (std::nothrow) PollNode{E(ev), chain, token, seq, nullptr};
  if (!n) return TB_E_NOMEM;
  PollNode *head = r->inbox.load(std::memory_order_relaxed);
  do {
    n->next = head;
  } while (!r->inbox.compare_exchange_weak(head, n, std::memory_order_release,
                                           std::memory_order_relaxed));
  r->pending_n.fetch_add(1, std::memory_order_relaxed);
  return TB_OK;
}

int tb_poll(tb_poll_t reg, uint64_t *fired, int32_t *status, int cap, int *nfired) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r || !nfired || cap < 0 || (cap > 0 && !fired)) return TB_E_INVALID;
  *nfired = 0;
  if (r->guard.exchange(true, std::memory_order_acquire)) return TB_NOT_READY;
  nvtxRangePushA("tb_poll");
  const int e = r->entries.fetch_add(1) + 1;
  int hw = r->high_water.load();
  while (e > hw && !r->high_water.compare_exchange_weak(hw, e)) {
  }
  int n = 0;
  r->drain_inbox();
  // Unchained entries: query each, keep the incomplete ones in order.
  {
    std::vector<PollNode *> &u = r->unchained;
    size_t keep = 0;
    for (size_t i = 0; i < u.size(); ++i) {
      PollNode *p = u[i];
      // A device fault fires the entry with its error code (status), so
      // the waiting future faults instead of hanging or reading garbage.
      const cudaError_t q = n < cap ? cudaEventQuery(p->ev) : cudaErrorNotReady;
      if (q != cudaErrorNotReady) {
        if (status) status[n] = q == cudaSuccess ? 0 : -(int)q;
        fired[n++] = p->token;
        delete p;
      } else {
        u[keep++] = p;
      }
    }
    u.resize(keep);
  }
  // Chains: pop completed heads; the first incomplete head blocks the chain.
  for (auto it = r->chains.begin(); it != r->chains.end();) {
    std::deque<PollNode *> &dq = it->second;
    while (!dq.empty() && n < cap) {
      const cudaError_t q = cudaEventQuery(dq.front()->ev);
      if (q == cudaErrorNotReady) break;
      if (status) status[n] = q == cudaSuccess ? 0 : -(int)q;
      fired[n++] = dq.front()->token;
      delete dq.front();
      dq.pop_front();
    }
    if (dq.empty())
      it = r->chains.erase(it);
    else
      ++it;
  }
  r->pending_n.fetch_sub(n, std::memory_order_relaxed);
  *nfired = n;
  r->entries.fetch_sub(1);
  r->guard.store(false, std::memory_order_release);
  nvtxRangePop();
  return TB_OK;
}

int tb_poll_pending(tb_poll_t reg, int64_t *n) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r || !n) return TB_E_INVALID;
  *n = r->pending_n.load(std::memory_order_relaxed);
  return TB_OK;
}

int tb_poll_drain(tb_poll_t reg, uint64_t *tokens, uint8_t *complete, int cap,
                  int *n) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r || !n || cap < 0 || (cap > 0 && (!tokens || !complete))) return TB_E_INVALID;
  *n = 0;
  // Blocking acquire of the guard (the reference takes it with `with`).
  while (r->guard.exchange(true, std::memory_order_acquire)) {
  }
  r->drain_inbox();
  int k = 0;
  auto take = [&](PollNode *p) -> bool {
    if (k >= cap) return false;
    tokens[k] = p->token;
    const cudaError_t q = cudaEventQuery(p->ev);
    complete[k] = q == cudaSuccess ? 1 : (q == cudaErrorNotReady ? 0 : 2);
    ++k;
    delete p;
    return true;
  };
  {
    std::vector<PollNode *> &u = r->unchained;
    size_t keep = 0;
    for (size_t i = 0; i < u.size(); ++i)
      if (!take(u[i])) u[keep++] = u[i];
    u.resize(keep);
  }
  for (auto it = r->chains.begin(); it != r->chains.end();) {
    std::deque<PollNode *> &dq = it->second;
    while (!dq.empty() && take(dq.front())) dq.pop_front();
    if (dq.empty())
      it = r->chains.erase(it);
    else
      ++it;
  }
  r->pending_n.fetch_sub(k, std::memory_order_relaxed);
  *n = k;
  r->guard.store(false, std::memory_order_release);
  return TB_OK;
}

int tb_poll_entry_high_water(tb_poll_t reg, int *hw) {
  Registry *r = reinterpret_cast<Registry *>(reg);
  if (!r || !hw) return TB_E_INVALID;
  *hw = r->high_water.load();
  return TB_OK;
}

// ------------------------------------------------------------- host tasks
int tb_htq_create(int side_streams, tb_htq_t *q) {
  if (!q || side_streams < 1 || side_streams > 64) return TB_E_INVALID;
  ensure_device();
  Htq *h = new (std::nothrow) Htq();
  if (!h) return TB_E_NOMEM;
  for (int i = 0; i < side_streams; ++i) {
    cudaStream_t st;
    const int r = rc(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (r != TB_OK) {
      for (auto s : h->side) cudaStreamDestroy(s);
      delete h;
      return r;
    }
    h->side.push_back(st);
  }
  *q = reinterpret_cast<tb_htq_t>(h);
  return TB_OK;
}

int tb_host_task(tb_htq_t q, tb_event_t ev, uint64_t token) {
  Htq *h = reinterpret_cast<Htq *>(q);
  if (!h || !ev) return TB_E_INVALID;
  {
    std::lock_guard<std::mutex> g(h->mu);
    if (h->closed) return TB_E_CLOSED;
  }
  ensure_device();
  cudaStream_t side = h->side[h->rr.fetch_add(1) % h->side.size()];
  int r = rc(cudaStreamWaitEvent(side, E(ev), 0));
  if (r != TB_OK) return r;
  HtItem *it = new (std::nothrow) HtItem{h, token};
  if (!it) return TB_E_NOMEM;
  r = rc(cudaStreamAddCallback(side, ht_trampoline, it, 0));
  if (r != TB_OK) delete it;
  return r;
}

int tb_htq_next(tb_htq_t q, uint64_t *token, int *status, int64_t timeout_us) {
  Htq *h = reinterpret_cast<Htq *>(q);
  if (!h || !token) return TB_E_INVALID;
  std::unique_lock<std::mutex> lk(h->mu);
  if (h->ready.empty() && !h->closed && timeout_us > 0)
    h->cv.wait_for(lk, std::chrono::microseconds(timeout_us),
                   [&] { return !h->ready.empty() || h->closed; });
  if (!h->ready.empty()) {
    *token = h->ready.front().first;
    if (status) *status = h->ready.front().second;
    h->ready.pop_front();
    return TB_OK;
  }
  return h->closed ? TB_E_CLOSED : TB_NOT_READY;
}

int tb_htq_close(tb_htq_t q) {
  Htq *h = reinterpret_cast<Htq *>(q);
  if (!h) return TB_E_INVALID;
  {
    std::lock_guard<std::mutex> g(h->mu);
    h->closed = true;
  }
  h->cv.notify_all();
  return TB_OK;
}

int tb_htq_destroy(tb_htq_t q) {
  Htq *h = reinterpret_cast<Htq *>(q);
  if (!h) return TB_E_INVALID;
  tb_htq_close(q);
  ensure_device();
  // Pending host funcs reference h: drain the side streams first.
  for (auto s : h->side) cudaStreamSynchronize(s);
  for (auto s : h->side) cudaStreamDestroy(s);
  delete h;
  return TB_OK;
}

}  // extern "C"
