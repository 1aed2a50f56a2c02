// tb_machine.cu — the paper's machine rebuilt natively: a work-stealing C++
// task runtime whose workers poll CUDA events between tasks (or, for the
// ablation, complete them from host-task threads or by fencing), per-executor
// dynamic kernel aggregation on CUDA streams, and the mini-app step driver.
//
// Same structure and semantics as the reference machine, without the GIL:
//   runtime/pool.py      -> Pool (per-worker deques, injector, random-victim
//                           steal, idle hook after every task + 5..100 us
//                           backoff while idle)
//   runtime/polling.py   -> Poller (MPSC inbox, single-entrant try-lock body,
//                           only each in-order stream's head queried)
//   bridge.py            -> bridge(): POLLING | HOSTTASK | FENCE
//   executors.py:147-304 -> Aggregator (launch on Full or on Idle via one
//                           queue-marker probe per batch; one tb_agg_launch)
//   miniapp.py:116-171   -> SubTask state machine + step driver (host ghost
//                           fold / post-process, exact fsum, min-tree dt)
// Results are bit-identical to the reference (the kernels are K1; the host
// reductions follow numpy's pairwise order and math.fsum exactly).
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <deque>
#include <map>
#include <mutex>
#include <random>
#include <thread>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/tb.h"
#include "tb_internal.h"

namespace tbm {

using Clock = std::chrono::steady_clock;

inline int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now().time_since_epoch())
      .count();
}

// TB_MACHINE_DIAG=1: per-run counters of where the host threads spend the
// step (tasks, poll bodies, event queries, enqueue calls, fences, idle
// loops), kept per thread and summed when the workers exit, printed to
// stderr at the end of the run. Off: one predictable branch per site.
enum DiagField {
  kTasks, kTaskNs, kHookNs, kSteals, kBodies, kQueries, kNotReady, kBodyNs, kEnqueues,
  kEnqueueNs, kFenceNs, kIdleLoops, kSleeps, kStartNs, kFinishNs, kLaunchNs, kBatchDoneNs,
  kScheduleNs, kDiagFields
};
const char *const kDiagNames[kDiagFields] = {
    "tasks", "task_ms", "hook_ms", "steals", "poll_bodies", "queries", "not_ready", "body_ms",
    "enqueues", "enqueue_ms", "fence_ms", "idle_loops", "sleeps", "start_ms", "finish_ms",
    "launch_ms", "batch_done_ms", "schedule_ms"};
const bool g_diag = [] {
  const char *e = getenv("TB_MACHINE_DIAG");
  return e && *e && *e != '0';
}();
std::atomic<int64_t> g_diag_sum[kDiagFields];
thread_local int64_t t_diag[kDiagFields];
inline void diag_add(DiagField f, int64_t v) {
  if (g_diag) t_diag[f] += v;
}
// time of a scope into field f (diag on)
struct DiagScope {
  DiagField f;
  int64_t t0;
  explicit DiagScope(DiagField f_) : f(f_), t0(g_diag ? now_ns() : 0) {}
  ~DiagScope() {
    if (g_diag) t_diag[f] += now_ns() - t0;
  }
};

// a worker's counters into the run's sums (at thread exit)
inline void diag_flush() {
  if (!g_diag) return;
  for (int f = 0; f < kDiagFields; ++f) {
    g_diag_sum[f].fetch_add(t_diag[f]);
    t_diag[f] = 0;
  }
}

void diag_reset() {
  if (!g_diag) return;
  for (auto &c : g_diag_sum) c.store(0);
}

void diag_print(int mode, int64_t workers, int64_t executors, int64_t max_agg, int64_t steps) {
  if (!g_diag) return;
  fprintf(stderr, "{\"diag\": \"machine\", \"mode\": %d, \"workers\": %lld, \"executors\": %lld, "
          "\"max_agg\": %lld, \"steps\": %lld", mode, (long long)workers, (long long)executors,
          (long long)max_agg, (long long)steps);
  for (int f = 0; f < kDiagFields; ++f) {
    const int64_t v = g_diag_sum[f].load();
    if (strstr(kDiagNames[f], "_ms"))
      fprintf(stderr, ", \"%s\": %.3f", kDiagNames[f], v * 1e-6);
    else
      fprintf(stderr, ", \"%s\": %lld", kDiagNames[f], (long long)v);
  }
  fprintf(stderr, "}\n");
}

struct Task {
  void (*fn)(void *);
  void *arg;
};

// ------------------------------------------------------------------ pool --
class Pool;
constexpr int kIdleSpins = 256;
thread_local Pool *t_pool = nullptr;
thread_local int t_worker = -1;

class Pool {
 public:
  Pool(int workers, int device, uint64_t seed) : device_(device) {
    qs_.resize(workers);
    for (int i = 0; i < workers; ++i) qs_[i].reset(new Queue());
    for (int i = 0; i < workers; ++i)
      threads_.emplace_back([this, i, seed] { run(i, seed + i); });
  }
  ~Pool() { stop(); }

  void set_idle_hook(int (*hook)(void *), void *arg) {
    hook_ = hook;
    hook_arg_ = arg;
  }

  void push(Task t) {
    if (t_pool == this && t_worker >= 0) {
      Queue &q = *qs_[t_worker];
      std::lock_guard<std::mutex> g(q.mu);
      q.dq.push_back(t);
      q.n.store((int64_t)q.dq.size(), std::memory_order_release);
    } else {
      std::lock_guard<std::mutex> g(inj_mu_);
      inj_.push_back(t);
      inj_n_.store((int64_t)inj_.size(), std::memory_order_release);
    }
  }

  // Many ready tasks at once (a finished batch's members, a step's tasks).
  // More than 2 per worker: dealt in contiguous runs across every worker's
  // deque from a rotating start — one lock per worker instead of the others
  // stealing them one at a time from the pusher's deque (with FENCE, whose
  // worker then blocks in the next batch's probe, that trickle shrank C4's
  // batches to ~1 member). Fewer: kept on the pusher's deque, where its
  // members' next requests meet the same executor without contention.
  void push_spread(const Task *t, size_t n) {
    const size_t W = qs_.size();
    if (n == 0) return;
    static const size_t min_spread = [] {
      const char *e = getenv("TB_PUSH_SPREAD_MIN");   // A/B: 0 = always, huge = never
      return e ? (size_t)atoll(e) : (size_t)0;
    }();
    const size_t threshold = min_spread ? min_spread : 2 * W + 1;
    if (W == 1 || n < threshold) {
      for (size_t i = 0; i < n; ++i) push(t[i]);
      return;
    }
    const size_t start = spread_rr_.fetch_add(1, std::memory_order_relaxed) % W;
    const size_t per = (n + W - 1) / W;
    for (size_t k = 0, i = 0; i < n; ++k) {
      const size_t m = std::min(per, n - i);
      Queue &q = *qs_[(start + k) % W];
      std::lock_guard<std::mutex> g(q.mu);
      q.dq.insert(q.dq.end(), t + i, t + i + m);
      q.n.store((int64_t)q.dq.size(), std::memory_order_release);
      i += m;
    }
  }

  // Executor-affine dealing: the ready tasks of executor group g (of G) go
  // to the workers w with w % G == g (W >= G), or all to worker g % W, in
  // contiguous runs. A task's next request then meets its executor's lock
  // on one of ~W/G workers instead of on all W, and the members of one
  // batch do not bounce the executor's lines across every core; stealing
  // still balances the load. TB_AFFINITY=0 restores push_spread.
  void push_group(const Task *t, size_t n, size_t g, size_t G) {
    const size_t W = qs_.size();
    if (n == 0) return;
    if (!affinity() || W == 1 || G <= 1) {
      push_spread(t, n);
      return;
    }
    if (W < G) {
      Queue &q = *qs_[g % W];
      std::lock_guard<std::mutex> lk(q.mu);
      q.dq.insert(q.dq.end(), t, t + n);
      q.n.store((int64_t)q.dq.size(), std::memory_order_release);
      return;
    }
    g %= G;
    const size_t cnt = (W - g + G - 1) / G;   // workers g, g + G, g + 2G, ...
    const size_t start = spread_rr_.fetch_add(1, std::memory_order_relaxed) % cnt;
    const size_t per = (n + cnt - 1) / cnt;
    for (size_t k = 0, i = 0; i < n; ++k) {
      const size_t m = std::min(per, n - i);
      Queue &q = *qs_[g + ((start + k) % cnt) * G];
      std::lock_guard<std::mutex> lk(q.mu);
      q.dq.insert(q.dq.end(), t + i, t + i + m);
      q.n.store((int64_t)q.dq.size(), std::memory_order_release);
      i += m;
    }
  }

  static bool affinity() {
    static const bool on = [] {
      const char *e = getenv("TB_AFFINITY");
      return !(e && *e == '0');
    }();
    return on;
  }

  void stop() {
    if (!alive_.exchange(false)) return;
    for (auto &t : threads_) t.join();
  }

 private:
  // n mirrors dq.size() (written under mu): idle workers read it before
  // taking a lock, so 16 spinning workers do not turn every queue's and the
  // injector's mutex into a contended line for the workers that have tasks.
  // A stale 0 only delays a take to the next loop iteration.
  struct Queue {
    std::mutex mu;
    std::deque<Task> dq;
    std::atomic<int64_t> n{0};
  };

  static bool pop(Queue &q, bool front, Task *out) {
    if (q.n.load(std::memory_order_acquire) == 0) return false;
    std::lock_guard<std::mutex> g(q.mu);
    if (q.dq.empty()) return false;
    if (front) {
      *out = q.dq.front();
      q.dq.pop_front();
    } else {
      *out = q.dq.back();
      q.dq.pop_back();
    }
    q.n.store((int64_t)q.dq.size(), std::memory_order_release);
    return true;
  }

  bool take(int w, std::mt19937_64 &rng, Task *out) {
    if (pop(*qs_[w], true, out)) return true;
    if (inj_n_.load(std::memory_order_acquire) > 0) {
      std::lock_guard<std::mutex> g(inj_mu_);
      if (!inj_.empty()) {
        *out = inj_.front();
        inj_.pop_front();
        inj_n_.store((int64_t)inj_.size(), std::memory_order_release);
        return true;
      }
    }
    // steal: scan every other worker once, from a random start (a single
    // random victim, as in src/runtime/pool.py:212-217, leaves fired
    // continuations stranded on the polling worker's deque)
    const int n = (int)qs_.size();
    const int start = n > 1 ? (int)(rng() % n) : 0;
    for (int k = 0; k < n; ++k) {
      const int v = (start + k) % n;
      if (v != w && pop(*qs_[v], false, out)) {
        diag_add(kSteals, 1);
        return true;
      }
    }
    return false;
  }

  void run(int w, uint64_t seed) {
    cudaSetDevice(device_);
    pin(w);
    t_pool = this;
    t_worker = w;
    std::mt19937_64 rng(seed);
    int nap_us = 5;
    int spins = 0;
    while (alive_.load(std::memory_order_relaxed)) {
      Task t;
      if (take(w, rng, &t)) {
        spins = 0;
        if (g_diag) {
          const int64_t t0 = now_ns();
          t.fn(t.arg);
          const int64_t t1 = now_ns();
          if (hook_) hook_(hook_arg_);
          diag_add(kTasks, 1);
          diag_add(kTaskNs, t1 - t0);
          diag_add(kHookNs, now_ns() - t1);
        } else {
          t.fn(t.arg);
          if (hook_) hook_(hook_arg_);
        }
        nap_us = 5;
        continue;
      }
      if (hook_ && hook_(hook_arg_)) {
        nap_us = 5;
        spins = 0;
        continue;
      }
      // Idle: yield-spin first (a Linux sleep is >= ~50 us of timer slack,
      // far longer than a B200 batch), then the reference's 5..100 us backoff.
      diag_add(kIdleLoops, 1);
      if (++spins < kIdleSpins) {
        std::this_thread::yield();
        continue;
      }
      diag_add(kSleeps, 1);
      std::this_thread::sleep_for(std::chrono::microseconds(nap_us));
      nap_us = std::min(nap_us * 2, 100);
    }
    diag_flush();
    t_pool = nullptr;
    t_worker = -1;
  }

  // TB_PIN_WORKERS=1: worker w runs on the w-th CPU of the process's
  // affinity mask (modulo its size)
  static void pin(int w) {
    static const bool on = [] {
      const char *e = getenv("TB_PIN_WORKERS");
      return e && *e == '1';
    }();
    if (!on) return;
    cpu_set_t mask;
    if (sched_getaffinity(0, sizeof(mask), &mask) != 0) return;
    std::vector<int> cpus;
    for (int c = 0; c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &mask)) cpus.push_back(c);
    if (cpus.empty()) return;
    cpu_set_t one;
    CPU_ZERO(&one);
    CPU_SET(cpus[(size_t)w % cpus.size()], &one);
    pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
  }

  int device_;
  std::vector<std::unique_ptr<Queue>> qs_;
  std::mutex inj_mu_;
  std::deque<Task> inj_;
  std::atomic<int64_t> inj_n_{0};
  std::vector<std::thread> threads_;
  std::atomic<bool> alive_{true};
  std::atomic<size_t> spread_rr_{0};
  int (*hook_)(void *) = nullptr;
  void *hook_arg_ = nullptr;
};

// ---------------------------------------------------------------- poller --
// Completion callbacks keyed to CUDA events; the body runs on whichever worker
// wins the try-lock, queries only each stream's head, and pushes the fired
// continuations as pool tasks.
class Poller {
 public:
  // fault: where a device error seen by the poll body is recorded (first
  // error wins); the continuation still runs and sees the machine failed
  Poller(Pool *pool, std::atomic<int> *fault) : pool_(pool), fault_(fault) {}

  void add(cudaEvent_t ev, uint64_t chain, Task cont) {
    std::lock_guard<std::mutex> g(inbox_mu_);
    inbox_.push_back(Entry{ev, chain, cont, nullptr, 0});
    waiting_.fetch_add(1, std::memory_order_relaxed);
  }

  // completion = words: fire cont once *word >= target (chain = the stream
  // that will store it; targets arrive in nondecreasing order per chain)
  void add_word(const uint64_t *word, uint64_t target, uint64_t chain, Task cont) {
    std::lock_guard<std::mutex> g(inbox_mu_);
    inbox_.push_back(Entry{nullptr, chain, cont, word, target});
    waiting_.fetch_add(1, std::memory_order_relaxed);
  }

  static int hook(void *self) { return static_cast<Poller *>(self)->poll(); }

  int poll() {
    // each thread looks at the shared lines (waiting_, last_ns_, the body
    // lock) at most once per half gap: after every task the check is one
    // clock read, not a cache miss on lines the body and add() write
    thread_local int64_t next_try = 0;
    const int64_t t = now_ns();
    if (t < next_try) return 0;
    next_try = t + gap_ns_ / 2;
    if (waiting_.load(std::memory_order_relaxed) == 0) return 0;
    // Every worker calls this after every task; with many workers the
    // try-lock itself becomes the contended line. A body started less than
    // gap_ns_ ago (~1/10 of the shortest batch round trip) makes the
    // call a read of one clock and one atomic.
    const int64_t now = t;
    if (now - last_ns_.load(std::memory_order_relaxed) < gap_.load(std::memory_order_relaxed))
      return 0;
    std::unique_lock<std::mutex> guard(body_, std::try_to_lock);
    if (!guard.owns_lock()) return 0;
    last_ns_.store(now, std::memory_order_relaxed);
    struct Range {   // NVTX range over the poll body (profilers only)
      Range() { nvtxRangePushA("machine poll body"); }
      ~Range() { nvtxRangePop(); }
    } range;
    {
      std::lock_guard<std::mutex> g(inbox_mu_);
      for (const Entry &e : inbox_) chains_[e.chain].push_back(e);
      inbox_.clear();
    }
    int fired = 0;
    int64_t queries = 0, not_ready = 0;
    for (auto it = chains_.begin(); it != chains_.end();) {
      auto &dq = it->second;
      while (!dq.empty()) {
        cudaError_t q;
        if (dq.front().word) {
          // a memory read; the stream is asked (a driver call) only when a
          // word has not moved for a millisecond: a faulted kernel never
          // stores its word
          q = __atomic_load_n(dq.front().word, __ATOMIC_ACQUIRE) >= dq.front().target
                  ? cudaSuccess
                  : stalled_stream_error(it->first, now);
        } else {
          q = cudaEventQuery(dq.front().ev);
        }
        ++queries;
        if (q == cudaErrorNotReady) {
          ++not_ready;
          break;
        }
        if (q != cudaSuccess) {
          int expect = 0;
          fault_->compare_exchange_strong(expect, -(int)q);
        }
        Entry e = dq.front();
        dq.pop_front();
        if (e.ev) tb_event_release(reinterpret_cast<tb_event_t>(e.ev));
        stalled_since_.erase(it->first);
        pool_->push(e.cont);
        ++fired;
      }
      it = dq.empty() ? chains_.erase(it) : std::next(it);
    }
    waiting_.fetch_sub(fired, std::memory_order_relaxed);
    // TB_POLL_GAP_MAX_NS > gap: a body that found nothing complete doubles
    // the gap to the next one (up to the max), one that fired resets it.
    // Off by default: at C4 it cut 96 %-not-ready queries without changing
    // the step time, and it slowed 2-worker polling (profiles/r02/
    // machine_env_ab.txt)
    gap_.store(fired ? gap_ns_ : std::min<int64_t>(2 * gap_.load(std::memory_order_relaxed),
                                                    gap_max_ns_),
               std::memory_order_relaxed);
    if (g_diag) {
      diag_add(kBodies, 1);
      diag_add(kQueries, queries);
      diag_add(kNotReady, not_ready);
      diag_add(kBodyNs, now_ns() - now);
    }
    return fired;
  }

 private:
  struct Entry {
    cudaEvent_t ev;
    uint64_t chain;
    Task cont;
    const uint64_t *word;
    uint64_t target;
  };
  // a word head not reached: cudaErrorNotReady, unless the chain's stream
  // (chain = its cudaStream_t) reports an error after >= 1 ms of waiting
  cudaError_t stalled_stream_error(uint64_t chain, int64_t now) {
    auto ins = stalled_since_.emplace(chain, now);
    if (now - ins.first->second < 1000000) return cudaErrorNotReady;
    ins.first->second = now;
    const cudaError_t q = cudaStreamQuery(reinterpret_cast<cudaStream_t>(chain));
    return (q == cudaSuccess || q == cudaErrorNotReady) ? cudaErrorNotReady : q;
  }
  std::unordered_map<uint64_t, int64_t> stalled_since_;
  Pool *pool_;
  std::atomic<int> *fault_;
  std::mutex inbox_mu_;
  std::vector<Entry> inbox_;
  std::mutex body_;
  std::unordered_map<uint64_t, std::deque<Entry>> chains_;
  std::atomic<int64_t> waiting_{0};
  const int64_t gap_ns_ = [] {
    const char *e = getenv("TB_POLL_GAP_NS");
    return e ? (int64_t)atoll(e) : (int64_t)2000;
  }();
  const int64_t gap_max_ns_ = [this] {
    const char *e = getenv("TB_POLL_GAP_MAX_NS");
    return std::max<int64_t>(gap_ns_, e ? (int64_t)atoll(e) : (int64_t)0);
  }();
  std::atomic<int64_t> gap_{gap_ns_};
  std::atomic<int64_t> last_ns_{0};
};

// ------------------------------------------------------ host-task threads --
class HostTasks {
 public:
  HostTasks(Pool *pool, int threads, int device, int side_streams, std::atomic<int> *fault)
      : pool_(pool), fault_(fault) {
    cudaSetDevice(device);
    for (int i = 0; i < side_streams; ++i) {
      cudaStream_t s;
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      side_.push_back(s);
    }
    for (int i = 0; i < threads; ++i) threads_.emplace_back([this] { run(); });
  }
  ~HostTasks() {
    for (auto s : side_) cudaStreamSynchronize(s);
    {
      std::lock_guard<std::mutex> g(mu_);
      closed_ = true;
    }
    cv_.notify_all();
    for (auto &t : threads_) t.join();
    for (auto s : side_) cudaStreamDestroy(s);
  }
  void add(cudaEvent_t ev, Task cont) {
    auto *item = new Item{this, ev, cont, cudaSuccess};
    cudaStream_t side = side_[rr_.fetch_add(1) % side_.size()];
    cudaStreamWaitEvent(side, ev, 0);
    // a stream callback is called with the stream's status even after a
    // device fault (cudaLaunchHostFunc is not), so the fault reaches the
    // machine instead of leaving its step waiting forever
    if (cudaStreamAddCallback(side, &HostTasks::trampoline, item, 0) != cudaSuccess) {
      item->status = cudaErrorLaunchFailure;
      trampoline(side, cudaErrorLaunchFailure, item);
    }
  }
  int64_t dispatched() const { return dispatched_.load(); }

 private:
  struct Item {
    HostTasks *self;
    cudaEvent_t ev;
    Task cont;
    cudaError_t status;
  };
  static void CUDART_CB trampoline(cudaStream_t, cudaError_t status, void *p) {
    // CUDA driver thread: enqueue only
    Item *it = static_cast<Item *>(p);
    it->status = status;
    HostTasks *self = it->self;   // `it` may be consumed as soon as it is queued
    {
      std::lock_guard<std::mutex> g(self->mu_);
      self->ready_.push_back(it);
    }
    self->cv_.notify_one();
  }
  void run() {
    for (;;) {
      Item *it = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return closed_ || !ready_.empty(); });
        if (ready_.empty()) return;
        it = ready_.front();
        ready_.pop_front();
      }
      if (it->status != cudaSuccess) {
        int expect = 0;
        fault_->compare_exchange_strong(expect, -(int)it->status);
      }
      tb_event_release(reinterpret_cast<tb_event_t>(it->ev));
      pool_->push(it->cont);   // foreign thread -> pool injector
      dispatched_.fetch_add(1);
      delete it;
    }
  }
  Pool *pool_;
  std::atomic<int> *fault_;
  std::vector<cudaStream_t> side_;
  std::atomic<unsigned> rr_{0};
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Item *> ready_;
  bool closed_ = false;
  std::vector<std::thread> threads_;
  std::atomic<int64_t> dispatched_{0};
};

// ---------------------------------------------------------------- machine --
constexpr int kCells = TB_CELLS;
constexpr int kFace = TB_FACE;
constexpr int64_t kGhosted = 5 * 1728;      // one ghosted hydro sub-grid [5][12^3]
constexpr int64_t kInterior = 5 * 512;      // its dU/dt [5][8^3]
constexpr int64_t kHydroOut = kInterior + 1;   // + amax

struct Machine;
struct SubTask;

struct Staging {
  size_t bytes;
  double *host;   // pinned
  double *dev;
};

struct Req {
  const double *src;
  double *dst;
  int64_t n;
  SubTask *task;
  uint8_t flags = 0;   // direct mode: bit 0 first round (fold), bit 1 last (reduce)
};

struct Executor;

// A batch is referenced by its launch (released in batch_done) and, when it
// opened with an idleness probe, by that probe (released in idle_fire) — the
// probe may complete long after a full launch finished.
struct Batch {
  Executor *ex;
  int kind;
  std::vector<Req> members;
  bool launched = false;
  bool idle = false;
  Staging *staging = nullptr;
  std::atomic<int> refs{1};
};

inline void batch_release(Batch *b) {
  if (b->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete b;
}

struct Executor {
  Machine *m;
  int id;
  cudaStream_t stream;
  std::mutex mu;
  // POLLING: an event is recorded and registered with the poller under this
  // lock, so each stream's poll chain is in record order (the poll body
  // queries only the chain head)
  std::mutex rec_mu;
  // per-executor batch statistics of the running step: [0, max_agg] = batches
  // by member count, then full- and idle-triggered launches (the
  // AggregationExecutor's batch_sizes / reasons, src/executors.py:166-169)
  std::unique_ptr<std::atomic<int64_t>[]> stats;
  Batch *open[TB_KINDS] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // completion = words: the mapped word this stream's batch kernels store
  // their sequence numbers in, its CTA counter, the last number issued
  // (under rec_mu)
  uint64_t *word = nullptr;
  unsigned *ctas = nullptr;
  uint64_t issued = 0;
};

// A task's state, 88 B, held contiguously in Machine::tasks (a chunk's
// members are a fixed stride apart, so resuming them streams through memory
// instead of chasing heap objects). Work buffers: the machine's task_bufs
// (staged / in place), its pinned arena (gather / resident) or the caller's
// rows (direct); d0 / d1 the device ping-pong rows (resident / direct).
struct SubTask {
  Machine *m;
  Executor *ex;
  int64_t lo, n;          // sub-grids [lo, lo+n)
  int32_t round;
  double *abuf, *bbuf;
  double *work, *out;
  double *d0 = nullptr, *d1 = nullptr;
};

struct Machine {
  tb_machine_config cfg;
  double *cells = nullptr;         // [S][512]: the caller's (run_cells) or own_cells
  std::vector<double> own_cells;
  std::vector<double> faces_v, mins_v, sums_v;
  double *faces = nullptr;         // [S][2][8] previous generation
  double *mins = nullptr, *sums = nullptr;   // per sub-grid, this step
  double *pinned_small = nullptr;  // zero_copy = 4: faces | mins | sums, mapped
  bool words = false;              // completion = TB_COMPLETION_WORDS
  uint64_t *words_host = nullptr;  // executors' completion words (mapped)
  unsigned *ctas_dev = nullptr;    // their CTA counters
  bool own_cells_pinned = false;   // zero_copy = 4 without caller cells
  std::unique_ptr<Pool> pool;
  std::unique_ptr<Poller> poller;
  std::unique_ptr<HostTasks> hosttasks;
  std::vector<std::unique_ptr<Executor>> execs;
  std::vector<SubTask> tasks;       // reserved up front: addresses stay put
  std::vector<double> task_bufs;    // staged / in-place modes and hydro: per-task buffers
  std::mutex staging_mu;
  std::map<size_t, std::vector<Staging *>> staging_free;
  std::vector<Staging *> staging_all;
  // step completion
  std::mutex done_mu;
  std::condition_variable done_cv;
  std::atomic<int64_t> remaining{0};
  // metrics
  std::atomic<int64_t> launches{0}, transfers{0}, event_waits{0}, full{0}, idle{0},
      members{0}, kernels{0};
  // first device fault / API error (0 = none); once set, tasks stop
  // scheduling and finish, the step loop stops, and the run returns it
  std::atomic<int> fault{0};
  std::atomic<int64_t> launch_seq{0};   // fault_at_launch counter
  double *arena = nullptr;              // zero_copy = 2: pinned task buffers
                                        // zero_copy = 3: one pinned buffer per task
  double *dev_arena = nullptr;          // zero_copy = 3: two device buffers per task
  void fail(int rc) {
    int expect = 0;
    if (rc != TB_OK) fault.compare_exchange_strong(expect, rc);
  }
  bool failed() const { return fault.load(std::memory_order_relaxed) != 0; }
  // hydro workload (tb_machine_run_hydro)
  bool hydro = false;
  int64_t nb = 0;                  // sub-grids per lattice edge
  double dx = 0.0, gamma = 0.0, dt = 0.0;
  std::vector<double> U;           // [S][5][512] interior state
  std::vector<double> dudt;        // [S][5][512]
  std::vector<double> amax;        // [S]
};

// Task arenas outlive a run: the pinned (device-mapped) and the device arena
// are taken from this cache when large enough and handed back at the end of
// the run, so repeated run_scenario calls do not re-pin 128 MiB each time. A
// run that finds the cache empty (another run holds it) allocates its own.
struct ArenaCache {
  std::mutex mu;
  double *host = nullptr;
  size_t host_bytes = 0;
  double *dev = nullptr;
  size_t dev_bytes = 0;
  int dev_id = -1;
};
ArenaCache g_arena;

double *arena_take_host(size_t bytes) {
  {
    std::lock_guard<std::mutex> g(g_arena.mu);
    if (g_arena.host && g_arena.host_bytes >= bytes) {
      double *p = g_arena.host;
      g_arena.host = nullptr;
      return p;
    }
  }
  double *p = nullptr;
  if (cudaHostAlloc(reinterpret_cast<void **>(&p), bytes,
                    cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess)
    return nullptr;
  return p;
}

double *arena_take_dev(size_t bytes, int dev) {
  {
    std::lock_guard<std::mutex> g(g_arena.mu);
    if (g_arena.dev && g_arena.dev_bytes >= bytes && g_arena.dev_id == dev) {
      double *p = g_arena.dev;
      g_arena.dev = nullptr;
      return p;
    }
  }
  double *p = nullptr;
  if (cudaMalloc(reinterpret_cast<void **>(&p), bytes) != cudaSuccess) return nullptr;
  return p;
}

// Hand arenas back (the cache keeps the larger of the cached and the
// returned one of each kind and frees the other).
void arena_give(double *host, size_t host_bytes, double *dev, size_t dev_bytes, int dev_id) {
  double *free_host = nullptr, *free_dev = nullptr;
  {
    std::lock_guard<std::mutex> g(g_arena.mu);
    if (host) {
      if (!g_arena.host || g_arena.host_bytes < host_bytes) {
        free_host = g_arena.host;
        g_arena.host = host;
        g_arena.host_bytes = host_bytes;
      } else {
        free_host = host;
      }
    }
    if (dev) {
      if (!g_arena.dev || g_arena.dev_bytes < dev_bytes || g_arena.dev_id != dev_id) {
        free_dev = g_arena.dev;
        g_arena.dev = dev;
        g_arena.dev_bytes = dev_bytes;
        g_arena.dev_id = dev_id;
      } else {
        free_dev = dev;
      }
    }
  }
  if (free_host) cudaFreeHost(free_host);
  if (free_dev) cudaFree(free_dev);
}

// Pooled pinned + device staging in power-of-two size classes (>= 4 KiB):
// batches of every member count share a handful of classes, so a C4 step
// reuses buffers instead of pinning new ones for each new batch size (the
// reference BufferPool's exact-size buckets, src/executors.py:86-121, stay
// the Python mirror's semantics). Null on an allocation failure.
Staging *staging_alloc(Machine *m, size_t bytes) {
  size_t cls = 4096;
  while (cls < bytes) cls <<= 1;
  {
    std::lock_guard<std::mutex> g(m->staging_mu);
    auto &v = m->staging_free[cls];
    if (!v.empty()) {
      Staging *s = v.back();
      v.pop_back();
      return s;
    }
  }
  Staging *s = new Staging{cls, nullptr, nullptr};
  if (cudaHostAlloc(reinterpret_cast<void **>(&s->host), cls, cudaHostAllocPortable) !=
          cudaSuccess ||
      cudaMalloc(reinterpret_cast<void **>(&s->dev), cls) != cudaSuccess) {
    if (s->host) cudaFreeHost(s->host);
    delete s;
    return nullptr;
  }
  std::lock_guard<std::mutex> g(m->staging_mu);
  m->staging_all.push_back(s);
  return s;
}

size_t hydro_staging_bytes(const Machine *m) {
  return sizeof(double) * (size_t)(m->cfg.max_agg * m->cfg.task_subgrids) *
         (size_t)(kGhosted + kHydroOut);
}

void staging_release(Machine *m, Staging *s) {
  std::lock_guard<std::mutex> g(m->staging_mu);
  m->staging_free[s->bytes].push_back(s);
}

// Bridge a recorded event into the runtime: the continuation `cont` becomes
// a pool task once the event completes (src/bridge.py:54-101). A device
// fault does not fail the continuation's scheduling — the continuation runs
// and finds the machine failed (errors surface as the run's result, never as
// a hang; src/executors.py:50-55, src/runtime/polling.py:71-75).
void bridge(Machine *m, Executor *ex, cudaEvent_t ev, Task cont) {
  switch (m->cfg.mode) {
    case TB_MODE_POLLING:
      m->poller->add(ev, reinterpret_cast<uint64_t>(ex->stream), cont);
      break;
    case TB_MODE_HOSTTASK:
      m->hosttasks->add(ev, cont);
      break;
    default: {  // FENCE: block this worker, then the future is ready
      m->event_waits.fetch_add(1, std::memory_order_relaxed);
      const int64_t t0 = g_diag ? now_ns() : 0;
      const cudaError_t e = cudaEventSynchronize(ev);
      if (g_diag) diag_add(kFenceNs, now_ns() - t0);
      if (e != cudaSuccess) m->fail(-(int)e);
      tb_event_release(reinterpret_cast<tb_event_t>(ev));
      m->pool->push(cont);
      break;
    }
  }
}

// Enqueue work on the executor's stream (`enqueue` records the completion
// event into *ev) and bridge that event. POLLING keeps record + register
// under the executor's record lock (poll chains in record order); a failed
// enqueue still bridges (ev may be 0: the query reports an error) so the
// continuation runs and sees the failure.
template <typename F>
void enqueue_and_bridge(Machine *m, Executor *ex, Task cont, F enqueue_) {
  auto enqueue = [&](tb_event_t *ev) {
    if (!g_diag) return enqueue_(ev);
    const int64_t t0 = now_ns();
    const int rc = enqueue_(ev);
    diag_add(kEnqueues, 1);
    diag_add(kEnqueueNs, now_ns() - t0);
    return rc;
  };
  tb_event_t ev = 0;
  if (m->cfg.mode == TB_MODE_POLLING) {
    std::lock_guard<std::mutex> g(ex->rec_mu);
    const int rc = enqueue(&ev);
    if (rc != TB_OK) m->fail(rc);
    if (!ev) {
      m->pool->push(cont);
      return;
    }
    bridge(m, ex, reinterpret_cast<cudaEvent_t>(ev), cont);
    return;
  }
  const int rc = enqueue(&ev);
  if (rc != TB_OK) m->fail(rc);
  if (!ev) {
    m->pool->push(cont);
    return;
  }
  bridge(m, ex, reinterpret_cast<cudaEvent_t>(ev), cont);
}

void resume_task(void *p);
void hydro_resume(void *p);

// A run of one batch's member continuations executed as one pool task: the
// pool's per-task work (deque lock, pop, steal, poll hook) is paid once per
// kResumeChunk members instead of once per member. Each member's
// continuation still runs exactly once, on a worker, after the batch
// completed (src/executors.py:300-301); the chunks are stealable. 64: a full
// C4 batch (256) is 4 chunks (C4 resident/direct 15.2 -> 14.0 ms/step against
// 16 at 8 workers, profiles/r02/machine_chunk_ab.txt; 4 was worse).
constexpr size_t kResumeChunk = 64;
struct ResumeChunk {
  void (*fn)(void *);
  uint32_t n;
  SubTask *t[kResumeChunk];
};

void resume_task_chunk(SubTask *const *ts, uint32_t n);

void resume_chunk(void *p) {
  ResumeChunk *c = static_cast<ResumeChunk *>(p);
  if (c->fn == resume_task)
    resume_task_chunk(c->t, c->n);
  else
    for (uint32_t i = 0; i < c->n; ++i) c->fn(c->t[i]);
  delete c;
}

size_t resume_chunk_size() {
  static const size_t k = [] {
    const char *e = getenv("TB_RESUME_CHUNK");   // A/B: 1 = one pool task per member
    const long v = e ? atol(e) : (long)kResumeChunk;
    return (size_t)std::max<long>(1, std::min<long>(v, (long)kResumeChunk));
  }();
  return k;
}

// The members' continuations (src/executors.py:300-301: every member's
// promise completes), dealt to the executor's worker group in chunks.
void resume_members(const Batch *b) {
  Machine *m = b->ex->m;
  void (*fn)(void *) = m->hydro ? hydro_resume : resume_task;
  const size_t n = b->members.size(), k = resume_chunk_size();
  std::vector<Task> ts;
  if (k == 1) {
    ts.reserve(n);
    for (const Req &r : b->members) ts.push_back(Task{fn, r.task});
  } else {
    ts.reserve((n + k - 1) / k);
    for (size_t i = 0; i < n; i += k) {
      ResumeChunk *c = new ResumeChunk;
      c->fn = fn;
      c->n = (uint32_t)std::min(k, n - i);
      for (uint32_t j = 0; j < c->n; ++j) c->t[j] = b->members[i + j].task;
      ts.push_back(Task{resume_chunk, c});
    }
  }
  m->pool->push_group(ts.data(), ts.size(), (size_t)b->ex->id, m->execs.size());
}

void batch_done(void *p) {   // AggregationExecutor finish (src/executors.py:286-301)
  DiagScope ds(kBatchDoneNs);
  Batch *b = static_cast<Batch *>(p);
  Machine *m = b->ex->m;
  if (m->failed()) {
    // the batch's outputs are garbage: skip the scatter, let members finish
  } else if (m->hydro) {   // scatter each member's dU/dt rows and amax entries
    int64_t total = 0;
    for (const Req &r : b->members) total += r.n;
    const int64_t nsub = total / kGhosted;
    const double *du = b->staging->host + total, *am = du + nsub * kInterior;
    int64_t o = 0;
    for (const Req &r : b->members) {
      const int64_t k = r.n / kGhosted;
      std::memcpy(r.dst, du + o * kInterior, sizeof(double) * k * kInterior);
      std::memcpy(r.dst + k * kInterior, am + o, sizeof(double) * k);
      o += k;
    }
  } else if (b->staging) {
    int64_t off = 0;
    for (const Req &r : b->members) {
      std::memcpy(r.dst, b->staging->host + off, sizeof(double) * r.n);
      off += r.n;
    }
  }
  if (b->staging) staging_release(m, b->staging);
  m->launches.fetch_add(1, std::memory_order_relaxed);
  m->members.fetch_add((int64_t)b->members.size(), std::memory_order_relaxed);
  (b->idle ? m->idle : m->full).fetch_add(1, std::memory_order_relaxed);
  if (b->ex->stats) {
    const int64_t M = m->cfg.max_agg;
    const int64_t k = std::min<int64_t>((int64_t)b->members.size(), M);
    b->ex->stats[k].fetch_add(1, std::memory_order_relaxed);
    b->ex->stats[M + 1 + (b->idle ? 1 : 0)].fetch_add(1, std::memory_order_relaxed);
  }
  resume_members(b);
  batch_release(b);
}

// A gather / direct batch's kernel launches (TB_GATHER_MAX members each);
// done (completion = words) is signalled by the last one — the earlier ones
// precede it on the stream.
int launch_gather_kernels(Batch *b, tb_stream_t st, int op, const tb_done *done) {
  Machine *m = b->ex->m;
  const bool direct = m->cfg.zero_copy == 4 && op != TB_OP_TRAP;
  const double *src[TB_GATHER_MAX];
  double *dst[TB_GATHER_MAX];
  int64_t n[TB_GATHER_MAX], g0[TB_GATHER_MAX];
  int32_t nsub[TB_GATHER_MAX];
  uint8_t flags[TB_GATHER_MAX];
  int rc = TB_OK;
  for (size_t i0 = 0; i0 < b->members.size() && rc == TB_OK; i0 += TB_GATHER_MAX) {
    const int k = (int)std::min<size_t>(TB_GATHER_MAX, b->members.size() - i0);
    const tb_done *d = i0 + (size_t)k >= b->members.size() ? done : nullptr;
    for (int i = 0; i < k; ++i) {
      const Req &r = b->members[i0 + i];
      src[i] = r.src;
      dst[i] = r.dst;
      n[i] = r.n;
      g0[i] = r.task->lo;
      nsub[i] = (int32_t)r.task->n;
      flags[i] = r.flags;
    }
    rc = direct ? tb_launch_gather_edge(st, b->kind, src, dst, g0, nsub, flags, k, m->faces,
                                        m->mins, m->sums, m->cfg.subgrids, d)
                : tb_launch_gather_done(st, op, b->kind, 0.0, 0.0, src, dst, n, k, d);
  }
  return rc;
}

// completion = words, FENCE: block this worker until the executor's word
// reaches target (spin, then yield); a stream that reports an error after a
// millisecond without progress fails the machine instead of hanging it
void wait_word(Machine *m, Executor *ex, uint64_t target) {
  m->event_waits.fetch_add(1, std::memory_order_relaxed);
  const int64_t t0 = now_ns();
  int64_t last_check = t0;
  for (uint64_t spins = 0;; ++spins) {
    if (__atomic_load_n(ex->word, __ATOMIC_ACQUIRE) >= target) break;
    if ((spins & 255) == 255) {
      const int64_t t = now_ns();
      if (t - last_check > 1000000) {
        last_check = t;
        const cudaError_t q = cudaStreamQuery(ex->stream);
        if (q != cudaSuccess && q != cudaErrorNotReady) {
          m->fail(-(int)q);
          break;
        }
      }
      if (t - t0 > 50000) std::this_thread::yield();
    }
  }
  if (g_diag) diag_add(kFenceNs, now_ns() - t0);
}

// completion = words: continuation cont runs once ex's word reaches target
// (POLLING: registered with the poller under rec_mu, which the caller holds;
// FENCE: the caller waits after releasing it)
void bridge_word_locked(Machine *m, Executor *ex, uint64_t target, Task cont) {
  if (__atomic_load_n(ex->word, __ATOMIC_ACQUIRE) >= target) {
    m->pool->push(cont);
    return;
  }
  m->poller->add_word(ex->word, target, reinterpret_cast<uint64_t>(ex->stream), cont);
}

void launch(Batch *b, bool idle) {   // src/executors.py:257-284 as one launch
  DiagScope ds(kLaunchNs);
  struct Range {   // NVTX range over the batch launch (profilers only)
    Range() { nvtxRangePushA("machine batch launch"); }
    ~Range() { nvtxRangePop(); }
  } range;
  Executor *ex = b->ex;
  Machine *m = ex->m;
  b->idle = idle;
  if (m->failed()) {   // the device is gone: no launch, members finish
    resume_members(b);
    batch_release(b);
    return;
  }
  const int64_t fat = m->cfg.fault_at_launch;
  const bool trap = fat > 0 && m->launch_seq.fetch_add(1) + 1 == fat;
  const int op = trap ? TB_OP_TRAP : TB_OP_KIND;
  const int do_barrier = m->cfg.inject_barriers && !m->cfg.barrier_elision;
  const tb_stream_t st = reinterpret_cast<tb_stream_t>(ex->stream);
  m->kernels.fetch_add(1, std::memory_order_relaxed);
  if (m->words) {
    // completion = words (zero_copy >= 2): the batch kernel itself stores
    // the batch's number in the executor's word; no event
    uint64_t seq = 0;
    int rc;
    {
      std::lock_guard<std::mutex> g(ex->rec_mu);
      const int64_t t0 = g_diag ? now_ns() : 0;
      seq = ++ex->issued;
      const tb_done d{ex->word, seq, ex->ctas};
      rc = launch_gather_kernels(b, st, op, &d);
      if (rc == TB_OK && do_barrier) rc = tb_barrier(st);
      if (g_diag) {
        diag_add(kEnqueues, 1);
        diag_add(kEnqueueNs, now_ns() - t0);
      }
      if (rc != TB_OK) {
        m->fail(rc);
      } else if (m->cfg.mode == TB_MODE_POLLING) {
        bridge_word_locked(m, ex, seq, Task{batch_done, b});
        return;
      }
    }
    if (rc == TB_OK) wait_word(m, ex, seq);
    m->pool->push(Task{batch_done, b});
    return;
  }
  if (m->cfg.zero_copy == 4 && !m->hydro && !trap) {
    // direct: members' rows where they live; first / last rounds fold and
    // reduce in the kernel (tb_launch_gather_edge)
    enqueue_and_bridge(m, ex, Task{batch_done, b}, [&](tb_event_t *ev) {
      const double *src[TB_GATHER_MAX];
      double *dst[TB_GATHER_MAX];
      int64_t g0[TB_GATHER_MAX];
      int32_t nsub[TB_GATHER_MAX];
      uint8_t flags[TB_GATHER_MAX];
      int rc = TB_OK;
      for (size_t i0 = 0; i0 < b->members.size() && rc == TB_OK; i0 += TB_GATHER_MAX) {
        const int k = (int)std::min<size_t>(TB_GATHER_MAX, b->members.size() - i0);
        for (int i = 0; i < k; ++i) {
          const Req &r = b->members[i0 + i];
          src[i] = r.src;
          dst[i] = r.dst;
          g0[i] = r.task->lo;
          nsub[i] = (int32_t)r.task->n;
          flags[i] = r.flags;
        }
        rc = tb_launch_gather_edge(st, b->kind, src, dst, g0, nsub, flags, k, m->faces, m->mins,
                                   m->sums, m->cfg.subgrids, nullptr);
      }
      if (rc == TB_OK && do_barrier) rc = tb_barrier(st);
      if (rc == TB_OK) rc = tb_event_record(st, ev);
      return rc;
    });
    return;
  }
  if (m->cfg.zero_copy >= 2 && !m->hydro) {
    // members read and written where they live (the pinned task arena)
    enqueue_and_bridge(m, ex, Task{batch_done, b}, [&](tb_event_t *ev) {
      const double *src[TB_GATHER_MAX];
      double *dst[TB_GATHER_MAX];
      int64_t n[TB_GATHER_MAX];
      int rc = TB_OK;
      for (size_t i0 = 0; i0 < b->members.size() && rc == TB_OK; i0 += TB_GATHER_MAX) {
        const int k = (int)std::min<size_t>(TB_GATHER_MAX, b->members.size() - i0);
        for (int i = 0; i < k; ++i) {
          const Req &r = b->members[i0 + i];
          src[i] = r.src;
          dst[i] = r.dst;
          n[i] = r.n;
        }
        rc = tb_launch_gather(st, op, b->kind, 0.0, 0.0, src, dst, n, k);
      }
      if (rc == TB_OK && do_barrier) rc = tb_barrier(st);
      if (rc == TB_OK) rc = tb_event_record(st, ev);
      return rc;
    });
    return;
  }
  int64_t total = 0;
  for (const Req &r : b->members) total += r.n;
  // hydro: staging = [ghosted inputs | dU/dt + amax outputs], one size class
  // (a full batch) so buffers are always reused
  const size_t bytes = m->hydro ? hydro_staging_bytes(m) : sizeof(double) * total;
  b->staging = staging_alloc(m, bytes);
  if (!b->staging) {   // out of pinned/device memory: the run fails, members finish
    const int rc = tb::rc(cudaGetLastError());
    m->fail(rc != TB_OK ? rc : -(int)cudaErrorMemoryAllocation);
    resume_members(b);
    batch_release(b);
    return;
  }
  int64_t off = 0;
  for (const Req &r : b->members) {
    std::memcpy(b->staging->host + off, r.src, sizeof(double) * r.n);
    off += r.n;
  }
  if (m->cfg.zero_copy && !m->hydro) {
    // the batch kernel in place on the pinned staging buffer (mapped host
    // memory, read and written over PCIe): one launch + one event, no copies
    enqueue_and_bridge(m, ex, Task{batch_done, b}, [&](tb_event_t *ev) {
      int rc = tb_launch(st, op, b->kind, 0.0, 0.0, b->staging->host, total);
      if (rc == TB_OK && do_barrier) rc = tb_barrier(st);
      if (rc == TB_OK) rc = tb_event_record(st, ev);
      return rc;
    });
    return;
  }
  m->transfers.fetch_add(2, std::memory_order_relaxed);
  enqueue_and_bridge(m, ex, Task{batch_done, b}, [&](tb_event_t *ev) {
    if (m->hydro && trap) {
      const int rc = tb_launch(st, TB_OP_TRAP, 0, 0.0, 0.0, nullptr, 0);
      return rc == TB_OK ? tb_event_record(st, ev) : rc;
    }
    if (m->hydro)
      return tb_agg_launch_hydro(st, b->staging->dev, b->staging->host, total / kGhosted,
                                        b->staging->dev + total, b->staging->host + total,
                                        m->dx, m->gamma, ev);
    return tb_agg_launch(st, op, b->kind, 0.0, 0.0, b->staging->dev, b->staging->host, bytes,
                         do_barrier, ev);
  });
}

void idle_fire(void *p) {   // the idleness probe completed (src/executors.py:209-218)
  Batch *b = static_cast<Batch *>(p);
  Executor *ex = b->ex;
  bool mine = false;
  {
    std::lock_guard<std::mutex> g(ex->mu);
    if (!b->launched) {                 // else the full trigger won
      if (ex->open[b->kind] == b) ex->open[b->kind] = nullptr;
      b->launched = true;
      mine = true;
    }
  }
  if (mine) launch(b, true);
  batch_release(b);                     // the probe's reference
}

// n requests of one kind on one executor under ONE acquisition of its lock
// (a resumed chunk's members all come from one batch, so their next
// requests share executor and kind): each joins the open batch or opens one
// (with its idleness probe), and a batch that reaches max_agg launches —
// src/executors.py:174-221 applied to each request in order.
void schedule_many(Executor *ex, int kind, const Req *reqs, int n) {
  DiagScope ds(kScheduleNs);
  Machine *m = ex->m;
  Batch *opened[kResumeChunk + 1], *full[kResumeChunk + 1];
  bool filled_here[kResumeChunk + 1];   // opened[i] also filled by this call
  int nopened = 0, nfull = 0;
  {
    std::lock_guard<std::mutex> g(ex->mu);
    for (int i = 0; i < n; ++i) {
      Batch *b = ex->open[kind];
      if (!b) {
        b = new Batch();
        b->ex = ex;
        b->kind = kind;
        b->members.reserve((size_t)std::min<int64_t>(m->cfg.max_agg, 1024));
        if (m->cfg.max_agg > 1) {
          ex->open[kind] = b;
          b->refs.store(2, std::memory_order_relaxed);   // launch + idleness probe
        }
        filled_here[nopened] = false;
        opened[nopened++] = b;
      }
      b->members.push_back(reqs[i]);
      if ((int64_t)b->members.size() >= m->cfg.max_agg) {
        if (ex->open[kind] == b) ex->open[kind] = nullptr;
        b->launched = true;
        full[nfull++] = b;
        for (int j = 0; j < nopened; ++j)
          if (opened[j] == b) filled_here[j] = true;
      }
    }
  }
  for (int i = 0; i < nopened; ++i) {
    Batch *b = opened[i];
    if (m->cfg.max_agg <= 1) continue;   // M = 1: launched at once, no probe
    if (filled_here[i]) {                // opened and filled by this call: no probe
      b->refs.fetch_sub(1, std::memory_order_relaxed);
      continue;
    }
    if (m->words) {
      // the queue is idle once its word reaches the last number issued
      uint64_t target;
      {
        std::lock_guard<std::mutex> g(ex->rec_mu);
        target = ex->issued;
        if (m->cfg.mode == TB_MODE_POLLING) {
          bridge_word_locked(m, ex, target, Task{idle_fire, b});
          continue;
        }
      }
      wait_word(m, ex, target);
      m->pool->push(Task{idle_fire, b});
      continue;
    }
    // One idleness probe per batch: a queue marker event (src/bridge.py:92-101).
    enqueue_and_bridge(m, ex, Task{idle_fire, b}, [&](tb_event_t *ev) {
      return tb_event_record(reinterpret_cast<tb_stream_t>(ex->stream), ev);
    });
  }
  for (int i = 0; i < nfull; ++i) launch(full[i], false);
}

void schedule(Executor *ex, int kind, const double *src, double *dst, int64_t n,
              SubTask *t) {   // src/executors.py:174-221
  const Req r{src, dst, n, t};
  schedule_many(ex, kind, &r, 1);
}

void task_finished(Machine *m) {
  if (m->remaining.fetch_sub(1) == 1) {
    std::lock_guard<std::mutex> g(m->done_mu);
    m->done_cv.notify_all();
  }
}

// numpy's pairwise sum of 512 contiguous doubles (see oracle/tb_oracle.c)
double pairwise512(const double *a) {
  double bsum[4];
  for (int blk = 0; blk < 4; ++blk) {
    const double *p = a + 128 * blk;
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = p[j];
    for (int i = 8; i < 128; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += p[i + j];
    bsum[blk] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  }
  return (bsum[0] + bsum[1]) + (bsum[2] + bsum[3]);
}

void start_task(void *p) {   // ghost fold + first round (src/miniapp.py:116-130)
  DiagScope ds(kStartNs);
  SubTask *t = static_cast<SubTask *>(p);
  Machine *m = t->m;
  if (m->failed()) {
    task_finished(m);
    return;
  }
  const int64_t S = m->cfg.subgrids;
  t->work = t->abuf;
  t->out = t->bbuf;
  t->round = 0;
  if (m->cfg.zero_copy == 4) {
    // direct: round 0's batch kernel reads the task's rows of the caller's
    // (pinned) cells and folds the neighbour faces itself; the last round
    // writes the rows back with their min and pairwise sum
    const bool one = m->cfg.chains * m->cfg.kernels_per_chain <= 1;
    t->out = one ? t->abuf : t->d0;
    Req r{t->work, t->out, t->n * kCells, t, (uint8_t)(one ? 3 : 1)};
    schedule_many(t->ex, 0, &r, 1);
    return;
  }
  for (int64_t k = 0; k < t->n; ++k) {
    const int64_t g = t->lo + k;
    double *w = t->work + k * kCells;
    std::memcpy(w, m->cells + g * kCells, sizeof(double) * kCells);
    const double *left = m->faces + ((g - 1 + S) % S) * 2 * kFace + kFace;
    const double *right = m->faces + ((g + 1) % S) * 2 * kFace;
    for (int i = 0; i < kFace; ++i) w[i] = 0.5 * (w[i] + left[i]);
    for (int i = 0; i < kFace; ++i)
      w[kCells - kFace + i] = 0.5 * (w[kCells - kFace + i] + right[i]);
  }
  // zero_copy = 3: round 0 reads the folded rows from pinned host memory and
  // writes device memory; the rounds in between stay in HBM
  if (m->dev_arena)
    t->out = m->cfg.chains * m->cfg.kernels_per_chain <= 1 ? t->abuf : t->d0;
  schedule(t->ex, 0, t->work, t->out, t->n * kCells, t);
}

// A task's continuation after its batch: the next round's request into *r
// (returns its kind), or -1 after the write-back + post-process of the last
// round (src/miniapp.py:127-133).
int advance_task(SubTask *t, Req *r) {
  Machine *m = t->m;
  if (m->failed()) {
    task_finished(m);
    return -1;
  }
  const int kpc = (int)m->cfg.kernels_per_chain;
  const int rounds = (int)(m->cfg.chains * kpc);
  if (m->dev_arena) {
    // zero_copy = 3: device ping-pong; the last round writes the host rows
    t->work = t->out;
    if (++t->round < rounds) {
      const bool last = t->round == rounds - 1;
      t->out = last ? t->abuf : (t->work == t->d0 ? t->d1 : t->d0);
      *r = Req{t->work, t->out, t->n * kCells, t,
               (uint8_t)(last && m->cfg.zero_copy == 4 ? 2 : 0)};
      return t->round % kpc;
    }
    if (m->cfg.zero_copy == 4) {   // direct: rows, min and sum written by the kernel
      task_finished(m);
      return -1;
    }
  } else {
    std::swap(t->work, t->out);
    if (++t->round < rounds) {
      *r = Req{t->work, t->out, t->n * kCells, t};
      return t->round % kpc;
    }
  }
  DiagScope ds(kFinishNs);
  for (int64_t k = 0; k < t->n; ++k) {
    const int64_t g = t->lo + k;
    const double *w = t->work + k * kCells;
    std::memcpy(m->cells + g * kCells, w, sizeof(double) * kCells);
    double mn = w[0];
    for (int i = 1; i < kCells; ++i) mn = w[i] < mn ? w[i] : mn;
    m->mins[g] = mn;
    m->sums[g] = pairwise512(w);
  }
  task_finished(m);
  return -1;
}

void resume_task(void *p) {   // next round, or write-back + post-process
  SubTask *t = static_cast<SubTask *>(p);
  Req r;
  const int kind = advance_task(t, &r);
  if (kind >= 0) schedule_many(t->ex, kind, &r, 1);
}

// A chunk of one batch's members (all on one executor; their next requests
// share one kind): advanced in turn, the continuing ones scheduled together.
void resume_task_chunk(SubTask *const *ts, uint32_t n) {
  Req reqs[kResumeChunk];
  int nreq = 0, kind = -1;
  Executor *ex = nullptr;
  for (uint32_t i = 0; i < n; ++i) {
    Req r;
    const int k = advance_task(ts[i], &r);
    if (k < 0) continue;
    if (nreq && (k != kind || ts[i]->ex != ex)) {   // not expected; keep order anyway
      schedule_many(ex, kind, reqs, nreq);
      nreq = 0;
    }
    kind = k;
    ex = ts[i]->ex;
    reqs[nreq++] = r;
  }
  if (nreq) schedule_many(ex, kind, reqs, nreq);
}

// ------------------------------------------------------- hydro workload --
// Host ghost exchange: sub-grid g's [5][12][12][12] block from the periodic
// lattice of interiors (what Octo-Tiger's HPX channels provide), row by row.
void ghost_fill(const Machine *m, int64_t g, double *out) {
  const int64_t n = m->nb, N = 8 * n;
  const int64_t bx = g % n, by = (g / n) % n, bz = g / (n * n);
  for (int f = 0; f < 5; ++f)
    for (int k = 0; k < 12; ++k) {
      const int64_t Z = (8 * bz - 2 + k + N) % N;
      for (int j = 0; j < 12; ++j) {
        const int64_t Y = (8 * by - 2 + j + N) % N;
        double *row = out + ((f * 12 + k) * 12 + j) * 12;
        const int64_t sb = ((Z / 8) * n + Y / 8) * n;
        const int64_t lrow = ((int64_t)f * 8 + Z % 8) * 64 + (Y % 8) * 8;
        // x: 2 ghosts from the left neighbour, 8 interior, 2 from the right
        const int64_t xl = (bx - 1 + n) % n, xr = (bx + 1) % n;
        const double *L = m->U.data() + (sb + xl) * kInterior + lrow;
        const double *C = m->U.data() + (sb + bx) * kInterior + lrow;
        const double *R = m->U.data() + (sb + xr) * kInterior + lrow;
        row[0] = L[6];
        row[1] = L[7];
        std::memcpy(row + 2, C, 8 * sizeof(double));
        row[10] = R[0];
        row[11] = R[1];
      }
    }
}

void hydro_done(Machine *m) { task_finished(m); }

void hydro_resume(void *p) {   // outputs landed in t->b: keep dU/dt and amax
  SubTask *t = static_cast<SubTask *>(p);
  Machine *m = t->m;
  std::memcpy(m->dudt.data() + t->lo * kInterior, t->bbuf,
              sizeof(double) * t->n * kInterior);
  std::memcpy(m->amax.data() + t->lo, t->bbuf + t->n * kInterior, sizeof(double) * t->n);
  hydro_done(m);
}

void hydro_start(void *p) {    // ghost exchange + one K6 request
  SubTask *t = static_cast<SubTask *>(p);
  if (t->m->failed()) {
    hydro_done(t->m);
    return;
  }
  for (int64_t k = 0; k < t->n; ++k) ghost_fill(t->m, t->lo + k, t->abuf + k * kGhosted);
  schedule(t->ex, 0, t->abuf, t->bbuf, t->n * kGhosted, t);
}

void hydro_update(void *p) {   // U += dt * dU/dt (two roundings, as the oracle)
  SubTask *t = static_cast<SubTask *>(p);
  Machine *m = t->m;
  double *u = m->U.data() + t->lo * kInterior;
  const double *du = m->dudt.data() + t->lo * kInterior;
  const double dt = m->dt;
  for (int64_t i = 0; i < t->n * kInterior; ++i) {
    const volatile double inc = dt * du[i];   // no contraction into an FMA
    u[i] = u[i] + inc;
  }
  hydro_done(m);
}

// exact sum (== math.fsum): 32-bit digits in int64 limbs, half-even rounding
double exact_sum(const double *x, int64_t n) {
  long long acc[TB_ACC_LIMBS + 2] = {0};
  for (int64_t i = 0; i < n; ++i) {
    const double v = x[i];
    if (v == 0.0) continue;
    unsigned long long bits;
    std::memcpy(&bits, &v, 8);
    const int ex = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & ((1ULL << 52) - 1);
    int p = 0;
    if (ex) {
      mant |= 1ULL << 52;
      p = ex - 1;
    }
    const int limb = p >> 5, off = p & 31;
    const unsigned __int128 w = (unsigned __int128)mant << off;
    const long long s = (long long)(bits >> 63) ? -1 : 1;
    acc[limb] += s * (long long)(uint64_t)(w & 0xffffffffu);
    acc[limb + 1] += s * (long long)(uint64_t)((w >> 32) & 0xffffffffu);
    acc[limb + 2] += s * (long long)(uint64_t)(w >> 64);
  }
  constexpr int ND = TB_ACC_LIMBS + 4;
  uint32_t d[ND];
  long long carry = 0;
  for (int i = 0; i < ND; ++i) {
    const long long v = (i < TB_ACC_LIMBS + 2 ? acc[i] : 0) + carry;
    d[i] = (uint32_t)(v & 0xffffffffLL);
    carry = v >> 32;
  }
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
  const int nbits = top * 32 + (32 - __builtin_clz(d[top]));
  auto bit = [&](int k) -> unsigned { return (d[k >> 5] >> (k & 31)) & 1u; };
  const int shift = nbits > 53 ? nbits - 53 : 0;
  unsigned long long mant = 0;
  for (int k = nbits - 1; k >= shift; --k) mant = (mant << 1) | bit(k);
  if (shift > 0) {
    const unsigned guard = bit(shift - 1);
    bool sticky = false;
    for (int k = shift - 2; k >= 0 && !sticky; --k) sticky = bit(k);
    if (guard && (sticky || (mant & 1ULL))) mant += 1;
  }
  const double r = std::ldexp((double)mant, shift - TB_ACC_BIAS);
  return neg ? -r : r;
}

}  // namespace tbm

using namespace tbm;

namespace tbm {

// cells_io: the caller's [S][512] cells, advanced in place (as the
// reference's tasks write each grid back, src/miniapp.py:132); null = the
// closed-form initial state in machine-owned memory, copied to cells_out.
int run_machine(const tb_machine_config *cfg_in, double *cells_io, double *checksum,
                tb_machine_step *steps_out, double *cells_out, int64_t *exec_stats) {
  if (!cfg_in || !checksum) return TB_E_INVALID;
  const tb_machine_config &c = *cfg_in;
  if (c.subgrids < 1 || c.steps < 0 || c.workers < 1 || c.executors < 1 || c.max_agg < 1 ||
      c.chains < 0 || c.kernels_per_chain < 1 || c.kernels_per_chain > TB_KINDS ||
      c.task_subgrids < 1 || c.mode < TB_MODE_POLLING || c.mode > TB_MODE_FENCE ||
      c.zero_copy < 0 || c.zero_copy > 4 || c.fault_at_launch < 0 ||
      (c.completion != TB_COMPLETION_EVENTS && c.completion != TB_COMPLETION_WORDS))
    return TB_E_INVALID;
  // completion words are stored by the gather kernels: kernel-only batches,
  // and a worker (not a host-task thread) must observe them
  if (c.completion == TB_COMPLETION_WORDS &&
      (c.zero_copy < 2 || c.mode == TB_MODE_HOSTTASK))
    return TB_E_INVALID;
  int dev = 0;
  cudaGetDevice(&dev);
  Machine m;
  m.cfg = c;
  const int64_t S = c.subgrids;
  const bool direct = c.zero_copy == 4;
  if (direct && cells_io) {
    // the batch kernels read and write the caller's rows: they must be
    // pinned host memory mapped at the same address (UVA)
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, cells_io) != cudaSuccess ||
        pa.type != cudaMemoryTypeHost || pa.devicePointer != cells_io) {
      cudaGetLastError();
      return TB_E_INVALID;
    }
  }
  size_t own_bytes = 0;
  if (cells_io) {
    m.cells = cells_io;
  } else {
    if (direct) {   // machine-owned rows, pinned (the cached host arena)
      own_bytes = sizeof(double) * S * kCells;
      if (!(m.cells = arena_take_host(own_bytes))) return tb::rc(cudaGetLastError());
      m.own_cells_pinned = true;
    } else {
      m.own_cells.resize(S * kCells);
      m.cells = m.own_cells.data();
    }
    const double scale = (double)(S * 1000 + kCells);
    for (int64_t g = 0; g < S; ++g)   // src/miniapp.py:72-77
      for (int i = 0; i < kCells; ++i)
        m.cells[g * kCells + i] = ((double)g * 1000.0 + (double)i) / scale;
  }
  size_t arena_bytes = 0, dev_arena_bytes = 0;
  if (direct) {
    // faces | mins | sums where the batch kernels read and write them
    if (cudaHostAlloc(reinterpret_cast<void **>(&m.pinned_small),
                      sizeof(double) * S * (2 * kFace + 2),
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      if (m.own_cells_pinned) arena_give(m.cells, own_bytes, nullptr, 0, dev);
      return tb::rc(cudaGetLastError());
    }
    m.faces = m.pinned_small;
    m.mins = m.faces + S * 2 * kFace;
    m.sums = m.mins + S;
    dev_arena_bytes = sizeof(double) * 2 * S * kCells;
    if (!(m.dev_arena = arena_take_dev(dev_arena_bytes, dev))) {
      cudaFreeHost(m.pinned_small);
      if (m.own_cells_pinned) arena_give(m.cells, own_bytes, nullptr, 0, dev);
      return tb::rc(cudaGetLastError());
    }
  } else {
    m.faces_v.resize(S * 2 * kFace);
    m.mins_v.resize(S);
    m.sums_v.resize(S);
    m.faces = m.faces_v.data();
    m.mins = m.mins_v.data();
    m.sums = m.sums_v.data();
  }
  if (c.zero_copy == 2) {
    // every task's two work buffers in one pinned, device-mapped arena
    arena_bytes = sizeof(double) * 2 * S * kCells;
    if (!(m.arena = arena_take_host(arena_bytes))) return tb::rc(cudaGetLastError());
  } else if (c.zero_copy == 3) {
    // one pinned, device-mapped row block per task (the host fold's input
    // and the last round's output) + two device blocks per task
    arena_bytes = sizeof(double) * S * kCells;
    dev_arena_bytes = 2 * arena_bytes;
    if (!(m.arena = arena_take_host(arena_bytes))) return tb::rc(cudaGetLastError());
    if (!(m.dev_arena = arena_take_dev(dev_arena_bytes, dev))) {
      arena_give(m.arena, arena_bytes, nullptr, 0, dev);
      return tb::rc(cudaGetLastError());
    }
  }
  diag_reset();
  m.pool.reset(new Pool((int)c.workers, dev, 1234));
  m.poller.reset(new Poller(m.pool.get(), &m.fault));
  if (c.mode == TB_MODE_POLLING) m.pool->set_idle_hook(&Poller::hook, m.poller.get());
  m.hosttasks.reset(new HostTasks(m.pool.get(), (int)std::max<int64_t>(1, c.hosttask_threads),
                                  dev, 4, &m.fault));
  if (c.completion == TB_COMPLETION_WORDS) {
    // one 64-B line per executor for its word, one 128-B line for its counter
    m.words = true;
    if (cudaHostAlloc(reinterpret_cast<void **>(&m.words_host), 64 * c.executors,
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void **>(&m.ctas_dev), 128 * c.executors) != cudaSuccess ||
        cudaMemset(m.ctas_dev, 0, 128 * c.executors) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      m.fail(tb::rc(cudaGetLastError()));
    } else {
      std::memset(m.words_host, 0, 64 * c.executors);
    }
  }
  for (int64_t e = 0; e < c.executors; ++e) {
    auto ex = std::make_unique<Executor>();
    ex->m = &m;
    ex->id = (int)e;
    cudaStreamCreateWithFlags(&ex->stream, cudaStreamNonBlocking);
    if (m.words && m.words_host && m.ctas_dev) {
      ex->word = m.words_host + 8 * e;
      ex->ctas = m.ctas_dev + 32 * e;
    }
    if (exec_stats) {
      ex->stats.reset(new std::atomic<int64_t>[c.max_agg + 3]);
      for (int64_t i = 0; i < c.max_agg + 3; ++i) ex->stats[i].store(0);
    }
    m.execs.push_back(std::move(ex));
  }
  // tasks: contiguous blocks of task_subgrids, round-robin over executors
  // (src/cli.py:224 aggs_by_grid)
  const int64_t ntasks = (S + c.task_subgrids - 1) / c.task_subgrids;
  m.tasks.reserve((size_t)ntasks);
  if (!direct && !m.dev_arena && !m.arena) m.task_bufs.resize((size_t)(2 * S * kCells));
  // executor-major order: task i (executor i mod E) sits among its
  // executor's tasks, so a batch's members — consecutive tasks of one
  // executor — are neighbours in memory when their continuations run
  for (int64_t k = 0; k < ntasks; ++k) {
    const int64_t E = c.executors, q = ntasks / E, r = ntasks % E;
    // k-th slot of the executor-major layout -> task index i
    const int64_t e = k < r * (q + 1) ? k / (q + 1) : r + (k - r * (q + 1)) / q;
    const int64_t j = k < r * (q + 1) ? k % (q + 1) : (k - r * (q + 1)) % q;
    const int64_t lo = (j * E + e) * c.task_subgrids;
    m.tasks.emplace_back();
    SubTask *t = &m.tasks.back();
    t->m = &m;
    t->lo = lo;
    t->n = std::min<int64_t>(c.task_subgrids, S - lo);
    t->ex = m.execs[(size_t)(lo % c.executors)].get();
    if (direct) {   // the caller's rows in, the caller's rows out
      t->abuf = t->bbuf = m.cells + lo * kCells;
      t->d0 = m.dev_arena + 2 * lo * kCells;
      t->d1 = t->d0 + t->n * kCells;
    } else if (m.dev_arena) {
      t->abuf = t->bbuf = m.arena + lo * kCells;
      t->d0 = m.dev_arena + 2 * lo * kCells;
      t->d1 = t->d0 + t->n * kCells;
    } else if (m.arena) {
      t->abuf = m.arena + 2 * lo * kCells;
      t->bbuf = t->abuf + t->n * kCells;
    } else {
      t->abuf = m.task_bufs.data() + 2 * lo * kCells;
      t->bbuf = t->abuf + t->n * kCells;
    }
  }
  double cs = 0.0;
  for (int64_t step = 0; step < c.steps && !m.failed(); ++step) {
    const int64_t k0 = m.kernels, t0n = m.transfers, w0 = m.event_waits, f0 = m.full,
                  i0 = m.idle, mb0 = m.members;
    const auto t0 = Clock::now();
    for (int64_t g = 0; g < S; ++g) {   // face snapshot (src/miniapp.py:89-93)
      std::memcpy(m.faces + g * 2 * kFace, &m.cells[g * kCells], sizeof(double) * kFace);
      std::memcpy(m.faces + g * 2 * kFace + kFace, &m.cells[g * kCells + kCells - kFace],
                  sizeof(double) * kFace);
    }
    m.remaining.store((int64_t)m.tasks.size());
    {
      // each executor's tasks to its worker group (Pool::push_group)
      const size_t E = m.execs.size();
      std::vector<std::vector<Task>> by(E);
      for (auto &t : m.tasks) by[(size_t)t.ex->id].push_back(Task{start_task, &t});
      for (size_t e = 0; e < E; ++e) m.pool->push_group(by[e].data(), by[e].size(), e, E);
    }
    {
      std::unique_lock<std::mutex> lk(m.done_mu);
      m.done_cv.wait(lk, [&] { return m.remaining.load() == 0; });
    }
    if (m.failed()) break;
    double dt = m.mins[0];
    for (int64_t g = 1; g < S; ++g) dt = m.mins[g] < dt ? m.mins[g] : dt;
    const double piece = exact_sum(m.sums, S);
    const auto t1 = Clock::now();
    cs += piece;
    if (steps_out) {
      tb_machine_step &o = steps_out[step];
      o.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      o.dt = dt;
      o.piece = piece;
      o.launches = m.kernels - k0;
      o.transfers = m.transfers - t0n;
      o.event_waits = m.event_waits - w0;
      o.full = m.full - f0;
      o.idle = m.idle - i0;
      o.members = m.members - mb0;
    }
    if (exec_stats) {   // [steps][executors][max_agg + 3], then reset
      const int64_t W = c.max_agg + 3;
      for (int64_t e = 0; e < c.executors; ++e)
        for (int64_t i = 0; i < W; ++i)
          exec_stats[(step * c.executors + e) * W + i] = m.execs[e]->stats[i].exchange(0);
    }
  }
  *checksum = cs;
  if (cells_out && cells_out != m.cells && !m.failed())
    std::memcpy(cells_out, m.cells, sizeof(double) * S * kCells);
  m.pool->stop();
  diag_print((int)c.mode, c.workers, c.executors, c.max_agg, c.steps);
  m.hosttasks.reset();
  for (auto &ex : m.execs) {
    cudaStreamSynchronize(ex->stream);
    cudaStreamDestroy(ex->stream);
  }
  for (Staging *s : m.staging_all) {
    cudaFreeHost(s->host);
    cudaFree(s->dev);
    delete s;
  }
  const int err = tb::rc(cudaGetLastError());
  // direct mode: the machine-owned pinned rows go back as the host arena
  double *host_arena = m.own_cells_pinned ? m.cells : m.arena;
  const size_t host_bytes = m.own_cells_pinned ? own_bytes : arena_bytes;
  if (!m.failed()) {
    arena_give(host_arena, host_bytes, m.dev_arena, dev_arena_bytes, dev);
  } else {   // a faulted context: do not keep its memory
    if (host_arena) cudaFreeHost(host_arena);
    if (m.dev_arena) cudaFree(m.dev_arena);
  }
  if (m.pinned_small) cudaFreeHost(m.pinned_small);
  if (m.words_host) cudaFreeHost(m.words_host);
  if (m.ctas_dev) cudaFree(m.ctas_dev);
  return m.failed() ? m.fault.load() : err;
}

}  // namespace tbm

extern "C" int tb_machine_run(const tb_machine_config *cfg_in, double *checksum,
                              tb_machine_step *steps_out, double *cells_out) {
  return run_machine(cfg_in, nullptr, checksum, steps_out, cells_out, nullptr);
}

extern "C" int tb_machine_run_cells(const tb_machine_config *cfg_in, double *cells,
                                    double *checksum, tb_machine_step *steps_out,
                                    int64_t *exec_stats) {
  if (!cells) return TB_E_INVALID;
  return run_machine(cfg_in, cells, checksum, steps_out, cells, exec_stats);
}

extern "C" int tb_machine_run_hydro(const tb_machine_config *cfg_in, const double *U_in,
                                    double *U_out, double cfl, double gamma,
                                    tb_machine_step *steps_out) {
  if (!cfg_in || !U_in || !(cfl > 0.0) || !(gamma > 1.0)) return TB_E_INVALID;
  const tb_machine_config &c = *cfg_in;
  int64_t nb = 1;
  while (nb * nb * nb < c.subgrids) ++nb;
  if (c.subgrids < 1 || nb * nb * nb != c.subgrids || c.steps < 0 || c.workers < 1 ||
      c.executors < 1 || c.max_agg < 1 || c.task_subgrids < 1 || c.mode < TB_MODE_POLLING ||
      c.mode > TB_MODE_FENCE || c.completion != TB_COMPLETION_EVENTS)
    return TB_E_INVALID;
  int dev = 0;
  cudaGetDevice(&dev);
  Machine m;
  m.cfg = c;
  m.hydro = true;
  m.nb = nb;
  m.dx = 1.0 / (8.0 * (double)nb);
  m.gamma = gamma;
  const int64_t S = c.subgrids;
  m.U.assign(U_in, U_in + S * kInterior);
  m.dudt.resize(S * kInterior);
  m.amax.resize(S);
  diag_reset();
  m.pool.reset(new Pool((int)c.workers, dev, 1234));
  m.poller.reset(new Poller(m.pool.get(), &m.fault));
  if (c.mode == TB_MODE_POLLING) m.pool->set_idle_hook(&Poller::hook, m.poller.get());
  m.hosttasks.reset(new HostTasks(m.pool.get(), (int)std::max<int64_t>(1, c.hosttask_threads),
                                  dev, 4, &m.fault));
  for (int64_t e = 0; e < c.executors; ++e) {
    auto ex = std::make_unique<Executor>();
    ex->m = &m;
    ex->id = (int)e;
    cudaStreamCreateWithFlags(&ex->stream, cudaStreamNonBlocking);
    m.execs.push_back(std::move(ex));
  }
  m.tasks.reserve((size_t)((S + c.task_subgrids - 1) / c.task_subgrids));
  m.task_bufs.resize((size_t)(S * (kGhosted + kHydroOut)));
  for (int64_t lo = 0; lo < S; lo += c.task_subgrids) {
    m.tasks.emplace_back();
    SubTask *t = &m.tasks.back();
    t->m = &m;
    t->lo = lo;
    t->n = std::min<int64_t>(c.task_subgrids, S - lo);
    t->ex = m.execs[(size_t)((lo / c.task_subgrids) % c.executors)].get();
    t->abuf = m.task_bufs.data() + lo * (kGhosted + kHydroOut);   // ghosted inputs
    t->bbuf = t->abuf + t->n * kGhosted;                           // dU/dt + amax
  }
  {  // pre-allocate the pinned/device staging pool (two full batches per stream)
    std::vector<Staging *> warm;
    for (int64_t i = 0; i < 2 * c.executors; ++i) warm.push_back(staging_alloc(&m, hydro_staging_bytes(&m)));
    for (Staging *st : warm) staging_release(&m, st);
  }
  std::vector<double> rho(S * 512);
  for (int64_t step = 0; step < c.steps && !m.failed(); ++step) {
    const int64_t k0 = m.kernels, t0n = m.transfers, w0 = m.event_waits, f0 = m.full,
                  i0 = m.idle, mb0 = m.members;
    const auto t0 = Clock::now();
    for (int phase = 0; phase < 2 && !m.failed(); ++phase) {   // fluxes, then the update
      m.remaining.store((int64_t)m.tasks.size());
      std::vector<Task> ts;
      ts.reserve(m.tasks.size());
      for (auto &t : m.tasks) ts.push_back(Task{phase ? hydro_update : hydro_start, &t});
      m.pool->push_spread(ts.data(), ts.size());   // hydro_update is host work: any worker
      std::unique_lock<std::mutex> lk(m.done_mu);
      m.done_cv.wait(lk, [&] { return m.remaining.load() == 0; });
      if (phase == 0) {
        double am = m.amax[0];
        for (int64_t g = 1; g < S; ++g) am = m.amax[g] > am ? m.amax[g] : am;
        m.dt = (cfl * m.dx) / am;
      }
    }
    const auto t1 = Clock::now();
    for (int64_t g = 0; g < S; ++g)
      std::memcpy(rho.data() + g * 512, m.U.data() + g * kInterior, 512 * sizeof(double));
    if (steps_out) {
      tb_machine_step &o = steps_out[step];
      o.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      o.dt = m.dt;
      o.piece = exact_sum(rho.data(), S * 512);
      o.launches = m.kernels - k0;
      o.transfers = m.transfers - t0n;
      o.event_waits = m.event_waits - w0;
      o.full = m.full - f0;
      o.idle = m.idle - i0;
      o.members = m.members - mb0;
    }
  }
  if (U_out && !m.failed()) std::memcpy(U_out, m.U.data(), sizeof(double) * S * kInterior);
  m.pool->stop();
  m.hosttasks.reset();
  for (auto &ex : m.execs) {
    cudaStreamSynchronize(ex->stream);
    cudaStreamDestroy(ex->stream);
  }
  for (Staging *st : m.staging_all) {
    cudaFreeHost(st->host);
    cudaFree(st->dev);
    delete st;
  }
  const int err = tb::rc(cudaGetLastError());
  return m.failed() ? m.fault.load() : err;
}
