/* A plain-C consumer of libtb.so (tests only): what a reference-side binding
 * (ctypes / cgo / JNI) does, with no Python or torch in the
 * process. Exit 0 and "OK" on stdout when every check passes.
 *
 *  1. the ring (src/reference.py:23-50 at S = 4, 2 steps) through
 *     tb_init_cells + tb_step_final: checksum and both dts bit-equal to the
 *     reference's GOLDEN_4X2 / GOLDEN_4X2_DTS (pkg/tests/test_miniapp.py:21-23);
 *  2. event polling (src/runtime/polling.py:101 needs only is_complete()):
 *     tb_event_record behind a tb_spin, tb_event_query until TB_OK;
 *  3. one aggregation batch (src/executors.py:257-284) through tb_agg_launch
 *     from pinned host memory, polled to completion, against the transform
 *     restated here (two roundings, no FMA: build with -ffp-contract=off).
 *
 * cc -std=c99 -O2 -ffp-contract=off -I include tests/c/ring_client.c \
 *    -L paper_2303_08058_b200 -ltb -Wl,-rpath,<dir of libtb.so> -o ring_client
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "tb.h"

#define CHECK(call)                                                          \
  do {                                                                       \
    int rc_ = (call);                                                        \
    if (rc_ != TB_OK) {                                                      \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #call,    \
              rc_, tb_error_string(rc_));                                    \
      return 1;                                                              \
    }                                                                        \
  } while (0)

static int same(double a, double b) { return memcmp(&a, &b, sizeof a) == 0; }

static int ring(tb_stream_t s) {
  enum { S = 4, STEPS = 2 };
  const double golden = 0x1.8e6968eb86d56p+10;
  const double golden_dts[STEPS] = {0x1.d0d57314f3d28p-10, 0x1.d0df8d332e761p-10};
  double *state[2], *dev_out;   /* dev_out: piece[2], dt[2], checksum */
  int64_t *acc;
  CHECK(tb_malloc((void **)&state[0], S * TB_CELLS * sizeof(double)));
  CHECK(tb_malloc((void **)&state[1], S * TB_CELLS * sizeof(double)));
  CHECK(tb_malloc((void **)&dev_out, 5 * sizeof(double)));
  CHECK(tb_malloc((void **)&acc, TB_ACC_WORDS * sizeof(int64_t)));
  CHECK(tb_memset(s, dev_out, 0, 5 * sizeof(double)));
  CHECK(tb_init_cells(s, state[0], S, 0, S));
  CHECK(tb_acc_reset(s, acc));
  for (int k = 0; k < STEPS; ++k) {
    const double *old = state[k & 1];
    /* single-device ring: the wrap faces come from the state itself */
    CHECK(tb_step_final(s, old, state[1 - (k & 1)], S, old + (S - 1) * TB_CELLS + 504, old,
                        3, 5, NULL, NULL, acc, dev_out + k, dev_out + 2 + k, dev_out + 4));
  }
  double host[5];
  CHECK(tb_memcpy_d2h(s, host, dev_out, sizeof host));
  CHECK(tb_stream_sync(s));
  if (!same(host[4], golden) || !same(host[2], golden_dts[0]) || !same(host[3], golden_dts[1])) {
    fprintf(stderr, "ring: checksum %a dts %a %a (want %a, %a %a)\n", host[4], host[2],
            host[3], golden, golden_dts[0], golden_dts[1]);
    return 1;
  }
  tb_free(state[0]);
  tb_free(state[1]);
  tb_free(dev_out);
  tb_free(acc);
  return 0;
}

static int polling(tb_stream_t s) {
  tb_event_t ev;
  CHECK(tb_spin(s, 2000000));           /* keep the queue busy for ~2 ms */
  CHECK(tb_event_record(s, &ev));
  long polls = 0;
  int rc;
  while ((rc = tb_event_query(ev)) == TB_NOT_READY) ++polls;
  CHECK(rc);
  if (polls == 0) {
    fprintf(stderr, "polling: event complete on the first query behind a 2 ms spin\n");
    return 1;
  }
  CHECK(tb_event_release(ev));
  return 0;
}

static int batch(tb_stream_t s) {
  enum { MEMBERS = 3, N = MEMBERS * TB_CELLS };
  const double c1 = 1.0000003, c2 = 1e-7;   /* kind 0 (src/miniapp.py:36-37) */
  double *h, *d, want[N];
  CHECK(tb_host_alloc((void **)&h, N * sizeof(double)));
  CHECK(tb_malloc((void **)&d, N * sizeof(double)));
  for (int i = 0; i < N; ++i) {
    h[i] = (double)i / 7.0 - 100.0;
    volatile double p = h[i] * c1;      /* two roundings, as numpy does */
    want[i] = p + c2;
  }
  tb_event_t done;
  CHECK(tb_agg_launch(s, TB_OP_KIND, 0, 0.0, 0.0, d, h, N * sizeof(double), 1, &done));
  int rc;
  while ((rc = tb_event_query(done)) == TB_NOT_READY) {
  }
  CHECK(rc);
  CHECK(tb_event_release(done));
  for (int i = 0; i < N; ++i)
    if (!same(h[i], want[i])) {
      fprintf(stderr, "batch: cell %d = %a, want %a\n", i, h[i], want[i]);
      return 1;
    }
  tb_host_free(h);
  tb_free(d);
  return 0;
}

int main(void) {
  CHECK(tb_init(0));
  tb_stream_t s;
  CHECK(tb_stream_create(&s));
  if (ring(s) || polling(s) || batch(s)) return 1;
  CHECK(tb_stream_destroy(s));
  printf("OK abi %d\n", tb_abi_version());
  return 0;
}
