/*
 * abi_smoke.c -- the C ABI used from plain C (no Python, no torch): route a C3-like hand-off on
 * the host, then (if a GPU is present) stream a small cache out to pinned host memory and back
 * into a cache with another max_seq, and check every word against the writer's definition
 * (computed here independently: word = low 16 bits of a simple coordinate code).
 *
 *   build:  gcc -O2 -I include tests/c/abi_smoke.c -L paper_2403_01876_b200 -ldvstream
 *           -Wl,-rpath,paper_2403_01876_b200 -o tests/c/abi_smoke   (done by __graft_entry__.build)
 *   run:    tests/c/abi_smoke [--route-only | --enqueue-bench | --token-bench | --partition]
 *           (--partition: the same stream check on the streaming stream of an 8-SM partition,
 *           dv_partition_create, then dv_partition_destroy)
 * Exit code 0 = pass.
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dv.h"

#define CHECK(x)                                                                        \
  do {                                                                                  \
    dv_status _s = (x);                                                                 \
    if (_s != DV_OK) {                                                                  \
      fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #x, dv_status_str(_s), \
              dv_last_error());                                                         \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

/* cudaMemcpy without including CUDA headers: use the library's own host/device buffers and its
 * flush/fetch (contiguous copies) so this file needs nothing but dv.h. */

static int route_check(void) {
  const int32_t pb[] = {0, 16, 32, 48, 64}, tb[] = {0, 13, 30, 47, 64}, rb[] = {0, 8};
  dv_setup ps = {4, pb, 1, rb, 1024, 0, NULL}, ts = {4, tb, 1, rb, 2048, 0, NULL};
  dv_region reg = {0, 64, 0, 8, 0, 1000, 0, 0};
  uint64_t n = 0;
  CHECK(dv_route(&ps, &ts, &reg, 72, 128, 2, NULL, 0, &n));
  if (n != 7) {
    fprintf(stderr, "C3 route: %llu pieces, expected 7\n", (unsigned long long)n);
    return 1;
  }
  dv_piece pieces[7];
  CHECK(dv_route(&ps, &ts, &reg, 72, 128, 2, pieces, 7, &n));
  const int32_t exp[7][4] = {{0, 0, 0, 13}, {0, 1, 13, 16}, {1, 1, 16, 30}, {1, 2, 30, 32},
                             {2, 2, 32, 47}, {2, 3, 47, 48}, {3, 3, 48, 64}};
  for (int i = 0; i < 7; ++i)
    if (pieces[i].src_stage != exp[i][0] || pieces[i].dst_stage != exp[i][1] ||
        pieces[i].layer_begin != exp[i][2] || pieces[i].layer_end != exp[i][3]) {
      fprintf(stderr, "C3 piece %d wrong\n", i);
      return 1;
    }
  /* a position beyond max_seq is a range error naming the limit */
  dv_region bad = {0, 64, 0, 8, 0, 1025, 0, 0};
  if (dv_route(&ps, &ps, &bad, 72, 128, 2, NULL, 0, &n) != DV_ERANGE ||
      !strstr(dv_last_error(), "1024")) {
    fprintf(stderr, "expected DV_ERANGE naming 1024\n");
    return 1;
  }
  printf("route ok\n");
  return 0;
}

static uint16_t word(int kv, int l, int r, int h, int s, int d) {
  return (uint16_t)(((((kv * 7 + l) * 13 + r) * 11 + h) * 101 + s) * 17 + d);
}

static int stream_check(void* st) {
  const int L = 2, B = 2, H = 4, S = 40, S2 = 64, D = 16, P = 40;
  dv_ctx* ctx;
  CHECK(dv_create(0, NULL, &ctx));
  const size_t n5 = (size_t)L * B * H * S * D, n6 = (size_t)L * B * H * S2 * D;
  uint16_t *hk, *hv, *log, *ok2, *ov2;
  void *dk, *dvv, *dk2, *dv2;
  uint64_t* flags;
  CHECK(dv_host_alloc(n5 * 2, (void**)&hk));
  CHECK(dv_host_alloc(n5 * 2, (void**)&hv));
  CHECK(dv_host_alloc(n5 * 4, (void**)&log));
  CHECK(dv_host_alloc(n6 * 2, (void**)&ok2));
  CHECK(dv_host_alloc(n6 * 2, (void**)&ov2));
  CHECK(dv_host_alloc(64, (void**)&flags));
  memset(flags, 0, 64);
  for (int l = 0; l < L; ++l)
    for (int r = 0; r < B; ++r)
      for (int h = 0; h < H; ++h)
        for (int s = 0; s < S; ++s)
          for (int d = 0; d < D; ++d) {
            const size_t i = ((((size_t)l * B + r) * H + h) * S + s) * D + d;
            hk[i] = word(0, l, r, h, s, d);
            hv[i] = word(1, l, r, h, s, d);
          }
  for (size_t i = 0; i < n6; ++i) ok2[i] = ov2[i] = 0xFFFF;
  CHECK(dv_device_alloc(0, n5 * 2, &dk));
  CHECK(dv_device_alloc(0, n5 * 2, &dvv));
  CHECK(dv_device_alloc(0, n6 * 2, &dk2));
  CHECK(dv_device_alloc(0, n6 * 2, &dv2));
  /* upload with level-3 flushes into device endpoints */
  dv_endpoint ek = {DV_EP_DEVICE, 0, dk, n5 * 2, NULL, 0, 0};
  dv_endpoint ev = {DV_EP_DEVICE, 0, dvv, n5 * 2, NULL, 0, 0};
  dv_endpoint ek2 = {DV_EP_DEVICE, 0, dk2, n6 * 2, NULL, 0, 0};
  dv_endpoint ev2 = {DV_EP_DEVICE, 0, dv2, n6 * 2, NULL, 0, 0};
  CHECK(dv_flush(ctx, hk, n5 * 2, &ek, 0, -1, 0, DV_XFER_STAGED, st));
  CHECK(dv_flush(ctx, hv, n5 * 2, &ev, 0, -1, 0, DV_XFER_STAGED, st));
  CHECK(dv_flush(ctx, ok2, n6 * 2, &ek2, 0, -1, 0, DV_XFER_STAGED, st));
  CHECK(dv_flush(ctx, ov2, n6 * 2, &ev2, 0, -1, 0, DV_XFER_STAGED, st));
  dv_cache src = {dk, dvv, 0, DV_LAYOUT_KV5D, 2, 0, L, 0, B, H, S, D, 0};
  dv_cache dst = {dk2, dv2, 0, DV_LAYOUT_KV5D, 2, 0, L, 0, B, H, S2, D, 0};
  const int32_t lb[] = {0, 2}, rb[] = {0, 2};
  dv_setup one = {1, lb, 1, rb, S, 0, NULL}, big = {1, lb, 1, rb, S2, 0, NULL};
  dv_region reg = {0, L, 0, B, 0, P, 0, 0};
  dv_endpoint inbox = {DV_EP_HOST, -1, log, n5 * 4, flags, 1, 0};
  CHECK(dv_stream_out(ctx, &src, &reg, &one, 0, 0, 0, &big, &inbox, 1, 1, DV_XFER_AUTO, st));
  CHECK(dv_stream_in(ctx, &dst, &reg, &one, &big, 0, 0, 0, &inbox, 1, DV_XFER_AUTO, st));
  /* download with level-3 fetches, then wait for everything */
  dv_endpoint hk_ep = {DV_EP_HOST, -1, ok2, n6 * 2, NULL, 0, 0};
  CHECK(dv_fetch(ctx, &ek2, 0, -1, 0, ok2, n6 * 2, DV_XFER_STAGED, st));
  CHECK(dv_fetch(ctx, &ev2, 0, -1, 0, ov2, n6 * 2, DV_XFER_STAGED, st));
  (void)hk_ep;
  dv_endpoint fl = {DV_EP_HOST, -1, flags, 64, flags, 8, 0};
  CHECK(dv_signal(ctx, &fl, 1, 42, st));
  int32_t done = 0;
  for (long spin = 0; spin < 2000000000L && !done; ++spin) CHECK(dv_query(ctx, &fl, 1, 42, &done));
  if (!done || flags[0] != 1) {
    fprintf(stderr, "flags not published (%llu)\n", (unsigned long long)flags[0]);
    return 1;
  }
  size_t bad = 0;
  for (int l = 0; l < L; ++l)
    for (int r = 0; r < B; ++r)
      for (int h = 0; h < H; ++h)
        for (int s = 0; s < S2; ++s)
          for (int d = 0; d < D; ++d) {
            const size_t i = ((((size_t)l * B + r) * H + h) * S2 + s) * D + d;
            const uint16_t ek_ = s < P ? word(0, l, r, h, s, d) : 0xFFFF;
            const uint16_t ev_ = s < P ? word(1, l, r, h, s, d) : 0xFFFF;
            bad += (ok2[i] != ek_) + (ov2[i] != ev_);
          }
  CHECK(dv_destroy(ctx));
  if (bad) {
    fprintf(stderr, "%zu words differ\n", bad);
    return 1;
  }
  printf("stream ok\n");
  return 0;
}

#include <time.h>

/* Host-side enqueue cost of one dv_scatter call (validation + plan + kernel launch), measured from
 * C with no Python in the loop: a C2-shaped per-layer token update (640 runs of 256 B) into a
 * device buffer; batches of 500 calls (well inside the launch queue, so no call blocks on a
 * full queue), synchronised between batches through a host-visible flag. */
static int enqueue_bench(void) {
  const int L = 40, B = 8, H = 40, S = 2048, D = 128;
  dv_ctx* ctx;
  CHECK(dv_create(0, NULL, &ctx));
  const size_t n = (size_t)L * B * H * S * D * 2;
  void *k, *v, *buf;
  CHECK(dv_device_alloc(0, n, &k));
  CHECK(dv_device_alloc(0, n, &v));
  CHECK(dv_device_alloc(0, 1 << 20, &buf));
  uint64_t* fl;
  CHECK(dv_device_alloc(0, 64, (void**)&fl));
  dv_cache c = {k, v, 0, DV_LAYOUT_KV5D, 2, 0, L, 0, B, H, S, D, 0};
  dv_endpoint ep = {DV_EP_DEVICE, 0, buf, 1 << 20, fl, 1, 0};
  const int N = 500, REP = 20;
  uint64_t* hf;
  CHECK(dv_host_alloc(64, (void**)&hf));
  memset(hf, 0, 64);
  dv_endpoint hep = {DV_EP_HOST, -1, hf, 64, hf, 1, 0};
  /* a second (destination) cache and a 1-stage setup for the level-1 direct form */
  void *k2, *v2;
  CHECK(dv_device_alloc(0, n, &k2));
  CHECK(dv_device_alloc(0, n, &v2));
  dv_cache c2 = {k2, v2, 0, DV_LAYOUT_KV5D, 2, 0, L, 0, B, H, S, D, 0};
  int32_t lbnd[2] = {0, L}, rbnd[2] = {0, B};
  dv_setup su = {1, lbnd, 1, rbnd, S, 0, NULL};
  const char* names[3] = {"dv_scatter_flag", "dv_scatter_noflag", "dv_stream_out_direct_flag"};
  uint64_t seq = 1, sig = 1;
  printf("{");
  for (int variant = 0; variant < 3; ++variant) {
    double total_ns = 0;
    for (int rep = 0; rep < REP + 1; ++rep) {
      struct timespec t0, t1;
      clock_gettime(CLOCK_MONOTONIC, &t0);
      for (int i = 0; i < N; ++i) {
        dv_region r = {i % L, i % L + 1, 0, B, 1000 + i % 1000, 1001 + i % 1000, 0, 0};
        if (variant == 0)
          CHECK(dv_scatter(ctx, &c, &r, &ep, 0, 0, seq++, DV_XFER_FUSED, NULL));
        else if (variant == 1)
          CHECK(dv_scatter(ctx, &c, &r, &ep, 0, -1, 0, DV_XFER_FUSED, NULL));
        else
          CHECK(dv_stream_out_direct(ctx, &c, &r, &su, 0, 0, 0, &su, &c2, &ep, 1, seq++, DV_XFER_FUSED, NULL));
      }
      clock_gettime(CLOCK_MONOTONIC, &t1);
      if (rep > 0) total_ns += (t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec);
      CHECK(dv_signal(ctx, &hep, 0, sig, NULL));   /* drain before the next batch */
      int32_t done = 0;
      while (!done) CHECK(dv_query(ctx, &hep, 0, sig, &done));
      ++sig;
    }
    const double us = total_ns / 1e3 / ((double)N * REP);
    printf("%s\"host_enqueue_us_%s\": %.3f", variant ? ", " : "", names[variant], us);
  }
  printf(", \"calls_each\": %d}\n", N * REP);
  /* the first key keeps the historical name read by DESIGN.md */
  CHECK(dv_destroy(ctx));
  return 0;
}

/* The headline workload from plain C: C2 token steps (40 layers x 8 requests x 40 heads x one
 * position x head_dim 128, fp16 words = 6,553,600 B) streamed to a pinned host log with
 * DV_XFER_DECOUPLED and a seq flag per step; wall time from the first call to the last flag seen
 * by dv_query. The cache content is whatever dv_device_alloc returned (bytes are opaque). */
static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}
static int token_bench(void) {
  const int L = 40, B = 8, H = 40, S = 2048, D = 128, RING = 64, N = 500, W = 10;
  const uint64_t step = 2ull * L * B * H * D * 2;
  dv_ctx* ctx;
  CHECK(dv_create(0, NULL, &ctx));
  void *k, *v, *log;
  const size_t n = (size_t)L * B * H * S * D * 2;
  CHECK(dv_device_alloc(0, n, &k));
  CHECK(dv_device_alloc(0, n, &v));
  CHECK(dv_host_alloc_near(0, step * RING, &log, NULL));
  uint64_t* fl;
  CHECK(dv_host_alloc(64, (void**)&fl));
  memset(fl, 0, 64);
  dv_cache c = {k, v, 0, DV_LAYOUT_KV5D, 2, 0, L, 0, B, H, S, D, 0};
  dv_endpoint ep = {DV_EP_HOST, -1, log, step * RING, fl, 1, 0};
  double t0 = 0;
  for (int t = 1; t <= W + N; ++t) {
    if (t == W + 1) {
      int32_t done = 0;
      while (!done) CHECK(dv_query(ctx, &ep, 0, (uint64_t)W, &done));
      t0 = now_s();
    }
    const int32_t q = 1000 + t % 1000;
    dv_region r = {0, L, 0, B, q, q + 1, 0, 0};
    CHECK(dv_scatter(ctx, &c, &r, &ep, (uint64_t)(t % RING) * step, 0, (uint64_t)t, DV_XFER_DECOUPLED, NULL));
  }
  int32_t done = 0;
  while (!done) CHECK(dv_query(ctx, &ep, 0, (uint64_t)(W + N), &done));
  const double dt = now_s() - t0;
  printf("{\"c2_token_steps_from_C_gbs\": %.2f, \"us_per_step\": %.2f, \"steps\": %d}\n",
         N * (double)step / dt / 1e9, dt / N * 1e6, N);
  CHECK(dv_destroy(ctx));
  return 0;
}

int main(int argc, char** argv) {
  if (dv_abi_version() != DV_ABI_VERSION) return 1;
  if (route_check()) return 1;
  if (argc > 1 && !strcmp(argv[1], "--route-only")) return 0;
  if (argc > 1 && !strcmp(argv[1], "--enqueue-bench")) return enqueue_bench();
  if (argc > 1 && !strcmp(argv[1], "--token-bench")) return token_bench();
  if (argc > 1 && !strcmp(argv[1], "--partition")) {
    dv_partition* part;
    void *st_stream, *st_compute;
    int32_t n0 = 0, n1 = 0;
    CHECK(dv_partition_create(0, 8, 0, &part, &st_stream, &st_compute, &n0, &n1));
    if (n0 < 8 || n1 < 1) {
      fprintf(stderr, "partition %d + %d SMs\n", n0, n1);
      return 1;
    }
    const int rc = stream_check(st_stream);   /* ends with dv_destroy: the device is idle after it */
    CHECK(dv_partition_destroy(part));
    if (!rc) printf("partition ok (%d + %d SMs)\n", n0, n1);
    return rc;
  }
  return stream_check(NULL);
}
