// Prior-art baselines (include/dv_baselines.h): the paper's per-run copies and buffered copies
// expressed with CUDA runtime DMA, for measurement next to the dvstream kernels.
#include "../../include/dv_baselines.h"
#include "dv_internal.h"

using namespace dv;

namespace {
struct Geo {
  const uint8_t* k;
  const uint8_t* v;
  int64_t row, sh, sr, sl, run;
  int nL, nR, H;
};
dv_status geo(const dv_cache* c, const dv_region* r0, Geo* g) {
  DV_TRY(check_cache(c, "source"));
  if (c->layout != DV_LAYOUT_KV5D) return fail(DV_ENOTSUP, "baselines support KV5D only");
  DV_TRY(check_region_shape(r0));
  DV_TRY(check_cache_holds(c, r0, "source"));
  const dv_region rr = resolve_heads(r0, c);
  const dv_region* r = &rr;
  g->row = (int64_t)c->head_dim * c->elem_bytes;
  g->sh = (int64_t)c->max_seq * g->row;
  g->sr = g->sh * c->n_heads;
  g->sl = g->sr * c->n_reqs;
  const int64_t off = (int64_t)(r->layer_begin - c->layer_begin) * g->sl +
                      (int64_t)(r->req_begin - c->req_begin) * g->sr +
                      (int64_t)(r->head_begin - c->head_begin) * g->sh + (int64_t)r->pos_begin * g->row;
  g->k = (const uint8_t*)c->k + off;
  g->v = (const uint8_t*)c->v + off;
  g->run = (int64_t)(r->pos_end - r->pos_begin) * g->row;
  g->nL = r->layer_end - r->layer_begin;
  g->nR = r->req_end - r->req_begin;
  g->H = r->head_end - r->head_begin;
  return DV_OK;
}
}  // namespace

extern "C" dv_status dvb_per_run_copy(const dv_cache* src, const dv_region* region, void* dst,
                                      void* stream, uint64_t* n_calls) {
  Geo g;
  DV_TRY(geo(src, region, &g));
  uint8_t* w = (uint8_t*)dst;
  uint64_t calls = 0;
  if (g.run)
    for (int l = 0; l < g.nL; ++l)
      for (int kv = 0; kv < 2; ++kv)
        for (int r = 0; r < g.nR; ++r)
          for (int h = 0; h < g.H; ++h) {
            const uint8_t* s = (kv ? g.v : g.k) + l * g.sl + r * g.sr + h * g.sh;
            DV_CUDA(cudaMemcpyAsync(w, s, g.run, cudaMemcpyDefault, (cudaStream_t)stream));
            w += g.run;
            ++calls;
          }
  if (n_calls) *n_calls = calls;
  return DV_OK;
}

extern "C" dv_status dvb_buffered_copy(const dv_cache* src, const dv_region* region, void* staging,
                                       void* dst, void* stream, uint64_t* n_calls) {
  Geo g;
  DV_TRY(geo(src, region, &g));
  uint8_t* w = (uint8_t*)staging;
  uint64_t calls = 0;
  const uint64_t total = 2ull * g.nL * g.nR * g.H * g.run;
  if (g.run) {
    for (int l = 0; l < g.nL; ++l)
      for (int kv = 0; kv < 2; ++kv)
        for (int r = 0; r < g.nR; ++r) {
          const uint8_t* s = (kv ? g.v : g.k) + l * g.sl + r * g.sr;
          DV_CUDA(cudaMemcpy2DAsync(w, g.run, s, g.sh, g.run, g.H, cudaMemcpyDefault,
                                    (cudaStream_t)stream));
          w += g.run * g.H;
          ++calls;
        }
    DV_CUDA(cudaMemcpyAsync(dst, staging, total, cudaMemcpyDefault, (cudaStream_t)stream));
    ++calls;
  }
  if (n_calls) *n_calls = calls;
  return DV_OK;
}
