// Host-only parts of dvstream: error state, validation, region sizes and the route planner
// (the stream_out / stream_in level of PAPER.md:169-172, Table 1; split/merge of §4.2.1,
// PAPER.md:266). Pure functions; usable without a GPU.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "dv_internal.h"

namespace dv {

static thread_local std::string g_err;

dv_status fail(dv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

dv_status cuda_fail(cudaError_t e, const char* what) {
  (void)cudaGetLastError();  // do not leave a (non-sticky) error behind for the caller's next check
  return fail(DV_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

dv_status check_setup(const dv_setup* s, const char* name) {
  if (!s) return fail(DV_EINVAL, "%s: NULL setup", name);
  if (s->n_stages < 1 || !s->layer_bounds) return fail(DV_EINVAL, "%s: need >= 1 stage", name);
  if (s->n_micro < 1 || !s->req_bounds) return fail(DV_EINVAL, "%s: need >= 1 microbatch", name);
  if (s->max_seq < 1) return fail(DV_EINVAL, "%s: max_seq must be >= 1", name);
  if (s->n_tp < 0 || (s->n_tp > 0) != (s->head_bounds != nullptr))
    return fail(DV_EINVAL, "%s: n_tp > 0 requires head_bounds (and n_tp = 0 none)", name);
  if (s->layer_bounds[0] < 0 || s->req_bounds[0] < 0 || (s->n_tp && s->head_bounds[0] < 0))
    return fail(DV_EINVAL, "%s: negative bound", name);
  for (int i = 0; i < s->n_stages; ++i)
    if (s->layer_bounds[i + 1] <= s->layer_bounds[i])
      return fail(DV_EINVAL, "%s: layer_bounds not strictly increasing at %d", name, i);
  for (int i = 0; i < s->n_micro; ++i)
    if (s->req_bounds[i + 1] <= s->req_bounds[i])
      return fail(DV_EINVAL, "%s: req_bounds not strictly increasing at %d", name, i);
  for (int i = 0; i < s->n_tp; ++i)
    if (s->head_bounds[i + 1] <= s->head_bounds[i])
      return fail(DV_EINVAL, "%s: head_bounds not strictly increasing at %d", name, i);
  return DV_OK;
}

bool all_heads(const dv_region* r) { return r->head_begin == 0 && r->head_end == 0; }

dv_status check_region_shape(const dv_region* r) {
  if (!r) return fail(DV_EINVAL, "NULL region");
  if (r->layer_begin < 0 || r->req_begin < 0 || r->pos_begin < 0 || r->head_begin < 0 ||
      r->layer_end < r->layer_begin || r->req_end < r->req_begin || r->pos_end < r->pos_begin ||
      r->head_end < r->head_begin)
    return fail(DV_EINVAL, "malformed region [%d,%d)x[%d,%d)x[%d,%d)x[%d,%d)", r->layer_begin,
                r->layer_end, r->req_begin, r->req_end, r->pos_begin, r->pos_end, r->head_begin,
                r->head_end);
  return DV_OK;
}

bool region_empty(const dv_region* r) {
  return r->layer_end == r->layer_begin || r->req_end == r->req_begin ||
         r->pos_end == r->pos_begin || (!all_heads(r) && r->head_end == r->head_begin);
}

dv_region resolve_heads(const dv_region* r, const dv_cache* c) {
  dv_region x = *r;
  if (all_heads(r)) {
    x.head_begin = c->head_begin;
    x.head_end = c->head_begin + c->n_heads;
  }
  return x;
}

dv_status check_cache(const dv_cache* c, const char* name) {
  if (!c) return fail(DV_EINVAL, "%s: NULL cache", name);
  if (!c->k || !c->v) return fail(DV_EINVAL, "%s: NULL k or v base", name);
  if (c->layout != DV_LAYOUT_KV5D && c->layout != DV_LAYOUT_FT6D)
    return fail(DV_ENOTSUP, "%s: unknown layout %d", name, c->layout);
  if (c->elem_bytes != 1 && c->elem_bytes != 2 && c->elem_bytes != 4 && c->elem_bytes != 8)
    return fail(DV_EINVAL, "%s: elem_bytes %d not in {1,2,4,8}", name, c->elem_bytes);
  if (c->n_layers < 0 || c->n_reqs < 0 || c->n_heads < 1 || c->max_seq < 1 || c->head_dim < 1 ||
      c->layer_begin < 0 || c->req_begin < 0 || c->head_begin < 0)
    return fail(DV_EINVAL, "%s: bad extents", name);
  if (((uint64_t)c->head_dim * c->elem_bytes) % 16)
    return fail(DV_EALIGN, "%s: head_dim*elem_bytes = %d is not a multiple of 16", name,
                c->head_dim * c->elem_bytes);
  if (((uintptr_t)c->k | (uintptr_t)c->v) % 16)
    return fail(DV_EALIGN, "%s: k/v base not 16-byte aligned", name);
  return DV_OK;
}

dv_status check_cache_holds(const dv_cache* c, const dv_region* r0, const char* name) {
  const dv_region rr = resolve_heads(r0, c);
  const dv_region* r = &rr;
  if (region_empty(r)) {
    if (r->pos_end > c->max_seq)
      return fail(DV_ERANGE, "pos_end %d exceeds %s max_seq %d", r->pos_end, name, c->max_seq);
    return DV_OK;
  }
  if (r->layer_begin < c->layer_begin || r->layer_end > c->layer_begin + c->n_layers)
    return fail(DV_EMAP, "%s cache holds layers [%d,%d), region needs [%d,%d)", name,
                c->layer_begin, c->layer_begin + c->n_layers, r->layer_begin, r->layer_end);
  if (r->req_begin < c->req_begin || r->req_end > c->req_begin + c->n_reqs)
    return fail(DV_EMAP, "%s cache holds requests [%d,%d), region needs [%d,%d)", name,
                c->req_begin, c->req_begin + c->n_reqs, r->req_begin, r->req_end);
  if (r->head_begin < c->head_begin || r->head_end > c->head_begin + c->n_heads)
    return fail(DV_EMAP, "%s cache holds heads [%d,%d), region needs [%d,%d)", name,
                c->head_begin, c->head_begin + c->n_heads, r->head_begin, r->head_end);
  if (r->pos_end > c->max_seq)
    return fail(DV_ERANGE, "pos_end %d exceeds %s max_seq %d", r->pos_end, name, c->max_seq);
  return DV_OK;
}

// Bytes of a region whose head range is explicit (or `H` heads when it is "all heads").
uint64_t region_bytes_h(const dv_region* r, int32_t H, int32_t D, int32_t e) {
  const uint64_t nh = all_heads(r) ? (uint64_t)H : (uint64_t)(r->head_end - r->head_begin);
  return 2ull * (uint64_t)(r->layer_end - r->layer_begin) * (uint64_t)(r->req_end - r->req_begin) *
         (uint64_t)(r->pos_end - r->pos_begin) * nh * (uint64_t)D * (uint64_t)e;
}

dv_status route(const dv_setup* src, const dv_setup* dst, const dv_region* r0, int32_t H,
                int32_t D, int32_t e, std::vector<dv_piece>* out) {
  out->clear();
  DV_TRY(check_setup(src, "source setup"));
  DV_TRY(check_setup(dst, "destination setup"));
  DV_TRY(check_region_shape(r0));
  if (H < 1 || D < 1 || e < 1) return fail(DV_EINVAL, "n_heads/head_dim/elem_bytes must be >= 1");
  if ((src->n_tp > 0) != (dst->n_tp > 0))
    return fail(DV_EINVAL, "both setups or neither must split heads");
  const bool tp = src->n_tp > 0;
  dv_region rr = *r0;
  if (tp && all_heads(&rr)) {
    rr.head_begin = src->head_bounds[0];
    rr.head_end = src->head_bounds[src->n_tp];
  }
  const dv_region* r = &rr;
  if (region_empty(r)) return DV_OK;
  const dv_setup* sides[2] = {src, dst};
  const char* names[2] = {"source", "destination"};
  for (int k = 0; k < 2; ++k) {
    const dv_setup* s = sides[k];
    if (r->layer_begin < s->layer_bounds[0] || r->layer_end > s->layer_bounds[s->n_stages])
      return fail(DV_EMAP, "%s setup holds layers [%d,%d), region needs [%d,%d)", names[k],
                  s->layer_bounds[0], s->layer_bounds[s->n_stages], r->layer_begin, r->layer_end);
    if (r->req_begin < s->req_bounds[0] || r->req_end > s->req_bounds[s->n_micro])
      return fail(DV_EMAP, "%s setup holds requests [%d,%d), region needs [%d,%d)", names[k],
                  s->req_bounds[0], s->req_bounds[s->n_micro], r->req_begin, r->req_end);
    if (tp && (r->head_begin < s->head_bounds[0] || r->head_end > s->head_bounds[s->n_tp]))
      return fail(DV_EMAP, "%s setup holds heads [%d,%d), region needs [%d,%d)", names[k],
                  s->head_bounds[0], s->head_bounds[s->n_tp], r->head_begin, r->head_end);
  }
  for (int k = 0; k < 2; ++k)
    if (r->pos_end > sides[k]->max_seq)
      return fail(DV_ERANGE, "pos_end %d exceeds %s max_seq %d", r->pos_end, names[k],
                  sides[k]->max_seq);

  // Block ranges that intersect the region on each side (bounds are sorted, so the blocks
  // overlapping [a,b) form one contiguous index range; found by binary search).
  auto span = [](const int32_t* b, int n, int32_t lo, int32_t hi, int* first, int* last) {
    *first = int(std::upper_bound(b, b + n + 1, lo) - b) - 1;
    *last = int(std::lower_bound(b, b + n + 1, hi) - b);  // exclusive
    if (*first < 0) *first = 0;
    if (*last > n) *last = n;
  };
  int si0, si1, su0, su1, dj0, dj1, dw0, dw1, st0 = 0, st1 = 1, dt0 = 0, dt1 = 1;
  span(src->layer_bounds, src->n_stages, r->layer_begin, r->layer_end, &si0, &si1);
  span(src->req_bounds, src->n_micro, r->req_begin, r->req_end, &su0, &su1);
  span(dst->layer_bounds, dst->n_stages, r->layer_begin, r->layer_end, &dj0, &dj1);
  span(dst->req_bounds, dst->n_micro, r->req_begin, r->req_end, &dw0, &dw1);
  if (tp) {
    span(src->head_bounds, src->n_tp, r->head_begin, r->head_end, &st0, &st1);
    span(dst->head_bounds, dst->n_tp, r->head_begin, r->head_end, &dt0, &dt1);
  }
  for (int i = si0; i < si1; ++i)
    for (int u = su0; u < su1; ++u)
      for (int t = st0; t < st1; ++t)
        for (int j = dj0; j < dj1; ++j)
          for (int w = dw0; w < dw1; ++w)
            for (int v = dt0; v < dt1; ++v) {
              int32_t a = std::max({r->layer_begin, src->layer_bounds[i], dst->layer_bounds[j]});
              int32_t b = std::min({r->layer_end, src->layer_bounds[i + 1], dst->layer_bounds[j + 1]});
              int32_t c = std::max({r->req_begin, src->req_bounds[u], dst->req_bounds[w]});
              int32_t d = std::min({r->req_end, src->req_bounds[u + 1], dst->req_bounds[w + 1]});
              int32_t hb = r->head_begin, he = r->head_end;
              if (tp) {
                hb = std::max({hb, src->head_bounds[t], dst->head_bounds[v]});
                he = std::min({he, src->head_bounds[t + 1], dst->head_bounds[v + 1]});
                if (hb >= he) continue;
              }
              if (a >= b || c >= d) continue;
              dv_piece p{};
              p.src_stage = i;
              p.src_micro = u;
              p.src_tp = t;
              p.dst_stage = j;
              p.dst_micro = w;
              p.dst_tp = v;
              p.layer_begin = a;
              p.layer_end = b;
              p.req_begin = c;
              p.req_end = d;
              p.pos_begin = r->pos_begin;
              p.pos_end = r->pos_end;
              p.head_begin = hb;
              p.head_end = he;
              dv_region pr{a, b, c, d, r->pos_begin, r->pos_end, hb, he};
              p.bytes = region_bytes_h(&pr, H, D, e);
              out->push_back(p);
            }
  // Wire offsets: cumulative per source block and per destination block, in piece order.
  const int stp = std::max(src->n_tp, 1), dtp = std::max(dst->n_tp, 1);
  std::vector<uint64_t> src_acc((size_t)src->n_stages * src->n_micro * stp, 0);
  std::vector<uint64_t> dst_acc((size_t)dst->n_stages * dst->n_micro * dtp, 0);
  for (auto& p : *out) {
    uint64_t& sa = src_acc[((size_t)p.src_stage * src->n_micro + p.src_micro) * stp + p.src_tp];
    uint64_t& da = dst_acc[((size_t)p.dst_stage * dst->n_micro + p.dst_micro) * dtp + p.dst_tp];
    p.src_wire_off = sa;
    sa += p.bytes;
    p.dst_wire_off = da;
    da += p.bytes;
  }
  return DV_OK;
}

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;          // ceil(log2 d)
  uint64_t p = 31 + l;
  f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
  f.shr = (uint32_t)(p - 32);
  return f;
}

void collapse(CopyPlan& p) {
  // 1) fold innermost dims into the run while both sides are contiguous across them
  for (int k = kDims - 1; k >= 0; --k) {
    if (p.n[k] == 1) continue;
    if (p.ss[k] == (int64_t)p.run_bytes && p.ds[k] == (int64_t)p.run_bytes) {
      p.run_bytes *= p.n[k];
      p.n[k] = 1;
      p.ss[k] = p.ds[k] = 0;
    } else {
      break;
    }
  }
  // 2) drop unit dims, keep order; then merge adjacent dims (outer j, inner i) when
  //    stride_j == n_i * stride_i on both sides
  uint32_t n[kDims];
  int64_t ss[kDims], ds[kDims];
  int m = 0;
  for (int k = 0; k < kDims; ++k)
    if (p.n[k] != 1) {
      n[m] = p.n[k];
      ss[m] = p.ss[k];
      ds[m] = p.ds[k];
      ++m;
    }
  int w = 0;
  for (int k = 0; k < m; ++k) {
    if (w > 0 && ss[w - 1] == (int64_t)n[k] * ss[k] && ds[w - 1] == (int64_t)n[k] * ds[k] &&
        (uint64_t)n[w - 1] * n[k] < (1ull << 31)) {
      n[w - 1] *= n[k];
      ss[w - 1] = ss[k];
      ds[w - 1] = ds[k];
    } else {
      n[w] = n[k];
      ss[w] = ss[k];
      ds[w] = ds[k];
      ++w;
    }
  }
  // right-align into kDims slots (outer padding with unit dims)
  for (int k = 0; k < kDims; ++k) {
    int src_k = k - (kDims - w);
    if (src_k < 0) {
      p.n[k] = 1;
      p.ss[k] = p.ds[k] = 0;
    } else {
      p.n[k] = n[src_k];
      p.ss[k] = ss[src_k];
      p.ds[k] = ds[src_k];
    }
  }
}

}  // namespace dv

extern "C" {

const char* dv_last_error(void) { return dv::g_err.c_str(); }

const char* dv_status_str(dv_status s) {
  switch (s) {
    case DV_OK: return "DV_OK";
    case DV_EINVAL: return "DV_EINVAL";
    case DV_EMAP: return "DV_EMAP";
    case DV_ERANGE: return "DV_ERANGE";
    case DV_EALIGN: return "DV_EALIGN";
    case DV_ENOMEM: return "DV_ENOMEM";
    case DV_EPEER: return "DV_EPEER";
    case DV_EBUSY: return "DV_EBUSY";
    case DV_ECUDA: return "DV_ECUDA";
    case DV_ENOTSUP: return "DV_ENOTSUP";
  }
  return "DV_?";
}

int32_t dv_abi_version(void) { return DV_ABI_VERSION; }

dv_status dv_region_bytes(const dv_region* region, int32_t n_heads, int32_t head_dim,
                          int32_t elem_bytes, uint64_t* out_bytes) {
  DV_TRY(dv::check_region_shape(region));
  if (!out_bytes) return dv::fail(DV_EINVAL, "NULL out_bytes");
  if (n_heads < 1 || head_dim < 1 || elem_bytes < 1)
    return dv::fail(DV_EINVAL, "n_heads/head_dim/elem_bytes must be >= 1");
  *out_bytes = dv::region_bytes_h(region, n_heads, head_dim, elem_bytes);
  return DV_OK;
}

dv_status dv_route(const dv_setup* src, const dv_setup* dst, const dv_region* region,
                   int32_t n_heads, int32_t head_dim, int32_t elem_bytes, dv_piece* out,
                   uint64_t cap, uint64_t* n) {
  if (!n) return dv::fail(DV_EINVAL, "NULL count pointer");
  std::vector<dv_piece> ps;
  DV_TRY(dv::route(src, dst, region, n_heads, head_dim, elem_bytes, &ps));
  *n = ps.size();
  if (cap && !out) return dv::fail(DV_EINVAL, "NULL out with cap > 0");
  for (uint64_t k = 0; k < std::min<uint64_t>(cap, ps.size()); ++k) out[k] = ps[k];
  return DV_OK;
}

}  // extern "C"
