/* _dvfast: a CPython fast path for the per-call entry points of include/dv.h (argument
 * marshalling only -- every call goes straight to libdvstream). The Python binding
 * (paper_2403_01876_b200/__init__.py) keeps its ctypes structures; it passes their ADDRESSES and
 * plain integers here, so a call costs one METH_FASTCALL dispatch instead of a ctypes foreign
 * call with per-argument conversion. Each function returns the dv_status; the binding raises on
 * a non-zero status with dv_last_error(). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "../../include/dv.h"

static int get_ptr(PyObject* o, void** out) {
  if (o == Py_None) {
    *out = NULL;
    return 0;
  }
  *out = PyLong_AsVoidPtr(o);
  return (*out == NULL && PyErr_Occurred()) ? -1 : 0;
}
static int get_u64(PyObject* o, uint64_t* out) {
  *out = (uint64_t)PyLong_AsUnsignedLongLongMask(o);
  return PyErr_Occurred() ? -1 : 0;
}
static int get_i32(PyObject* o, int32_t* out) {
  const long v = PyLong_AsLong(o);
  if (v == -1 && PyErr_Occurred()) return -1;
  *out = (int32_t)v;
  return 0;
}

/* A region is either the address of a dv_region or a tuple (layer_begin, layer_end, req_begin,
 * req_end, pos_begin, pos_end[, head_begin, head_end]) -- the tuple form skips building a ctypes
 * structure per call. */
static int get_region(PyObject* o, dv_region* tmp, void** out) {
  if (!PyTuple_Check(o)) return get_ptr(o, out);
  const Py_ssize_t n = PyTuple_GET_SIZE(o);
  if (n != 6 && n != 8) {
    PyErr_SetString(PyExc_ValueError, "region tuple needs 6 or 8 entries");
    return -1;
  }
  int32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (Py_ssize_t i = 0; i < n; ++i)
    if (get_i32(PyTuple_GET_ITEM(o, i), &v[i])) return -1;
  tmp->layer_begin = v[0];
  tmp->layer_end = v[1];
  tmp->req_begin = v[2];
  tmp->req_end = v[3];
  tmp->pos_begin = v[4];
  tmp->pos_end = v[5];
  tmp->head_begin = v[6];
  tmp->head_end = v[7];
  *out = tmp;
  return 0;
}

#define NARGS(n)                                                              \
  if (nargs != (n)) {                                                         \
    PyErr_Format(PyExc_TypeError, "expected %d arguments, got %zd", (n), nargs); \
    return NULL;                                                              \
  }

/* scatter(ctx, src_cache*, region*, dst_ep*, dst_off, flag_slot, seq, xfer, stream) */
static PyObject* f_scatter(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(9);
  void *ctx, *src, *reg, *dst, *st;
  dv_region rt;
  uint64_t off, seq, xfer;
  int32_t slot;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &src) || get_region(a[2], &rt, &reg) || get_ptr(a[3], &dst) ||
      get_u64(a[4], &off) || get_i32(a[5], &slot) || get_u64(a[6], &seq) || get_u64(a[7], &xfer) ||
      get_ptr(a[8], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_scatter((dv_ctx*)ctx, (const dv_cache*)src, (const dv_region*)reg, (const dv_endpoint*)dst,
                 off, slot, seq, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* gather(ctx, src_ep*, src_off, flag_slot, wait_seq, dst_cache*, region*, xfer, stream) */
static PyObject* f_gather(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(9);
  void *ctx, *src, *dst, *reg, *st;
  dv_region rt;
  uint64_t off, seq, xfer;
  int32_t slot;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &src) || get_u64(a[2], &off) || get_i32(a[3], &slot) ||
      get_u64(a[4], &seq) || get_ptr(a[5], &dst) || get_region(a[6], &rt, &reg) || get_u64(a[7], &xfer) ||
      get_ptr(a[8], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_gather((dv_ctx*)ctx, (const dv_endpoint*)src, off, slot, seq, (const dv_cache*)dst,
                (const dv_region*)reg, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* remap(ctx, src_cache*, dst_cache*, region*, signal_ep* or None, flag_slot, seq, xfer, stream) */
static PyObject* f_remap(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(9);
  void *ctx, *src, *dst, *reg, *sig, *st;
  dv_region rt;
  uint64_t seq, xfer;
  int32_t slot;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &src) || get_ptr(a[2], &dst) || get_region(a[3], &rt, &reg) ||
      get_ptr(a[4], &sig) || get_i32(a[5], &slot) || get_u64(a[6], &seq) || get_u64(a[7], &xfer) ||
      get_ptr(a[8], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_remap((dv_ctx*)ctx, (const dv_cache*)src, (const dv_cache*)dst, (const dv_region*)reg,
               (const dv_endpoint*)sig, slot, seq, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* stream_out_direct(ctx, src*, region*, src_setup*, my_stage, my_micro, my_tp, dst_setup*,
 *                   dst_caches*, signals* or None, n_dst, seq, xfer, stream) */
static PyObject* f_stream_out_direct(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(14);
  void *ctx, *src, *reg, *ss, *ds, *dc, *sig, *st;
  dv_region rt;
  int32_t stage, micro, tp, n;
  uint64_t seq, xfer;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &src) || get_region(a[2], &rt, &reg) || get_ptr(a[3], &ss) ||
      get_i32(a[4], &stage) || get_i32(a[5], &micro) || get_i32(a[6], &tp) || get_ptr(a[7], &ds) ||
      get_ptr(a[8], &dc) || get_ptr(a[9], &sig) || get_i32(a[10], &n) || get_u64(a[11], &seq) ||
      get_u64(a[12], &xfer) || get_ptr(a[13], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_stream_out_direct((dv_ctx*)ctx, (const dv_cache*)src, (const dv_region*)reg,
                           (const dv_setup*)ss, stage, micro, tp, (const dv_setup*)ds,
                           (const dv_cache*)dc, (const dv_endpoint*)sig, n, seq, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* stream_out(ctx, src*, region*, src_setup*, my_stage, my_micro, my_tp, dst_setup*, inboxes*,
 *            n_inboxes, seq, xfer, stream) */
static PyObject* f_stream_out(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(13);
  void *ctx, *src, *reg, *ss, *ds, *ib, *st;
  dv_region rt;
  int32_t stage, micro, tp, n;
  uint64_t seq, xfer;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &src) || get_region(a[2], &rt, &reg) || get_ptr(a[3], &ss) ||
      get_i32(a[4], &stage) || get_i32(a[5], &micro) || get_i32(a[6], &tp) || get_ptr(a[7], &ds) ||
      get_ptr(a[8], &ib) || get_i32(a[9], &n) || get_u64(a[10], &seq) || get_u64(a[11], &xfer) ||
      get_ptr(a[12], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_stream_out((dv_ctx*)ctx, (const dv_cache*)src, (const dv_region*)reg, (const dv_setup*)ss, stage,
                    micro, tp, (const dv_setup*)ds, (const dv_endpoint*)ib, n, seq, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* stream_in(ctx, dst*, region*, src_setup*, dst_setup*, my_stage, my_micro, my_tp, inbox*, wait_seq,
 *           xfer, stream) */
static PyObject* f_stream_in(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  NARGS(12);
  void *ctx, *dst, *reg, *ss, *ds, *ib, *st;
  dv_region rt;
  int32_t stage, micro, tp;
  uint64_t seq, xfer;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &dst) || get_region(a[2], &rt, &reg) || get_ptr(a[3], &ss) ||
      get_ptr(a[4], &ds) || get_i32(a[5], &stage) || get_i32(a[6], &micro) || get_i32(a[7], &tp) ||
      get_ptr(a[8], &ib) || get_u64(a[9], &seq) || get_u64(a[10], &xfer) || get_ptr(a[11], &st))
    return NULL;
  dv_status s;
  Py_BEGIN_ALLOW_THREADS
  s = dv_stream_in((dv_ctx*)ctx, (const dv_cache*)dst, (const dv_region*)reg, (const dv_setup*)ss,
                   (const dv_setup*)ds, stage, micro, tp, (const dv_endpoint*)ib, seq, (uint32_t)xfer, st);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(s);
}

/* wait(ctx, ep*, flag_slot, seq, stream) and signal(...) */
static PyObject* f_wait_signal(PyObject* const* a, Py_ssize_t nargs, int signal) {
  NARGS(5);
  void *ctx, *ep, *st;
  int32_t slot;
  uint64_t seq;
  if (get_ptr(a[0], &ctx) || get_ptr(a[1], &ep) || get_i32(a[2], &slot) || get_u64(a[3], &seq) ||
      get_ptr(a[4], &st))
    return NULL;
  dv_status s = signal ? dv_signal((dv_ctx*)ctx, (const dv_endpoint*)ep, slot, seq, st)
                       : dv_wait((dv_ctx*)ctx, (const dv_endpoint*)ep, slot, seq, st);
  return PyLong_FromLong(s);
}
static PyObject* f_wait(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  return f_wait_signal(a, nargs, 0);
}
static PyObject* f_signal(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  return f_wait_signal(a, nargs, 1);
}

static PyMethodDef methods[] = {
    {"scatter", (PyCFunction)(void (*)(void))f_scatter, METH_FASTCALL, "dv_scatter"},
    {"gather", (PyCFunction)(void (*)(void))f_gather, METH_FASTCALL, "dv_gather"},
    {"remap", (PyCFunction)(void (*)(void))f_remap, METH_FASTCALL, "dv_remap"},
    {"stream_out_direct", (PyCFunction)(void (*)(void))f_stream_out_direct, METH_FASTCALL,
     "dv_stream_out_direct"},
    {"stream_out", (PyCFunction)(void (*)(void))f_stream_out, METH_FASTCALL, "dv_stream_out"},
    {"stream_in", (PyCFunction)(void (*)(void))f_stream_in, METH_FASTCALL, "dv_stream_in"},
    {"wait", (PyCFunction)(void (*)(void))f_wait, METH_FASTCALL, "dv_wait"},
    {"signal", (PyCFunction)(void (*)(void))f_signal, METH_FASTCALL, "dv_signal"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_dvfast",
                                    "CPython fast path of the dvstream per-call entry points", -1,
                                    methods};

PyMODINIT_FUNC PyInit__dvfast(void) { return PyModule_Create(&module); }
