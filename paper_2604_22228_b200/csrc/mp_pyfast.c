/* mp_pyfast.c — CPython fast path for the per-message call of the Python
 * API: `send(ctx, src, dst, size, src_dev, dst_dev, cfg, stream) -> status`
 * with plain integers (pointers as ints), calling mp_send (include/mpb200.h)
 * directly.  A ctypes call with eight converted arguments costs ~1.5 us, more
 * than a cached-graph launch; this METH_FASTCALL entry costs ~0.1 us.  The GIL
 * is released around mp_send (a launch may block on a full launch queue).
 * Errors keep the C ABI contract: the status is returned and the message is
 * read with mp_last_error() on the same thread (engine.py re-raises). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stddef.h>

#include "mpb200.h"

static PyObject* fast_send(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 8) {
    PyErr_SetString(PyExc_TypeError, "send(ctx, src, dst, size, src_dev, dst_dev, cfg, stream)");
    return NULL;
  }
  mp_ctx* ctx = (mp_ctx*)PyLong_AsVoidPtr(args[0]);
  const void* src = PyLong_AsVoidPtr(args[1]);
  void* dst = PyLong_AsVoidPtr(args[2]);
  unsigned long long size = PyLong_AsUnsignedLongLong(args[3]);
  long sd = PyLong_AsLong(args[4]);
  long dd = PyLong_AsLong(args[5]);
  const mp_config* cfg = (const mp_config*)PyLong_AsVoidPtr(args[6]);
  void* stream = PyLong_AsVoidPtr(args[7]);
  if (PyErr_Occurred()) return NULL;
  if (sd < INT32_MIN || sd > INT32_MAX || dd < INT32_MIN || dd > INT32_MAX) {
    PyErr_SetString(PyExc_OverflowError, "device index out of range");
    return NULL;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = mp_send(ctx, src, dst, (uint64_t)size, (int32_t)sd, (int32_t)dd, cfg, stream);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

/* A send bound once to its arguments (Engine.prepare): calling the object
 * replays it — one mp_send, no argument conversion at all. */
typedef struct {
  PyObject_HEAD
  mp_ctx* ctx;
  const void* src;
  void* dst;
  uint64_t size;
  int32_t sd, dd;
  const mp_config* cfg;
  void* stream;
  PyObject* keep;     /* objects that must outlive the binding (tensors, config, stream) */
  PyObject* on_error; /* on_error(rc) raises the mapped exception; NULL: return rc */
  PyObject* weaklist; /* Engine keeps weak references to invalidate on close() */
} BoundSend;

static void bound_dealloc(BoundSend* self) {
  if (self->weaklist) PyObject_ClearWeakRefs((PyObject*)self);
  Py_XDECREF(self->keep);
  Py_XDECREF(self->on_error);
  Py_TYPE(self)->tp_free((PyObject*)self);
}

/* Success returns None with no Python-level work at all; a failure (or a
 * binding invalidated by Engine.close(): rc = -1000, the context is never
 * touched) goes to on_error, which maps the status to the reference's
 * exception classes.  Without on_error the status is returned. */
static PyObject* bound_call(BoundSend* self, PyObject* args, PyObject* kw) {
  (void)args;
  (void)kw;
  int rc = -1000;
  if (self->ctx) {
    Py_BEGIN_ALLOW_THREADS
    rc = mp_send(self->ctx, self->src, self->dst, self->size, self->sd, self->dd, self->cfg,
                 self->stream);
    Py_END_ALLOW_THREADS
  }
  if (!self->on_error) return PyLong_FromLong(rc);
  if (rc == 0) Py_RETURN_NONE;
  return PyObject_CallFunction(self->on_error, "i", rc);
}

static PyObject* bound_invalidate(BoundSend* self, PyObject* unused) {
  (void)unused;
  self->ctx = NULL;
  Py_RETURN_NONE;
}

static PyMethodDef bound_methods[] = {
    {"invalidate", (PyCFunction)bound_invalidate, METH_NOARGS,
     "forget the context (Engine.close): later calls fail without touching it"},
    {NULL, NULL, 0, NULL},
};

static PyTypeObject BoundSendType = {
    PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_mpfast.BoundSend",
    .tp_basicsize = sizeof(BoundSend),
    .tp_dealloc = (destructor)bound_dealloc,
    .tp_call = (ternaryfunc)bound_call,
    .tp_methods = bound_methods,
    .tp_weaklistoffset = offsetof(BoundSend, weaklist),
    .tp_flags = Py_TPFLAGS_DEFAULT,
    .tp_doc = "a send bound to its arguments; call() -> MP_* status",
};

static PyObject* fast_bind(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 9 && nargs != 10) {
    PyErr_SetString(PyExc_TypeError,
                    "bind(ctx, src, dst, size, src_dev, dst_dev, cfg, stream, keep[, on_error])");
    return NULL;
  }
  BoundSend* b = PyObject_New(BoundSend, &BoundSendType);
  if (!b) return NULL;
  b->keep = NULL;
  b->on_error = NULL;
  b->weaklist = NULL;
  b->ctx = (mp_ctx*)PyLong_AsVoidPtr(args[0]);
  b->src = PyLong_AsVoidPtr(args[1]);
  b->dst = PyLong_AsVoidPtr(args[2]);
  b->size = (uint64_t)PyLong_AsUnsignedLongLong(args[3]);
  long sd = PyLong_AsLong(args[4]), dd = PyLong_AsLong(args[5]);
  b->cfg = (const mp_config*)PyLong_AsVoidPtr(args[6]);
  b->stream = PyLong_AsVoidPtr(args[7]);
  if (PyErr_Occurred() || sd < INT32_MIN || sd > INT32_MAX || dd < INT32_MIN || dd > INT32_MAX) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_OverflowError, "device index out of range");
    Py_DECREF(b);
    return NULL;
  }
  b->sd = (int32_t)sd;
  b->dd = (int32_t)dd;
  Py_INCREF(args[8]);
  b->keep = args[8];
  if (nargs == 10 && args[9] != Py_None) {
    Py_INCREF(args[9]);
    b->on_error = args[9];
  }
  return (PyObject*)b;
}

/* mp_send_many over a caller-owned mp_xfer array (Engine.prepare_many keeps
 * the array and config alive): send_many(ctx, xfers, n, cfg, joint, stream). */
static PyObject* fast_send_many(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "send_many(ctx, xfers, n, cfg, joint, stream)");
    return NULL;
  }
  mp_ctx* ctx = (mp_ctx*)PyLong_AsVoidPtr(args[0]);
  const mp_xfer* xs = (const mp_xfer*)PyLong_AsVoidPtr(args[1]);
  long n = PyLong_AsLong(args[2]);
  const mp_config* cfg = (const mp_config*)PyLong_AsVoidPtr(args[3]);
  long joint = PyLong_AsLong(args[4]);
  void* stream = PyLong_AsVoidPtr(args[5]);
  if (PyErr_Occurred()) return NULL;
  if (n < INT32_MIN || n > INT32_MAX) {
    PyErr_SetString(PyExc_OverflowError, "transfer count out of range");
    return NULL;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = mp_send_many(ctx, xs, (int32_t)n, cfg, joint ? 1 : 0, stream);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"send_many", (PyCFunction)(void (*)(void))fast_send_many, METH_FASTCALL,
     "mp_send_many over an mp_xfer array address; returns the MP_* status"},
    {"send", (PyCFunction)(void (*)(void))fast_send, METH_FASTCALL,
     "mp_send with integer arguments; returns the MP_* status"},
    {"bind", (PyCFunction)(void (*)(void))fast_bind, METH_FASTCALL,
     "bind(ctx, src, dst, size, src_dev, dst_dev, cfg, stream, keep) -> BoundSend"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_mpfast", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__mpfast(void) {
  if (PyType_Ready(&BoundSendType) < 0) return NULL;
  return PyModule_Create(&module);
}
