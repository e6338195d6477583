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

static PyMethodDef methods[] = {
    {"send", (PyCFunction)(void (*)(void))fast_send, METH_FASTCALL,
     "mp_send with integer arguments; returns the MP_* status"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_mpfast", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__mpfast(void) { return PyModule_Create(&module); }
