/* host_submit.c — CPython fast path for the pipelined host submission.
 *
 * One async batch through the public API costs two copies, one graph launch
 * and one event record in the driver (≈4 µs of host time), but through ctypes
 * another 3–5 µs went to argument conversion and numpy's __array_interface__
 * dict (tools/e2e_probe.py).  On a box whose copies take ≈11.5 µs per batch
 * (tools/submit_probe.cu) that made the e2e loop host-bound on slower host
 * CPUs.  This module calls lcp_query_host_packed_async (include/lcp_b200.h)
 * directly: the queries' address comes from the buffer protocol, the function
 * address from the loaded C-ABI library (no link-time dependency on it), and
 * the GIL is released around the call so serving threads overlap.
 * submit_wait() adds the wait (the single-query API's whole round trip).
 *
 * Built in-tree by _build.py (gcc, Python headers); _native.py uses ctypes
 * when the module is absent, so this is a speed path, never a semantic one.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*submit_fn)(const void* index, void* ws, const uint16_t* queries, int32_t count,
                         int32_t k, int32_t mode, int32_t out_stride, void* out_block,
                         int32_t flags);

typedef int (*wait_fn)(void* ws);
typedef int (*server_fn)(void* server, const uint16_t* row);

static submit_fn g_submit = NULL;
static wait_fn g_wait = NULL;
static server_fn g_server = NULL;

/* bind(addresses of lcp_query_host_packed_async, lcp_workspace_wait,
 *      lcp_server_query_row) */
static PyObject* bind(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 3) {
    PyErr_SetString(PyExc_TypeError, "bind() takes 3 arguments");
    return NULL;
  }
  void* s = PyLong_AsVoidPtr(args[0]);
  void* w = PyLong_AsVoidPtr(args[1]);
  void* q = PyLong_AsVoidPtr(args[2]);
  if (PyErr_Occurred()) return NULL;
  g_submit = (submit_fn)s;
  g_wait = (wait_fn)w;
  g_server = (server_fn)q;
  Py_RETURN_NONE;
}

/* server_query(server, row) -> rc: one latency-mode query (lcp_server_query_row)
 * with the row taken through the buffer protocol (1-D, 2-byte items) */
static PyObject* server_query(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 2) {
    PyErr_SetString(PyExc_TypeError, "server_query() takes 2 arguments");
    return NULL;
  }
  if (!g_server) {
    PyErr_SetString(PyExc_RuntimeError, "server_query(): bind() the C-ABI entry points first");
    return NULL;
  }
  void* srv = PyLong_AsVoidPtr(args[0]);
  if (PyErr_Occurred()) return NULL;
  Py_buffer v;
  if (PyObject_GetBuffer(args[1], &v, PyBUF_C_CONTIGUOUS | PyBUF_ND) < 0) return NULL;
  if (v.ndim != 1 || v.itemsize != 2) {
    PyBuffer_Release(&v);
    PyErr_SetString(PyExc_ValueError, "the query must be a C-contiguous 1-D 2-byte array");
    return NULL;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = g_server(srv, (const uint16_t*)v.buf);
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&v);
  return PyLong_FromLong(rc);
}

/* submit(index, ws, queries, length, k, mode, out_stride, out_block, flags) -> rc
 * queries: C-contiguous 2-D buffer of 2-byte items with `length` columns.
 * With `wait`, the workspace's batch is also waited for (one round trip). */
static PyObject* submit_impl(PyObject* const* args, Py_ssize_t nargs, int wait) {
  if (nargs != 9) {
    PyErr_SetString(PyExc_TypeError, "submit() takes 9 arguments");
    return NULL;
  }
  if (!g_submit || !g_wait) {
    PyErr_SetString(PyExc_RuntimeError, "submit(): bind() the C-ABI entry point first");
    return NULL;
  }
  void* ix = PyLong_AsVoidPtr(args[0]);
  void* ws = PyLong_AsVoidPtr(args[1]);
  const long length = PyLong_AsLong(args[3]);
  const long k = PyLong_AsLong(args[4]);
  const long mode = PyLong_AsLong(args[5]);
  const long stride = PyLong_AsLong(args[6]);
  void* out = PyLong_AsVoidPtr(args[7]);
  const long flags = PyLong_AsLong(args[8]);
  if (PyErr_Occurred()) return NULL;
  Py_buffer v;
  if (PyObject_GetBuffer(args[2], &v, PyBUF_C_CONTIGUOUS | PyBUF_ND) < 0) return NULL;
  if (v.ndim != 2 || v.itemsize != 2 || v.shape[1] != length || v.shape[0] > INT32_MAX) {
    PyBuffer_Release(&v);
    PyErr_SetString(PyExc_ValueError, "queries must be a C-contiguous (count, L) 2-byte array");
    return NULL;
  }
  const int32_t count = (int32_t)v.shape[0];
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = g_submit(ix, ws, (const uint16_t*)v.buf, count, (int32_t)k, (int32_t)mode, (int32_t)stride, out,
                (int32_t)flags);
  if (rc == 0 && wait) rc = g_wait(ws);
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&v);
  return PyLong_FromLong(rc);
}

static PyObject* submit(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  return submit_impl(args, nargs, 0);
}

static PyObject* submit_wait(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  return submit_impl(args, nargs, 1);
}

static PyMethodDef methods[] = {
    {"bind", (PyCFunction)(void (*)(void))bind, METH_FASTCALL,
     "bind(addresses of lcp_query_host_packed_async, lcp_workspace_wait, lcp_server_query_row)"},
    {"server_query", (PyCFunction)(void (*)(void))server_query, METH_FASTCALL,
     "server_query(server, row) -> rc (lcp_server_query_row)"},
    {"submit", (PyCFunction)(void (*)(void))submit, METH_FASTCALL,
     "submit(index, ws, queries, length, k, mode, out_stride, out_block, flags) -> rc"},
    {"submit_wait", (PyCFunction)(void (*)(void))submit_wait, METH_FASTCALL,
     "submit_wait(...): submit, then lcp_workspace_wait(ws) -> rc"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_lcp_host", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__lcp_host(void) { return PyModule_Create(&module); }
