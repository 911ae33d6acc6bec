/* K9 host side: native packing of StepSequence lists into the CSR layout.
 *
 * Replaces the per-chunk padding of the reference (tuner.py:36-52 _pack,
 * features.py:70-92 StepSequence) for the device path.  The Python API takes
 * a list of objects with `.steps` (T, d0) and `.context` (C,); numpy's
 * concatenate over 10^5-10^6 small arrays costs ~0.5 us per array, which made
 * packing the largest host cost of `fit` / `predict`.  This module walks the
 * list once (numpy C API: array headers are read directly, no buffer
 * exports), converts to the output dtype while copying, and writes straight
 * into caller-provided (pinned) buffers.
 *
 *   lens = _ttpack.pack(seqs, d0, C, alloc)
 *
 * d0 / C = -1 take the widths of the first item.  alloc(rows, n, d0, C) ->
 * (steps_buf, ctx_buf): writable C-contiguous buffers of rows*d0 and n*C
 * elements, float64 or float32 ndarrays.
 * Returns an int64 `bytes` of per-program step counts, or None when any item
 * is malformed or not a float32/float64 ndarray (wrong rank/width, empty
 * program, lists, integer arrays);
 * the caller then takes its checked per-item path for the exact error.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static PyObject *s_steps, *s_context;

static int float_type(int t) { return t == NPY_DOUBLE || t == NPY_FLOAT; }

/* copy a (rows, cols) strided float array into dense out of type out_t */
static void copy2d(PyArrayObject *a, npy_intp rows, npy_intp cols, char *out, int out_t) {
  const int in_t = PyArray_TYPE(a);
  const npy_intp isz = in_t == NPY_DOUBLE ? 8 : 4;
  const npy_intp *st = PyArray_STRIDES(a);
  const npy_intp rs = PyArray_NDIM(a) > 1 ? st[0] : 0;
  const npy_intp cs = PyArray_NDIM(a) > 1 ? st[1] : st[0];
  const char *src = (const char *)PyArray_DATA(a);
  if (in_t == out_t && cs == isz && (rows == 1 || rs == cols * isz)) {
    memcpy(out, src, (size_t)(rows * cols * isz));
    return;
  }
  for (npy_intp r = 0; r < rows; ++r) {
    const char *row = src + r * rs;
    for (npy_intp c = 0; c < cols; ++c) {
      const char *e = row + c * cs;
      const double v = in_t == NPY_DOUBLE ? *(const double *)e : (double)*(const float *)e;
      if (out_t == NPY_DOUBLE)
        ((double *)out)[r * cols + c] = v;
      else
        ((float *)out)[r * cols + c] = (float)v;
    }
  }
}

static void release(PyObject **held, Py_ssize_t n) {
  for (Py_ssize_t i = 0; i < n; ++i) Py_XDECREF(held[i]);
  free(held);
}

static int out_ok(PyObject *o, npy_intp need) {
  if (!PyArray_Check(o)) return 0;
  PyArrayObject *a = (PyArrayObject *)o;
  return float_type(PyArray_TYPE(a)) && PyArray_IS_C_CONTIGUOUS(a) && PyArray_ISWRITEABLE(a) &&
         PyArray_SIZE(a) >= need;
}

static PyObject *pack(PyObject *self, PyObject *args) {
  (void)self;
  PyObject *seqs, *alloc;
  Py_ssize_t d0, C;
  if (!PyArg_ParseTuple(args, "OnnO", &seqs, &d0, &C, &alloc)) return NULL;
  PyObject *fast = PySequence_Fast(seqs, "seqs must be a sequence");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject **objs = PySequence_Fast_ITEMS(fast);
  if (n == 0) {
    Py_DECREF(fast);
    Py_RETURN_NONE;
  }
  /* held[2i] = steps array, held[2i+1] = context array (owned references) */
  PyObject **held = (PyObject **)calloc((size_t)(2 * n), sizeof(PyObject *));
  PyObject *lens = PyBytes_FromStringAndSize(NULL, n * (Py_ssize_t)sizeof(int64_t));
  if (!held || !lens) {
    free(held);
    Py_XDECREF(lens);
    Py_DECREF(fast);
    return PyErr_NoMemory();
  }
  int64_t *L = (int64_t *)PyBytes_AS_STRING(lens);
  npy_intp rows = 0;
  int bad = 0;
  for (Py_ssize_t i = 0; i < n && !bad; ++i) {
    PyObject *so = held[2 * i] = PyObject_GetAttr(objs[i], s_steps);
    PyObject *co = held[2 * i + 1] = so ? PyObject_GetAttr(objs[i], s_context) : NULL;
    if (!so || !co || !PyArray_Check(so) || !PyArray_Check(co)) {
      bad = 1;
      break;
    }
    PyArrayObject *sa = (PyArrayObject *)so, *ca = (PyArrayObject *)co;
    if (d0 < 0 && PyArray_NDIM(sa) == 2) d0 = PyArray_DIM(sa, 1);
    if (C < 0 && PyArray_NDIM(ca) == 1) C = PyArray_DIM(ca, 0);
    if (PyArray_NDIM(sa) != 2 || PyArray_DIM(sa, 1) != d0 || PyArray_DIM(sa, 0) < 1 ||
        !float_type(PyArray_TYPE(sa)) || PyArray_NDIM(ca) != 1 || PyArray_DIM(ca, 0) != C ||
        !float_type(PyArray_TYPE(ca))) {
      bad = 1;
      break;
    }
    L[i] = PyArray_DIM(sa, 0);
    rows += PyArray_DIM(sa, 0);
  }
  if (bad) {
    /* malformed (or attribute error): the caller's checked path reports it */
    PyErr_Clear();
    release(held, 2 * n);
    Py_DECREF(lens);
    Py_DECREF(fast);
    Py_RETURN_NONE;
  }
  PyObject *bufs = PyObject_CallFunction(alloc, "nnnn", (Py_ssize_t)rows, n, d0, C);
  int ok = 0;
  if (bufs) {
    if (PyTuple_Check(bufs) && PyTuple_GET_SIZE(bufs) == 2 &&
        out_ok(PyTuple_GET_ITEM(bufs, 0), rows * d0) && out_ok(PyTuple_GET_ITEM(bufs, 1), n * C)) {
      PyArrayObject *os = (PyArrayObject *)PyTuple_GET_ITEM(bufs, 0);
      PyArrayObject *oc = (PyArrayObject *)PyTuple_GET_ITEM(bufs, 1);
      const int ts = PyArray_TYPE(os), tc = PyArray_TYPE(oc);
      const npy_intp ss = ts == NPY_DOUBLE ? 8 : 4, sc = tc == NPY_DOUBLE ? 8 : 4;
      char *ps = (char *)PyArray_DATA(os), *pc = (char *)PyArray_DATA(oc);
      for (Py_ssize_t j = 0; j < n; ++j) {
        const npy_intp T = (npy_intp)L[j];
        copy2d((PyArrayObject *)held[2 * j], T, d0, ps, ts);
        ps += T * d0 * ss;
        copy2d((PyArrayObject *)held[2 * j + 1], 1, C, pc, tc);
        pc += C * sc;
      }
      ok = 1;
    } else {
      PyErr_SetString(PyExc_ValueError,
                      "alloc() must return two writable C-contiguous float32/float64 arrays of "
                      "rows*d0 and n*C elements");
    }
    Py_DECREF(bufs);
  }
  release(held, 2 * n);
  Py_DECREF(fast);
  if (!ok) {
    Py_DECREF(lens);
    return NULL;
  }
  return lens;
}

static PyMethodDef methods[] = {
    {"pack", pack, METH_VARARGS, "pack(seqs, d0, C, alloc) -> int64 lens bytes | None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_ttpack", NULL, -1, methods};

PyMODINIT_FUNC PyInit__ttpack(void) {
  import_array();
  s_steps = PyUnicode_InternFromString("steps");
  s_context = PyUnicode_InternFromString("context");
  return PyModule_Create(&mod);
}
