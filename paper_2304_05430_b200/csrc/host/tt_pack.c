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
#include <structmember.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static PyObject *s_steps, *s_context;
enum { kMaxThreads = 32 }; /* conversion copy threads */

static int float_type(int t) { return t == NPY_DOUBLE || t == NPY_FLOAT; }
/* a source array the raw copy loops may read: float32/64 in native byte order
 * and aligned (anything else -- '>f8', unaligned views -- makes pack() return
 * None so the numpy path converts it) */
static int readable_src(PyArrayObject *a) {
  return float_type(PyArray_TYPE(a)) && PyArray_ISNOTSWAPPED(a) && PyArray_ISALIGNED(a);
}

/* one strided float source block (rows x cols) */
typedef struct {
  const char *src;
  npy_intp rs, cs;
  int in_t;
} Src;

/* copy a (rows, cols) strided float block into dense out of type out_t */
static void copy2d(const Src *a, npy_intp rows, npy_intp cols, char *out, int out_t) {
  const npy_intp isz = a->in_t == NPY_DOUBLE ? 8 : 4;
  const npy_intp n = rows * cols;
  if (a->cs == isz && (rows == 1 || a->rs == cols * isz)) {  /* contiguous source */
    if (a->in_t == out_t) {
      memcpy(out, a->src, (size_t)(n * isz));
    } else if (out_t == NPY_FLOAT) {
      const double *in = (const double *)a->src;
      float *o = (float *)out;
      for (npy_intp i = 0; i < n; ++i) o[i] = (float)in[i];
    } else {
      const float *in = (const float *)a->src;
      double *o = (double *)out;
      for (npy_intp i = 0; i < n; ++i) o[i] = (double)in[i];
    }
    return;
  }
  for (npy_intp r = 0; r < rows; ++r) {
    const char *row = a->src + r * a->rs;
    for (npy_intp c = 0; c < cols; ++c) {
      const char *e = row + c * a->cs;
      const double v = a->in_t == NPY_DOUBLE ? *(const double *)e : (double)*(const float *)e;
      if (out_t == NPY_DOUBLE)
        ((double *)out)[r * cols + c] = v;
      else
        ((float *)out)[r * cols + c] = (float)v;
    }
  }
}

typedef struct {
  const Src *st, *cx;
  const int64_t *L, *roff; /* step counts, first output row of each item */
  Py_ssize_t i0, i1;
  npy_intp d0, C, ss, sc;
  char *ps, *pc;
  int ts, tc;
} Job;

static void *run_job(void *arg) {
  const Job *j = (const Job *)arg;
  for (Py_ssize_t i = j->i0; i < j->i1; ++i) {
    copy2d(&j->st[i], (npy_intp)j->L[i], j->d0, j->ps + (npy_intp)j->roff[i] * j->d0 * j->ss, j->ts);
    copy2d(&j->cx[i], 1, j->C, j->pc + (npy_intp)i * j->C * j->sc, j->tc);
  }
  return NULL;
}

/* Attribute fast path: objects of one type whose `steps` / `context` are
 * __slots__ members are read at the members' offsets (what the member
 * descriptor would do); any other layout goes through PyObject_GetAttr. */
typedef struct {
  PyTypeObject *tp;
  Py_ssize_t off_s, off_c; /* > 0: slot offsets */
} AttrCache;

static void attr_cache_init(AttrCache *c, PyObject *obj) {
  c->tp = Py_TYPE(obj);
  c->off_s = c->off_c = 0;
  PyObject *d1 = _PyType_Lookup(c->tp, s_steps), *d2 = _PyType_Lookup(c->tp, s_context);
  if (d1 && d2 && Py_IS_TYPE(d1, &PyMemberDescr_Type) && Py_IS_TYPE(d2, &PyMemberDescr_Type)) {
    PyMemberDef *m1 = ((PyMemberDescrObject *)d1)->d_member, *m2 = ((PyMemberDescrObject *)d2)->d_member;
    if (m1->type == Py_T_OBJECT_EX && m2->type == Py_T_OBJECT_EX) {
      c->off_s = m1->offset;
      c->off_c = m2->offset;
    }
  }
}

/* new reference or NULL (exception set) */
static PyObject *get_attr(const AttrCache *c, PyObject *obj, PyObject *name, Py_ssize_t off) {
  if (Py_TYPE(obj) == c->tp && off > 0) {
    PyObject *v = *(PyObject **)((char *)obj + off);
    if (v) {
      Py_INCREF(v);
      return v;
    }
  }
  return PyObject_GetAttr(obj, name);
}

static void release(PyObject **held, Py_ssize_t n) {
  for (Py_ssize_t i = 0; i < n; ++i) Py_XDECREF(held[i]);
  free(held);
}

static int out_ok(PyObject *o, npy_intp need) {
  if (!PyArray_Check(o)) return 0;
  PyArrayObject *a = (PyArrayObject *)o;
  return float_type(PyArray_TYPE(a)) && PyArray_ISNOTSWAPPED(a) && PyArray_IS_C_CONTIGUOUS(a) &&
         PyArray_ISWRITEABLE(a) &&
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
  AttrCache ac;
  for (Py_ssize_t i = 0; i < n && !bad; ++i) {
    if (i == 0) attr_cache_init(&ac, objs[0]);
    PyObject *so = held[2 * i] = get_attr(&ac, objs[i], s_steps, ac.off_s);
    PyObject *co = held[2 * i + 1] = so ? get_attr(&ac, objs[i], s_context, ac.off_c) : NULL;
    if (!so || !co || !PyArray_Check(so) || !PyArray_Check(co)) {
      bad = 1;
      break;
    }
    PyArrayObject *sa = (PyArrayObject *)so, *ca = (PyArrayObject *)co;
    if (d0 < 0 && PyArray_NDIM(sa) == 2) d0 = PyArray_DIM(sa, 1);
    if (C < 0 && PyArray_NDIM(ca) == 1) C = PyArray_DIM(ca, 0);
    if (PyArray_NDIM(sa) != 2 || PyArray_DIM(sa, 1) != d0 || PyArray_DIM(sa, 0) < 1 ||
        !readable_src(sa) || PyArray_NDIM(ca) != 1 || PyArray_DIM(ca, 0) != C ||
        !readable_src(ca)) {
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
      Src *src = (Src *)malloc((size_t)(2 * n) * sizeof(Src));
      int64_t *roff = (int64_t *)malloc((size_t)n * sizeof(int64_t));
      if (!src || !roff) {
        free(src);
        free(roff);
        PyErr_NoMemory();
      } else {
        /* gather the source descriptors under the GIL, copy without it */
        int64_t acc = 0;
        for (Py_ssize_t j = 0; j < n; ++j) {
          PyArrayObject *sa = (PyArrayObject *)held[2 * j], *ca = (PyArrayObject *)held[2 * j + 1];
          src[j] = (Src){(const char *)PyArray_DATA(sa), PyArray_STRIDE(sa, 0), PyArray_STRIDE(sa, 1),
                         PyArray_TYPE(sa)};
          src[n + j] = (Src){(const char *)PyArray_DATA(ca), 0, PyArray_STRIDE(ca, 0), PyArray_TYPE(ca)};
          roff[j] = acc;
          acc += L[j];
        }
        Job base;
        base.st = src;
        base.cx = src + n;
        base.L = L;
        base.roff = roff;
        base.d0 = d0;
        base.C = C;
        base.ts = PyArray_TYPE(os);
        base.tc = PyArray_TYPE(oc);
        base.ss = base.ts == NPY_DOUBLE ? 8 : 4;
        base.sc = base.tc == NPY_DOUBLE ? 8 : 4;
        base.ps = (char *)PyArray_DATA(os);
        base.pc = (char *)PyArray_DATA(oc);
        long ncpu = sysconf(_SC_NPROCESSORS_ONLN);
        int nth = (int)(ncpu < 1 ? 1 : ncpu > kMaxThreads ? kMaxThreads : ncpu);
        if (n < 4096) nth = 1;
        Job jobs[kMaxThreads];
        pthread_t tids[kMaxThreads];
        int started[kMaxThreads] = {0};
        Py_BEGIN_ALLOW_THREADS
        for (int t = 0; t < nth; ++t) {
          jobs[t] = base;
          jobs[t].i0 = n * t / nth;
          jobs[t].i1 = n * (t + 1) / nth;
          if (t > 0) started[t] = pthread_create(&tids[t], NULL, run_job, &jobs[t]) == 0;
        }
        run_job(&jobs[0]);
        for (int t = 1; t < nth; ++t) {
          if (started[t])
            pthread_join(tids[t], NULL);
          else
            run_job(&jobs[t]);
        }
        Py_END_ALLOW_THREADS
        free(src);
        free(roff);
        ok = 1;
      }
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
