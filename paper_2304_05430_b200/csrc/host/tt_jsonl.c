/* Dataset I/O: native codec for the record lines of the
 * tensortune.v1 JSONL format (data.py:507-657), byte-compatible with the
 * reference's writer and equivalent to its reader.
 *
 *   recs = _ttjsonl.parse_records(buf, start, end, ScheduleConfig, MeasurementRecord)
 *       Parse the '\n'-separated record lines in buf[start:end) -- each one
 *       exactly in the canonical shape dumps_dataset writes:
 *         {"type": "record", "record_id": S, "task_id": S, "schedule":
 *          {"tile_factors": [[i, ...], ...], "unroll_factor": i,
 *           "vectorize_width": i[, "thread_binding": [i, i]]},
 *          "measured_flops": i, "error_flag": true|false[, "mean_cost": f]}
 *       -- and build the reference's own dataclasses with the values
 *       MeasurementRecord.from_json / ScheduleConfig.from_json would produce
 *       (data.py:74-98, :199-228).  Returns a list, or None as soon as any
 *       line deviates from the canonical shape (other key order, escapes in
 *       strings, whitespace, unknown fields...): the caller then runs the
 *       reference's own json path, which yields the same objects or the
 *       exact same error.
 *
 *   text = _ttjsonl.dump_records(records)
 *       The record lines of dumps_dataset (data.py:535-560): json.dumps with
 *       separators (", ", ": ") and the cost spliced in by format_cost
 *       (repr if it has >= 9 significant digits, else "%.8e").  Returns None
 *       if any record needs what only the reference does (non-ASCII or
 *       escaped characters in an id, the cost sentinel, non-int fields).
 *
 * Integers go through PyLong_FromString (arbitrary size, like json), floats
 * through PyOS_string_to_double (correctly rounded, like float()), repr
 * through PyOS_double_to_string(.., 'r', ..) (Python's float repr).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <string.h>

typedef struct {
  const char *p, *end;
} Cur;

static int lit(Cur *c, const char *s) {
  const size_t n = strlen(s);
  if ((size_t)(c->end - c->p) < n || memcmp(c->p, s, n) != 0) return 0;
  c->p += n;
  return 1;
}

/* a JSON string without escapes or control characters, ASCII only */
static PyObject *plain_str(Cur *c) {
  if (c->p >= c->end || *c->p != '"') return NULL;
  const char *s = ++c->p;
  while (c->p < c->end && *c->p != '"') {
    const unsigned char ch = (unsigned char)*c->p;
    if (ch == '\\' || ch < 0x20 || ch >= 0x80) return NULL;
    ++c->p;
  }
  if (c->p >= c->end) return NULL;
  PyObject *o = PyUnicode_FromStringAndSize(s, c->p - s);
  ++c->p;
  return o;
}

/* a JSON integer: -?(0|[1-9][0-9]*) */
static PyObject *json_int(Cur *c) {
  const char *s = c->p;
  if (c->p < c->end && *c->p == '-') ++c->p;
  if (c->p >= c->end || *c->p < '0' || *c->p > '9') return NULL;
  if (*c->p == '0' && c->p + 1 < c->end && c->p[1] >= '0' && c->p[1] <= '9') return NULL;
  while (c->p < c->end && *c->p >= '0' && *c->p <= '9') ++c->p;
  if (c->p < c->end && (*c->p == '.' || *c->p == 'e' || *c->p == 'E')) return NULL; /* a float */
  char tmp[64];
  const size_t n = (size_t)(c->p - s);
  if (n >= sizeof tmp) return NULL;
  memcpy(tmp, s, n);
  tmp[n] = 0;
  return PyLong_FromString(tmp, NULL, 10);
}

/* a JSON number as float (json.loads gives int or float; float() of either
 * is what from_json stores) */
static PyObject *json_float(Cur *c) {
  const char *s = c->p;
  if (c->p < c->end && *c->p == '-') ++c->p;
  if (c->p >= c->end || *c->p < '0' || *c->p > '9') return NULL;
  while (c->p < c->end && ((*c->p >= '0' && *c->p <= '9') || *c->p == '.' || *c->p == 'e' ||
                           *c->p == 'E' || *c->p == '+' || *c->p == '-'))
    ++c->p;
  char tmp[64];
  const size_t n = (size_t)(c->p - s);
  if (n >= sizeof tmp) return NULL;
  memcpy(tmp, s, n);
  tmp[n] = 0;
  char *endp = NULL;
  const double v = PyOS_string_to_double(tmp, &endp, NULL);
  if (v == -1.0 && PyErr_Occurred()) {
    PyErr_Clear();
    return NULL;
  }
  if (endp != tmp + n) return NULL;
  return PyFloat_FromDouble(v);
}

/* [i, i, ...] -> tuple of ints (at least one element) */
static PyObject *int_tuple(Cur *c) {
  if (!lit(c, "[")) return NULL;
  PyObject *items = PyList_New(0);
  if (!items) return NULL;
  for (;;) {
    PyObject *v = json_int(c);
    if (!v) {
      Py_DECREF(items);
      return NULL;
    }
    PyList_Append(items, v);
    Py_DECREF(v);
    if (lit(c, "]")) break;
    if (!lit(c, ", ")) {
      Py_DECREF(items);
      return NULL;
    }
  }
  PyObject *t = PyList_AsTuple(items);
  Py_DECREF(items);
  return t;
}

/* one record line (without the newline) -> MeasurementRecord, or NULL */
static PyObject *parse_line(Cur *c, PyObject *Sched, PyObject *Rec) {
  PyObject *rid = NULL, *tid = NULL, *tiles = NULL, *unroll = NULL, *vec = NULL, *bind = Py_None,
           *flops = NULL, *cost = Py_None, *sched = NULL, *out = NULL;
  int err_flag = 0;
  Py_INCREF(Py_None);
  Py_INCREF(Py_None);
  if (!lit(c, "{\"type\": \"record\", \"record_id\": ") || !(rid = plain_str(c))) goto done;
  if (!lit(c, ", \"task_id\": ") || !(tid = plain_str(c))) goto done;
  if (!lit(c, ", \"schedule\": {\"tile_factors\": [")) goto done;
  {
    PyObject *lst = PyList_New(0);
    if (!lst) goto done;
    for (;;) {
      PyObject *t = int_tuple(c);
      if (!t) {
        Py_DECREF(lst);
        goto done;
      }
      PyList_Append(lst, t);
      Py_DECREF(t);
      if (lit(c, "]")) break;
      if (!lit(c, ", ")) {
        Py_DECREF(lst);
        goto done;
      }
    }
    tiles = PyList_AsTuple(lst);
    Py_DECREF(lst);
    if (!tiles) goto done;
  }
  if (!lit(c, ", \"unroll_factor\": ") || !(unroll = json_int(c))) goto done;
  if (!lit(c, ", \"vectorize_width\": ") || !(vec = json_int(c))) goto done;
  if (lit(c, ", \"thread_binding\": ")) {
    PyObject *b = int_tuple(c);
    if (!b) goto done;
    if (PyTuple_GET_SIZE(b) != 2) { /* the reference raises: let it */
      Py_DECREF(b);
      goto done;
    }
    Py_DECREF(bind);
    bind = b;
  }
  if (!lit(c, "}, \"measured_flops\": ") || !(flops = json_int(c))) goto done;
  if (lit(c, ", \"error_flag\": true")) {
    err_flag = 1;
  } else if (!lit(c, ", \"error_flag\": false")) {
    goto done;
  }
  if (lit(c, ", \"mean_cost\": ")) {
    PyObject *f = json_float(c);
    if (!f) goto done;
    Py_DECREF(cost);
    cost = f;
  }
  if (!lit(c, "}")) goto done;
  if (c->p != c->end) goto done;
  sched = PyObject_CallFunctionObjArgs(Sched, tiles, unroll, vec, bind, NULL);
  if (!sched) goto done;
  out = PyObject_CallFunctionObjArgs(Rec, rid, tid, sched, cost, flops, err_flag ? Py_True : Py_False,
                                     NULL);
done:
  Py_XDECREF(rid);
  Py_XDECREF(tid);
  Py_XDECREF(tiles);
  Py_XDECREF(unroll);
  Py_XDECREF(vec);
  Py_XDECREF(bind);
  Py_XDECREF(flops);
  Py_XDECREF(cost);
  Py_XDECREF(sched);
  if (!out && PyErr_Occurred()) PyErr_Clear(); /* fall back: the reference reports it */
  return out;
}

static PyObject *parse_records(PyObject *self, PyObject *args) {
  Py_buffer buf;
  Py_ssize_t start, end;
  PyObject *Sched, *Rec;
  if (!PyArg_ParseTuple(args, "y*nnOO", &buf, &start, &end, &Sched, &Rec)) return NULL;
  if (start < 0 || end > buf.len || start > end) {
    PyBuffer_Release(&buf);
    PyErr_SetString(PyExc_ValueError, "bad range");
    return NULL;
  }
  const char *b = (const char *)buf.buf;
  PyObject *out = PyList_New(0);
  if (!out) {
    PyBuffer_Release(&buf);
    return NULL;
  }
  Py_ssize_t pos = start;
  while (pos < end) {
    const char *nl = memchr(b + pos, '\n', (size_t)(end - pos));
    const Py_ssize_t stop = nl ? (Py_ssize_t)(nl - b) : end;
    Cur c = {b + pos, b + stop};
    PyObject *r = parse_line(&c, Sched, Rec);
    if (!r) {
      Py_DECREF(out);
      PyBuffer_Release(&buf);
      Py_RETURN_NONE;
    }
    PyList_Append(out, r);
    Py_DECREF(r);
    pos = stop + 1;
  }
  PyBuffer_Release(&buf);
  return out;
}

/* ----------------------------------------------------------- writer -- */

typedef struct {
  char *d;
  size_t n, cap;
} Buf;

static int put(Buf *w, const char *s, size_t n) {
  if (w->n + n > w->cap) {
    size_t cap = w->cap ? w->cap * 2 : 1 << 16;
    while (cap < w->n + n) cap *= 2;
    char *d = (char *)realloc(w->d, cap);
    if (!d) return 0;
    w->d = d;
    w->cap = cap;
  }
  memcpy(w->d + w->n, s, n);
  w->n += n;
  return 1;
}
static int puts_(Buf *w, const char *s) { return put(w, s, strlen(s)); }

static int put_str(Buf *w, PyObject *o) { /* plain ASCII, no escapes needed */
  if (!PyUnicode_Check(o)) return 0;
  Py_ssize_t n;
  const char *s = PyUnicode_AsUTF8AndSize(o, &n);
  if (!s) {
    PyErr_Clear();
    return 0;
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    const unsigned char ch = (unsigned char)s[i];
    if (ch == '"' || ch == '\\' || ch < 0x20 || ch >= 0x80) return 0;
  }
  if (strstr(s, "@@MEAN-COST-SENTINEL@@")) return 0; /* the reference raises */
  return put(w, "\"", 1) && put(w, s, (size_t)n) && put(w, "\"", 1);
}

static int put_int(Buf *w, PyObject *o) { /* exact int (not bool) -> str(o) */
  if (!PyLong_CheckExact(o)) return 0;
  PyObject *s = PyObject_Str(o);
  if (!s) {
    PyErr_Clear();
    return 0;
  }
  Py_ssize_t n;
  const char *t = PyUnicode_AsUTF8AndSize(s, &n);
  const int ok = t && put(w, t, (size_t)n);
  Py_DECREF(s);
  return ok;
}

static int put_int_list(Buf *w, PyObject *seq) {
  PyObject *f = PySequence_Fast(seq, "");
  if (!f) {
    PyErr_Clear();
    return 0;
  }
  int ok = puts_(w, "[");
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(f);
  for (Py_ssize_t i = 0; ok && i < n; ++i) {
    if (i) ok = puts_(w, ", ");
    ok = ok && put_int(w, PySequence_Fast_GET_ITEM(f, i));
  }
  Py_DECREF(f);
  return ok && puts_(w, "]");
}

/* format_cost (data.py:517-528) */
static int put_cost(Buf *w, double v) {
  char *r = PyOS_double_to_string(v, 'r', 0, Py_DTSF_ADD_DOT_0, NULL);
  if (!r) {
    PyErr_Clear();
    return 0;
  }
  /* significant digits of the mantissa: digits only, leading zeros stripped */
  int digits = 0, lead = 1;
  for (const char *p = r; *p && *p != 'e' && *p != 'E'; ++p) {
    if (*p < '0' || *p > '9') continue;
    if (lead && *p == '0') continue;
    lead = 0;
    ++digits;
  }
  int ok;
  if (digits >= 9 || !isfinite(v)) {
    ok = puts_(w, r);
  } else {
    char *e = PyOS_double_to_string(v, 'e', 8, 0, NULL);
    ok = e && puts_(w, e);
    if (e) PyMem_Free(e);
  }
  PyMem_Free(r);
  return ok;
}

static PyObject *a_record_id, *a_task_id, *a_schedule, *a_mean_cost, *a_measured_flops, *a_error_flag,
    *a_tile_factors, *a_unroll, *a_vec, *a_binding;

static int put_record(Buf *w, PyObject *rec) {
  int ok = 0;
  PyObject *rid = PyObject_GetAttr(rec, a_record_id), *tid = PyObject_GetAttr(rec, a_task_id),
           *sch = PyObject_GetAttr(rec, a_schedule), *cost = PyObject_GetAttr(rec, a_mean_cost),
           *flops = PyObject_GetAttr(rec, a_measured_flops), *ef = PyObject_GetAttr(rec, a_error_flag);
  PyObject *tiles = NULL, *unr = NULL, *vec = NULL, *bind = NULL;
  if (!rid || !tid || !sch || !cost || !flops || !ef) goto done;
  if (!(tiles = PyObject_GetAttr(sch, a_tile_factors)) || !(unr = PyObject_GetAttr(sch, a_unroll)) ||
      !(vec = PyObject_GetAttr(sch, a_vec)) || !(bind = PyObject_GetAttr(sch, a_binding)))
    goto done;
  if (ef != Py_True && ef != Py_False) goto done; /* json.dumps of a non-bool differs */
  if (!(puts_(w, "{\"type\": \"record\", \"record_id\": ") && put_str(w, rid) &&
        puts_(w, ", \"task_id\": ") && put_str(w, tid) &&
        puts_(w, ", \"schedule\": {\"tile_factors\": [")))
    goto done;
  {
    PyObject *f = PySequence_Fast(tiles, "");
    if (!f) goto done;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(f);
    int k = 1;
    for (Py_ssize_t i = 0; k && i < n; ++i) {
      if (i) k = puts_(w, ", ");
      k = k && put_int_list(w, PySequence_Fast_GET_ITEM(f, i));
    }
    Py_DECREF(f);
    if (!k) goto done;
  }
  if (!(puts_(w, "], \"unroll_factor\": ") && put_int(w, unr) && puts_(w, ", \"vectorize_width\": ") &&
        put_int(w, vec)))
    goto done;
  if (bind != Py_None && !(puts_(w, ", \"thread_binding\": ") && put_int_list(w, bind))) goto done;
  if (!(puts_(w, "}, \"measured_flops\": ") && put_int(w, flops) &&
        puts_(w, ef == Py_True ? ", \"error_flag\": true" : ", \"error_flag\": false")))
    goto done;
  if (ef == Py_False && cost != Py_None) {
    if (!PyFloat_CheckExact(cost)) goto done;
    if (!(puts_(w, ", \"mean_cost\": ") && put_cost(w, PyFloat_AS_DOUBLE(cost)))) goto done;
  }
  ok = puts_(w, "}\n");
done:
  Py_XDECREF(rid);
  Py_XDECREF(tid);
  Py_XDECREF(sch);
  Py_XDECREF(cost);
  Py_XDECREF(flops);
  Py_XDECREF(ef);
  Py_XDECREF(tiles);
  Py_XDECREF(unr);
  Py_XDECREF(vec);
  Py_XDECREF(bind);
  if (!ok && PyErr_Occurred()) PyErr_Clear();
  return ok;
}

static PyObject *dump_records(PyObject *self, PyObject *args) {
  PyObject *records;
  if (!PyArg_ParseTuple(args, "O", &records)) return NULL;
  PyObject *f = PySequence_Fast(records, "records must be a sequence");
  if (!f) return NULL;
  Buf w = {NULL, 0, 0};
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(f);
  for (Py_ssize_t i = 0; i < n; ++i) {
    if (!put_record(&w, PySequence_Fast_GET_ITEM(f, i))) {
      Py_DECREF(f);
      free(w.d);
      Py_RETURN_NONE;
    }
  }
  Py_DECREF(f);
  PyObject *out = PyUnicode_DecodeASCII(w.d ? w.d : "", (Py_ssize_t)w.n, NULL);
  free(w.d);
  return out;
}

static PyMethodDef methods[] = {
    {"parse_records", parse_records, METH_VARARGS,
     "parse_records(buf, start, end, ScheduleConfig, MeasurementRecord) -> list | None"},
    {"dump_records", dump_records, METH_VARARGS, "dump_records(records) -> str | None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_ttjsonl", NULL, -1, methods};

PyMODINIT_FUNC PyInit__ttjsonl(void) {
  a_record_id = PyUnicode_InternFromString("record_id");
  a_task_id = PyUnicode_InternFromString("task_id");
  a_schedule = PyUnicode_InternFromString("schedule");
  a_mean_cost = PyUnicode_InternFromString("mean_cost");
  a_measured_flops = PyUnicode_InternFromString("measured_flops");
  a_error_flag = PyUnicode_InternFromString("error_flag");
  a_tile_factors = PyUnicode_InternFromString("tile_factors");
  a_unroll = PyUnicode_InternFromString("unroll_factor");
  a_vec = PyUnicode_InternFromString("vectorize_width");
  a_binding = PyUnicode_InternFromString("thread_binding");
  return PyModule_Create(&mod);
}
