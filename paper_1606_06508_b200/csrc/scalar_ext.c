/* CPython fast path for the reference's scalar kernel signatures.
 *
 * scalar(op, dim, dtype, nout, sq_first, args) converts the Python numbers in `args`
 * (ka[6] then x1..xn for the scaling families, x1..xn otherwise), calls fn_scalar of
 * libfastnorm_b200.so and builds the result: a float for one output, else a tuple
 * (squared length first for normalize{n}_sq, like the Python wrapper).  On a library
 * error it returns the fn_status code as an int; the caller raises.  The entry point
 * is bound at run time from the address ctypes resolved (bind()), so this module
 * shares the one loaded copy of the library.  It replaces a ctypes call (about 3 us)
 * with a METH_FASTCALL call (well under 1 us); the work itself is the same launch.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*scalar_fn)(int, int, int, const double*, double*, const double*);
typedef int (*run_fn)(int, int, int, const void*, int64_t, void*, void*, void*, const double*, void*);
typedef int (*host_fn)(int, int, int, const void*, int64_t, void*, void*, void*, const double*);
static scalar_fn g_fn = NULL;
static run_fn g_run = NULL;
static host_fn g_host = NULL;

static PyObject* bind(PyObject* self, PyObject* arg) {
    (void)self;
    void* p = PyLong_AsVoidPtr(arg);
    if (!p && PyErr_Occurred()) return NULL;
    g_fn = (scalar_fn)p;
    Py_RETURN_NONE;
}

static PyObject* scalar(PyObject* self, PyObject* const* a, Py_ssize_t na) {
    (void)self;
    if (na != 6 || !PyTuple_Check(a[5])) {
        PyErr_SetString(PyExc_TypeError, "scalar(op, dim, dtype, nout, sq_first, args: tuple)");
        return NULL;
    }
    if (!g_fn) {
        PyErr_SetString(PyExc_RuntimeError, "fn_scalar is not bound");
        return NULL;
    }
    const int op = (int)PyLong_AsLong(a[0]), dim = (int)PyLong_AsLong(a[1]);
    const int dtype = (int)PyLong_AsLong(a[2]), nout = (int)PyLong_AsLong(a[3]);
    const int sq_first = PyObject_IsTrue(a[4]);
    if (PyErr_Occurred()) return NULL;
    PyObject* args = a[5];
    const Py_ssize_t n = PyTuple_GET_SIZE(args);
    if (dim < 2 || dim > 4 || nout < 1 || nout > 16 || (n != dim && n != dim + 6)) {
        PyErr_SetString(PyExc_ValueError, "bad scalar call shape");
        return NULL;
    }
    double vals[10], out[16];
    for (Py_ssize_t i = 0; i < n; ++i) {
        vals[i] = PyFloat_AsDouble(PyTuple_GET_ITEM(args, i));
        if (vals[i] == -1.0 && PyErr_Occurred()) return NULL;
    }
    const int with_ka = n == dim + 6;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = g_fn(op, dim, dtype, with_ka ? vals + 6 : vals, out, with_ka ? vals : NULL);
    Py_END_ALLOW_THREADS
    if (rc) return PyLong_FromLong(rc);
    if (nout == 1) return PyFloat_FromDouble(out[0]);
    PyObject* t = PyTuple_New(nout);
    if (!t) return NULL;
    for (int k = 0; k < nout; ++k) {
        const int src = sq_first ? (k == 0 ? nout - 1 : k - 1) : k;
        PyObject* v = PyFloat_FromDouble(out[src]);
        if (!v) { Py_DECREF(t); return NULL; }
        PyTuple_SET_ITEM(t, k, v);
    }
    return t;
}

/* run(op, dim, dtype, x, n, head, body, sq, ka, stream) -> fn_status: fn_run with every
 * pointer (and the stream handle) passed as a Python int, None meaning NULL.  The batched
 * device path calls this instead of a ctypes prototype (about 1 us less per call). */
static void* as_ptr(PyObject* o) {
    if (o == Py_None) return NULL;
    return PyLong_AsVoidPtr(o);
}

static PyObject* bind_run(PyObject* self, PyObject* arg) {
    (void)self;
    void* p = PyLong_AsVoidPtr(arg);
    if (!p && PyErr_Occurred()) return NULL;
    g_run = (run_fn)p;
    Py_RETURN_NONE;
}

static PyObject* run(PyObject* self, PyObject* const* a, Py_ssize_t na) {
    (void)self;
    if (na != 10) {
        PyErr_SetString(PyExc_TypeError, "run(op, dim, dtype, x, n, head, body, sq, ka, stream)");
        return NULL;
    }
    if (!g_run) {
        PyErr_SetString(PyExc_RuntimeError, "fn_run is not bound");
        return NULL;
    }
    const int op = (int)PyLong_AsLong(a[0]), dim = (int)PyLong_AsLong(a[1]), dtype = (int)PyLong_AsLong(a[2]);
    const long long n = PyLong_AsLongLong(a[4]);
    void* x = as_ptr(a[3]);
    void* h = as_ptr(a[5]);
    void* b = as_ptr(a[6]);
    void* q = as_ptr(a[7]);
    void* ka = as_ptr(a[8]);
    void* st = as_ptr(a[9]);
    if (PyErr_Occurred()) return NULL;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = g_run(op, dim, dtype, x, (int64_t)n, h, b, q, (const double*)ka, st);
    Py_END_ALLOW_THREADS
    return PyLong_FromLong(rc);
}

static PyObject* bind_host(PyObject* self, PyObject* arg) {
    (void)self;
    void* p = PyLong_AsVoidPtr(arg);
    if (!p && PyErr_Occurred()) return NULL;
    g_host = (host_fn)p;
    Py_RETURN_NONE;
}

/* host_run(op, dim, dtype, x, n, head, body, sq, ka) -> fn_status: fn_host_run with the
 * arrays passed as C-contiguous buffer objects (numpy arrays; None = NULL) and ka as an
 * address.  Taking the buffers here avoids numpy's .ctypes objects on small calls. */
static PyObject* host_run(PyObject* self, PyObject* const* a, Py_ssize_t na) {
    (void)self;
    if (na != 9) {
        PyErr_SetString(PyExc_TypeError, "host_run(op, dim, dtype, x, n, head, body, sq, ka)");
        return NULL;
    }
    if (!g_host) {
        PyErr_SetString(PyExc_RuntimeError, "fn_host_run is not bound");
        return NULL;
    }
    const int op = (int)PyLong_AsLong(a[0]), dim = (int)PyLong_AsLong(a[1]), dtype = (int)PyLong_AsLong(a[2]);
    const long long n = PyLong_AsLongLong(a[4]);
    void* ka = as_ptr(a[8]);
    if (PyErr_Occurred()) return NULL;
    Py_buffer views[4];
    int held[4] = {0, 0, 0, 0};
    void* ptrs[4] = {NULL, NULL, NULL, NULL};
    const int slots[4] = {3, 5, 6, 7};
    PyObject* result = NULL;
    for (int k = 0; k < 4; ++k) {
        PyObject* o = a[slots[k]];
        if (o == Py_None) continue;
        const int flags = PyBUF_C_CONTIGUOUS | (k ? PyBUF_WRITABLE : 0);
        if (PyObject_GetBuffer(o, &views[k], flags) != 0) goto done;
        held[k] = 1;
        ptrs[k] = views[k].buf;
    }
    {
        int rc;
        Py_BEGIN_ALLOW_THREADS
        rc = g_host(op, dim, dtype, ptrs[0], (int64_t)n, ptrs[1], ptrs[2], ptrs[3], (const double*)ka);
        Py_END_ALLOW_THREADS
        result = PyLong_FromLong(rc);
    }
done:
    for (int k = 0; k < 4; ++k)
        if (held[k]) PyBuffer_Release(&views[k]);
    return result;
}

static PyMethodDef methods[] = {
    {"bind_host", bind_host, METH_O, "bind_host(address of fn_host_run)"},
    {"host_run", (PyCFunction)(void (*)(void))host_run, METH_FASTCALL, "fn_host_run on buffer objects"},
    {"bind", bind, METH_O, "bind(address of fn_scalar)"},
    {"bind_run", bind_run, METH_O, "bind_run(address of fn_run)"},
    {"run", (PyCFunction)(void (*)(void))run, METH_FASTCALL, "fn_run with integer pointers"},
    {"scalar", (PyCFunction)(void (*)(void))scalar, METH_FASTCALL, "one row through fn_scalar"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_scalar", NULL, -1, methods};

PyMODINIT_FUNC PyInit__scalar(void) { return PyModule_Create(&module); }
