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
static scalar_fn g_fn = NULL;

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

static PyMethodDef methods[] = {
    {"bind", bind, METH_O, "bind(address of fn_scalar)"},
    {"scalar", (PyCFunction)(void (*)(void))scalar, METH_FASTCALL, "one row through fn_scalar"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_scalar", NULL, -1, methods};

PyMODINIT_FUNC PyInit__scalar(void) { return PyModule_Create(&module); }
