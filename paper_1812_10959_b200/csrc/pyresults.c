/* pyresults.c — the MiningResult's frequent tuple built in C.
 *
 * The engine hands back F itemsets as three host arrays (masks uint64 [F][W],
 * LSW first; sizes int32 [F]; supports int64 [F]), already in the canonical
 * (size, mask) order of engine.py:446-455.  The reference's result is a tuple
 * of FrequentItemset(mask: int, size: int, support: int) NamedTuples
 * (engine.py:70-74), so every mask becomes an arbitrary-precision Python int.
 * Doing that in Python (int.from_bytes per row + tuple.__new__) costs about
 * 250 ns per itemset (2.5 ms for cfg4's 8.5k itemsets, half of cfg1's run);
 * here it is one pass in C.  Host-side formatting only: no counting happens
 * here, and the module is built with the library by _build.py. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

/* An arbitrary-precision int from `top` little-endian 64-bit words: the
 * interpreter's 30-bit digits cut out of the words directly
 * (_PyLong_FromDigits, CPython >= 3.12), instead of _PyLong_FromByteArray's
 * byte-by-byte loop (8 x top iterations; three times slower on a 16-word mask). */
static PyObject* mask_to_long(const uint64_t* w, Py_ssize_t top) {
#if PY_VERSION_HEX >= 0x030C0000 && PyLong_SHIFT == 30
    digit d[(64 * 64 + 29) / 30 + 1];
    if (top <= 64) {
        const Py_ssize_t bits = top * 64;
        Py_ssize_t nd = 0;
        for (Py_ssize_t b = 0; b < bits; b += 30) {
            const Py_ssize_t i = b >> 6, o = b & 63;
            uint64_t x = w[i] >> o;
            if (o > 34 && i + 1 < top) x |= w[i + 1] << (64 - o);
            d[nd++] = (digit)(x & 0x3FFFFFFFu);
        }
        while (nd > 0 && d[nd - 1] == 0) --nd;
        return (PyObject*)_PyLong_FromDigits(0, nd, d);
    }
#endif
    return _PyLong_FromByteArray((const unsigned char*)w, (size_t)top * 8u, 1, 0);
}

static PyObject* frequent_tuple(PyObject* self, PyObject* args) {
    PyObject* cls;
    Py_buffer masks, sizes, sups;
    Py_ssize_t W;
    (void)self;
    if (!PyArg_ParseTuple(args, "Oy*ny*y*", &cls, &masks, &W, &sizes, &sups)) return NULL;
    PyObject* out = NULL;
    if (!PyType_Check(cls) || !PyType_IsSubtype((PyTypeObject*)cls, &PyTuple_Type)) {
        PyErr_SetString(PyExc_TypeError, "frequent_tuple: cls must be a tuple subclass");
        goto done;
    }
    const Py_ssize_t F = sizes.len / (Py_ssize_t)sizeof(int32_t);
    if (W < 1 || masks.len != F * W * (Py_ssize_t)sizeof(uint64_t) ||
        sups.len != F * (Py_ssize_t)sizeof(int64_t)) {
        PyErr_SetString(PyExc_ValueError, "frequent_tuple: inconsistent array sizes");
        goto done;
    }
    PyTypeObject* tp = (PyTypeObject*)cls;
    const unsigned char* mb = (const unsigned char*)masks.buf;
    const int32_t* sz = (const int32_t*)sizes.buf;
    const int64_t* sp = (const int64_t*)sups.buf;
    out = PyTuple_New(F);
    if (!out) goto done;
    for (Py_ssize_t i = 0; i < F; ++i) {
        /* little-endian words == little-endian bytes on x86-64; only the
         * bytes up to the highest non-zero word (itemsets are sparse) */
        const uint64_t* row = (const uint64_t*)(mb + (size_t)i * (size_t)W * 8u);
        Py_ssize_t top = W;
        while (top > 1 && row[top - 1] == 0) --top;
        PyObject* mask = mask_to_long(row, top);
        PyObject* size = PyLong_FromLong(sz[i]);
        PyObject* sup = PyLong_FromLongLong(sp[i]);
        PyObject* item = tp->tp_alloc(tp, 3);
        if (!mask || !size || !sup || !item) {
            Py_XDECREF(mask);
            Py_XDECREF(size);
            Py_XDECREF(sup);
            Py_XDECREF(item);
            Py_CLEAR(out);
            goto done;
        }
        PyTuple_SET_ITEM(item, 0, mask);
        PyTuple_SET_ITEM(item, 1, size);
        PyTuple_SET_ITEM(item, 2, sup);
        PyTuple_SET_ITEM(out, i, item);
    }
done:
    PyBuffer_Release(&masks);
    PyBuffer_Release(&sizes);
    PyBuffer_Release(&sups);
    return out;
}

static PyMethodDef methods[] = {
    {"frequent_tuple", frequent_tuple, METH_VARARGS,
     "frequent_tuple(cls, masks_u64_bytes, W, sizes_i32_bytes, supports_i64_bytes) -> tuple of cls(mask, size, support)"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_dicpy", "MiningResult builders in C", -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__dicpy(void) { return PyModule_Create(&module); }
