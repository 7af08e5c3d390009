/* hostptrs.c -- host-side helper of the reference-shaped list API (batch_svd): one C pass over a Python
 * list of matrices that checks they are uniform (same element format, same 2-D shape, F-contiguous:
 * the column-major layout the C-ABI takes, src/core.py:54-60) and collects their data pointers for
 * bsvd_pack_host.  A Python-level loop over 10,000 arrays (attribute lookups, __array_interface__
 * dicts) costs ~8 ms on the B200 host; the ndarray pass below ~0.1 ms.  Not part of the C-ABI boundary
 * (include/bsvd_b200.h): it reads numpy's array struct (or, for other buffer exporters, uses the CPython
 * buffer protocol) and is loaded with ctypes.PyDLL, so it runs with the GIL held.  Built by
 * csrc/Makefile into _lib/libbsvd_hostptrs.so. */

#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>
#include <stdint.h>
#include <string.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/ndarraytypes.h>

/* Returns 0 when every item of `list` (a Python list of n >= 1 objects) exports an F-contiguous
 * 2-D buffer with the format, item size and shape of item 0; ptrs[i] = item i's data.  shape[0..1] and
 * *itemsize describe item 0; fmt receives its format string (truncated to fmt_len - 1).  Returns
 * i + 1 for the first item that differs or exports no such buffer, -1 for a bad argument.  Python
 * errors raised while probing are cleared (the caller falls back to its per-item path). */
int bsvd_py_gather_fortran(PyObject* list, Py_ssize_t n, uintptr_t* ptrs, Py_ssize_t* shape, Py_ssize_t* itemsize,
                           char* fmt, Py_ssize_t fmt_len) {
    if (!list || !PyList_Check(list) || PyList_GET_SIZE(list) != n || n < 1 || !ptrs || !shape || !itemsize)
        return -1;
    char f0[32] = {0};
    Py_ssize_t s0 = 0, s1 = 0, is = 0;
    for (Py_ssize_t i = 0; i < n; ++i) {
        PyObject* o = PyList_GET_ITEM(list, i);
        Py_buffer v;
        if (PyObject_GetBuffer(o, &v, PyBUF_F_CONTIGUOUS | PyBUF_FORMAT) != 0) {
            PyErr_Clear();
            return (int)(i + 1);
        }
        const char* f = v.format ? v.format : "B";
        int ok = v.ndim == 2 && v.shape != NULL;
        if (ok && i == 0) {
            strncpy(f0, f, sizeof(f0) - 1);
            s0 = v.shape[0];
            s1 = v.shape[1];
            is = v.itemsize;
        } else if (ok) {
            ok = v.shape[0] == s0 && v.shape[1] == s1 && v.itemsize == is && strcmp(f, f0) == 0;
        }
        ptrs[i] = (uintptr_t)v.buf;
        PyBuffer_Release(&v);
        if (!ok) return (int)(i + 1);
    }
    shape[0] = s0;
    shape[1] = s1;
    *itemsize = is;
    if (fmt && fmt_len > 0) {
        strncpy(fmt, f0, (size_t)fmt_len - 1);
        fmt[fmt_len - 1] = 0;
    }
    return 0;
}

/* The same check for exact numpy arrays straight from the array struct (numpy/ndarraytypes.h field
 * layout; no C-API table needed): every item's type is `ndarray_type`, its dtype object is item 0's,
 * 2-D with item 0's shape, flagged F-contiguous.  The buffer-protocol path above costs ~1 us per
 * array (numpy builds the format and shape per export); this one ~20 ns. */
int bsvd_py_gather_ndarray(PyObject* list, Py_ssize_t n, PyObject* ndarray_type, uintptr_t* ptrs, Py_ssize_t* shape) {
    if (!list || !PyList_Check(list) || PyList_GET_SIZE(list) != n || n < 1 || !ptrs || !shape || !ndarray_type)
        return -1;
    PyArrayObject_fields* a0 = NULL;
    for (Py_ssize_t i = 0; i < n; ++i) {
        PyObject* o = PyList_GET_ITEM(list, i);
        if ((PyObject*)Py_TYPE(o) != ndarray_type) return (int)(i + 1);
        PyArrayObject_fields* a = (PyArrayObject_fields*)o;
        if (i == 0) {
            if (a->nd != 2) return 1;
            a0 = a;
        } else if (a->nd != 2 || a->descr != a0->descr || a->dimensions[0] != a0->dimensions[0] ||
                   a->dimensions[1] != a0->dimensions[1]) {
            return (int)(i + 1);
        }
        if (!(a->flags & NPY_ARRAY_F_CONTIGUOUS)) return (int)(i + 1);
        ptrs[i] = (uintptr_t)a->data;
    }
    shape[0] = a0->dimensions[0];
    shape[1] = a0->dimensions[1];
    return 0;
}

/* list[start + j] = a fresh instance of `type` (allocated without __init__, like object.__new__) with its
 * slots _g = group, _j = j, for j < n: the lazy SvdResult records of one device launch (batch.py
 * _LazyResult, __slots__ = ("_g", "_j")).  The slot offsets come from the type's member descriptors, so a
 * record costs one allocation and two stores (no per-record instance dict until its first use).  Returns
 * 0, or -1 with a Python error set. */
static Py_ssize_t slot_offset(PyObject* type, const char* name) {
    PyObject* d = PyObject_GetAttrString(type, name);
    Py_ssize_t off = -1;
    if (d && Py_TYPE(d) == &PyMemberDescr_Type) {
        const PyMemberDef* mdef = ((PyMemberDescrObject*)d)->d_member;
        if (mdef->type == Py_T_OBJECT_EX) off = mdef->offset;
    }
    Py_XDECREF(d);
    PyErr_Clear();
    return off;
}

int bsvd_py_fill_lazy(PyObject* list, Py_ssize_t start, Py_ssize_t n, PyObject* type, PyObject* group) {
    static PyObject *key_g = NULL, *key_j = NULL, *cached = NULL;
    static Py_ssize_t off_g = -1, off_j = -1;
    if (!key_g) key_g = PyUnicode_InternFromString("_g");
    if (!key_j) key_j = PyUnicode_InternFromString("_j");
    if (!key_g || !key_j) return -1;
    if (!PyList_Check(list) || !PyType_Check(type) || start < 0 || start + n > PyList_GET_SIZE(list)) {
        PyErr_SetString(PyExc_ValueError, "bsvd_py_fill_lazy: bad arguments");
        return -1;
    }
    if (cached != type) {
        off_g = slot_offset(type, "_g");
        off_j = slot_offset(type, "_j");
        cached = type;  /* borrowed: the type lives as long as the module */
    }
    PyTypeObject* tp = (PyTypeObject*)type;
    for (Py_ssize_t j = 0; j < n; ++j) {
        PyObject* obj = tp->tp_alloc(tp, 0);
        PyObject* jj = PyLong_FromSsize_t(j);
        if (!obj || !jj) {
            Py_XDECREF(obj);
            Py_XDECREF(jj);
            return -1;
        }
        if (off_g >= 0 && off_j >= 0) {  /* fresh object: the slots are NULL */
            Py_INCREF(group);
            *(PyObject**)((char*)obj + off_g) = group;
            *(PyObject**)((char*)obj + off_j) = jj;
        } else if (PyObject_GenericSetAttr(obj, key_g, group) < 0 || PyObject_GenericSetAttr(obj, key_j, jj) < 0) {
            Py_DECREF(jj);
            Py_DECREF(obj);
            return -1;
        } else {
            Py_DECREF(jj);
        }
        PyList_SetItem(list, start + j, obj); /* steals obj, releases the old item */
    }
    return 0;
}

/* list[start + j] = [quiet] if last[j] == 0 else [(False, 1, last[j])] for j < n (the reference's
 * per-problem pair_stats of an unblocked problem's last sweep, src/batch.py:113-142); last: int32[n]. */
int bsvd_py_fill_pair_stats(PyObject* list, Py_ssize_t start, Py_ssize_t n, const int32_t* last, PyObject* quiet) {
    if (!PyList_Check(list) || start < 0 || start + n > PyList_GET_SIZE(list) || !last) {
        PyErr_SetString(PyExc_ValueError, "bsvd_py_fill_pair_stats: bad arguments");
        return -1;
    }
    for (Py_ssize_t j = 0; j < n; ++j) {
        PyObject* inner = PyList_New(1);
        if (!inner) return -1;
        PyObject* item;
        if (last[j] == 0) {
            Py_INCREF(quiet);
            item = quiet;
        } else {
            item = Py_BuildValue("(Oii)", Py_False, 1, (int)last[j]);
            if (!item) {
                Py_DECREF(inner);
                return -1;
            }
        }
        PyList_SET_ITEM(inner, 0, item);
        PyList_SetItem(list, start + j, inner);
    }
    return 0;
}
