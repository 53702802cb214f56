// _m4dfast: CPython fast path for the transport's per-message entry points.
//
// ctypes costs ~0.3 us per argument; m4d_transport_post_send takes ten, and
// the 1-byte ping-pong of the paper's Fig. 6 is dominated by exactly these
// calls (post, progress) plus the host-buffer address lookup.  This module
// calls the same C ABI (include/m4d.h) through function pointers handed over
// by the ctypes loader (bind), so there is one copy of libm4d.so and one
// transport state; it only removes the argument marshalling:
//
//   post(handle, is_send, channel, peer, tag, data, domain, device_len, req_id)
//       host payload:   data = buffer object (address via the buffer protocol), device_len = -1
//       device payload: data = int device address, device_len = its byte length
//       -> None when the request stays pending, else (status, bytes) of the
//       inline completion; raises OSError(status) when the post itself fails.
//   progress(handle) -> list of (req_id, status, bytes), or None when idle.
//
// Reference interface replaced: Transport.post_send / post_recv / progress
// (pkg/src/commshim/transport/base.py:267-284).
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "m4d.h"

namespace {

using post_send_fn = m4d_status (*)(m4d_transport*, uint32_t, int, uint32_t, const void*, uint64_t, int, int,
                                    uint64_t, m4d_completion*);
using post_recv_fn = m4d_status (*)(m4d_transport*, uint32_t, int, uint32_t, void*, uint64_t, int, int, uint64_t,
                                    m4d_completion*);
using progress_fn = int (*)(m4d_transport*, m4d_completion*, int);

post_send_fn g_send = nullptr;
post_recv_fn g_recv = nullptr;
progress_fn g_progress = nullptr;

constexpr int kBatch = 64;

PyObject* bind(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 3) {
        PyErr_SetString(PyExc_TypeError, "bind(post_send, post_recv, progress) takes 3 addresses");
        return nullptr;
    }
    void* p[3];
    for (int i = 0; i < 3; ++i) {
        p[i] = PyLong_AsVoidPtr(args[i]);
        if (!p[i]) {
            if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null function address");
            return nullptr;
        }
    }
    g_send = reinterpret_cast<post_send_fn>(p[0]);
    g_recv = reinterpret_cast<post_recv_fn>(p[1]);
    g_progress = reinterpret_cast<progress_fn>(p[2]);
    Py_RETURN_NONE;
}

// post(handle, is_send, channel, peer, tag, data, domain, device_len, req_id)
//   host payload : data = buffer object, device_len = -1
//   device payload: data = int address,  device_len = byte length
PyObject* post(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 9) {
        PyErr_SetString(PyExc_TypeError, "post takes 9 arguments");
        return nullptr;
    }
    if (!g_send) {
        PyErr_SetString(PyExc_RuntimeError, "_m4dfast.bind() was not called");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    const long is_send = PyLong_AsLong(args[1]);
    const unsigned long channel = PyLong_AsUnsignedLong(args[2]);
    const long peer = PyLong_AsLong(args[3]);
    const unsigned long tag = PyLong_AsUnsignedLong(args[4]);
    const long domain = PyLong_AsLong(args[6]);
    const long long device_len = PyLong_AsLongLong(args[7]);
    const unsigned long long req_id = PyLong_AsUnsignedLongLong(args[8]);
    if (PyErr_Occurred()) return nullptr;
    m4d_completion now;
    m4d_status st;
    if (device_len >= 0) {
        void* addr = PyLong_AsVoidPtr(args[5]);
        if (PyErr_Occurred()) return nullptr;
        st = is_send ? g_send(t, channel, static_cast<int>(peer), tag, addr, device_len, domain, 1, req_id, &now)
                     : g_recv(t, channel, static_cast<int>(peer), tag, addr, device_len, domain, 1, req_id, &now);
    } else {
        Py_buffer view;
        if (PyObject_GetBuffer(args[5], &view, is_send ? PyBUF_SIMPLE : PyBUF_WRITABLE) != 0) return nullptr;
        // The transport keeps the raw address while the request is pending; the
        // Python request object holds the exporter alive for that long.
        st = is_send ? g_send(t, channel, static_cast<int>(peer), tag, view.buf, view.len, domain, 0, req_id, &now)
                     : g_recv(t, channel, static_cast<int>(peer), tag, view.buf, view.len, domain, 0, req_id, &now);
        PyBuffer_Release(&view);
    }
    if (st != M4D_OK) {
        PyErr_SetObject(PyExc_OSError, PyLong_FromLong(st));
        return nullptr;
    }
    if (now.status == -1) Py_RETURN_NONE;
    return Py_BuildValue("(iK)", now.status, static_cast<unsigned long long>(now.bytes));
}

PyObject* progress(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 1) {
        PyErr_SetString(PyExc_TypeError, "progress(handle)");
        return nullptr;
    }
    if (!g_progress) {
        PyErr_SetString(PyExc_RuntimeError, "_m4dfast.bind() was not called");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    if (PyErr_Occurred()) return nullptr;
    m4d_completion batch[kBatch];
    PyObject* out = nullptr;
    for (;;) {
        const int n = g_progress(t, batch, kBatch);
        if (n > 0 && !out && !(out = PyList_New(0))) return nullptr;
        for (int k = 0; k < n; ++k) {
            PyObject* item = Py_BuildValue("(KiK)", static_cast<unsigned long long>(batch[k].req_id), batch[k].status,
                                           static_cast<unsigned long long>(batch[k].bytes));
            if (!item || PyList_Append(out, item) != 0) {
                Py_XDECREF(item);
                Py_DECREF(out);
                return nullptr;
            }
            Py_DECREF(item);
        }
        if (n < kBatch) break;
    }
    if (!out) Py_RETURN_NONE;
    return out;
}

PyMethodDef methods[] = {
    {"bind", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(bind)), METH_FASTCALL,
     "bind(post_send, post_recv, progress): C-ABI function addresses from the ctypes loader"},
    {"post", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(post)), METH_FASTCALL,
     "post(handle, is_send, channel, peer, tag, data, domain, device_len, req_id)"},
    {"progress", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(progress)), METH_FASTCALL,
     "progress(handle) -> [(req_id, status, bytes)] or None"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_m4dfast", "Fast path of the libm4d transport calls.", -1, methods,
                      nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__m4dfast(void) { return PyModule_Create(&module); }
