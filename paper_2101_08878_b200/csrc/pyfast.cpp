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
//
// Framed composites (the messaging layer's wire protocol done natively):
//
//   send_framed(handle, kind, channel, peer, tag, header, frames, max_chunk, req_id)
//   recv_framed(handle, kind, channel, peer, tag, max_chunk, req_id)
//   take_framed(req_id) -> (outcome, header bytes, payload, detail)
//
// Device frames: a message whose only frame is a device frame of at most
// dev_max bytes (the transport's eager device threshold, one chunk) is also
// done natively.  The sender passes that frame as (address, length) and it
// goes out as an eager device send; the receiver (recv_framed's dev_max
// argument) posts a loan-only device receive, and the payload it returns is
// the loan, (device address, token), of the ring bytes (or of a transport
// receive slot when the message came by rendezvous).
//
// kind 0 is send_payload/recv_payload (messaging.py:295-320 of the reference:
// a <QBB transfer header, then the payload in max_chunk slices, one tag);
// kind 1 is write_message/read_message (:325-388: a <I count + n x <QBB
// header on MESSAGE_TAG, then frame i in slices on tag 16 + i mod 2^15).  The
// composite posts exactly the transport messages the Python functions post,
// in the same order, so either side may use either path.  A receive
// composite reads the header, and for host frames posts the slice receives
// into one buffer itself; anything else (device frames, a malformed or EOS
// header) completes it early with the header bytes so Python finishes the
// message the generic way and raises the generic errors.  Sub-requests carry
// ids with kSubBit set and never reach Python.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstring>
#include <memory>
#include <unordered_map>
#include <vector>

#include "m4d.h"

namespace {

using post_send_fn = m4d_status (*)(m4d_transport*, uint32_t, int, uint32_t, const void*, uint64_t, int, int,
                                    uint64_t, m4d_completion*);
using post_recv_fn = m4d_status (*)(m4d_transport*, uint32_t, int, uint32_t, void*, uint64_t, int, int, uint64_t,
                                    m4d_completion*);
using progress_fn = int (*)(m4d_transport*, m4d_completion*, int);

using take_loan_fn = int (*)(m4d_transport*, uint64_t, uint64_t*, uint64_t*);
using post_many_fn = m4d_status (*)(m4d_transport*, int, uint32_t, int, uint32_t, void* const*, const uint64_t*, int,
                                    int, int, const uint64_t*, m4d_completion*, int*);
using release_loan_fn = m4d_status (*)(m4d_transport*, uint64_t);

post_send_fn g_send = nullptr;
take_loan_fn g_take_loan = nullptr;
release_loan_fn g_release_loan = nullptr;
post_many_fn g_post_many = nullptr;
post_recv_fn g_recv = nullptr;
progress_fn g_progress = nullptr;

constexpr int kBatch = 64;
constexpr uint64_t kSubBit = 1ull << 62;
constexpr int kTagMessage = 1;        // messaging.MESSAGE_TAG
constexpr int kDataTagBase = 16;      // messaging.DATA_TAG_BASE
constexpr int kDataTagSpan = 1 << 15;
constexpr uint32_t kEos = 0xffffffffu;
constexpr size_t kMaxFrames = 1024;
constexpr size_t kMsgHeaderCap = 4 + kMaxFrames * 10;
constexpr uint64_t kFramedLimit = 1u << 20;  // messaging.FRAMED_SEND_LIMIT

enum Outcome { kComplete = 0, kHeaderOnly = 1, kEndOfStream = 2, kShortChunk = 3 };

struct Framed {
    uint64_t id = 0;
    m4d_transport* t = nullptr;
    int kind = 0, peer = 0;
    uint32_t channel = 0, tag = 0;
    uint64_t max_chunk = 1;
    bool recv = false;
    std::vector<uint8_t> header;
    uint64_t header_got = 0;
    std::vector<uint8_t> payload;
    std::vector<Py_buffer> views;  // send: exporters held until the sends complete
    uint64_t dev_max = 0;          // recv: single device frames up to this size are received by loan
    bool dev = false;              // recv: the payload is a device frame, lent (loan_ptr, loan_token)
    bool has_loan = false;
    uint64_t loan_ptr = 0, loan_token = 0;
    int pending = 0;
    int status = M4D_OK;
    int outcome = kComplete;
    long long detail[3] = {0, 0, 0};  // short chunk: offset, expected, actual
    bool done = false;
    std::vector<std::pair<uint64_t, uint64_t>> expect;  // per sub id: (offset, piece)
    std::unordered_map<uint64_t, size_t> sub_slot;
};

std::unordered_map<uint64_t, std::shared_ptr<Framed>> g_framed;   // composite id -> state
std::unordered_map<uint64_t, std::shared_ptr<Framed>> g_by_sub;   // sub id -> composite
std::unordered_map<m4d_transport*, std::vector<m4d_completion>> g_ready;  // finished composites, per transport
uint64_t g_next_sub = 1;

void release_views(Framed& f) {
    for (Py_buffer& v : f.views) PyBuffer_Release(&v);
    f.views.clear();
}

void finish(const std::shared_ptr<Framed>& f, int status, bool inline_done, m4d_completion* now) {
    if (f->done) return;
    f->done = true;
    f->status = status;
    release_views(*f);
    m4d_completion c{f->id, status, f->recv ? 1 : 0, f->payload.size()};
    if (!f->recv) g_framed.erase(f->id);  // a send composite has no result to take
    if (inline_done && now) *now = c;
    else g_ready[f->t].push_back(c);
}

// A composite that finished while its own post call was still running is
// reported by that call, not by progress().
void unqueue(const std::shared_ptr<Framed>& f) {
    auto it = g_ready.find(f->t);
    if (it == g_ready.end()) return;
    auto& v = it->second;
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i].req_id == f->id) {
            v.erase(v.begin() + static_cast<long>(i));
            break;
        }
}

void on_sub(const std::shared_ptr<Framed>& f, uint64_t sub, int status, uint64_t bytes);

// Posts one sub-request; an inline completion is handled at once.
int post_sub(const std::shared_ptr<Framed>& f, bool send, uint32_t tag, void* ptr, uint64_t len, uint64_t offset,
             int on_device = 0) {
    const uint64_t sub = kSubBit | g_next_sub++;
    m4d_completion now;
    g_by_sub[sub] = f;
    f->sub_slot[sub] = f->expect.size();
    f->expect.emplace_back(offset, len);
    ++f->pending;
    const int domain = on_device ? 1 : 0;
    const m4d_status st = send ? g_send(f->t, f->channel, f->peer, tag, ptr, len, domain, on_device, sub, &now)
                               : g_recv(f->t, f->channel, f->peer, tag, ptr, len, domain, on_device, sub, &now);
    if (st != M4D_OK) {
        g_by_sub.erase(sub);
        --f->pending;
        return st;
    }
    if (now.status != -1) {
        g_by_sub.erase(sub);
        on_sub(f, sub, now.status, now.bytes);
    }
    return M4D_OK;
}

int data_tag(size_t i) { return kDataTagBase + static_cast<int>(i % kDataTagSpan); }

// The receive composite's header arrived: post the slice receives (host frames) or stop early.
void on_header(const std::shared_ptr<Framed>& f, uint64_t got) {
    f->header_got = got;
    f->header.resize(got);
    std::vector<std::pair<uint64_t, int>> frames;  // (length, tag)
    // A lone device frame small enough for the eager device protocol: one loan-only
    // device receive (the bytes stay where they land on this GPU).
    auto device_frame = [&](uint64_t len, int tag) {
        if (!f->dev_max || !g_take_loan || len == 0 || len > f->dev_max || len > f->max_chunk) {
            f->outcome = kHeaderOnly;
            return;
        }
        f->dev = true;
        f->outcome = kComplete;
        const int st = post_sub(f, false, static_cast<uint32_t>(tag), nullptr, len, 0, 1 | 4);
        if (st != M4D_OK) f->status = st;
    };
    if (f->kind == 0) {
        if (got != 10) { f->outcome = kHeaderOnly; return; }
        uint64_t len;
        std::memcpy(&len, f->header.data(), 8);
        if (f->header[9] != 0) { device_frame(len, static_cast<int>(f->tag)); return; }
        frames.emplace_back(len, static_cast<int>(f->tag));
    } else {
        if (got < 4) { f->outcome = kHeaderOnly; return; }
        uint32_t count;
        std::memcpy(&count, f->header.data(), 4);
        if (count == kEos) { f->outcome = kEndOfStream; return; }
        if (count > kMaxFrames || got != 4 + 10ull * count) { f->outcome = kHeaderOnly; return; }
        if (count == 1 && f->header[4 + 9] != 0) {
            uint64_t len;
            std::memcpy(&len, f->header.data() + 4, 8);
            device_frame(len, data_tag(0));
            return;
        }
        for (uint32_t i = 0; i < count; ++i) {
            const uint8_t* m = f->header.data() + 4 + 10 * i;
            uint64_t len;
            std::memcpy(&len, m, 8);
            if (m[9] != 0) { f->outcome = kHeaderOnly; return; }  // a device frame: Python allocates it
            frames.emplace_back(len, data_tag(i));
        }
    }
    uint64_t total = 0;
    for (auto& fr : frames) total += fr.first;
    // Bulk transfers are received slice by slice from Python (as the send side posts
    // them): one native call posting and assembling megabytes would stall the loop.
    if (total > kFramedLimit) { f->outcome = kHeaderOnly; return; }
    f->payload.resize(total);
    f->outcome = kComplete;
    uint64_t at = 0;
    for (auto& fr : frames) {
        for (uint64_t off = 0; off < fr.first; off += f->max_chunk) {
            const uint64_t piece = fr.first - off < f->max_chunk ? fr.first - off : f->max_chunk;
            const int st = post_sub(f, false, static_cast<uint32_t>(fr.second), f->payload.data() + at + off, piece, off);
            if (st != M4D_OK) { f->status = st; return; }
            if (f->done) return;
        }
        at += fr.first;
    }
}

void on_sub(const std::shared_ptr<Framed>& f, uint64_t sub, int status, uint64_t bytes) {
    --f->pending;
    const size_t slot = f->sub_slot[sub];
    f->sub_slot.erase(sub);
    if (f->done) return;
    if (status != M4D_OK) {
        finish(f, status, false, nullptr);
        return;
    }
    if (f->recv && slot == 0) {  // the header
        ++f->pending;  // guard: slices completing inline must not finish the composite early
        on_header(f, bytes);
        --f->pending;
        if (f->status != M4D_OK) { finish(f, f->status, false, nullptr); return; }
    } else if (f->recv && f->dev) {
        uint64_t ptr = 0, token = 0;
        if (g_take_loan(f->t, sub, &ptr, &token)) {
            f->has_loan = true;
            f->loan_ptr = ptr;
            f->loan_token = token;
        }
        if (bytes != f->expect[slot].second && f->outcome == kComplete) {
            f->outcome = kShortChunk;
            f->detail[0] = 0;
            f->detail[1] = static_cast<long long>(f->expect[slot].second);
            f->detail[2] = static_cast<long long>(bytes);
        }
    } else if (f->recv && bytes != f->expect[slot].second && f->outcome == kComplete) {
        f->outcome = kShortChunk;
        f->detail[0] = static_cast<long long>(f->expect[slot].first);
        f->detail[1] = static_cast<long long>(f->expect[slot].second);
        f->detail[2] = static_cast<long long>(bytes);
    }
    if (!f->pending && !f->done) finish(f, M4D_OK, false, nullptr);
}

PyObject* bind(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 3 && nargs != 5 && nargs != 6) {
        PyErr_SetString(PyExc_TypeError, "bind(post_send, post_recv, progress[, take_loan, release_loan[, post_many]])");
        return nullptr;
    }
    void* p[6];
    for (int i = 0; i < nargs; ++i) {
        p[i] = PyLong_AsVoidPtr(args[i]);
        if (!p[i]) {
            if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null function address");
            return nullptr;
        }
    }
    g_send = reinterpret_cast<post_send_fn>(p[0]);
    g_recv = reinterpret_cast<post_recv_fn>(p[1]);
    g_progress = reinterpret_cast<progress_fn>(p[2]);
    if (nargs >= 5) {
        g_take_loan = reinterpret_cast<take_loan_fn>(p[3]);
        g_release_loan = reinterpret_cast<release_loan_fn>(p[4]);
    }
    if (nargs == 6) g_post_many = reinterpret_cast<post_many_fn>(p[5]);
    Py_RETURN_NONE;
}

// post(handle, is_send, channel, peer, tag, data, domain, device_len, req_id)
//   host payload : data = buffer object, device_len = -1
//   device payload: data = int address,  device_len = byte length
PyObject* post(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 9 && nargs != 10) {
        PyErr_SetString(PyExc_TypeError, "post takes 9 or 10 arguments");
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
    const long flags = nargs == 10 ? PyLong_AsLong(args[9]) : 0;  // 1: eager send / loan receive allowed
    if (PyErr_Occurred()) return nullptr;
    m4d_completion now;
    m4d_status st;
    if (device_len >= 0) {
        void* addr = PyLong_AsVoidPtr(args[5]);
        if (PyErr_Occurred()) return nullptr;
        const int on_device = 1 | static_cast<int>((flags & 1) << 1);
        st = is_send ? g_send(t, channel, static_cast<int>(peer), tag, addr, device_len, domain, on_device, req_id, &now)
                     : g_recv(t, channel, static_cast<int>(peer), tag, addr, device_len, domain, on_device, req_id, &now);
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
            if (batch[k].req_id & kSubBit) {
                auto it = g_by_sub.find(batch[k].req_id);
                if (it != g_by_sub.end()) {
                    std::shared_ptr<Framed> f = it->second;
                    g_by_sub.erase(it);
                    on_sub(f, batch[k].req_id, batch[k].status, batch[k].bytes);
                }
                continue;
            }
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
    auto ready = g_ready.find(t);
    if (ready != g_ready.end() && !ready->second.empty()) {
        if (!out && !(out = PyList_New(0))) return nullptr;
        for (const m4d_completion& c : ready->second) {
            PyObject* item = Py_BuildValue("(KiK)", static_cast<unsigned long long>(c.req_id), c.status,
                                           static_cast<unsigned long long>(c.bytes));
            if (!item || PyList_Append(out, item) != 0) {
                Py_XDECREF(item);
                Py_DECREF(out);
                return nullptr;
            }
            Py_DECREF(item);
        }
        ready->second.clear();
    }
    if (!out) Py_RETURN_NONE;
    return out;
}

PyObject* inline_result(const std::shared_ptr<Framed>& f) {
    if (!f->done) Py_RETURN_NONE;
    return Py_BuildValue("(iK)", f->status, static_cast<unsigned long long>(f->payload.size()));
}

// recv_framed(handle, kind, channel, peer, tag, max_chunk, req_id)
PyObject* recv_framed(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if ((nargs != 7 && nargs != 8) || !g_recv) {
        PyErr_SetString(PyExc_TypeError, "recv_framed(handle, kind, channel, peer, tag, max_chunk, req_id[, dev_max])");
        return nullptr;
    }
    auto f = std::make_shared<Framed>();
    f->t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    f->kind = static_cast<int>(PyLong_AsLong(args[1]));
    f->channel = static_cast<uint32_t>(PyLong_AsUnsignedLong(args[2]));
    f->peer = static_cast<int>(PyLong_AsLong(args[3]));
    f->tag = static_cast<uint32_t>(PyLong_AsUnsignedLong(args[4]));
    f->max_chunk = PyLong_AsUnsignedLongLong(args[5]);
    f->id = PyLong_AsUnsignedLongLong(args[6]);
    if (nargs == 8) f->dev_max = PyLong_AsUnsignedLongLong(args[7]);
    if (PyErr_Occurred()) return nullptr;
    if (f->max_chunk < 1) f->max_chunk = 1;
    f->recv = true;
    f->header.resize(f->kind == 0 ? 10 : kMsgHeaderCap);
    g_framed[f->id] = f;
    const int st = post_sub(f, false, f->tag, f->header.data(), f->header.size(), 0);
    if (st != M4D_OK) {
        g_framed.erase(f->id);
        PyErr_SetObject(PyExc_OSError, PyLong_FromLong(st));
        return nullptr;
    }
    if (!f->pending && !f->done) finish(f, f->status, true, nullptr);
    if (f->done) unqueue(f);  // completed inline: reported here, not through progress()
    return inline_result(f);
}

// send_framed(handle, kind, channel, peer, tag, header, frames, max_chunk, req_id)
PyObject* send_framed(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 9 || !g_send) {
        PyErr_SetString(PyExc_TypeError, "send_framed(handle, kind, channel, peer, tag, header, frames, max_chunk, req_id)");
        return nullptr;
    }
    auto f = std::make_shared<Framed>();
    f->t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    f->kind = static_cast<int>(PyLong_AsLong(args[1]));
    f->channel = static_cast<uint32_t>(PyLong_AsUnsignedLong(args[2]));
    f->peer = static_cast<int>(PyLong_AsLong(args[3]));
    f->tag = static_cast<uint32_t>(PyLong_AsUnsignedLong(args[4]));
    f->max_chunk = PyLong_AsUnsignedLongLong(args[7]);
    f->id = PyLong_AsUnsignedLongLong(args[8]);
    if (PyErr_Occurred()) return nullptr;
    if (f->max_chunk < 1) f->max_chunk = 1;
    PyObject* frames = args[6];
    if (!PyTuple_Check(frames)) {
        PyErr_SetString(PyExc_TypeError, "frames must be a tuple of buffers");
        return nullptr;
    }
    const Py_ssize_t nf = PyTuple_GET_SIZE(frames);
    // a frame is a host buffer, or (device address, length): a device frame sent eagerly
    struct Body {
        uint8_t* ptr;
        uint64_t len;
        bool device;
    };
    std::vector<Body> bodies(static_cast<size_t>(nf));
    for (Py_ssize_t i = 0; i < nf; ++i) {
        PyObject* item = PyTuple_GET_ITEM(frames, i);
        if (PyTuple_Check(item)) {
            if (PyTuple_GET_SIZE(item) != 2) {
                PyErr_SetString(PyExc_TypeError, "a device frame is (address, length)");
                return nullptr;
            }
            bodies[static_cast<size_t>(i)] = Body{static_cast<uint8_t*>(PyLong_AsVoidPtr(PyTuple_GET_ITEM(item, 0))),
                                                  PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(item, 1)), true};
            if (PyErr_Occurred()) return nullptr;
        }
    }
    f->views.reserve(static_cast<size_t>(nf) + 1);
    auto fail_views = [&]() {
        release_views(*f);
        return nullptr;
    };
    f->views.emplace_back();
    if (PyObject_GetBuffer(args[5], &f->views.back(), PyBUF_SIMPLE) != 0) { f->views.clear(); return nullptr; }
    for (Py_ssize_t i = 0; i < nf; ++i) {
        Body& b = bodies[static_cast<size_t>(i)];
        if (b.device) continue;
        f->views.emplace_back();
        if (PyObject_GetBuffer(PyTuple_GET_ITEM(frames, i), &f->views.back(), PyBUF_SIMPLE) != 0) {
            f->views.pop_back();
            return fail_views();
        }
        b.ptr = static_cast<uint8_t*>(f->views.back().buf);
        b.len = static_cast<uint64_t>(f->views.back().len);
    }
    g_framed[f->id] = f;
    f->pending = 1;  // guard: the composite cannot finish while its sends are still being posted
    const uint32_t header_tag = f->kind == 0 ? f->tag : static_cast<uint32_t>(kTagMessage);
    int st = post_sub(f, true, header_tag, f->views[0].buf, static_cast<uint64_t>(f->views[0].len), 0);
    for (Py_ssize_t i = 0; i < nf && st == M4D_OK && !f->done; ++i) {
        const Body& b = bodies[static_cast<size_t>(i)];
        const uint32_t tag = f->kind == 0 ? f->tag : static_cast<uint32_t>(data_tag(static_cast<size_t>(i)));
        if (b.device) {  // one eager-capable device send (the caller checked it fits one chunk)
            st = post_sub(f, true, tag, b.ptr, b.len, 0, 1 | 2);
            continue;
        }
        for (uint64_t off = 0; off < b.len && st == M4D_OK && !f->done; off += f->max_chunk) {
            const uint64_t piece = b.len - off < f->max_chunk ? b.len - off : f->max_chunk;
            st = post_sub(f, true, tag, b.ptr + off, piece, off);
        }
    }
    --f->pending;
    if (st != M4D_OK && !f->done) {
        if (f->pending) {
            f->status = st;  // the remaining posted parts still complete; report the failure then
        } else {
            g_framed.erase(f->id);
            release_views(*f);
            PyErr_SetObject(PyExc_OSError, PyLong_FromLong(st));
            return nullptr;
        }
    }
    if (!f->pending && !f->done) finish(f, f->status, true, nullptr);
    if (f->done) unqueue(f);
    return inline_result(f);
}

// take_framed(req_id) -> (outcome, header, payload bytearray | None, (offset, expected, actual))
PyObject* take_framed(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 1) {
        PyErr_SetString(PyExc_TypeError, "take_framed(req_id)");
        return nullptr;
    }
    const uint64_t id = PyLong_AsUnsignedLongLong(args[0]);
    if (PyErr_Occurred()) return nullptr;
    auto it = g_framed.find(id);
    if (it == g_framed.end()) {
        PyErr_SetString(PyExc_KeyError, "no framed result for this request");
        return nullptr;
    }
    std::shared_ptr<Framed> f = it->second;
    g_framed.erase(it);
    PyObject* payload = nullptr;
    if (f->dev) {
        if (f->has_loan && f->outcome == kComplete) {
            payload = Py_BuildValue("(KK)", static_cast<unsigned long long>(f->loan_ptr),
                                    static_cast<unsigned long long>(f->loan_token));
            if (!payload) return nullptr;
        } else {
            if (f->has_loan && g_release_loan) g_release_loan(f->t, f->loan_token);
            Py_INCREF(Py_None);
            payload = Py_None;
        }
    } else if (f->outcome == kComplete) {
        payload = PyByteArray_FromStringAndSize(reinterpret_cast<const char*>(f->payload.data()),
                                                static_cast<Py_ssize_t>(f->payload.size()));
        if (!payload) return nullptr;
    } else {
        Py_INCREF(Py_None);
        payload = Py_None;
    }
    return Py_BuildValue("(iy#N(LLL))", f->outcome, reinterpret_cast<const char*>(f->header.data()),
                         static_cast<Py_ssize_t>(f->header_got), payload, f->detail[0], f->detail[1], f->detail[2]);
}

// forget(handle): drop the composite state of a transport that is closing.
PyObject* forget(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 1) {
        PyErr_SetString(PyExc_TypeError, "forget(handle)");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    if (PyErr_Occurred()) return nullptr;
    for (auto it = g_by_sub.begin(); it != g_by_sub.end();)
        it = it->second->t == t ? g_by_sub.erase(it) : std::next(it);
    for (auto it = g_framed.begin(); it != g_framed.end();) {
        if (it->second->t == t) {
            release_views(*it->second);
            it = g_framed.erase(it);
        } else {
            ++it;
        }
    }
    g_ready.erase(t);
    Py_RETURN_NONE;
}

// post_many(handle, is_send, channel, peer, tag, addrs, lens, domain, on_device, req_ids)
//   device payloads only (addrs: device addresses); one C call for the whole window.
//   -> list of (index, status, bytes) of the posts that completed inline; a failing
//   post raises OSError(status, posted).
PyObject* post_many(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 10 || !g_post_many) {
        PyErr_SetString(PyExc_TypeError, "post_many(handle, is_send, channel, peer, tag, addrs, lens, domain, "
                                         "on_device, req_ids) (bound with post_many)");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    const long is_send = PyLong_AsLong(args[1]);
    const unsigned long channel = PyLong_AsUnsignedLong(args[2]);
    const long peer = PyLong_AsLong(args[3]);
    const unsigned long tag = PyLong_AsUnsignedLong(args[4]);
    const long domain = PyLong_AsLong(args[7]);
    const long on_device = PyLong_AsLong(args[8]);
    if (PyErr_Occurred()) return nullptr;
    PyObject* addrs = args[5];
    PyObject* lens = args[6];
    PyObject* ids = args[9];
    if (!PyTuple_Check(addrs) || !PyTuple_Check(lens) || !PyTuple_Check(ids) ||
        PyTuple_GET_SIZE(addrs) != PyTuple_GET_SIZE(lens) || PyTuple_GET_SIZE(addrs) != PyTuple_GET_SIZE(ids)) {
        PyErr_SetString(PyExc_TypeError, "addrs, lens and req_ids must be tuples of one length");
        return nullptr;
    }
    const Py_ssize_t n = PyTuple_GET_SIZE(addrs);
    std::vector<void*> ptrs(static_cast<size_t>(n));
    std::vector<uint64_t> sizes(static_cast<size_t>(n)), rid(static_cast<size_t>(n));
    for (Py_ssize_t i = 0; i < n; ++i) {
        ptrs[static_cast<size_t>(i)] = PyLong_AsVoidPtr(PyTuple_GET_ITEM(addrs, i));
        sizes[static_cast<size_t>(i)] = PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(lens, i));
        rid[static_cast<size_t>(i)] = PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(ids, i));
    }
    if (PyErr_Occurred()) return nullptr;
    std::vector<m4d_completion> now(static_cast<size_t>(n));
    int posted = 0;
    const m4d_status st = g_post_many(t, is_send ? 1 : 0, static_cast<uint32_t>(channel), static_cast<int>(peer),
                                      static_cast<uint32_t>(tag), ptrs.data(), sizes.data(), static_cast<int>(n),
                                      static_cast<int>(domain), static_cast<int>(1 | (on_device & ~1)), rid.data(),
                                      now.data(), &posted);
    PyObject* out = PyList_New(0);
    if (!out) return nullptr;
    for (int i = 0; i < posted; ++i) {
        if (now[static_cast<size_t>(i)].status == -1) continue;
        PyObject* item = Py_BuildValue("(iiK)", i, now[static_cast<size_t>(i)].status,
                                       static_cast<unsigned long long>(now[static_cast<size_t>(i)].bytes));
        if (!item || PyList_Append(out, item) != 0) {
            Py_XDECREF(item);
            Py_DECREF(out);
            return nullptr;
        }
        Py_DECREF(item);
    }
    if (st != M4D_OK) {
        Py_DECREF(out);
        PyErr_SetObject(PyExc_OSError, Py_BuildValue("(ii)", st, posted));
        return nullptr;
    }
    return out;
}

// loan(handle, req_id) -> (device address, token) of a receive completed by loan, or None
PyObject* loan(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 2 || !g_take_loan) {
        PyErr_SetString(PyExc_TypeError, "loan(handle, req_id) (bound with take_loan)");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    const uint64_t id = PyLong_AsUnsignedLongLong(args[1]);
    if (PyErr_Occurred()) return nullptr;
    uint64_t ptr = 0, token = 0;
    if (!g_take_loan(t, id, &ptr, &token)) Py_RETURN_NONE;
    return Py_BuildValue("(KK)", static_cast<unsigned long long>(ptr), static_cast<unsigned long long>(token));
}

// unloan(handle, token): hand a loaned ring slot back
PyObject* unloan(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 2 || !g_release_loan) {
        PyErr_SetString(PyExc_TypeError, "unloan(handle, token) (bound with release_loan)");
        return nullptr;
    }
    auto* t = static_cast<m4d_transport*>(PyLong_AsVoidPtr(args[0]));
    const uint64_t token = PyLong_AsUnsignedLongLong(args[1]);
    if (PyErr_Occurred()) return nullptr;
    g_release_loan(t, token);
    Py_RETURN_NONE;
}

PyMethodDef methods[] = {
    {"post_many", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(post_many)), METH_FASTCALL,
     "post_many(handle, is_send, channel, peer, tag, addrs, lens, domain, on_device, req_ids) -> [(i, status, bytes)]"},
    {"loan", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(loan)), METH_FASTCALL,
     "loan(handle, req_id) -> (device address, token) | None"},
    {"unloan", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(unloan)), METH_FASTCALL,
     "unloan(handle, token)"},
    {"bind", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(bind)), METH_FASTCALL,
     "bind(post_send, post_recv, progress): C-ABI function addresses from the ctypes loader"},
    {"post", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(post)), METH_FASTCALL,
     "post(handle, is_send, channel, peer, tag, data, domain, device_len, req_id)"},
    {"progress", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(progress)), METH_FASTCALL,
     "progress(handle) -> [(req_id, status, bytes)] or None"},
    {"recv_framed", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(recv_framed)), METH_FASTCALL,
     "recv_framed(handle, kind, channel, peer, tag, max_chunk, req_id) -> None | (status, bytes)"},
    {"send_framed", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(send_framed)), METH_FASTCALL,
     "send_framed(handle, kind, channel, peer, tag, header, frames, max_chunk, req_id) -> None | (status, bytes)"},
    {"forget", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(forget)), METH_FASTCALL,
     "forget(handle): drop the composite state of a closing transport"},
    {"take_framed", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(take_framed)), METH_FASTCALL,
     "take_framed(req_id) -> (outcome, header, payload | None, (offset, expected, actual))"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_m4dfast", "Fast path of the libm4d transport calls.", -1, methods,
                      nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__m4dfast(void) { return PyModule_Create(&module); }
