// Native host-side KJT packing: records -> per-key (values, offsets) int64
// buffers, the CPU half of `build_kjt` (/root/reference/pkg/src/sessiondedup/
// tensors.py:228-254).  The reference walks every row
// with np.asarray per list (~48 ms for cfg1's 4096 rows x 8 keys); here one C++
// pass reads the Python lists in place (PyList/PyTuple fast paths, PyLong
// conversions) and writes each key's IDs into one contiguous int64 buffer,
// ready for the H2D copy.
//
//   pack_rows(rows, keys) -> [(values: bytes, offsets: bytes), ...] per key
//
// Semantics kept: a row is a Mapping or an object with a `.features` mapping
// (tensors.py:228-234); an absent key (or None) is an empty list (237-243); an
// ID list must be one-dimensional (47-51); lists that are not plain Python
// ints go through the optional `convert` callable (np.asarray + 1-D check), so
// floats, numpy arrays and scalars convert or fail exactly as in the reference.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

PyObject* row_features(PyObject* row) {
  // returns a NEW reference to the features mapping, or nullptr with an exception set
  if (PyDict_CheckExact(row)) {  // plain dict records: no attribute lookup
    Py_INCREF(row);
    return row;
  }
  PyObject* feats = PyObject_GetAttrString(row, "features");
  if (feats && feats != Py_None) return feats;
  Py_XDECREF(feats);
  PyErr_Clear();
  if (PyMapping_Check(row) && !PyList_Check(row) && !PyTuple_Check(row)) {
    Py_INCREF(row);
    return row;
  }
  PyErr_Format(PyExc_TypeError, "cannot extract features from %s", Py_TYPE(row)->tp_name);
  return nullptr;
}

// IDs of `seq` through the Python converter (the reference's _as_id_array,
// np.asarray(seq, dtype=int64) + the 1-D check, tensors.py:47-51): used for
// everything the fast path below does not take, so odd inputs (floats, numpy
// arrays of any shape, scalars) behave exactly like the reference.
int append_converted(PyObject* seq, std::vector<int64_t>& out, PyObject* conv) {
  if (!conv) {  // no converter: keep the pending error, or the reference's 1-D text
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "ID list must be one-dimensional");
    return -1;
  }
  PyErr_Clear();
  PyObject* arr = PyObject_CallFunctionObjArgs(conv, seq, nullptr);
  if (!arr) return -1;
  Py_buffer view;
  if (PyObject_GetBuffer(arr, &view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
    Py_DECREF(arr);
    return -1;
  }
  if (view.itemsize != (Py_ssize_t)sizeof(int64_t)) {
    PyBuffer_Release(&view);
    Py_DECREF(arr);
    PyErr_SetString(PyExc_TypeError, "ID converter must return an int64 array");
    return -1;
  }
  const size_t n = (size_t)(view.len / (Py_ssize_t)sizeof(int64_t)), base = out.size();
  out.resize(base + n);
  if (n) std::memcpy(out.data() + base, view.buf, n * sizeof(int64_t));
  PyBuffer_Release(&view);
  Py_DECREF(arr);
  return 0;
}

// append the IDs of `seq` to `out`; -1 with an exception on error.  Fast path:
// a list/tuple of Python ints (or index-like scalars); anything else goes
// through `conv`.
int append_ids(PyObject* seq, std::vector<int64_t>& out, PyObject* conv) {
  if (seq == Py_None) return 0;
  if (conv && !PyList_Check(seq) && !PyTuple_Check(seq)) return append_converted(seq, out, conv);
  PyObject* fast = PySequence_Fast(seq, "ID list must be a sequence");
  if (!fast) return -1;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  const size_t base = out.size();
  out.resize(base + (size_t)n);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* it = items[i];
    long long v = -1;
    bool ok = PyLong_Check(it) || PyIndex_Check(it);
    if (ok) {
      v = PyLong_AsLongLong(it);
      if (v == -1 && PyErr_Occurred()) {
        PyErr_Clear();
        PyObject* idx = PyNumber_Index(it);
        if (idx) {
          v = PyLong_AsLongLong(idx);
          Py_DECREF(idx);
        }
        ok = !(v == -1 && PyErr_Occurred());
      }
    }
    if (!ok) {  // float, nested list, overflow, ...: numpy's conversion decides
      Py_DECREF(fast);
      out.resize(base);
      return append_converted(seq, out, conv);
    }
    out[base + (size_t)i] = (int64_t)v;
  }
  Py_DECREF(fast);
  return 0;
}

PyObject* pack_rows(PyObject*, PyObject* args) {
  PyObject *rows, *keys, *conv = nullptr;
  if (!PyArg_ParseTuple(args, "OO|O", &rows, &keys, &conv)) return nullptr;
  PyObject* rfast = PySequence_Fast(rows, "rows must be a sequence");
  if (!rfast) return nullptr;
  PyObject* kfast = PySequence_Fast(keys, "keys must be a sequence");
  if (!kfast) {
    Py_DECREF(rfast);
    return nullptr;
  }
  const Py_ssize_t B = PySequence_Fast_GET_SIZE(rfast), K = PySequence_Fast_GET_SIZE(kfast);
  std::vector<std::vector<int64_t>> vals((size_t)K), offs((size_t)K);
  for (auto& o : offs) o.reserve((size_t)B);
  PyObject* result = nullptr;
  for (Py_ssize_t i = 0; i < B; ++i) {
    PyObject* feats = row_features(PySequence_Fast_GET_ITEM(rfast, i));
    if (!feats) goto done;
    for (Py_ssize_t k = 0; k < K; ++k) {
      offs[k].push_back((int64_t)vals[k].size());
      PyObject* key = PySequence_Fast_GET_ITEM(kfast, k);
      PyObject* seq;
      if (PyDict_CheckExact(feats)) {  // fast path: borrowed reference, no method call
        seq = PyDict_GetItemWithError(feats, key);
        if (!seq && PyErr_Occurred()) {
          Py_DECREF(feats);
          goto done;
        }
        Py_XINCREF(seq);
        if (!seq) {
          seq = Py_None;
          Py_INCREF(seq);
        }
      } else {
        seq = PyObject_CallMethod(feats, "get", "O", key);
        if (!seq) {
          Py_DECREF(feats);
          goto done;
        }
      }
      const int rc = append_ids(seq, vals[k], conv);
      Py_DECREF(seq);
      if (rc) {
        Py_DECREF(feats);
        goto done;
      }
    }
    Py_DECREF(feats);
  }
  result = PyList_New(K);
  if (!result) goto done;
  for (Py_ssize_t k = 0; k < K; ++k) {
    PyObject* v = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(vals[k].data()),
                                            (Py_ssize_t)(vals[k].size() * sizeof(int64_t)));
    PyObject* o = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(offs[k].data()),
                                            (Py_ssize_t)(offs[k].size() * sizeof(int64_t)));
    if (!v || !o) {
      Py_XDECREF(v);
      Py_XDECREF(o);
      Py_CLEAR(result);
      goto done;
    }
    PyObject* pair = PyTuple_Pack(2, v, o);
    Py_DECREF(v);
    Py_DECREF(o);
    if (!pair) {
      Py_CLEAR(result);
      goto done;
    }
    PyList_SET_ITEM(result, k, pair);
  }
done:
  Py_DECREF(rfast);
  Py_DECREF(kfast);
  return result;
}

PyMethodDef methods[] = {
    {"pack_rows", pack_rows, METH_VARARGS,
     "pack_rows(rows, keys[, convert]) -> [(values bytes, offsets bytes)] per key (int64 little-endian)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostpack", "Native KJT host packing", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__hostpack(void) { return PyModule_Create(&module); }
