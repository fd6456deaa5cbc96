// hostpy.cpp — native host side of the Python boundary (CPython C API).
//
// The device path starts from the reference's own term objects (src/inet/
// core.py:33-155: Var, Agent, Equation, Configuration — slotted classes) and
// must end in them (EvalResult.final). Walking them in Python costs ~30 us per
// net to flatten and ~1 us per agent to rebuild — more than the reduction
// itself for a 4096-net batch or an 8,190-agent tower. This module does both
// walks natively:
//
//   flatten_batch(configs, label_index, Var, Agent, Symbol)
//       -> (agents, agent_off, eqs, eq_off, iface, iface_off, n_vars, var_ids, fresh_base)
//      the flat device input of flat.flatten (same record layout, variables
//      renumbered densely in first-occurrence order, then by original id as
//      the reference's var = var keying needs, engine.py:150-153);
//   unflatten(agents, iface, eqs, syms, var_ids, fresh_base, Var, Agent, Equation, Configuration)
//      -> Configuration
//      the reverse of flat.unflatten (preorder records, children after parents).
//
// Objects are read and built through their slot offsets (member descriptors
// of the reference classes), as the interpreter itself does for __slots__; any
// object of another class takes the generic attribute path. Errors raise
// LookupError (an unknown symbol: the caller falls back to the Python path)
// or the usual Python exceptions.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

namespace {

constexpr uint32_t kVar = 0x80000000u;
constexpr uint32_t kNone = 0xFFFFFFFFu;

// Offset of slot `name` of `type` (a member descriptor), or -1.
Py_ssize_t slot_offset(PyObject* type, const char* name) {
  PyObject* d = PyObject_GetAttrString(type, name);
  if (!d) {
    PyErr_Clear();
    return -1;
  }
  Py_ssize_t off = -1;
  if (PyObject_TypeCheck(d, &PyMemberDescr_Type)) {
    PyMemberDef* m = reinterpret_cast<PyMemberDescrObject*>(d)->d_member;
    if (m->type == T_OBJECT_EX || m->type == T_OBJECT) off = m->offset;
  }
  Py_DECREF(d);
  return off;
}

struct Slot {
  PyTypeObject* type = nullptr;
  Py_ssize_t off = -1;
  PyObject* name = nullptr;  // interned attribute name (generic path)
  bool init(PyObject* t, const char* n) {
    type = reinterpret_cast<PyTypeObject*>(t);
    off = slot_offset(t, n);
    name = PyUnicode_InternFromString(n);
    return name != nullptr;
  }
  // new reference
  PyObject* get(PyObject* o) const {
    if (off >= 0 && Py_TYPE(o) == type) {
      PyObject* v = *reinterpret_cast<PyObject**>(reinterpret_cast<char*>(o) + off);
      if (v) {
        Py_INCREF(v);
        return v;
      }
    }
    return PyObject_GetAttr(o, name);
  }
  ~Slot() { Py_XDECREF(name); }
};

// An instance of a slotted class with its slots set (steals nothing; INCREFs values).
PyObject* make_slotted(PyTypeObject* type, const Py_ssize_t* offs, PyObject* const* vals, int n) {
  PyObject* o = type->tp_alloc(type, 0);
  if (!o) return nullptr;
  for (int k = 0; k < n; ++k) {
    Py_INCREF(vals[k]);
    *reinterpret_cast<PyObject**>(reinterpret_cast<char*>(o) + offs[k]) = vals[k];
  }
  return o;
}

PyObject* bytes_of(const void* p, size_t n) { return PyBytes_FromStringAndSize(static_cast<const char*>(p), n); }

// ---------------------------------------------------------------------------

PyObject* flatten_batch(PyObject*, PyObject* args) {
  PyObject *configs, *label_index, *var_t, *agent_t, *sym_t;
  if (!PyArg_ParseTuple(args, "OO!OOO", &configs, &PyDict_Type, &label_index, &var_t, &agent_t, &sym_t)) return nullptr;
  Slot s_id, s_sym, s_children, s_name, s_iface, s_eqs, s_lhs, s_rhs;
  if (!s_id.init(var_t, "id") || !s_sym.init(agent_t, "sym") || !s_children.init(agent_t, "children") ||
      !s_name.init(sym_t, "name"))
    return nullptr;
  PyObject* seq = PySequence_Fast(configs, "configs must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t N = PySequence_Fast_GET_SIZE(seq);
  std::vector<uint32_t> agents, eqs, iface, n_vars;
  std::vector<uint64_t> agent_off{0}, eq_off{0}, iface_off{0};
  PyObject* var_ids_all = PyList_New(N);
  PyObject* fresh_all = PyList_New(N);
  std::unordered_map<long long, uint32_t> dense;
  std::vector<long long> ids;
  std::vector<std::pair<PyObject*, uint32_t>> work;  // (term, record index)
  bool ok = var_ids_all && fresh_all;
  PyObject *attr_iface = PyUnicode_InternFromString("interface"), *attr_eqs = PyUnicode_InternFromString("equations"),
           *attr_lhs = PyUnicode_InternFromString("lhs"), *attr_rhs = PyUnicode_InternFromString("rhs");
  for (Py_ssize_t c = 0; ok && c < N; ++c) {
    PyObject* cfg = PySequence_Fast_GET_ITEM(seq, c);
    dense.clear();
    ids.clear();
    const size_t a0 = agents.size() / 4, e0 = eqs.size(), i0 = iface.size();
    // term -> ref; agents appended with their ports filled from a work list
    auto var_ref = [&](PyObject* t, uint32_t& out) -> bool {
      PyObject* idv = s_id.get(t);
      if (!idv) return false;
      const long long id = PyLong_AsLongLong(idv);
      Py_DECREF(idv);
      if (id == -1 && PyErr_Occurred()) return false;
      auto it = dense.find(id);
      if (it == dense.end()) {
        if (ids.size() >= kVar - 1) {
          PyErr_SetString(PyExc_OverflowError, "too many variables");
          return false;
        }
        it = dense.emplace(id, static_cast<uint32_t>(ids.size())).first;
        ids.push_back(id);
      }
      out = kVar | it->second;
      return true;
    };
    auto ref = [&](PyObject* t, uint32_t& out) -> bool {
      if (Py_TYPE(t) == reinterpret_cast<PyTypeObject*>(var_t) ||
          (Py_TYPE(t) != reinterpret_cast<PyTypeObject*>(agent_t) && !PyObject_HasAttr(t, s_sym.name)))
        return var_ref(t, out);
      const size_t root = agents.size() / 4 - a0;
      agents.insert(agents.end(), {0u, kNone, kNone, kNone});
      work.clear();
      work.emplace_back(t, static_cast<uint32_t>(root));
      while (!work.empty()) {
        auto [x, slot] = work.back();
        work.pop_back();
        PyObject* sym = s_sym.get(x);
        if (!sym) return false;
        PyObject* name = s_name.get(sym);
        Py_DECREF(sym);
        if (!name) return false;
        PyObject* lab = PyDict_GetItemWithError(label_index, name);
        Py_DECREF(name);
        if (!lab) {
          if (!PyErr_Occurred()) PyErr_SetString(PyExc_LookupError, "symbol not in the label table");
          return false;
        }
        const long labv = PyLong_AsLong(lab);
        PyObject* kids = s_children.get(x);
        if (!kids) return false;
        PyObject* kseq = PySequence_Fast(kids, "children must be a sequence");
        Py_DECREF(kids);
        if (!kseq) return false;
        const Py_ssize_t ar = PySequence_Fast_GET_SIZE(kseq);
        if (ar > 3) {
          Py_DECREF(kseq);
          PyErr_SetString(PyExc_LookupError, "arity > 3");
          return false;
        }
        uint32_t* rec = &agents[4 * (a0 + slot)];
        rec[0] = static_cast<uint32_t>(labv);
        for (Py_ssize_t k = 0; k < ar; ++k) {
          PyObject* ch = PySequence_Fast_GET_ITEM(kseq, k);
          uint32_t r;
          if (Py_TYPE(ch) == reinterpret_cast<PyTypeObject*>(agent_t) ||
              (Py_TYPE(ch) != reinterpret_cast<PyTypeObject*>(var_t) && PyObject_HasAttr(ch, s_sym.name))) {
            r = static_cast<uint32_t>(agents.size() / 4 - a0);
            agents.insert(agents.end(), {0u, kNone, kNone, kNone});
            work.emplace_back(ch, r);
          } else if (!var_ref(ch, r)) {
            Py_DECREF(kseq);
            return false;
          }
          agents[4 * (a0 + slot) + 1 + k] = r;  // (agents may have grown: index again)
        }
        Py_DECREF(kseq);
      }
      out = static_cast<uint32_t>(root);
      return true;
    };
    PyObject* ifc = PyObject_GetAttr(cfg, attr_iface);
    PyObject* eql = ifc ? PyObject_GetAttr(cfg, attr_eqs) : nullptr;
    PyObject* ifs = eql ? PySequence_Fast(ifc, "interface") : nullptr;
    PyObject* eqs_s = ifs ? PySequence_Fast(eql, "equations") : nullptr;
    ok = eqs_s != nullptr;
    for (Py_ssize_t k = 0; ok && k < PySequence_Fast_GET_SIZE(ifs); ++k) {
      uint32_t r;
      ok = ref(PySequence_Fast_GET_ITEM(ifs, k), r);
      if (ok) iface.push_back(r);
    }
    for (Py_ssize_t k = 0; ok && k < PySequence_Fast_GET_SIZE(eqs_s); ++k) {
      PyObject* e = PySequence_Fast_GET_ITEM(eqs_s, k);
      PyObject* l = PyObject_GetAttr(e, attr_lhs);
      PyObject* r = l ? PyObject_GetAttr(e, attr_rhs) : nullptr;
      uint32_t rl = 0, rr = 0;
      ok = r && ref(l, rl) && ref(r, rr);
      Py_XDECREF(l);
      Py_XDECREF(r);
      if (ok) {
        eqs.push_back(rl);
        eqs.push_back(rr);
      }
    }
    Py_XDECREF(ifc);
    Py_XDECREF(eql);
    Py_XDECREF(ifs);
    Py_XDECREF(eqs_s);
    if (!ok) break;
    // dense ids in the order of the original ids (the reference keys var = var on
    // the smaller id, engine.py:150-153)
    const size_t nv = ids.size();
    long long max_id = -1;
    for (long long v : ids) max_id = std::max(max_id, v);
    if (!std::is_sorted(ids.begin(), ids.end())) {
      std::vector<uint32_t> order(nv), rank(nv);
      std::iota(order.begin(), order.end(), 0u);
      std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ids[a] < ids[b]; });
      for (uint32_t k = 0; k < nv; ++k) rank[order[k]] = k;
      auto remap = [&](uint32_t& r) {
        if (r != kNone && (r & kVar)) r = kVar | rank[r & ~kVar];
      };
      for (size_t k = 4 * a0; k < agents.size(); ++k)
        if (k % 4) remap(agents[k]);
      for (size_t k = e0; k < eqs.size(); ++k) remap(eqs[k]);
      for (size_t k = i0; k < iface.size(); ++k) remap(iface[k]);
      std::vector<long long> sorted(nv);
      for (uint32_t k = 0; k < nv; ++k) sorted[k] = ids[order[k]];
      ids.swap(sorted);
    }
    PyObject* vl = PyList_New(static_cast<Py_ssize_t>(nv));
    if (!vl) {
      ok = false;
      break;
    }
    for (size_t k = 0; k < nv; ++k) PyList_SET_ITEM(vl, k, PyLong_FromLongLong(ids[k]));
    PyList_SET_ITEM(var_ids_all, c, vl);
    PyList_SET_ITEM(fresh_all, c, PyLong_FromLongLong(max_id + 1));
    n_vars.push_back(static_cast<uint32_t>(nv));
    agent_off.push_back(agents.size() / 4);
    eq_off.push_back(eqs.size() / 2);
    iface_off.push_back(iface.size());
  }
  Py_DECREF(attr_iface);
  Py_DECREF(attr_eqs);
  Py_DECREF(attr_lhs);
  Py_DECREF(attr_rhs);
  Py_DECREF(seq);
  if (!ok) {
    Py_XDECREF(var_ids_all);
    Py_XDECREF(fresh_all);
    return nullptr;
  }
  return Py_BuildValue("(NNNNNNNNN)", bytes_of(agents.data(), agents.size() * 4),
                       bytes_of(agent_off.data(), agent_off.size() * 8), bytes_of(eqs.data(), eqs.size() * 4),
                       bytes_of(eq_off.data(), eq_off.size() * 8), bytes_of(iface.data(), iface.size() * 4),
                       bytes_of(iface_off.data(), iface_off.size() * 8), bytes_of(n_vars.data(), n_vars.size() * 4),
                       var_ids_all, fresh_all);
}

// ---------------------------------------------------------------------------

PyObject* unflatten(PyObject*, PyObject* args) {
  Py_buffer ab{}, ib{}, eb{};
  PyObject *syms, *var_ids, *fresh_base, *var_t, *agent_t, *eq_t, *cfg_t;
  if (!PyArg_ParseTuple(args, "y*y*y*OOOOOOO", &ab, &ib, &eb, &syms, &var_ids, &fresh_base, &var_t, &agent_t, &eq_t,
                        &cfg_t))
    return nullptr;
  struct Release {
    Py_buffer* b[3];
    ~Release() {
      for (Py_buffer* x : b) PyBuffer_Release(x);
    }
  } rel{{&ab, &ib, &eb}};
  const uint32_t* ag = static_cast<const uint32_t*>(ab.buf);
  const uint32_t* ifc = static_cast<const uint32_t*>(ib.buf);
  const uint32_t* eq = static_cast<const uint32_t*>(eb.buf);
  const size_t na = ab.len / 16, ni = ib.len / 4, ne = eb.len / 8;
  const Py_ssize_t off_id = slot_offset(var_t, "id");
  const Py_ssize_t off_ag[2] = {slot_offset(agent_t, "sym"), slot_offset(agent_t, "children")};
  const Py_ssize_t off_eq[2] = {slot_offset(eq_t, "lhs"), slot_offset(eq_t, "rhs")};
  const Py_ssize_t off_cf[2] = {slot_offset(cfg_t, "interface"), slot_offset(cfg_t, "equations")};
  const bool fast = off_id >= 0 && off_ag[0] >= 0 && off_ag[1] >= 0 && off_eq[0] >= 0 && off_eq[1] >= 0 &&
                    off_cf[0] >= 0 && off_cf[1] >= 0;
  PyObject* sym_seq = PySequence_Fast(syms, "syms");
  PyObject* vid_seq = sym_seq ? PySequence_Fast(var_ids, "var_ids") : nullptr;
  if (!vid_seq) {
    Py_XDECREF(sym_seq);
    return nullptr;
  }
  const Py_ssize_t n_in = PySequence_Fast_GET_SIZE(vid_seq);
  const long long base = PyLong_AsLongLong(fresh_base);
  std::vector<PyObject*> arity_of;  // label -> arity (borrowed ints not needed: compute)
  const Py_ssize_t L = PySequence_Fast_GET_SIZE(sym_seq);
  std::vector<int> arity(L, 0);
  PyObject* s_ar = PyUnicode_InternFromString("arity");
  for (Py_ssize_t l = 0; l < L; ++l) {
    PyObject* a = PyObject_GetAttr(PySequence_Fast_GET_ITEM(sym_seq, l), s_ar);
    arity[l] = a ? static_cast<int>(PyLong_AsLong(a)) : 0;
    Py_XDECREF(a);
  }
  Py_DECREF(s_ar);
  std::unordered_map<uint32_t, PyObject*> vars;
  bool ok = true;
  auto var = [&](uint32_t d) -> PyObject* {  // borrowed (owned by `vars`)
    auto it = vars.find(d);
    if (it != vars.end()) return it->second;
    PyObject* idv = d < static_cast<uint32_t>(n_in) ? PySequence_Fast_GET_ITEM(vid_seq, d) : nullptr;
    PyObject* own = idv ? nullptr : PyLong_FromLongLong(base + (static_cast<long long>(d) - n_in));
    PyObject* idobj = idv ? idv : own;
    PyObject* v = nullptr;
    if (idobj) v = fast ? make_slotted(reinterpret_cast<PyTypeObject*>(var_t), &off_id, &idobj, 1)
                        : PyObject_CallOneArg(var_t, idobj);
    Py_XDECREF(own);
    if (!v) {
      ok = false;
      return nullptr;
    }
    vars.emplace(d, v);
    return v;
  };
  std::vector<PyObject*> built(na, nullptr);
  PyObject* empty = PyTuple_New(0);
  for (size_t a = na; ok && a-- > 0;) {
    const uint32_t* rec = ag + 4 * a;
    if (rec[0] >= static_cast<uint32_t>(L)) {
      PyErr_SetString(PyExc_ValueError, "label out of range");
      ok = false;
      break;
    }
    const int ar = arity[rec[0]];
    PyObject* kids = ar ? PyTuple_New(ar) : (Py_INCREF(empty), empty);
    for (int k = 0; ok && k < ar; ++k) {
      const uint32_t p = rec[1 + k];
      PyObject* ch = (p & kVar) ? var(p & ~kVar) : (p < na ? built[p] : nullptr);
      if (!ch) {
        if (ok) PyErr_SetString(PyExc_ValueError, "dangling port");
        ok = false;
        break;
      }
      Py_INCREF(ch);
      PyTuple_SET_ITEM(kids, k, ch);
    }
    if (!ok) {
      Py_DECREF(kids);
      break;
    }
    PyObject* vals[2] = {PySequence_Fast_GET_ITEM(sym_seq, rec[0]), kids};
    PyObject* o = fast ? make_slotted(reinterpret_cast<PyTypeObject*>(agent_t), off_ag, vals, 2)
                       : PyObject_CallFunctionObjArgs(agent_t, vals[0], kids, nullptr);
    Py_DECREF(kids);
    if (!o) ok = false;
    built[a] = o;
  }
  auto term = [&](uint32_t r) -> PyObject* {  // borrowed
    if (r & kVar) return var(r & ~kVar);
    return r < na ? built[r] : nullptr;
  };
  PyObject *ift = nullptr, *eqt = nullptr, *result = nullptr;
  if (ok) {
    ift = PyTuple_New(static_cast<Py_ssize_t>(ni));
    for (size_t k = 0; ok && k < ni; ++k) {
      PyObject* t = term(ifc[k]);
      if (!t) ok = false;
      else {
        Py_INCREF(t);
        PyTuple_SET_ITEM(ift, k, t);
      }
    }
  }
  if (ok) {
    eqt = PyTuple_New(static_cast<Py_ssize_t>(ne));
    for (size_t k = 0; ok && k < ne; ++k) {
      PyObject* sides[2] = {term(eq[2 * k]), term(eq[2 * k + 1])};
      if (!sides[0] || !sides[1]) {
        ok = false;
        break;
      }
      PyObject* e = fast ? make_slotted(reinterpret_cast<PyTypeObject*>(eq_t), off_eq, sides, 2)
                         : PyObject_CallFunctionObjArgs(eq_t, sides[0], sides[1], nullptr);
      if (!e) ok = false;
      else PyTuple_SET_ITEM(eqt, k, e);
    }
  }
  if (ok) {
    PyObject* parts[2] = {ift, eqt};
    result = fast ? make_slotted(reinterpret_cast<PyTypeObject*>(cfg_t), off_cf, parts, 2)
                  : PyObject_CallFunctionObjArgs(cfg_t, ift, eqt, nullptr);
  }
  if (!ok && !PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "malformed normal form");
  Py_XDECREF(ift);
  Py_XDECREF(eqt);
  for (PyObject* o : built) Py_XDECREF(o);
  for (auto& kv : vars) Py_DECREF(kv.second);
  Py_DECREF(empty);
  Py_DECREF(sym_seq);
  Py_DECREF(vid_seq);
  return result;
}

PyMethodDef methods[] = {
    {"flatten_batch", flatten_batch, METH_VARARGS, "configs -> flat device input (see hostpy.cpp)"},
    {"unflatten", unflatten, METH_VARARGS, "flat normal form -> Configuration of the given classes"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostpy", "native term flattening / rebuilding", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__hostpy(void) { return PyModule_Create(&module); }
