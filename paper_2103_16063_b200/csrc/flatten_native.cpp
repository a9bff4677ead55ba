#include <unordered_map>
// Host-side flattening of an AtomicPartition + CostModel into the atom-level
// arrays of partition_blocks (paper_2103_16063_b200/flatten.py:
// _flatten_atoms, blocks.py:73-124), natively: the same traversal of the
// reference's graph objects without the interpreter loop.  It covers the
// common case -- every byte count an exact integer that fits int64, no
// structural violation; anything else raises Fallback and the Python
// implementation runs (and raises the reference's errors).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <unordered_map>
#include <vector>

namespace py = pybind11;

namespace {

struct Fallback {};

// attribute names interned once; ga() = getattr with a new reference
struct Names {
    py::str value{"value"}, is_param{"is_param"}, fixed_bytes{"fixed_bytes"},
        bytes_per_sample{"bytes_per_sample"}, task{"task"}, flops_per_sample{"flops_per_sample"};
};
const Names &names() {
    static Names *n = new Names();
    return *n;
}
inline py::object ga(py::handle o, const py::str &name) {
    PyObject *r = PyObject_GetAttr(o.ptr(), name.ptr());
    if (!r) throw py::error_already_set();
    return py::reinterpret_steal<py::object>(r);
}
inline py::handle dget(py::handle dict, py::handle key) {   // borrowed
    PyObject *r = PyDict_GetItem(dict.ptr(), key.ptr());
    if (!r) throw Fallback();
    return r;
}

// an exact integer byte count (flatten.py: _as_int), else Fallback
int64_t as_int(PyObject *x) {
    if (PyLong_CheckExact(x)) {
        int overflow = 0;
        const long long v = PyLong_AsLongLongAndOverflow(x, &overflow);
        if (overflow) throw Fallback();
        return v;
    }
    if (PyFloat_Check(x)) {
        const double d = PyFloat_AS_DOUBLE(x);
        if (!(d == std::floor(d)) || std::fabs(d) >= 9007199254740992.0) throw Fallback();
        return (int64_t)d;
    }
    throw Fallback();
}

int64_t size1(const py::handle &info) {
    return as_int(ga(info, names().fixed_bytes).ptr()) + as_int(ga(info, names().bytes_per_sample).ptr());
}

template <class T>
py::array_t<T> arr(const std::vector<T> &v) {
    py::array_t<T> a(v.size());
    if (!v.empty()) std::copy(v.begin(), v.end(), a.mutable_data());
    return a;
}

void csr(const std::vector<std::vector<int32_t>> &lists, std::vector<int32_t> &off,
         std::vector<int32_t> &flat) {
    off.assign(lists.size() + 1, 0);
    flat.clear();
    for (size_t i = 0; i < lists.size(); ++i) {
        flat.insert(flat.end(), lists[i].begin(), lists[i].end());
        off[i + 1] = (int32_t)flat.size();
    }
}

py::dict flatten(py::object partition, py::object model) {
    py::object g = model.attr("graph");
    py::object pg = partition.attr("graph");
    py::list atoms = partition.attr("atoms");
    const int n = (int)py::len(atoms);
    py::dict nodes = g.attr("nodes");
    // the graph's adjacency dicts (graph.py:56-57: node id -> sorted tuple); a
    // different reference layout falls back to the Python path
    py::dict succ_d = g.attr("_succ"), pred_d = g.attr("_pred");
    py::object graph_inputs = g.attr("inputs");
    py::object none = py::none();

    // node id -> atom (atoms.py:259-305); duplicates are the Python path's error
    py::dict atom_of;
    for (int i = 0; i < n; ++i) {
        py::int_ idx(i);
        for (py::handle nid : py::reinterpret_borrow<py::object>(atoms[i].attr("node_ids")))
            if (PyDict_SetDefault(atom_of.ptr(), nid.ptr(), idx.ptr()) != idx.ptr()) throw Fallback();
    }
    auto atom_get = [&](py::handle k) -> int {
        PyObject *v = PyDict_GetItem(atom_of.ptr(), k.ptr());
        return v ? (int)PyLong_AsLong(v) : -1;
    };

    // per value node (keyed by the node object): is it a value, a parameter,
    // its bytes at microbatch 1 -- read once, used by every reader
    struct VInfo {
        bool is_value = false, is_param = false, size_ok = false;
        int64_t size = 0;
    };
    std::unordered_map<PyObject *, VInfo> vcache;
    vcache.reserve(2 * (size_t)py::len(nodes) + 16);
    auto vinfo = [&](py::handle node) -> const VInfo & {
        auto it = vcache.find(node.ptr());
        if (it != vcache.end()) return it->second;
        VInfo x;
        py::object value = ga(node, names().value);
        x.is_value = !value.is_none();
        if (x.is_value) {
            x.is_param = PyObject_IsTrue(ga(value, names().is_param).ptr()) == 1;
            try {
                x.size = size1(value);
                x.size_ok = true;
            } catch (Fallback &) {
            }
        }
        return vcache.emplace(node.ptr(), x).first->second;
    };
    auto vsize = [](const VInfo &x) -> int64_t {
        if (!x.size_ok) throw Fallback();
        return x.size;
    };

    std::vector<py::object> inputs_of_atom(n);
    py::dict listing;
    for (int a = 0; a < n; ++a) {
        py::int_ idx(a);
        inputs_of_atom[a] = py::reinterpret_steal<py::object>(
            PyFrozenSet_New(atoms[a].attr("input_values").ptr()));
        for (py::handle v : inputs_of_atom[a]) {
            PyObject *lst = PyDict_GetItem(listing.ptr(), v.ptr());
            if (!lst) {
                py::list l;
                l.append(idx);
                listing[v] = l;
            } else {
                PyList_Append(lst, idx.ptr());
            }
        }
    }
    py::list in_ids = py::module_::import("builtins").attr("sorted")(listing);
    py::dict in_index;
    std::vector<int32_t> in_owner, in_atoms_off{0}, in_atoms;
    std::vector<int64_t> in_size;
    for (size_t i = 0; i < py::len(in_ids); ++i) {
        py::handle v = in_ids[i];
        in_index[v] = py::int_(i);
        const VInfo &vi = vinfo(dget(nodes, v));
        if (!vi.is_value) throw Fallback();
        const int own = atom_get(v);
        const bool is_input = PySequence_Contains(graph_inputs.ptr(), v.ptr()) == 1;
        in_owner.push_back((is_input || own < 0) ? -1 : own);
        in_size.push_back(vsize(vi));
        for (py::handle a : py::reinterpret_borrow<py::list>(dget(listing, v)))
            in_atoms.push_back((int32_t)PyLong_AsLong(a.ptr()));
        in_atoms_off.push_back((int32_t)in_atoms.size());
    }
    auto in_index_of = [&](py::handle v) -> int {
        PyObject *x = PyDict_GetItem(in_index.ptr(), v.ptr());
        return x ? (int)PyLong_AsLong(x) : -1;
    };

    std::vector<int64_t> atom_param(n, 0), task_fp1, task_prod1, dep_size;
    std::vector<int32_t> task_atom, dep_off{0}, dep_owner;
    std::vector<double> task_flops;
    std::vector<std::vector<int32_t>> atom_tasks(n);
    py::list tnodes;
    for (auto item : nodes) {                       // sorted id order (graph.py:90-93)
        py::handle nid = item.first, node = item.second;
        const int a = atom_get(nid);
        if (a < 0) continue;
        const Names &N = names();
        const VInfo &self = vinfo(node);
        if (self.is_value) {
            if (self.is_param)
                atom_param[a] += as_int(ga(ga(node, N.value), N.fixed_bytes).ptr());
            continue;
        }
        int64_t fp = 0;
        for (py::handle vid : dget(succ_d, nid)) {
            const VInfo &x = vinfo(dget(nodes, vid));
            if (x.is_value && !x.is_param) fp += vsize(x);
        }
        task_prod1.push_back(fp);
        py::object task = ga(node, N.task);
        tnodes.append(task);
        const py::object &ins = inputs_of_atom[a];
        for (py::handle vid : dget(pred_d, nid)) {
            const VInfo &x = vinfo(dget(nodes, vid));
            if (!x.is_value || x.is_param) continue;
            if (PySet_Contains(ins.ptr(), vid.ptr()) == 1) {
                const int own = in_owner[in_index_of(vid)];
                if (own >= 0) {
                    dep_owner.push_back(own);
                    dep_size.push_back(vsize(x));
                }
            } else {
                if (atom_get(vid) != a) throw Fallback();     // cross-atom read: Python raises
                fp += vsize(x);
            }
        }
        dep_off.push_back((int32_t)dep_owner.size());
        atom_tasks[a].push_back((int32_t)task_atom.size());
        task_atom.push_back(a);
        task_flops.push_back(PyFloat_AsDouble(ga(task, N.flops_per_sample).ptr()));
        task_fp1.push_back(fp);
    }

    // atom dependencies (atoms.py:115-125) and traffic entries (blocks.py:96-102)
    // atoms.py:93-106: value id -> owner atom / frozenset of consumer atoms
    py::dict owner_d = partition.attr("_value_owner");
    py::dict cons_d = partition.attr("_consumer_atoms");
    py::dict ppred_d = pg.attr("_pred");
    py::dict pnodes = pg.attr("nodes");
    std::vector<int64_t> dep_keys;
    std::vector<int32_t> tr_owner;
    std::vector<int64_t> tr_size;
    std::vector<std::vector<int32_t>> tr_cons, atom_tr(n);
    for (auto item : pnodes) {                      // value_ids() (graph.py:140-141)
        py::handle vid = item.first;
        const VInfo &vi = vinfo(item.second);
        if (!vi.is_value) continue;
        const int owner = (int)PyLong_AsLong(dget(owner_d, vid).ptr());
        std::vector<int32_t> cons;
        for (py::handle c : dget(cons_d, vid)) cons.push_back((int32_t)PyLong_AsLong(c.ptr()));
        std::sort(cons.begin(), cons.end());
        if (PyTuple_GET_SIZE(dget(ppred_d, vid).ptr()) > 0)     // graph.py:84-88: a producer
            for (int c : cons)
                if (c != owner) dep_keys.push_back((int64_t)owner * n + c);
        std::vector<int32_t> foreign;
        for (int c : cons)
            if (c != owner) foreign.push_back(c);
        if (!foreign.empty()) {
            const int e = (int)tr_owner.size();
            tr_owner.push_back(owner);
            tr_size.push_back(vsize(vi));                  // value_size(vid, 1) (graph.py:151-155)
            std::vector<int32_t> members(foreign);
            members.push_back(owner);
            std::sort(members.begin(), members.end());
            members.erase(std::unique(members.begin(), members.end()), members.end());
            for (int x : members) atom_tr[x].push_back(e);
            tr_cons.push_back(std::move(foreign));
        }
    }
    std::sort(dep_keys.begin(), dep_keys.end());
    dep_keys.erase(std::unique(dep_keys.begin(), dep_keys.end()), dep_keys.end());
    std::vector<std::vector<int32_t>> succ(n), pred(n), nbr(n);
    for (int64_t k : dep_keys) {
        const int a = (int)(k / n), b = (int)(k % n);
        succ[a].push_back(b);
        pred[b].push_back(a);
    }
    for (int i = 0; i < n; ++i) {
        std::vector<int32_t> u(succ[i]);
        u.insert(u.end(), pred[i].begin(), pred[i].end());
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        nbr[i] = std::move(u);
    }

    // inputs of each atom by in_ids index, ascending (sorted(ins) then index)
    std::vector<std::vector<int32_t>> atom_in(n);
    for (int a = 0; a < n; ++a) {
        for (py::handle v : inputs_of_atom[a]) atom_in[a].push_back(in_index_of(v));
        std::sort(atom_in[a].begin(), atom_in[a].end());
    }

    py::dict out;
    std::vector<int32_t> off, flat;
    auto put_csr = [&](const char *o, const char *f, const std::vector<std::vector<int32_t>> &l) {
        csr(l, off, flat);
        out[o] = arr(off);
        out[f] = arr(flat);
    };
    out["n"] = n;
    out["atom_param"] = arr(atom_param);
    out["task_atom"] = arr(task_atom);
    out["task_flops"] = arr(task_flops);
    out["task_fp1"] = arr(task_fp1);
    out["task_prod1"] = arr(task_prod1);
    out["dep_off"] = arr(dep_off);
    out["dep_owner"] = arr(dep_owner);
    out["dep_size"] = arr(dep_size);
    put_csr("atom_task_off", "atom_tasks", atom_tasks);
    put_csr("atom_in_off", "atom_in", atom_in);
    out["in_owner"] = arr(in_owner);
    out["in_size"] = arr(in_size);
    out["in_atoms_off"] = arr(in_atoms_off);
    out["in_atoms"] = arr(in_atoms);
    put_csr("succ_off", "succ", succ);
    put_csr("pred_off", "pred", pred);
    put_csr("nbr_off", "nbr", nbr);
    out["tr_owner"] = arr(tr_owner);
    out["tr_size"] = arr(tr_size);
    put_csr("tr_cons_off", "tr_cons", tr_cons);
    put_csr("atom_tr_off", "atom_tr", atom_tr);
    out["tnodes"] = tnodes;
    return out;
}

// Block-level arrays of the span profile (flatten.py: flatten_blockset,
// costs.py:97-160 over BlockSet spans).  Same conventions: the common case
// natively, every structural violation -> Fallback (the Python restatement
// raises UnsupportedGraph with its message).
py::dict flatten_blocks(py::object bs) {
    const Names &N = names();
    py::object model = bs.attr("model");
    py::object g = model.attr("graph");
    py::object part = bs.attr("partition");
    py::list atoms = part.attr("atoms");
    const int n_atoms = (int)py::len(atoms);
    py::tuple block_atoms = bs.attr("block_atoms");
    const int nb = (int)py::len(block_atoms);
    py::dict nodes = g.attr("nodes");
    py::dict succ_d = g.attr("_succ"), pred_d = g.attr("_pred");
    py::object graph_inputs = g.attr("inputs");

    py::dict atom_of;
    for (int i = 0; i < n_atoms; ++i) {
        py::int_ idx(i);
        for (py::handle nid : py::reinterpret_borrow<py::object>(atoms[i].attr("node_ids")))
            if (PyDict_SetDefault(atom_of.ptr(), nid.ptr(), idx.ptr()) != idx.ptr()) throw Fallback();
    }
    // per value node (keyed by the node object): value?, parameter?, its two
    // byte counts -- read once, used by every reader
    struct VInfo {
        bool is_value = false, is_param = false, ok = false;
        int64_t fix = 0, ps = 0;
    };
    std::unordered_map<PyObject *, VInfo> vcache;
    vcache.reserve(2 * (size_t)py::len(nodes) + 16);
    auto vinfo = [&](py::handle node) -> const VInfo & {
        auto it = vcache.find(node.ptr());
        if (it != vcache.end()) return it->second;
        VInfo x;
        py::object value = ga(node, N.value);
        x.is_value = !value.is_none();
        if (x.is_value) {
            x.is_param = PyObject_IsTrue(ga(value, N.is_param).ptr()) == 1;
            try {
                x.fix = as_int(ga(value, N.fixed_bytes).ptr());
                x.ps = as_int(ga(value, N.bytes_per_sample).ptr());
                x.ok = true;
            } catch (Fallback &) {
            }
        }
        return vcache.emplace(node.ptr(), x).first->second;
    };
    auto need = [](const VInfo &x) -> const VInfo & {
        if (!x.ok) throw Fallback();
        return x;
    };
    std::vector<int> block_of_atom(n_atoms, -1);
    int covered = 0;
    for (int bi = 0; bi < nb; ++bi)
        for (py::handle a : py::reinterpret_borrow<py::object>(block_atoms[bi])) {
            const long ai = PyLong_AsLong(a.ptr());
            if (ai < 0 || ai >= n_atoms) throw Fallback();
            if (block_of_atom[ai] < 0) ++covered;
            block_of_atom[ai] = bi;
        }
    if (covered != n_atoms) throw Fallback();
    auto atom_get = [&](py::handle k) -> int {
        PyObject *v = PyDict_GetItem(atom_of.ptr(), k.ptr());
        return v ? (int)PyLong_AsLong(v) : -1;
    };
    auto blk_of = [&](py::handle k) -> int {
        const int a = atom_get(k);
        return a < 0 ? -1 : block_of_atom[a];
    };

    // values in some atom's input_values and their consumer blocks
    std::vector<py::object> inputs_of_atom(n_atoms);
    py::dict cons_of;                             // vid -> index into cons_sets
    std::vector<std::vector<int32_t>> cons_sets;
    for (int a = 0; a < n_atoms; ++a) {
        inputs_of_atom[a] = py::reinterpret_steal<py::object>(
            PyFrozenSet_New(atoms[a].attr("input_values").ptr()));
        for (py::handle v : inputs_of_atom[a]) {
            PyObject *k = PyDict_GetItem(cons_of.ptr(), v.ptr());
            int ci;
            if (!k) {
                ci = (int)cons_sets.size();
                cons_sets.emplace_back();
                cons_of[v] = py::int_(ci);
            } else {
                ci = (int)PyLong_AsLong(k);
            }
            cons_sets[ci].push_back(block_of_atom[a]);
        }
    }
    py::list in_ids = py::module_::import("builtins").attr("sorted")(cons_of);
    py::dict in_index;
    std::vector<int32_t> in_ob, in_off{0}, in_cons;
    std::vector<int64_t> in_fix, in_ps;
    for (size_t i = 0; i < py::len(in_ids); ++i) {
        py::handle vid = in_ids[i];
        in_index[vid] = py::int_(i);
        const VInfo &vi = vinfo(dget(nodes, vid));
        if (!vi.is_value) throw Fallback();                   // not a value
        std::vector<int32_t> cb = cons_sets[PyLong_AsLong(dget(cons_of, vid).ptr())];
        std::sort(cb.begin(), cb.end());
        cb.erase(std::unique(cb.begin(), cb.end()), cb.end());
        int ob;
        if (PySequence_Contains(graph_inputs.ptr(), vid.ptr()) == 1) {
            ob = -1;
            const int own = blk_of(vid);
            if (own >= 0 && !std::binary_search(cb.begin(), cb.end(), own)) throw Fallback();
        } else {
            ob = blk_of(vid);
            if (ob > cb[0]) throw Fallback();
        }
        in_ob.push_back(ob);
        in_cons.insert(in_cons.end(), cb.begin(), cb.end());
        in_off.push_back((int32_t)in_cons.size());
        in_fix.push_back(need(vi).fix);
        in_ps.push_back(vi.ps);
    }
    auto in_index_of = [&](py::handle v) -> int {
        PyObject *x = PyDict_GetItem(in_index.ptr(), v.ptr());
        return x ? (int)PyLong_AsLong(x) : -1;
    };

    std::vector<int64_t> blk_param(nb, 0), blk_res_fix(nb, 0), blk_res_ps(nb, 0);
    std::vector<int32_t> task_block, dep_off{0}, dep_ob;
    std::vector<double> task_flops;
    std::vector<int64_t> fp_fix, fp_ps, dep_fix, dep_ps, prod_fix, prod_ps;
    py::list task_nodes;
    for (auto kv : nodes) {                       // sorted id order (graph.py:90-93)
        py::handle nid = kv.first, node = kv.second;
        const int b = blk_of(nid);
        if (b < 0) continue;
        const VInfo &self = vinfo(node);
        if (self.is_value) {
            if (self.is_param) {
                blk_param[b] += as_int(ga(ga(node, N.value), N.fixed_bytes).ptr());
            } else if (PyTuple_GET_SIZE(dget(pred_d, nid).ptr()) == 0) {     // no producer
                const bool span_input = PySequence_Contains(graph_inputs.ptr(), nid.ptr()) == 1 &&
                                        in_index_of(nid) >= 0;
                if (!span_input) {
                    blk_res_fix[b] += need(self).fix;
                    blk_res_ps[b] += self.ps;
                }
            }
            continue;
        }
        py::object task = ga(node, N.task);
        const int a = atom_get(nid);
        int64_t pf = 0, pp = 0;
        for (py::handle vid : dget(succ_d, nid)) {
            const VInfo &vi = vinfo(dget(nodes, vid));
            if (vi.is_value && !vi.is_param) {
                pf += need(vi).fix;
                pp += vi.ps;
            }
        }
        blk_res_fix[b] += pf;
        blk_res_ps[b] += pp;
        int64_t bf = pf, bp = pp;
        const py::object &ins = inputs_of_atom[a];
        for (py::handle vid : dget(pred_d, nid)) {
            const VInfo &vi = vinfo(dget(nodes, vid));
            if (!vi.is_value || vi.is_param) continue;
            const int64_t vf = need(vi).fix;
            const int64_t vp = vi.ps;
            const int i = in_index_of(vid);
            if (i < 0) {
                bf += vf;
                bp += vp;
                continue;
            }
            const int ob = in_ob[i];
            if (PySet_Contains(ins.ptr(), vid.ptr()) != 1) {
                if (ob != b) throw Fallback();       // cross-atom read: Python raises
                bf += vf;
                bp += vp;
                continue;
            }
            if (ob < 0) continue;                    // model input / unowned
            dep_ob.push_back(ob);
            dep_fix.push_back(vf);
            dep_ps.push_back(vp);
        }
        task_block.push_back(b);
        task_flops.push_back(PyFloat_AsDouble(ga(task, N.flops_per_sample).ptr()));
        task_nodes.append(task);
        fp_fix.push_back(bf);
        fp_ps.push_back(bp);
        prod_fix.push_back(pf);
        prod_ps.push_back(pp);
        dep_off.push_back((int32_t)dep_ob.size());
    }
    if (PyErr_Occurred()) throw py::error_already_set();

    py::dict out;
    out["task_block"] = arr(task_block);
    out["task_flops"] = arr(task_flops);
    out["task_fp_fix"] = arr(fp_fix);
    out["task_fp_ps"] = arr(fp_ps);
    out["task_prod_fix"] = arr(prod_fix);
    out["task_prod_ps"] = arr(prod_ps);
    out["task_dep_off"] = arr(dep_off);
    out["dep_ob"] = arr(dep_ob);
    out["dep_fix"] = arr(dep_fix);
    out["dep_ps"] = arr(dep_ps);
    out["in_ob"] = arr(in_ob);
    out["in_cons_off"] = arr(in_off);
    out["in_cons"] = arr(in_cons);
    out["in_fix"] = arr(in_fix);
    out["in_ps"] = arr(in_ps);
    out["blk_param"] = arr(blk_param);
    out["blk_res_fix"] = arr(blk_res_fix);
    out["blk_res_ps"] = arr(blk_res_ps);
    out["task_nodes"] = task_nodes;
    return out;
}

}  // namespace

PYBIND11_MODULE(_flatten_native, m) {
    static py::exception<Fallback> fallback(m, "Fallback");
    py::register_exception_translator([](std::exception_ptr p) {
        try {
            if (p) std::rethrow_exception(p);
        } catch (const Fallback &) {
            PyErr_SetString(fallback.ptr(), "outside the native path's common case");
        }
    });
    m.def("flatten_atoms", &flatten, "atom-level arrays of partition_blocks (flatten.py)");
    m.def("flatten_blocks", &flatten_blocks, "block-level span-profile arrays (flatten.py)");
}
