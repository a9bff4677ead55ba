// Atomic decomposition (reference pkg/src/pipecut/atoms.py:38-305) natively:
// constant marking, per-anchor constant closures, clone expansion and atom
// assembly over integer node indices, then the reference's own host objects
// (TaskGraph, Node, Subcomponent, AtomicPartition) built directly.
// §8f rank 4: at the paper's ~15,000 atoms the Python pass takes ~1.2 s.
//
// Node index = position in g.nodes, which TaskGraph builds in ascending id
// order (graph.py:90-93), so index order is the reference's string order
// (checked on entry; UTF-8 byte order equals code-point order).  Every error
// the reference raises is raised here, first one first in the reference's
// order, with its class and message: CycleError (graph.py:170-172),
// NoNonConstantTask and DanglingOutput (atoms.py:179-198), the clone-id
// collision ValueError (atoms.py:209-210).  A TaskGraph whose internal layout
// is not the reference's (non-str ids, unsorted node dict, adjacency that is
// not id-sorted tuples) raises TypeError: there is no fallback path.
#include <pybind11/pybind11.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <queue>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace py = pybind11;

namespace {

inline void check(PyObject *o) {
    if (!o) throw py::error_already_set();
}

// the reference's exception classes (set by build() from its arguments)
struct RefErrors {
    PyObject *cycle = nullptr, *no_task = nullptr, *dangling = nullptr;
};
RefErrors g_err;

[[noreturn]] void raise_obj(PyObject *cls, PyObject *msg) {
    check(msg);
    PyErr_SetObject(cls, msg);
    Py_DECREF(msg);
    throw py::error_already_set();
}
// a TaskGraph not laid out like the reference's (graph.py:82-116)
[[noreturn]] void layout(const char *what) {
    PyErr_Format(PyExc_TypeError, "build_atomic_subcomponents: unsupported TaskGraph layout (%s)",
                 what);
    throw py::error_already_set();
}
inline py::object steal(PyObject *o) {
    check(o);
    return py::reinterpret_steal<py::object>(o);
}
inline std::string_view utf8(PyObject *s) {
    if (!PyUnicode_Check(s)) layout("node ids must be str");
    Py_ssize_t n = 0;
    const char *p = PyUnicode_AsUTF8AndSize(s, &n);
    check((PyObject *)p);
    return std::string_view(p, (size_t)n);
}

struct Graph {        // the input TaskGraph on indices
    int n = 0;
    std::vector<PyObject *> id, node;          // borrowed (g keeps them alive)
    std::vector<char> is_task, is_input, is_output;
    std::vector<std::vector<int>> pred, succ;  // ascending (= sorted ids)
};

// graph.py:157-173 (heap on index == heap on id)
std::vector<int> topo_order(const Graph &G) {
    std::vector<int> indeg(G.n), order;
    order.reserve(G.n);
    std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
    for (int i = 0; i < G.n; ++i)
        if ((indeg[i] = (int)G.pred[i].size()) == 0) ready.push(i);
    while (!ready.empty()) {
        int u = ready.top();
        ready.pop();
        order.push_back(u);
        for (int v : G.succ[u])
            if (--indeg[v] == 0) ready.push(v);
    }
    if ((int)order.size() != G.n) {
        // CycleError(f"graph contains a cycle through {stuck[:8]}"), stuck sorted
        py::list stuck;
        for (int i = 0; i < G.n && stuck.size() < 8; ++i)
            if (indeg[i] > 0) stuck.append(py::reinterpret_borrow<py::object>(G.id[i]));
        raise_obj(g_err.cycle, PyUnicode_FromFormat("graph contains a cycle through %R", stuck.ptr()));
    }
    return order;
}

py::tuple str_tuple(const std::vector<int> &idx, const std::vector<PyObject *> &ids) {
    PyObject *t = PyTuple_New((Py_ssize_t)idx.size());
    check(t);
    for (size_t k = 0; k < idx.size(); ++k) {
        Py_INCREF(ids[idx[k]]);
        PyTuple_SET_ITEM(t, (Py_ssize_t)k, ids[idx[k]]);
    }
    return py::reinterpret_steal<py::tuple>(t);
}

// an instance of a plain (frozen) dataclass with the given fields, set as its
// own __init__ would (object.__setattr__), without the per-field Python calls
py::object make(const py::object &cls, std::initializer_list<py::str> names,
                std::initializer_list<py::object> values) {
    PyTypeObject *tp = (PyTypeObject *)cls.ptr();
    py::tuple empty;
    py::object o = steal(tp->tp_new(tp, empty.ptr(), nullptr));
    auto v = values.begin();
    for (const py::str &nm : names) {
        if (PyObject_GenericSetAttr(o.ptr(), nm.ptr(), v->ptr()) != 0) throw py::error_already_set();
        ++v;
    }
    return o;
}

py::object build(py::object g, py::object node_cls, py::object graph_cls, py::object sub_cls,
                 py::object part_cls, py::object cycle_error, py::object no_task_error,
                 py::object dangling_error) {
    g_err.cycle = cycle_error.ptr();
    g_err.no_task = no_task_error.ptr();
    g_err.dangling = dangling_error.ptr();
    Graph G;
    PyObject *nodes = g.attr("nodes").ptr();
    py::object nodes_ref = g.attr("nodes");
    if (!PyDict_Check(nodes)) layout("nodes is not a dict");
    G.n = (int)PyDict_Size(nodes);
    const int n = G.n;
    G.id.resize(n);
    G.node.resize(n);
    G.is_task.assign(n, 0);
    G.is_input.assign(n, 0);
    G.is_output.assign(n, 0);
    G.pred.resize(n);
    G.succ.resize(n);
    std::unordered_map<PyObject *, int> ptr_index;          // ids are usually the key objects
    ptr_index.reserve((size_t)n * 2);
    py::dict index;                                          // by value, built on first miss
    py::str s_task("task"), s_value("value");
    {
        PyObject *k, *v;
        Py_ssize_t pos = 0;
        int i = 0;
        std::string_view prev;
        while (PyDict_Next(nodes, &pos, &k, &v)) {
            std::string_view cur = utf8(k);
            if (i > 0 && !(prev < cur)) layout("nodes not in sorted-id order");
            prev = cur;
            G.id[i] = k;
            G.node[i] = v;
            py::object task = steal(PyObject_GetAttr(v, s_task.ptr()));
            G.is_task[i] = !task.is_none();
            ptr_index.emplace(k, i);
            ++i;
        }
    }
    auto idx_of = [&](PyObject *key) -> int {
        auto hit = ptr_index.find(key);
        if (hit != ptr_index.end()) return hit->second;
        if (PyDict_Size(index.ptr()) == 0)
            for (int i = 0; i < n; ++i)
                check(PyDict_SetItem(index.ptr(), G.id[i], py::int_(i).ptr()) == 0 ? Py_None
                                                                                 : nullptr);
        PyObject *r = PyDict_GetItem(index.ptr(), key);
        if (!r) layout("an edge or input/output names an unknown node");
        return (int)PyLong_AsLong(r);
    };
    py::object pred_ref = g.attr("_pred"), succ_ref = g.attr("_succ");
    for (int i = 0; i < n; ++i) {
        for (int dir = 0; dir < 2; ++dir) {
            PyObject *t = PyDict_GetItem(dir ? succ_ref.ptr() : pred_ref.ptr(), G.id[i]);
            if (!t || !PyTuple_Check(t)) layout("adjacency is not a tuple per node");
            auto &dst = dir ? G.succ[i] : G.pred[i];
            const Py_ssize_t m = PyTuple_GET_SIZE(t);
            dst.resize((size_t)m);
            for (Py_ssize_t k = 0; k < m; ++k) dst[k] = idx_of(PyTuple_GET_ITEM(t, k));
            if (!std::is_sorted(dst.begin(), dst.end())) layout("adjacency not in sorted-id order");
        }
    }
    py::object inputs = g.attr("inputs"), outputs = g.attr("outputs");
    for (py::handle v : inputs) G.is_input[idx_of(v.ptr())] = 1;
    for (py::handle v : outputs) G.is_output[idx_of(v.ptr())] = 1;
    auto producer = [&](int v) { return G.pred[v].empty() ? -1 : G.pred[v][0]; };

    // mark_constant_tasks (atoms.py:38-59)
    const std::vector<int> topo = topo_order(G);
    std::vector<int> topo_pos(n);
    for (int i = 0; i < n; ++i) topo_pos[topo[i]] = i;
    std::vector<char> constant(n, 0);
    std::vector<int> anchors, anchor_of(n, -1);
    for (int u : topo) {
        if (!G.is_task[u]) continue;
        bool dep = false;
        for (int v : G.pred[u]) {
            const int p = producer(v);
            if (G.is_input[v] || (p >= 0 && !constant[p])) {
                dep = true;
                break;
            }
        }
        constant[u] = !dep;
        if (dep) {
            anchor_of[u] = (int)anchors.size();
            anchors.push_back(u);
        }
    }
    const int na = (int)anchors.size();
    if (na == 0)                                              // atoms.py:178-179
        raise_obj(g_err.no_task, PyUnicode_FromString("no task depends on a model input"));
    for (int v = 0; v < n; ++v)                               // sorted(g.outputs), atoms.py:181-187
        if (G.is_output[v]) {
            const int p = producer(v);
            if (p < 0 && !G.is_input[v])
                raise_obj(g_err.dangling, PyUnicode_FromFormat(
                    "output %R is not produced by any task", G.id[v]));
            if (p >= 0 && constant[p])
                raise_obj(g_err.dangling, PyUnicode_FromFormat(
                    "output %R depends on no model input", G.id[v]));
        }

    // _constant_closure per anchor (atoms.py:62-80); owners in anchor order
    std::vector<std::vector<int>> closure(na);
    std::vector<std::vector<int>> owners(n);
    {
        std::vector<int> stamp(n, -1), stack;
        for (int a = 0; a < na; ++a) {
            auto &cl = closure[a];
            auto add = [&](int x) {
                stamp[x] = a;
                cl.push_back(x);
            };
            stack.assign(G.pred[anchors[a]].begin(), G.pred[anchors[a]].end());
            while (!stack.empty()) {
                const int v = stack.back();
                stack.pop_back();
                if (stamp[v] == a || G.is_input[v]) continue;
                const int p = producer(v);
                if (p < 0) {
                    add(v);
                    continue;
                }
                if (!constant[p]) continue;
                add(v);
                if (stamp[p] != a) {
                    add(p);
                    stack.insert(stack.end(), G.pred[p].begin(), G.pred[p].end());
                }
            }
            for (int x : cl) owners[x].push_back(a);
        }
    }
    for (int u : topo)                                        // constant.items(), atoms.py:194-196
        if (G.is_task[u] && constant[u] && owners[u].empty())
            raise_obj(g_err.dangling, PyUnicode_FromFormat("constant task %R feeds no atom", G.id[u]));
    for (int u = 0; u < n; ++u)                               // g.value_ids(), atoms.py:197-199
        if (!G.is_task[u] && producer(u) < 0 && !G.is_input[u] && owners[u].empty())
            raise_obj(g_err.dangling, PyUnicode_FromFormat("constant value %R feeds no atom", G.id[u]));

    // clone ids (atoms.py:202-215): "<id>::c<rank>" per owning atom when shared
    bool cloned = false;
    for (int u = 0; u < n; ++u) cloned |= owners[u].size() > 1;

    // new graph: index space of the expanded graph (sorted by id)
    int nn = n;
    std::vector<PyObject *> nid;                             // new ids, borrowed / owned below
    std::vector<PyObject *> nnode;
    std::vector<int> old_to_new(n, -1);                      // non-owned and single-owned nodes
    std::vector<std::vector<int>> local_new(na);             // per atom: new index of closure[k]
    std::vector<std::vector<int>> npred, nsucc;
    std::vector<char> nis_task, nis_input, nis_output;
    py::list keep;                                           // owns clone ids / Nodes
    py::dict clone_origins;
    if (!cloned) {
        nid = G.id;
        nnode = G.node;
        for (int i = 0; i < n; ++i) old_to_new[i] = i;
        for (int a = 0; a < na; ++a)
            local_new[a].assign(closure[a].begin(), closure[a].end());
    } else {
        struct Item {
            std::string_view key;
            PyObject *id, *node;
            int orig, atom;          // atom = -1: the node keeps its id
        };
        std::vector<Item> items;
        items.reserve((size_t)n + 64);
        std::deque<std::string> store;
        std::vector<std::vector<int>> clone_slot(n);          // per shared node: item per rank
        for (int u = 0; u < n; ++u) {
            if (owners[u].size() <= 1) {
                items.push_back({utf8(G.id[u]), G.id[u], G.node[u], u, -1});
                continue;
            }
            py::object task = steal(PyObject_GetAttr(G.node[u], s_task.ptr()));
            py::object value = steal(PyObject_GetAttr(G.node[u], s_value.ptr()));
            for (size_t r = 0; r < owners[u].size(); ++r) {
                py::str cid = py::reinterpret_steal<py::str>(
                    steal(PyUnicode_FromFormat("%U::c%zu", G.id[u], r)).release());
                if (PyDict_Contains(nodes, cid.ptr()))               // atoms.py:209-210
                    raise_obj(PyExc_ValueError, PyUnicode_FromFormat(
                        "clone id %R collides with a node", cid.ptr()));
                py::object nd = node_cls(cid, task, value);
                keep.append(cid);
                keep.append(nd);
                check(PyDict_SetItem(clone_origins.ptr(), cid.ptr(), G.id[u]) == 0 ? Py_None
                                                                                  : nullptr);
                clone_slot[u].push_back((int)items.size());
                items.push_back({utf8(cid.ptr()), cid.ptr(), nd.ptr(), u, owners[u][r]});
            }
        }
        // clone_origins insertion order: sorted(owners) then rank (atoms.py:204-215)
        std::vector<int> order(items.size());
        for (size_t k = 0; k < items.size(); ++k) order[k] = (int)k;
        std::sort(order.begin(), order.end(),
                  [&](int x, int y) { return items[x].key < items[y].key; });
        nn = (int)items.size();
        std::vector<int> item_new(items.size());
        nid.resize(nn);
        nnode.resize(nn);
        for (int j = 0; j < nn; ++j) {
            const Item &it = items[order[j]];
            if (j > 0 && !(items[order[j - 1]].key < it.key)) layout("clone ids not unique");
            item_new[order[j]] = j;
            nid[j] = it.id;
            nnode[j] = it.node;
        }
        for (size_t k = 0; k < items.size(); ++k)
            if (items[k].atom < 0) old_to_new[items[k].orig] = item_new[k];
        auto ids = [&](int a, int u) -> int {                 // local_id[a][u] (new index)
            if (owners[u].size() <= 1) return old_to_new[u];
            const auto &ow = owners[u];
            const size_t r = (size_t)(std::lower_bound(ow.begin(), ow.end(), a) - ow.begin());
            if (r >= ow.size() || ow[r] != a) layout("closure ownership");   // unreachable
            return item_new[clone_slot[u][r]];
        };
        for (int a = 0; a < na; ++a) {
            local_new[a].resize(closure[a].size());
            for (size_t k = 0; k < closure[a].size(); ++k) local_new[a][k] = ids(a, closure[a][k]);
        }
        // edges (atoms.py:237-256), as (src, dst) in new indices
        std::vector<int64_t> edges;
        for (int u = 0; u < n; ++u) {
            if (!owners[u].empty()) continue;
            for (int v : G.succ[u])
                if (owners[v].empty())
                    edges.push_back((int64_t)old_to_new[u] * nn + old_to_new[v]);
        }
        std::vector<int> in_cl(n, -1);
        for (int a = 0; a < na; ++a) {
            for (int x : closure[a]) in_cl[x] = a;
            const int anchor = anchors[a];
            const int anchor_new = old_to_new[anchor];
            for (size_t k = 0; k < closure[a].size(); ++k) {
                const int x = closure[a][k], xn = local_new[a][k];
                if (G.is_task[x]) {
                    for (int v : G.pred[x]) edges.push_back((int64_t)ids(a, v) * nn + xn);
                    for (int v : G.succ[x])
                        if (in_cl[v] == a) edges.push_back((int64_t)xn * nn + ids(a, v));
                } else if (std::binary_search(G.succ[x].begin(), G.succ[x].end(), anchor)) {
                    edges.push_back((int64_t)xn * nn + anchor_new);
                }
            }
        }
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        npred.assign(nn, {});
        nsucc.assign(nn, {});
        for (int64_t e : edges) {                              // sorted: lists stay ascending
            nsucc[(int)(e / nn)].push_back((int)(e % nn));
            npred[(int)(e % nn)].push_back((int)(e / nn));
        }
        nis_task.assign(nn, 0);
        nis_input.assign(nn, 0);
        nis_output.assign(nn, 0);
        for (size_t k = 0; k < items.size(); ++k) {
            const int j = item_new[k], u = items[k].orig;
            nis_task[j] = G.is_task[u];
            nis_input[j] = G.is_input[u];
            nis_output[j] = G.is_output[u];
        }
        // the expanded TaskGraph (graph.py:82-116) without re-validating
        py::object ng = steal(PyObject_CallMethod(graph_cls.ptr(), "__new__", "O", graph_cls.ptr()));
        py::dict d_nodes, d_succ, d_pred;
        // adjacency tuples: the input graph's own tuple where a node kept its id
        // and its neighbours (tuples are immutable, so sharing is safe)
        auto adj = [&](const std::vector<int> &nl, int u, bool succ) -> py::object {
            if (u >= 0) {
                const std::vector<int> &ol = succ ? G.succ[u] : G.pred[u];
                bool same = nl.size() == ol.size();
                for (size_t k = 0; same && k < nl.size(); ++k) same = nid[nl[k]] == G.id[ol[k]];
                PyObject *t = same ? PyDict_GetItem((succ ? succ_ref : pred_ref).ptr(), G.id[u])
                                   : nullptr;
                if (t) return py::reinterpret_borrow<py::object>(t);
            }
            return str_tuple(nl, nid);
        };
        for (int j = 0; j < nn; ++j) {
            const Item &it = items[order[j]];
            const int u = it.atom < 0 ? it.orig : -1;
            check(PyDict_SetItem(d_nodes.ptr(), nid[j], nnode[j]) == 0 ? Py_None : nullptr);
            check(PyDict_SetItem(d_succ.ptr(), nid[j], adj(nsucc[j], u, true).ptr()) == 0
                      ? Py_None : nullptr);
            check(PyDict_SetItem(d_pred.ptr(), nid[j], adj(npred[j], u, false).ptr()) == 0
                      ? Py_None : nullptr);
        }
        PyObject *et = PyTuple_New((Py_ssize_t)edges.size());
        check(et);
        py::tuple etup = py::reinterpret_steal<py::tuple>(et);
        for (size_t k = 0; k < edges.size(); ++k) {
            PyObject *pair = PyTuple_Pack(2, nid[(int)(edges[k] / nn)], nid[(int)(edges[k] % nn)]);
            check(pair);
            PyTuple_SET_ITEM(et, (Py_ssize_t)k, pair);
        }
        ng.attr("nodes") = d_nodes;
        ng.attr("edges") = etup;
        ng.attr("inputs") = inputs;
        ng.attr("outputs") = outputs;
        ng.attr("_succ") = d_succ;
        ng.attr("_pred") = d_pred;
        keep.append(ng);
    }
    const auto &P = cloned ? npred : G.pred;
    const auto &S = cloned ? nsucc : G.succ;
    const auto &T = cloned ? nis_task : G.is_task;
    const auto &IN = cloned ? nis_input : G.is_input;
    const auto &OUT = cloned ? nis_output : G.is_output;
    py::object expanded = cloned ? py::object(keep[keep.size() - 1]) : g;

    // _assemble (atoms.py:259-305)
    std::vector<std::vector<int>> members(na);
    std::vector<int> task_atom(nn, -1);                      // anchors only
    for (int a = 0; a < na; ++a) {
        const int an = old_to_new[anchors[a]];
        auto &mb = members[a];
        mb.push_back(an);
        task_atom[an] = a;
        mb.insert(mb.end(), S[an].begin(), S[an].end());
        mb.insert(mb.end(), local_new[a].begin(), local_new[a].end());
    }
    for (int u = 0; u < n; ++u) {                             // inputs, sorted order
        if (!G.is_input[u]) continue;
        const int un = old_to_new[u];
        if (S[un].empty()) {
            members[0].push_back(un);
            continue;
        }
        int best = -1;
        for (int t : S[un]) {                                 // min (topo_pos, id)
            if (task_atom[t] < 0) layout("input consumed by a constant task");   // unreachable
            const int ot = anchors[task_atom[t]];
            if (best < 0 || topo_pos[ot] < topo_pos[anchors[task_atom[best]]]) best = t;
        }
        members[task_atom[best]].push_back(un);
    }
    std::vector<int> value_owner(nn, -1);
    for (int a = 0; a < na; ++a) {
        auto &mb = members[a];
        std::sort(mb.begin(), mb.end());
        mb.erase(std::unique(mb.begin(), mb.end()), mb.end());
        for (int x : mb)
            if (!T[x]) value_owner[x] = a;
    }
    const int width = std::max<int>(5, (int)std::to_string(na).size());
    PyObject *atoms_t = PyTuple_New(na);
    check(atoms_t);
    py::tuple atoms = py::reinterpret_steal<py::tuple>(atoms_t);
    std::vector<int> ins, outs;
    std::vector<char> in_seen(nn, 0);
    std::vector<py::object> member_sets(na);
    py::str f_id("id"), f_node_ids("node_ids"), f_input_values("input_values"),
        f_output_values("output_values");
    for (int a = 0; a < na; ++a) {
        const int an = old_to_new[anchors[a]];
        ins.clear();
        for (int v : P[an])
            if (IN[v] || value_owner[v] != a) ins.push_back(v);   // P sorted, unique
        outs.clear();
        for (int x : members[a]) {
            if (T[x]) continue;
            if (OUT[x]) {
                outs.push_back(x);
                continue;
            }
            for (int c : S[x])
                if (task_atom[c] >= 0 && task_atom[c] != a) {
                    outs.push_back(x);
                    break;
                }
        }
        PyObject *lst = PyList_New((Py_ssize_t)members[a].size());
        check(lst);
        py::object lref = py::reinterpret_steal<py::object>(lst);
        for (size_t k = 0; k < members[a].size(); ++k) {
            Py_INCREF(nid[members[a][k]]);
            PyList_SET_ITEM(lst, (Py_ssize_t)k, nid[members[a][k]]);
        }
        member_sets[a] = steal(PyFrozenSet_New(lst));
        std::string num = std::to_string(a);
        std::string sid = "A" + std::string((size_t)std::max(0, width - (int)num.size()), '0') + num;
        py::object sub = make(sub_cls, {f_id, f_node_ids, f_input_values, f_output_values},
                              {py::str(sid), member_sets[a], str_tuple(ins, nid),
                               str_tuple(outs, nid)});
        PyTuple_SET_ITEM(atoms_t, a, sub.release().ptr());
    }

    // AtomicPartition with its lookup tables (atoms.py:91-104) filled here
    py::object part = steal(PyObject_CallMethod(part_cls.ptr(), "__new__", "O", part_cls.ptr()));
    part.attr("graph") = expanded;
    part.attr("atoms") = atoms;
    part.attr("clone_origins") = clone_origins;
    py::dict d_task_atom, d_value_owner, d_consumers;
    std::vector<int> member_atom(nn, -1);                    // every member task's atom
    std::vector<py::int_> ints;
    ints.reserve(na);
    for (int a = 0; a < na; ++a) ints.emplace_back(a);
    for (int a = 0; a < na; ++a)
        for (int x : members[a]) {
            if (T[x]) member_atom[x] = a;
            check(PyDict_SetItem(T[x] ? d_task_atom.ptr() : d_value_owner.ptr(), nid[x],
                                 ints[a].ptr()) == 0 ? Py_None : nullptr);
        }
    for (int j = 0; j < nn; ++j) {
        if (T[j]) continue;
        PyObject *lst = PyList_New((Py_ssize_t)S[j].size());
        check(lst);
        py::object lref = py::reinterpret_steal<py::object>(lst);
        for (size_t k = 0; k < S[j].size(); ++k) {
            const int c = member_atom[S[j][k]];
            if (c < 0) {                                     // self._task_atom[t] (atoms.py:103)
                PyErr_SetObject(PyExc_KeyError, nid[S[j][k]]);
                throw py::error_already_set();
            }
            Py_INCREF(ints[c].ptr());
            PyList_SET_ITEM(lst, (Py_ssize_t)k, ints[c].ptr());
        }
        py::object fs = steal(PyFrozenSet_New(lst));
        check(PyDict_SetItem(d_consumers.ptr(), nid[j], fs.ptr()) == 0 ? Py_None : nullptr);
    }
    part.attr("_task_atom") = d_task_atom;
    part.attr("_value_owner") = d_value_owner;
    part.attr("_consumer_atoms") = d_consumers;
    return part;
}

}  // namespace

PYBIND11_MODULE(_atoms_native, m) {
    m.def("build_atomic_subcomponents", &build,
          "atoms.py:164-222 over the reference's host objects; raises the reference's errors");
}
