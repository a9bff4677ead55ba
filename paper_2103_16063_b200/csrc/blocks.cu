// K6: block coarsening -- partition_blocks (pkg/src/pipecut/blocks.py:361-397).
//
// The reference is a sequential greedy multilevel algorithm whose decisions
// must be reproduced exactly (SURVEY.md finding 7).  Its cost is in the
// predicates it evaluates: the memory of merged atom sets (a full
// CostModel.profile each, blocks.py:107-116), convexity (blocks.py:45-70),
// group compute times (blocks.py:104-105) and cut traffic (blocks.py:118-124).
// Every candidate of a coarsening pass (all adjacent group pairs of a level)
// is independent of the greedy state it is tested in, so the device evaluates
// the whole pass in one batch and the host replays the greedy order over the
// device's answers (one sync per level).  Uncoarsening changes state after
// every accepted move, so it runs entirely on the device: k_refine walks all
// levels' pairs in one resident CTA or cluster (accepted moves are rare: 62
// on BERT, 0 on ResNet).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <queue>
#include <set>
#include <vector>

#include <cooperative_groups.h>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace pcb {

struct DevAtoms {
    int n, T, V, E;
    int64_t budget;
    double factor, flops, beta;
    const int64_t *atom_param;
    const int32_t *task_atom;
    const double *task_flops;
    const int64_t *task_fp1;
    const int32_t *dep_off, *dep_owner;
    const int64_t *dep_size;
    const int32_t *atom_task_off, *atom_tasks;
    const int32_t *atom_in_off, *atom_in;
    const int32_t *in_owner;
    const int64_t *in_size;
    const int32_t *in_atoms_off, *in_atoms;
    const int32_t *pred_off, *pred;
    const int32_t *tr_owner;
    const int64_t *tr_size;
    const int32_t *tr_cons_off, *tr_cons;
    const int32_t *atom_tr_off, *atom_tr;
    const int64_t *task_prod1;
    const uint8_t *ov_has;          // null without a cost table
    const double *ov_tf, *ov_tb;
    const int64_t *ov_act;
    const int32_t *nbr_off, *nbr;   // sorted(succ | pred) per atom (blocks.py:87-88)
};

// per-task time at m = 1, cost-table entry first (costs.py:130-140)
__device__ __forceinline__ void atom_task_times(const DevAtoms &A, int t, double &x, double &y) {
    if (A.ov_has && A.ov_has[t]) {
        x = A.ov_tf[t];
        y = isnan(A.ov_tb[t]) ? __dmul_rn(A.beta, x) : A.ov_tb[t];
    } else {
        x = __ddiv_rn(__dmul_rn(A.task_flops[t], 1.0), A.flops);
        y = __dmul_rn(A.beta, x);
    }
}

// Group memberships of the coarsening levels: grp[l*n + x] = group of atom x
// at level l; CSR goff[l*(n+1) + g] / gat[l*n + j] lists each group's atoms
// ascending (groups ordered by first atom, as the reference keeps them).
struct DevLevels {
    const int32_t *grp, *goff, *gat;
    int n;
};

// mode 0: group (la, ga) union group (lb, gb) (gb < 0: just (la, ga));
// mode 1: group (la, ga) minus group (lb, gb)
struct SetDesc {
    int32_t la, ga, lb, gb, mode;
};

__device__ __forceinline__ bool in_set(const DevLevels &L, const SetDesc &s, int x) {
    const bool a = L.grp[(int64_t)s.la * L.n + x] == s.ga;
    if (s.mode == 0) return a || (s.gb >= 0 && L.grp[(int64_t)s.lb * L.n + x] == s.gb);
    return a && L.grp[(int64_t)s.lb * L.n + x] != s.gb;
}

template <class F>
__device__ __forceinline__ void for_each_member(const DevLevels &L, const SetDesc &s, F f) {
    const int32_t *off = L.goff + (int64_t)s.la * (L.n + 1);
    const int32_t *at = L.gat + (int64_t)s.la * L.n;
    for (int j = off[s.ga]; j < off[s.ga + 1]; ++j) {
        const int x = at[j];
        if (s.mode == 1 && L.grp[(int64_t)s.lb * L.n + x] == s.gb) continue;
        f(x);
    }
    if (s.mode == 0 && s.gb >= 0) {
        const int32_t *offb = L.goff + (int64_t)s.lb * (L.n + 1);
        const int32_t *atb = L.gat + (int64_t)s.lb * L.n;
        for (int j = offb[s.gb]; j < offb[s.gb + 1]; ++j) {
            const int x = atb[j];
            if (L.grp[(int64_t)s.la * L.n + x] == s.ga) continue;
            f(x);
        }
    }
}

// CostModel.profile(merged(G), 1, checkpointing=True).mem_bytes (costs.py:97-160)
__device__ int64_t set_mem(const DevAtoms &A, const DevLevels &L, const SetDesc &s) {
    int64_t param = 0, inb = 0, mfp = 0;
    for_each_member(L, s, [&](int x) {
        param += A.atom_param[x];
        for (int q = A.atom_in_off[x]; q < A.atom_in_off[x + 1]; ++q) {
            const int iv = A.atom_in[q];
            const int own = A.in_owner[iv];
            if (own >= 0 && in_set(L, s, own)) continue;          // owned inside: not an input
            for (int r = A.in_atoms_off[iv]; r < A.in_atoms_off[iv + 1]; ++r) {
                const int y = A.in_atoms[r];
                if (in_set(L, s, y)) {                              // count at the first lister
                    if (y == x) inb += A.in_size[iv];
                    break;
                }
            }
        }
        for (int q = A.atom_task_off[x]; q < A.atom_task_off[x + 1]; ++q) {
            const int t = A.atom_tasks[q];
            int64_t fp = A.task_fp1[t];
            if (A.ov_has && A.ov_has[t] && A.ov_act[t] >= 0) fp += A.ov_act[t] - A.task_prod1[t];
            for (int d = A.dep_off[t]; d < A.dep_off[t + 1]; ++d)
                if (in_set(L, s, A.dep_owner[d])) fp += A.dep_size[d];
            mfp = fp > mfp ? fp : mfp;
        }
    });
    const double memd = __dadd_rn(__dmul_rn((double)param, A.factor), (double)(inb + mfp));
    return (int64_t)memd;
}

// k_eval_sets: memory and convexity of implicit atom sets, one warp per set
// (is_convex, blocks.py:45-70, as a sweep in index order: atom indices are a
// topological order, so the reference's DFS "reached" set is: x in (lo, hi),
// not a member, with a member or reached predecessor).  Memory: lanes stride over
// the set's members and reduce exact integer partial sums (param, inputs) and
// the footprint max, so the value is the one set_mem computes.  Convexity: the
// index-order sweep, 32 consecutive atoms at a time --
// reachability from earlier chunks comes from the bitmap, inside the chunk it
// propagates by ballots until nothing changes (edges only go forward); a member
// with a reached predecessor makes the set non-convex.
__device__ __forceinline__ bool bit_at(const uint32_t *bits, int i) {
    return (bits[i >> 5] >> (i & 31)) & 1u;
}

// One warp evaluates set s: member count, memory, convexity (bits: the
// warp's bitmap scratch, >= n/32 + 1 words).  All lanes return the results.
__device__ __noinline__ void eval_set_warp(const DevAtoms &A, const DevLevels &L, const SetDesc s,
                                           uint32_t *bits, int &count_out, int64_t &mem_out,
                                           bool &convex_out) {
    const int lane = threadIdx.x & 31;
    const int n = L.n;
    const int32_t *offa = L.goff + (int64_t)s.la * (n + 1);
    const int32_t *ata = L.gat + (int64_t)s.la * n;
    const int a0 = offa[s.ga], na = offa[s.ga + 1] - a0;
    int b0 = 0, nbm = 0;
    const int32_t *atb = ata;
    if (s.mode == 0 && s.gb >= 0) {
        const int32_t *offb = L.goff + (int64_t)s.lb * (n + 1);
        atb = L.gat + (int64_t)s.lb * n;
        b0 = offb[s.gb];
        nbm = offb[s.gb + 1] - b0;
    }
    int lo = 0x7fffffff, hi = -1, count = 0;
    long long param = 0, inb = 0, mfp = 0;
    for (int j = lane; j < na + nbm; j += 32) {
        int x;
        if (j < na) {
            x = ata[a0 + j];
            if (s.mode == 1 && L.grp[(int64_t)s.lb * n + x] == s.gb) continue;
        } else {
            x = atb[b0 + j - na];
            if (L.grp[(int64_t)s.la * n + x] == s.ga) continue;
        }
        lo = min(lo, x);
        hi = max(hi, x);
        ++count;
        param += A.atom_param[x];
        for (int q = A.atom_in_off[x]; q < A.atom_in_off[x + 1]; ++q) {
            const int iv = A.atom_in[q];
            const int own = A.in_owner[iv];
            if (own >= 0 && in_set(L, s, own)) continue;          // owned inside: not an input
            for (int r = A.in_atoms_off[iv]; r < A.in_atoms_off[iv + 1]; ++r) {
                const int y = A.in_atoms[r];
                if (in_set(L, s, y)) {                              // count at the first lister
                    if (y == x) inb += A.in_size[iv];
                    break;
                }
            }
        }
        for (int q = A.atom_task_off[x]; q < A.atom_task_off[x + 1]; ++q) {
            const int t = A.atom_tasks[q];
            long long fp = A.task_fp1[t];
            if (A.ov_has && A.ov_has[t] && A.ov_act[t] >= 0) fp += A.ov_act[t] - A.task_prod1[t];
            for (int d = A.dep_off[t]; d < A.dep_off[t + 1]; ++d)
                if (in_set(L, s, A.dep_owner[d])) fp += A.dep_size[d];
            mfp = fp > mfp ? fp : mfp;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        count += __shfl_xor_sync(0xffffffffu, count, o);
        param += __shfl_xor_sync(0xffffffffu, param, o);
        inb += __shfl_xor_sync(0xffffffffu, inb, o);
        const long long m2 = __shfl_xor_sync(0xffffffffu, mfp, o);
        mfp = m2 > mfp ? m2 : mfp;
    }
    if (count == 0) {
        count_out = 0;
        mem_out = 0;
        convex_out = true;
        return;
    }
    bool convex = true;
    if (hi - lo + 1 != count) {
        const int span = hi - lo + 1;
        for (int w = lane; w < (span + 31) / 32; w += 32) bits[w] = 0u;
        __syncwarp();
        for (int base = lo + 1; base <= hi; base += 32) {
            const int x = base + lane;
            const bool valid = x <= hi;
            const bool mem = valid && in_set(L, s, x);
            const bool open = valid && !mem && x < hi;           // may become reached
            bool reached = false, bad = false;
            if (mem) {
                for (int q = A.pred_off[x]; q < A.pred_off[x + 1]; ++q) {
                    const int p = A.pred[q];
                    if (p > lo && p < base && bit_at(bits, p - lo)) bad = true;
                }
            } else if (open) {
                for (int q = A.pred_off[x]; q < A.pred_off[x + 1]; ++q) {
                    const int p = A.pred[q];
                    if (p < lo) continue;
                    if (in_set(L, s, p) || (p > lo && p < base && bit_at(bits, p - lo))) {
                        reached = true;
                        break;
                    }
                }
            }
            uint32_t rmask = __ballot_sync(0xffffffffu, reached);
            for (;;) {                                          // in-chunk propagation
                bool nr = reached;
                if (open && !reached)
                    for (int q = A.pred_off[x]; q < A.pred_off[x + 1]; ++q) {
                        const int p = A.pred[q];
                        if (p >= base && p < x && ((rmask >> (p - base)) & 1u)) {
                            nr = true;
                            break;
                        }
                    }
                const uint32_t nm = __ballot_sync(0xffffffffu, nr);
                reached = nr;
                if (nm == rmask) break;
                rmask = nm;
            }
            if (mem)
                for (int q = A.pred_off[x]; q < A.pred_off[x + 1]; ++q) {
                    const int p = A.pred[q];
                    if (p >= base && p < x && ((rmask >> (p - base)) & 1u)) bad = true;
                }
            if (__any_sync(0xffffffffu, bad)) {
                convex = false;
                break;
            }
            if (reached) atomicOr(&bits[(x - lo) >> 5], 1u << ((x - lo) & 31));
            __syncwarp();
        }
    }
    count_out = count;
    const double memd = __dadd_rn(__dmul_rn((double)param, A.factor), (double)(inb + mfp));
    mem_out = (int64_t)memd;
    convex_out = convex;
}

__global__ void k_eval_sets_warp(DevAtoms A, DevLevels L, const SetDesc *sets, int nsets,
                                 uint32_t *scratch, int words, int64_t *out_mem,
                                 int32_t *out_count, uint8_t *out_convex) {
    const int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= nsets) return;                                   // warp-uniform
    int count;
    int64_t mem;
    bool convex;
    eval_set_warp(A, L, sets[i], scratch + (int64_t)i * words, count, mem, convex);
    if ((threadIdx.x & 31) == 0) {
        out_count[i] = count;
        out_mem[i] = mem;
        out_convex[i] = convex ? 1 : 0;
    }
}

// sum(atom_comp[i] for i in group) with CPython 3.12's float sum: the first
// term enters as 0 + x0, the rest by Neumaier compensation (bltinmodule.c).
__global__ void k_group_comps(DevLevels L, int level, int ngroups, const double *atom_comp,
                              double *out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const int32_t *off = L.goff + (int64_t)level * (L.n + 1);
    const int32_t *at = L.gat + (int64_t)level * L.n;
    double f = __dadd_rn(0.0, atom_comp[at[off[g]]]);
    double c = 0.0;
    for (int j = off[g] + 1; j < off[g + 1]; ++j) {
        const double x = atom_comp[at[j]];
        const double t = __dadd_rn(f, x);
        if (fabs(f) >= fabs(x))
            c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else
            c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
    out[g] = f;
}

// CostModel.profile(atom, 1, checkpointing=True) for every atom (level 0)
__global__ void k_atom_profiles(DevAtoms A, DevLevels L, int level, int ngroups, double *out_tf,
                                double *out_tb, double *out_comp, int64_t *out_mem) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    double tf = 0.0, tb = 0.0;
    const int x = L.gat[(int64_t)level * L.n + L.goff[(int64_t)level * (L.n + 1) + g]];
    for (int q = A.atom_task_off[x]; q < A.atom_task_off[x + 1]; ++q) {
        const int t = A.atom_tasks[q];
        double v, w;
        atom_task_times(A, t, v, w);
        tf = __dadd_rn(tf, v);
        tb = __dadd_rn(tb, w);
    }
    out_tf[g] = tf;
    out_tb[g] = tb;
    out_comp[g] = __dadd_rn(tf, tb);                      // blocks.py:93
    out_mem[g] = set_mem(A, L, SetDesc{level, g, level, -1, 0});
}

// CostModel.profile(group, 1, checkpointing=True) for every group of a level,
// one warp per group: the time folds over the group's tasks in global sorted
// node-id order -- the warp scans the tasks 32 at a time, a ballot picks the
// members, and their times are added one by one in index order.
__global__ void k_group_profiles(DevAtoms A, DevLevels L, int level, int ngroups, double *out_tf,
                                 double *out_tb, double *out_comp, int64_t *out_mem) {
    const int g = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= ngroups) return;                             // warp-uniform
    const int32_t *grp = L.grp + (int64_t)level * L.n;
    double tf = 0.0, tb = 0.0;
    for (int base = 0; base < A.T; base += 32) {
        const int t = base + lane;
        const bool in = t < A.T && grp[A.task_atom[t]] == g;
        double v = 0.0, w = 0.0;
        if (in) atom_task_times(A, t, v, w);
        unsigned m = __ballot_sync(0xffffffffu, in);
        while (m) {
            const int src = __ffs(m) - 1;
            tf = __dadd_rn(tf, __shfl_sync(0xffffffffu, v, src));
            tb = __dadd_rn(tb, __shfl_sync(0xffffffffu, w, src));
            m &= m - 1;
        }
    }
    if (lane == 0) {
        out_tf[g] = tf;
        out_tb[g] = tb;
        out_comp[g] = __dadd_rn(tf, tb);                  // blocks.py:93
        out_mem[g] = set_mem(A, L, SetDesc{level, g, level, -1, 0});
    }
}

// ---------------------------------------------------------------- refinement
// _uncoarsen (blocks.py:173-232) as one resident CTA, or one thread-block
// cluster (up to 16 CTAs, one per SM) when there are many pairs: no host
// round trip per pair.  For each transition level li (coarsest first) the
// pairs are walked in order; a pair moves one side (mover, a level-li group)
// into a neighbouring level-li group's block when that strictly cuts the
// top-level traffic and both touched groups stay convex and inside memory at
// every coarser level.  The reference tests fit first and saving second; the
// choice is the same if the saving is computed first: the answer is the
// candidate with the largest positive saving among those that fit, the
// earliest (side v before w, target index ascending) on ties.  So the kernel
//   1. computes, for a window of pairs at once (one warp per pair side), the
//      best positive-saving candidate of every side -- savings depend only on
//      the top-level labels, which change only when a move is applied;
//   2. takes the first pair of the window with a positive candidate and tests
//      that candidate's fit (2 sets per coarser level, one warp each); if it
//      does not fit, the next candidate in (saving desc, side, target) order
//      is recomputed and tested, and so on;
//   3. applies an accepted move on the device (relabel the mover's atoms and
//      splice its atoms between the two groups' member lists at every coarser
//      level) and restarts the window after the pair; a pair without an
//      accepted move leaves the state as it was, so the window's other
//      results stay valid.
// Every CTA of the cluster runs the same control flow over the same global
// data (window results, fit verdicts), so all reach the same decisions; the
// cluster barrier orders the exchanges.  Member order inside a group is free
// at levels above li (every set predicate is order-independent), so the
// splice appends the mover.
constexpr int RF_THREADS = 512;
constexpr int RF_WARPS = RF_THREADS / 32;
constexpr int RF_WMAX = 1024;         // pairs per window (2 sides each)
constexpr size_t RF_CLUSTER_MIN_PAIRS = 2048;   // fewer recorded merges: one CTA

struct Cand {
    long long s;                      // saving; 0 = none
    int side, ti;
};

struct RefineArgs {
    int ntrans, top;
    const int32_t *pair_off;          // [ntrans + 1]
    const int2 *pairs;                // level-li group indices (v, w)
    int32_t *grp, *goff, *gat;        // the level arrays (written by moves)
    uint32_t *bits;                   // [cluster warps][words] convexity bitmaps
    int words;
    int32_t *tmp;                     // [min(cluster warps, top)][n] splice scratch
    int32_t *src, *dst;               // [top] a move's groups per coarser level
    long long *sav;                   // [2][2 * RF_WMAX] window: best saving per side
    int32_t *sti;                     // [2][2 * RF_WMAX] window: its target
    int32_t *ok;                      // [2 * top] a fit test's per-set verdicts
    Cand *next;                       // [2] next candidates after a rejected one
    int64_t budget;
    long long *stats;                 // windows, side evaluations, fit tests, moves
};

// a ranks before b: larger saving, then side v, then smaller target index
__device__ __forceinline__ bool cand_before(const Cand &a, const Cand &b) {
    if (a.s != b.s) return a.s > b.s;
    if (a.side != b.side) return a.side < b.side;
    return a.ti < b.ti;
}

// base_traffic - traffic(moved) for level-li group `mover` moving into
// top-level block `dest` (blocks.py:193-201), summed exactly over the value
// entries the mover touches (each entry once, at its smallest mover atom);
// the warp's lanes split the mover's atoms
__device__ long long move_saving_warp(const DevAtoms &A, const DevLevels &L, int li, int top,
                                      int mover, int dest) {
    const int lane = threadIdx.x & 31;
    const int32_t *gl = L.grp + (int64_t)li * L.n;
    const int32_t *gt = L.grp + (int64_t)top * L.n;
    const int32_t *off = L.goff + (int64_t)li * (L.n + 1);
    const int32_t *at = L.gat + (int64_t)li * L.n;
    long long saving = 0;
    for (int j = off[mover] + lane; j < off[mover + 1]; j += 32) {
        const int x = at[j];
        for (int q = A.atom_tr_off[x]; q < A.atom_tr_off[x + 1]; ++q) {
            const int e = A.atom_tr[q];
            const int owner = A.tr_owner[e];
            int first = gl[owner] == mover ? owner : 0x7fffffff;
            for (int r = A.tr_cons_off[e]; r < A.tr_cons_off[e + 1]; ++r) {
                const int c = A.tr_cons[r];
                if (gl[c] == mover && c < first) first = c;
            }
            if (first != x) continue;
            const int home0 = gt[owner];
            const int home1 = gl[owner] == mover ? dest : home0;
            int before = 0, after = 0;
            const int c0 = A.tr_cons_off[e], c1 = A.tr_cons_off[e + 1];
            for (int r = c0; r < c1; ++r) {
                const int c = A.tr_cons[r];
                const int b0 = gt[c];
                const int b1 = gl[c] == mover ? dest : b0;
                bool seen0 = b0 == home0, seen1 = b1 == home1;
                for (int u = c0; u < r && !(seen0 && seen1); ++u) {
                    const int cu = A.tr_cons[u];
                    if (gt[cu] == b0) seen0 = true;
                    if ((gl[cu] == mover ? dest : gt[cu]) == b1) seen1 = true;
                }
                before += !seen0;
                after += !seen1;
            }
            saving += A.tr_size[e] * (long long)(before - after);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) saving += __shfl_xor_sync(0xffffffffu, saving, o);
    return saving;
}

// Best positive-saving candidate of one pair side ranking after `after`
// (after.s < 0: no bound).  Targets are visited in ascending index: each
// step takes the smallest neighbouring group index above the last one.
__device__ Cand side_best(const DevAtoms &A, const DevLevels &L, int li, int top, int mover,
                          int side, const Cand &after) {
    const int lane = threadIdx.x & 31;
    const int32_t *gl = L.grp + (int64_t)li * L.n;
    const int32_t *gt = L.grp + (int64_t)top * L.n;
    const int32_t *off = L.goff + (int64_t)li * (L.n + 1);
    const int32_t *at = L.gat + (int64_t)li * L.n;
    const int here = gt[at[off[mover]]];
    Cand best{0, side, 0x7fffffff};
    int last = -1;
    for (;;) {
        int cur = 0x7fffffff;
        for (int j = off[mover] + lane; j < off[mover + 1]; j += 32) {
            const int x = at[j];
            for (int r = A.nbr_off[x]; r < A.nbr_off[x + 1]; ++r) {
                const int t = gl[A.nbr[r]];
                if (t > last && t < cur && t != mover) cur = t;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cur = min(cur, __shfl_xor_sync(0xffffffffu, cur, o));
        if (cur == 0x7fffffff) break;
        last = cur;
        const int dest = gt[at[off[cur]]];
        if (dest == here) continue;                              // blocks.py:189
        const Cand c{move_saving_warp(A, L, li, top, mover, dest), side, cur};
        if (c.s > 0 && (after.s < 0 || cand_before(after, c)) && (best.s == 0 || cand_before(c, best)))
            best = c;
    }
    return best;
}

// move `cnt` atoms (mover) from group src to group dst in one level's CSR
// (labels already rewritten): the groups between the two shift by cnt
__device__ void splice_warp(int32_t *off, int32_t *at, const int32_t *grp, int src, int dst,
                            const int32_t *mover, int cnt, int32_t *tmp) {
    const int lane = threadIdx.x & 31;
    const int s0 = off[src], s1 = off[src + 1], d0 = off[dst], d1 = off[dst + 1];
    const int base = min(s0, d0), end = max(s1, d1);
    int w = 0;
    auto copy_range = [&](int b, int e) {
        for (int j = b + lane; j < e; j += 32) tmp[w + j - b] = at[j];
        w += e - b;
    };
    auto keep_src = [&]() {                                      // src minus the mover
        for (int j0 = s0; j0 < s1; j0 += 32) {
            const int j = j0 + lane;
            const int x = j < s1 ? at[j] : -1;
            const bool keep = j < s1 && grp[x] == src;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) tmp[w + __popc(m & ((1u << lane) - 1u))] = x;
            w += __popc(m);
        }
    };
    auto add_mover = [&]() {
        for (int j = lane; j < cnt; j += 32) tmp[w + j] = mover[j];
        w += cnt;
    };
    if (src < dst) {
        keep_src();
        copy_range(s1, d1);
        add_mover();
    } else {
        copy_range(d0, d1);
        add_mover();
        copy_range(d1, s0);
        keep_src();
    }
    __syncwarp();
    for (int j = lane; j < end - base; j += 32) at[base + j] = tmp[j];
    const int lo = min(src, dst), hi = max(src, dst), delta = src < dst ? -cnt : cnt;
    for (int g = lo + 1 + lane; g <= hi; g += 32) off[g] += delta;
    __syncwarp();
}

__global__ void __launch_bounds__(RF_THREADS, 1) k_refine(DevAtoms A, DevLevels L, RefineArgs R) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank(), nct = (int)cluster.num_blocks();
    // a one-CTA cluster exchanges through its own L1: a CTA barrier suffices
    // (the cluster barrier's acquire would also drop the L1's atom arrays)
    auto csync = [&]() {
        if (nct == 1) __syncthreads();
        else cluster.sync();
    };
    __shared__ int s_first, s_bad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gw = rank * RF_WARPS + warp, NW = nct * RF_WARPS;     // cluster-wide warp
    const int gt = rank * RF_THREADS + tid, NT = nct * RF_THREADS;  // cluster-wide thread
    const int n = L.n;
    const int W0 = max(1, NW / 2);                 // pairs of a window after a move
    uint32_t *bits = R.bits + (int64_t)gw * R.words;
    long long n_win = 0, n_side = 0, n_fit = 0, n_move = 0;
    int buf = 0;                                   // window results double-buffered
    for (int li = R.ntrans - 1; li >= 0; --li) {
        const int2 *pairs = R.pairs + R.pair_off[li];
        const int np = R.pair_off[li + 1] - R.pair_off[li];
        const int nlev = R.top - li;
        const int32_t *offl = L.goff + (int64_t)li * (n + 1);
        const int32_t *atl = L.gat + (int64_t)li * n;
        int p = 0, ws = 0, we = 0, W = W0;
        long long *sav = R.sav;
        int *sti = R.sti;
        while (p < np) {
            if (p >= we) {                                       // 1. a new window
                buf ^= 1;
                sav = R.sav + buf * 2 * RF_WMAX;
                sti = R.sti + buf * 2 * RF_WMAX;
                ws = p;
                we = min(np, p + W);
                for (int it = gw; it < 2 * (we - ws); it += NW) {
                    const int2 pr = pairs[ws + (it >> 1)];
                    const Cand c = side_best(A, L, li, R.top, (it & 1) ? pr.y : pr.x, it & 1,
                                             Cand{-1, 0, 0});
                    if (lane == 0) {
                        sav[it] = c.s;
                        sti[it] = c.ti;
                    }
                }
                ++n_win;
                n_side += 2 * (we - ws);
                csync();
            }
            // the first pair of the window with a candidate (every CTA alike)
            if (tid == 0) s_first = 0x7fffffff;
            __syncthreads();
            for (int it = 2 * (p - ws) + tid; it < 2 * (we - ws); it += RF_THREADS)
                if (sav[it] > 0) atomicMin(&s_first, it >> 1);
            __syncthreads();
            const int fq = s_first;
            __syncthreads();                                     // s_first is reset next
            if (fq == 0x7fffffff) {                              // no candidate in the window
                p = we;
                W = min(2 * W, RF_WMAX);
                continue;
            }
            // 2. test that pair's candidates in rank order
            const int q = ws + fq;
            const int2 pr = pairs[q];
            Cand c0{sav[2 * fq], 0, sti[2 * fq]}, c1{sav[2 * fq + 1], 1, sti[2 * fq + 1]};
            Cand c = c0.s > 0 && (c1.s <= 0 || cand_before(c0, c1)) ? c0 : c1;
            bool moved = false;
            while (c.s > 0) {
                const int mv = c.side ? pr.y : pr.x;
                if (rank == 0) {
                    const int a0 = atl[offl[mv]], t0 = atl[offl[c.ti]];
                    for (int e = tid; e < nlev; e += RF_THREADS) {
                        const int ell = li + 1 + e;
                        R.src[e] = L.grp[(int64_t)ell * n + a0];
                        R.dst[e] = L.grp[(int64_t)ell * n + t0];
                    }
                }
                csync();
                for (int k = gw; k < 2 * nlev; k += NW) {        // _move_fits (blocks.py:206-221)
                    const int e = k >> 1, ell = li + 1 + e;
                    const SetDesc sd = (k & 1) ? SetDesc{ell, R.dst[e], li, mv, 0}     // grown
                                               : SetDesc{ell, R.src[e], li, mv, 1};    // shrunk
                    int cnt;
                    int64_t mem;
                    bool convex;
                    eval_set_warp(A, L, sd, bits, cnt, mem, convex);
                    if (lane == 0) R.ok[k] = convex && mem < R.budget && ((k & 1) || cnt > 0);
                }
                ++n_fit;
                csync();
                if (tid == 0) s_bad = 0;
                __syncthreads();
                for (int k = tid; k < 2 * nlev; k += RF_THREADS)
                    if (!R.ok[k]) s_bad = 1;
                __syncthreads();
                const bool bad = s_bad;
                __syncthreads();
                if (!bad) {                                      // 3. _apply_move (blocks.py:224-232)
                    const int m0 = offl[mv], cnt = offl[mv + 1] - m0;
                    for (int k = gt; k < nlev * cnt; k += NT) {
                        const int e = k / cnt;
                        R.grp[(int64_t)(li + 1 + e) * n + atl[m0 + k % cnt]] = R.dst[e];
                    }
                    csync();
                    for (int e = gw; e < nlev; e += NW) {
                        const int ell = li + 1 + e;
                        splice_warp(R.goff + (int64_t)ell * (n + 1), R.gat + (int64_t)ell * n,
                                    R.grp + (int64_t)ell * n, R.src[e], R.dst[e], atl + m0, cnt,
                                    R.tmp + (int64_t)gw * n);
                    }
                    csync();
                    moved = true;
                    ++n_move;
                    break;
                }
                // next candidate of this pair after the rejected one
                if (gw < 2) {
                    const Cand b = side_best(A, L, li, R.top, gw ? pr.y : pr.x, gw, c);
                    if (lane == 0) R.next[gw] = b;
                }
                csync();
                const Cand b0 = R.next[0], b1 = R.next[1];
                c = b0.s > 0 && (b1.s <= 0 || cand_before(b0, b1)) ? b0 : b1;
                n_side += 2;
            }
            p = q + 1;
            if (moved) {                                         // later savings changed
                we = p;
                W = W0;
            }
        }
    }
    if (rank == 0 && tid == 0) {
        R.stats[0] = n_win;
        R.stats[1] = n_side;
        R.stats[2] = n_fit;
        R.stats[3] = n_move;
    }
}

// ====================================================================== host side
namespace {

struct Coarsener {
    pc_ctx *ctx;
    const pc_atoms *H;
    DevAtoms A{};
    int n;
    // device buffers and pinned level staging live in the context (cb)
    DBuf &atoms_d, &lev_grp, &lev_off, &lev_at, &sets_d, &scratch_d, &out_d, &comp_d;
    int &lev_cap;
    int32_t *&pin;                    // [lev_cap][3n + 1] (grp | off | at)
    std::vector<std::vector<std::vector<int>>> levels;
    std::vector<double> atom_comp;

    Coarsener(pc_ctx *c, const pc_atoms *h)
        : ctx(c), H(h), n(h->n), atoms_d(c->cb.atoms_d), lev_grp(c->cb.lev_grp),
          lev_off(c->cb.lev_off), lev_at(c->cb.lev_at), sets_d(c->cb.sets_d),
          scratch_d(c->cb.scratch_d), out_d(c->cb.out_d), comp_d(c->cb.comp_d),
          lev_cap(c->cb.lev_cap), pin(c->cb.pin) {
        if (c->cb.lev_n != n) {          // slot layout depends on n: re-slice, keep the memory
            cudaStreamSynchronize(c->st);
            const size_t fit_g = c->cb.lev_grp.n / (sizeof(int32_t) * (size_t)std::max(n, 1));
            const size_t fit_o = c->cb.lev_off.n / (sizeof(int32_t) * (size_t)(n + 1));
            const size_t fit_a = c->cb.lev_at.n / (sizeof(int32_t) * (size_t)std::max(n, 1));
            const size_t fit_p = c->cb.pin_bytes / (sizeof(int32_t) * (3 * (size_t)n + 1));
            lev_cap = (int)std::min(std::min(fit_g, fit_o), std::min(fit_a, fit_p));
            c->cb.lev_n = n;
        }
    }

    int upload_atoms() {
        struct Part { const void *src; size_t bytes; size_t off; };
        std::vector<Part> parts;
        size_t total = 0;
        auto add = [&](const void *src, size_t bytes) {
            size_t off = (total + 15) & ~size_t(15);
            parts.push_back({src, bytes, off});
            total = off + bytes;
            return parts.size() - 1;
        };
        const size_t T = H->n_tasks, V = H->n_in, E = H->n_traffic, N = H->n;
        const size_t nd = H->dep_off[T], nin = H->atom_in_off[N], nia = H->in_atoms_off[V];
        const size_t np = H->pred_off[N], nc = H->tr_cons_off[E], ntr = H->atom_tr_off[N];
        size_t i0 = add(H->atom_param, 8 * N), i1 = add(H->task_atom, 4 * T), i2 = add(H->task_flops, 8 * T);
        size_t i3 = add(H->task_fp1, 8 * T), i4 = add(H->dep_off, 4 * (T + 1)), i5 = add(H->dep_owner, 4 * nd);
        size_t i6 = add(H->dep_size, 8 * nd), i7 = add(H->atom_task_off, 4 * (N + 1)), i8 = add(H->atom_tasks, 4 * T);
        size_t i9 = add(H->atom_in_off, 4 * (N + 1)), i10 = add(H->atom_in, 4 * nin), i11 = add(H->in_owner, 4 * V);
        size_t i12 = add(H->in_size, 8 * V), i13 = add(H->in_atoms_off, 4 * (V + 1)), i14 = add(H->in_atoms, 4 * nia);
        size_t i15 = add(H->pred_off, 4 * (N + 1)), i16 = add(H->pred, 4 * np), i17 = add(H->tr_owner, 4 * E);
        size_t i18 = add(H->tr_size, 8 * E), i19 = add(H->tr_cons_off, 4 * (E + 1)), i20 = add(H->tr_cons, 4 * nc);
        size_t i21 = add(H->atom_tr_off, 4 * (N + 1)), i22 = add(H->atom_tr, 4 * ntr);
        size_t i23 = add(H->task_prod1, 8 * T);
        const bool ov = H->ov_has != nullptr;
        size_t i24 = ov ? add(H->ov_has, T) : 0, i25 = ov ? add(H->ov_tf, 8 * T) : 0;
        size_t i26 = ov ? add(H->ov_tb, 8 * T) : 0, i27 = ov ? add(H->ov_act, 8 * T) : 0;
        const size_t nnb = H->nbr_off[N];
        size_t i28 = add(H->nbr_off, 4 * (N + 1)), i29 = add(H->nbr, 4 * nnb);
        CUDA_TRY(ctx, atoms_d.ensure(total + 64));
        std::vector<char> staging(total + 64, 0);
        for (auto &p : parts)
            if (p.bytes) memcpy(staging.data() + p.off, p.src, p.bytes);
        CUDA_TRY(ctx, cudaMemcpy(atoms_d.p, staging.data(), total, cudaMemcpyHostToDevice));
        char *b = atoms_d.as<char>();
        auto at = [&](size_t i) { return (void *)(b + parts[i].off); };
        A.n = (int)N;
        A.T = (int)T;
        A.V = (int)V;
        A.E = (int)E;
        A.budget = H->budget;
        A.factor = (1.0 + H->grad_factor) + H->opt_factor;
        A.flops = H->flops_per_sec;
        A.beta = H->bwd_fwd_ratio;
        A.atom_param = (const int64_t *)at(i0);
        A.task_atom = (const int32_t *)at(i1);
        A.task_flops = (const double *)at(i2);
        A.task_fp1 = (const int64_t *)at(i3);
        A.dep_off = (const int32_t *)at(i4);
        A.dep_owner = (const int32_t *)at(i5);
        A.dep_size = (const int64_t *)at(i6);
        A.atom_task_off = (const int32_t *)at(i7);
        A.atom_tasks = (const int32_t *)at(i8);
        A.atom_in_off = (const int32_t *)at(i9);
        A.atom_in = (const int32_t *)at(i10);
        A.in_owner = (const int32_t *)at(i11);
        A.in_size = (const int64_t *)at(i12);
        A.in_atoms_off = (const int32_t *)at(i13);
        A.in_atoms = (const int32_t *)at(i14);
        A.pred_off = (const int32_t *)at(i15);
        A.pred = (const int32_t *)at(i16);
        A.tr_owner = (const int32_t *)at(i17);
        A.tr_size = (const int64_t *)at(i18);
        A.tr_cons_off = (const int32_t *)at(i19);
        A.tr_cons = (const int32_t *)at(i20);
        A.atom_tr_off = (const int32_t *)at(i21);
        A.atom_tr = (const int32_t *)at(i22);
        A.task_prod1 = (const int64_t *)at(i23);
        A.ov_has = ov ? (const uint8_t *)at(i24) : nullptr;
        A.ov_tf = ov ? (const double *)at(i25) : nullptr;
        A.ov_tb = ov ? (const double *)at(i26) : nullptr;
        A.ov_act = ov ? (const int64_t *)at(i27) : nullptr;
        A.nbr_off = (const int32_t *)at(i28);
        A.nbr = (const int32_t *)at(i29);
        return PC_OK;
    }

    DevLevels dev_levels() const {
        return DevLevels{lev_grp.as<int32_t>(), lev_off.as<int32_t>(), lev_at.as<int32_t>(), n};
    }

    // copy level `l` (list of ascending atom groups) into device slot l: the
    // level's pinned staging slot is only rewritten after a later sync, so the
    // copies stay asynchronous
    int upload_level(int l, const std::vector<std::vector<int>> &groups) {
        const size_t per = 3 * (size_t)n + 1;
        if (l >= lev_cap) {
            CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
            int cap = std::max(16, 2 * (l + 1));
            DBuf g2, o2, a2;
            CUDA_TRY(ctx, g2.ensure(sizeof(int32_t) * (size_t)cap * n));
            CUDA_TRY(ctx, o2.ensure(sizeof(int32_t) * (size_t)cap * (n + 1)));
            CUDA_TRY(ctx, a2.ensure(sizeof(int32_t) * (size_t)cap * n));
            int32_t *p2 = nullptr;
            CUDA_TRY(ctx, cudaMallocHost(&p2, sizeof(int32_t) * per * cap));
            ctx->cb.pin_bytes = sizeof(int32_t) * per * cap;
            if (lev_cap) {
                CUDA_TRY(ctx, cudaMemcpy(g2.p, lev_grp.p, sizeof(int32_t) * (size_t)lev_cap * n, cudaMemcpyDeviceToDevice));
                CUDA_TRY(ctx, cudaMemcpy(o2.p, lev_off.p, sizeof(int32_t) * (size_t)lev_cap * (n + 1), cudaMemcpyDeviceToDevice));
                CUDA_TRY(ctx, cudaMemcpy(a2.p, lev_at.p, sizeof(int32_t) * (size_t)lev_cap * n, cudaMemcpyDeviceToDevice));
            }
            if (pin) cudaFreeHost(pin);
            pin = p2;
            std::swap(lev_grp.p, g2.p); std::swap(lev_grp.n, g2.n);
            std::swap(lev_off.p, o2.p); std::swap(lev_off.n, o2.n);
            std::swap(lev_at.p, a2.p); std::swap(lev_at.n, a2.n);
            lev_cap = cap;
        }
        int32_t *grp = pin + per * l, *off = grp + n, *at = off + n + 1;
        std::fill(grp, grp + n, -1);
        off[0] = 0;
        int32_t pos = 0;
        for (size_t g = 0; g < groups.size(); ++g) {
            for (int x : groups[g]) {
                grp[x] = (int32_t)g;
                at[pos++] = x;
            }
            off[g + 1] = pos;
        }
        for (size_t g = groups.size(); g < (size_t)n; ++g) off[g + 1] = pos;
        for (int32_t q = pos; q < n; ++q) at[q] = 0;
        CUDA_TRY(ctx, cudaMemcpyAsync(lev_grp.as<int32_t>() + (size_t)l * n, grp, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(lev_off.as<int32_t>() + (size_t)l * (n + 1), off, 4 * (size_t)(n + 1), cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(lev_at.as<int32_t>() + (size_t)l * n, at, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
        return PC_OK;
    }

    // pinned read-back staging (pageable D2H copies would each block)
    char *pinned_out(size_t bytes) {
        CoarsenBufs &cb = ctx->cb;
        if (cb.pout_bytes < bytes) {
            cudaStreamSynchronize(ctx->st);
            if (cb.pout) cudaFreeHost(cb.pout);
            cb.pout = nullptr;
            cb.pout_bytes = 0;
            const size_t want = std::max(bytes, (size_t)1 << 20);
            if (cudaMallocHost(&cb.pout, want) != cudaSuccess) return nullptr;
            cb.pout_bytes = want;
        }
        return cb.pout;
    }

    // k_eval_sets over `sets` (launch only; outputs in out_d)
    int eval_launch(const std::vector<SetDesc> &sets) {
        const int ns = (int)sets.size();
        if (!ns) return PC_OK;
        const int words = (n + 31) / 32 + 1;
        CUDA_TRY(ctx, sets_d.ensure(sizeof(SetDesc) * ns));
        CUDA_TRY(ctx, scratch_d.ensure(sizeof(uint32_t) * (size_t)ns * words));
        CUDA_TRY(ctx, out_d.ensure((8 + 4 + 1) * (size_t)ns + 64));
        CUDA_TRY(ctx, cudaMemcpyAsync(sets_d.p, sets.data(), sizeof(SetDesc) * ns, cudaMemcpyHostToDevice, ctx->st));
        int64_t *om = out_d.as<int64_t>();
        int32_t *oc = (int32_t *)(om + ns);
        uint8_t *ov = (uint8_t *)(oc + ns);
        k_eval_sets_warp<<<(unsigned)(((int64_t)ns * 32 + 127) / 128), 128, 0, ctx->st>>>(
            A, dev_levels(), sets_d.as<SetDesc>(), ns, scratch_d.as<uint32_t>(), words, om, oc, ov);
        ctx->launches++;
        return check_launch(ctx, "eval_sets");
    }

    // group compute times of level l and the set evaluations, one sync
    int comps_eval(int l, int ngroups, std::vector<double> &gc, const std::vector<SetDesc> &sets,
                   std::vector<int64_t> &mem, std::vector<int32_t> &count, std::vector<uint8_t> &convex) {
        const size_t ns = sets.size();
        CUDA_TRY(ctx, ctx->cb.gc_d.ensure(sizeof(double) * ngroups + 64));
        k_group_comps<<<(ngroups + 127) / 128, 128, 0, ctx->st>>>(dev_levels(), l, ngroups, comp_d.as<double>(),
                                                                 ctx->cb.gc_d.as<double>());
        ctx->launches++;
        if (int rc = check_launch(ctx, "group_comps")) return rc;
        if (int rc = eval_launch(sets)) return rc;
        const size_t gbytes = sizeof(double) * (size_t)ngroups, sbytes = 13 * ns;
        char *h = pinned_out(gbytes + sbytes + 16);
        if (!h) return fail(ctx, PC_ERR_CUDA, "pinned staging");
        CUDA_TRY(ctx, cudaMemcpyAsync(h, ctx->cb.gc_d.p, gbytes, cudaMemcpyDeviceToHost, ctx->st));
        if (ns) CUDA_TRY(ctx, cudaMemcpyAsync(h + gbytes, out_d.p, sbytes, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        gc.assign((const double *)h, (const double *)h + ngroups);
        const int64_t *om = (const int64_t *)(h + gbytes);
        const int32_t *oc = (const int32_t *)(om + ns);
        const uint8_t *ov = (const uint8_t *)(oc + ns);
        mem.assign(om, om + ns);
        count.assign(oc, oc + ns);
        convex.assign(ov, ov + ns);
        return PC_OK;
    }

    int eval(const std::vector<SetDesc> &sets, std::vector<int64_t> &mem, std::vector<int32_t> &count,
             std::vector<uint8_t> &convex) {
        const size_t ns = sets.size();
        mem.assign(ns, 0);
        count.assign(ns, 0);
        convex.assign(ns, 0);
        if (!ns) return PC_OK;
        if (int rc = eval_launch(sets)) return rc;
        char *h = pinned_out(13 * ns + 16);
        if (!h) return fail(ctx, PC_ERR_CUDA, "pinned staging");
        CUDA_TRY(ctx, cudaMemcpyAsync(h, out_d.p, 13 * ns, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        const int64_t *om = (const int64_t *)h;
        const int32_t *oc = (const int32_t *)(om + ns);
        const uint8_t *ov = (const uint8_t *)(oc + ns);
        mem.assign(om, om + ns);
        count.assign(oc, oc + ns);
        convex.assign(ov, ov + ns);
        return PC_OK;
    }

    int profiles(int l, int ngroups, bool single, std::vector<double> &tf, std::vector<double> &tb,
                 std::vector<double> &comp, std::vector<int64_t> &mem) {
        CUDA_TRY(ctx, out_d.ensure(32 * (size_t)ngroups + 64));
        double *a = out_d.as<double>();
        if (single)
            k_atom_profiles<<<(ngroups + 127) / 128, 128, 0, ctx->st>>>(A, dev_levels(), l, ngroups, a, a + ngroups,
                                                                       a + 2 * ngroups, (int64_t *)(a + 3 * ngroups));
        else
            k_group_profiles<<<(unsigned)(((int64_t)ngroups * 32 + 127) / 128), 128, 0, ctx->st>>>(
                A, dev_levels(), l, ngroups, a, a + ngroups, a + 2 * ngroups, (int64_t *)(a + 3 * ngroups));
        ctx->launches++;
        if (int rc = check_launch(ctx, "group_profiles")) return rc;
        char *h = pinned_out(32 * (size_t)ngroups + 16);
        if (!h) return fail(ctx, PC_ERR_CUDA, "pinned staging");
        CUDA_TRY(ctx, cudaMemcpyAsync(h, a, 32 * (size_t)ngroups, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        const double *hd = (const double *)h;
        tf.assign(hd, hd + ngroups);
        tb.assign(hd + ngroups, hd + 2 * ngroups);
        comp.assign(hd + 2 * ngroups, hd + 3 * ngroups);
        mem.assign((const int64_t *)(hd + 3 * ngroups), (const int64_t *)(hd + 4 * ngroups));
        return PC_OK;
    }
};

std::vector<int> member_map(int n, const std::vector<std::vector<int>> &level);
void sort_by_first(std::vector<std::vector<int>> &level);

using Transitions = std::vector<std::vector<int2>>;   // per level: merged (v, w) group indices

// _uncoarsen on the device (k_refine): the recorded merges go up as level
// group-index pairs, one launch walks every level, and the top level's labels
// come back (the only level used afterwards).  stats: windows, side
// evaluations, fit tests, moves.
int refine_on_device(Coarsener &co, const Transitions &tr, long long stats[4]) {
    pc_ctx *ctx = co.ctx;
    const int n = co.n, top = (int)co.levels.size() - 1, nt = (int)tr.size();
    std::vector<int32_t> head(nt + 1, 0);
    std::vector<int2> pairs;
    for (int li = 0; li < nt; ++li) {
        pairs.insert(pairs.end(), tr[li].begin(), tr[li].end());
        head[li + 1] = (int32_t)pairs.size();
    }
    // the cluster: as many CTAs (one per SM) as the device co-schedules, <= 16
    int &ncl = ctx->cb.refine_cluster;
    if (ncl == 0) {
        ncl = 1;
        if (cudaFuncSetAttribute(k_refine, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            cudaGetLastError();
        for (int c = 16; c > 1; c /= 2) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(c);
            cfg.blockDim = dim3(RF_THREADS);
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, k_refine, &cfg) == cudaSuccess && nc > 0) {
                ncl = c;
                break;
            }
            cudaGetLastError();
        }
    }
    // A cluster barrier costs a few microseconds per window or move (its
    // acquire also drops the L1's atom arrays), one CTA's barrier almost
    // nothing; the cluster pays off once windows are wide, i.e. on many pairs
    // (measured, r2be: C1 / C2 with 211 / 931 pairs 1.22 / 1.83 ms on one CTA
    // vs 1.68 / 1.98 on 16; C4 with 2,531 pairs 2.87 vs 2.43; 15,362 pairs
    // 12.2 vs 6.6 ms).
    int cl = pairs.size() >= RF_CLUSTER_MIN_PAIRS ? ncl : 1;
    if (const char *e = getenv("PIPECUT_B200_REFINE_CLUSTER"))     // tests / A-B
        cl = std::max(1, std::min(ncl, atoi(e)));
    const int NW = cl * RF_WARPS;
    const int words = (n + 31) / 32 + 1;
    size_t total = 0;
    auto carve = [&](size_t bytes) { const size_t o = (total + 15) & ~size_t(15); total = o + bytes; return o; };
    const size_t o_stats = carve(4 * sizeof(long long)), o_head = carve(4 * head.size());
    const size_t o_pairs = carve(sizeof(int2) * pairs.size()), o_src = carve(4 * (size_t)top);
    const size_t o_dst = carve(4 * (size_t)top), o_bits = carve(4 * (size_t)NW * words);
    const size_t o_tmp = carve(4 * (size_t)std::min(NW, top) * n);
    const size_t o_sav = carve(sizeof(long long) * 4 * RF_WMAX), o_sti = carve(4 * 4 * RF_WMAX);
    const size_t o_ok = carve(4 * 2 * (size_t)top), o_next = carve(2 * sizeof(Cand));
    CUDA_TRY(ctx, ctx->cb.refine_d.ensure(total + 64));
    char *b = ctx->cb.refine_d.as<char>();
    std::vector<char> up(o_src - o_head);
    memcpy(up.data(), head.data(), 4 * head.size());
    if (!pairs.empty()) memcpy(up.data() + (o_pairs - o_head), pairs.data(), sizeof(int2) * pairs.size());
    CUDA_TRY(ctx, cudaMemcpyAsync(b + o_head, up.data(), up.size(), cudaMemcpyHostToDevice, ctx->st));
    RefineArgs R;
    R.ntrans = nt;
    R.top = top;
    R.pair_off = (const int32_t *)(b + o_head);
    R.pairs = (const int2 *)(b + o_pairs);
    R.grp = co.lev_grp.as<int32_t>();
    R.goff = co.lev_off.as<int32_t>();
    R.gat = co.lev_at.as<int32_t>();
    R.bits = (uint32_t *)(b + o_bits);
    R.words = words;
    R.tmp = (int32_t *)(b + o_tmp);
    R.src = (int32_t *)(b + o_src);
    R.dst = (int32_t *)(b + o_dst);
    R.sav = (long long *)(b + o_sav);
    R.sti = (int32_t *)(b + o_sti);
    R.ok = (int32_t *)(b + o_ok);
    R.next = (Cand *)(b + o_next);
    R.budget = co.H->budget;
    R.stats = (long long *)(b + o_stats);
    {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(RF_THREADS);
        cfg.stream = ctx->st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const DevLevels L = co.dev_levels();
        CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k_refine, co.A, L, R));
    }
    ctx->launches++;
    if (int rc = check_launch(ctx, "refine")) return rc;
    std::vector<int32_t> lab(n);
    CUDA_TRY(ctx, cudaMemcpyAsync(lab.data(), co.lev_grp.as<int32_t>() + (size_t)top * n, 4 * (size_t)n,
                                  cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(stats, b + o_stats, 4 * sizeof(long long), cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    // the top level from its labels; levels 1..top-1 are stale on the host
    // from here (moves changed them on the device) and are not read again
    std::vector<std::vector<int>> groups(co.levels[top].size());
    for (int x = 0; x < n; ++x) groups[lab[x]].push_back(x);
    sort_by_first(groups);
    co.levels[top] = groups;
    return PC_OK;
}

std::vector<int> member_map(int n, const std::vector<std::vector<int>> &level) {
    std::vector<int> m(n, -1);
    for (size_t g = 0; g < level.size(); ++g)
        for (int x : level[g]) m[x] = (int)g;
    return m;
}

void sort_by_first(std::vector<std::vector<int>> &level) {
    std::sort(level.begin(), level.end(),
              [](const std::vector<int> &a, const std::vector<int> &b) { return a[0] < b[0]; });
}

}  // namespace
}  // namespace pcb

using namespace pcb;

extern "C" int pc_partition_blocks(pc_ctx *ctx, const pc_atoms *H, int32_t k, int32_t *n_blocks,
                                   int32_t *block_off, int32_t *block_atoms, double *out_tf,
                                   double *out_tb, int64_t *out_mem, int64_t *err) {
    if (k < 1) return fail(ctx, PC_ERR_INVALID, "k must be at least 1");
    if (H->n < 1) return fail(ctx, PC_ERR_INVALID, "no atoms");
    cudaSetDevice(ctx->device);
    Coarsener co(ctx, H);
    const int n = H->n;
    const int64_t budget = H->budget;
    // PIPECUT_B200_BLOCKS_TIMES: host wall time per phase (debug)
    const bool phase_times = getenv("PIPECUT_B200_BLOCKS_TIMES") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto phase = [&](const char *what) {
        if (!phase_times) return;
        cudaStreamSynchronize(ctx->st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[pipecut_b200] blocks %-12s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t_prev).count());
        t_prev = now;
    };
    if (int rc = co.upload_atoms()) return rc;
    phase("upload");

    // ---- level 0 and the atoms' own profiles (blocks.py:89-94, 366-369)
    std::vector<std::vector<int>> l0(n);
    for (int i = 0; i < n; ++i) l0[i] = {i};
    co.levels.push_back(l0);
    if (int rc = co.upload_level(0, l0)) return rc;
    std::vector<double> tf, tb, comp;
    std::vector<int64_t> mem;
    if (int rc = co.profiles(0, n, true, tf, tb, comp, mem)) return rc;
    co.atom_comp = comp;
    CUDA_TRY(ctx, co.comp_d.ensure(sizeof(double) * n));
    CUDA_TRY(ctx, cudaMemcpy(co.comp_d.p, comp.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    for (int i = 0; i < n; ++i) {
        if (mem[i] >= budget) {                                 // InfeasibleAtom
            err[0] = i;
            err[1] = mem[i];
            return fail(ctx, PC_ERR_ATOM, "atom exceeds device memory");
        }
    }
    const int32_t *nbr_off = H->nbr_off, *nbr = H->nbr;

    phase("level0");
    // ---- coarsening passes (blocks.py:127-166, 371-378)
    Transitions transitions;
    double t_adj = 0, t_dev = 0, t_greedy = 0, t_next = 0;     // PIPECUT_B200_BLOCKS_TIMES split
    auto tick = [&]() { return phase_times ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point(); };
    auto since = [&](std::chrono::steady_clock::time_point t) {
        return phase_times ? std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count() : 0.0;
    };
    while ((int)co.levels.back().size() > k) {
        auto tc = tick();
        const int L = (int)co.levels.size() - 1;
        const std::vector<std::vector<int>> &G = co.levels[L];
        const int m = (int)G.size();
        const std::vector<int> gmap = member_map(n, G);
        // every adjacent pair (CSR, ascending per group), evaluated once on
        // the device; aset = the pair's set index from either side
        std::vector<int> aoff(m + 1, 0), adj, aset;
        std::vector<int> c;
        for (int gi = 0; gi < m; ++gi) {
            c.clear();
            for (int a : G[gi])
                for (int q = nbr_off[a]; q < nbr_off[a + 1]; ++q) {
                    const int gj = gmap[nbr[q]];
                    if (gj != gi) c.push_back(gj);
                }
            std::sort(c.begin(), c.end());
            c.erase(std::unique(c.begin(), c.end()), c.end());
            adj.insert(adj.end(), c.begin(), c.end());
            aoff[gi + 1] = (int)adj.size();
        }
        std::vector<SetDesc> sets;
        aset.assign(adj.size(), -1);
        for (int gi = 0; gi < m; ++gi)
            for (int e = aoff[gi]; e < aoff[gi + 1]; ++e)
                if (gi < adj[e]) {
                    aset[e] = (int)sets.size();
                    sets.push_back(SetDesc{L, gi, L, adj[e], 0});
                }
        for (int gi = 0; gi < m; ++gi)
            for (int e = aoff[gi]; e < aoff[gi + 1]; ++e)
                if (gi > adj[e]) {
                    const int gj = adj[e];
                    const int f = (int)(std::lower_bound(adj.begin() + aoff[gj], adj.begin() + aoff[gj + 1], gi) -
                                        adj.begin());
                    aset[e] = aset[f];
                }
        std::vector<double> gc;
        std::vector<int64_t> smem;
        std::vector<int32_t> scount;
        std::vector<uint8_t> sconv;
        t_adj += since(tc);
        tc = tick();
        if (int rc = co.comps_eval(L, m, gc, sets, smem, scount, sconv)) return rc;
        t_dev += since(tc);
        tc = tick();
        auto key_less = [&](int a, int b) {
            if (gc[a] != gc[b]) return gc[a] < gc[b];
            return G[a][0] < G[b][0];
        };
        std::vector<int> order(m);
        for (int i = 0; i < m; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), key_less);
        // the greedy pass over the device's answers
        std::vector<char> used(m, 0);
        std::vector<int> partner(m, -1);
        int count = m;
        std::vector<std::pair<int, int>> cands;                 // (group, set)
        for (int gi : order) {
            if (count <= k) break;
            if (used[gi]) continue;
            cands.clear();
            for (int e = aoff[gi]; e < aoff[gi + 1]; ++e)
                if (!used[adj[e]]) cands.push_back({adj[e], aset[e]});
            std::sort(cands.begin(), cands.end(),
                      [&](const std::pair<int, int> &a, const std::pair<int, int> &b) { return key_less(a.first, b.first); });
            for (const auto &gs : cands) {
                const int gj = gs.first, si = gs.second;
                if (sconv[si] && smem[si] < budget) {           // is_convex and fits (blocks.py:115-116)
                    partner[gi] = gj;
                    used[gi] = used[gj] = 1;
                    --count;
                    break;
                }
            }
        }
        t_greedy += since(tc);
        tc = tick();
        std::vector<char> absorbed(m, 0);
        for (int gi = 0; gi < m; ++gi)
            if (partner[gi] >= 0) absorbed[partner[gi]] = 1;
        std::vector<std::vector<int>> next;
        std::vector<int2> merges;                               // (v, w) as level-L group indices
        next.reserve(m);
        for (int gi = 0; gi < m; ++gi) {
            if (absorbed[gi]) continue;
            if (partner[gi] < 0) {
                next.push_back(G[gi]);
            } else {
                const std::vector<int> &v = G[gi], &w = G[partner[gi]];
                std::vector<int> u(v.size() + w.size());
                std::merge(v.begin(), v.end(), w.begin(), w.end(), u.begin());
                next.push_back(std::move(u));
                merges.push_back(make_int2(gi, partner[gi]));
            }
        }
        if (merges.empty()) break;
        sort_by_first(next);
        co.levels.push_back(std::move(next));
        transitions.push_back(std::move(merges));
        if (int rc = co.upload_level(L + 1, co.levels.back())) return rc;
        t_next += since(tc);
    }

    if (phase_times)
        fprintf(stderr, "[pipecut_b200] coarsen: %d levels, adjacency %.2f ms, device + sync %.2f ms, "
                        "greedy %.2f ms, next level %.2f ms\n", (int)co.levels.size(), t_adj, t_dev, t_greedy, t_next);
    phase("coarsen");
    const int top = (int)co.levels.size() - 1;
    if (!transitions.empty()) {
        long long st[4];
        if (int rc = refine_on_device(co, transitions, st)) return rc;
        if (phase_times)
            fprintf(stderr, "[pipecut_b200] refine: %lld windows, %lld side evaluations, "
                            "%lld fit tests, %lld moves\n", st[0], st[1], st[2], st[3]);
    }
    phase("refine");
    // ---- dependency order (blocks.py:235-255) and compaction (267-292)
    auto topo = [&](const std::vector<std::vector<int>> &groups) {
        const int m = (int)groups.size();
        const std::vector<int> gm = member_map(n, groups);
        std::vector<std::set<int>> out(m);
        std::vector<int> indeg(m, 0);
        for (int a = 0; a < n; ++a)
            for (int q = H->succ_off[a]; q < H->succ_off[a + 1]; ++q) {
                const int ga = gm[a], gb = gm[H->succ[q]];
                if (ga != gb && out[ga].insert(gb).second) indeg[gb]++;
            }
        std::priority_queue<std::pair<int, int>, std::vector<std::pair<int, int>>, std::greater<>> heap;
        for (int g = 0; g < m; ++g)
            if (indeg[g] == 0) heap.push({groups[g][0], g});
        std::vector<std::vector<int>> order;
        while (!heap.empty()) {
            const int g = heap.top().second;
            heap.pop();
            order.push_back(groups[g]);
            for (int nbg : out[g])
                if (--indeg[nbg] == 0) heap.push({groups[nbg][0], nbg});
        }
        return order;
    };
    std::vector<std::vector<int>> glist = topo(co.levels[top]);
    if ((int)glist.size() != (int)co.levels[top].size())
        return fail(ctx, PC_ERR_INVALID, "group contraction must stay acyclic");
    if ((int)glist.size() > k) {
        const int scratch = (int)co.levels.size();
        while ((int)glist.size() > k) {
            if (int rc = co.upload_level(scratch, glist)) return rc;
            const int m = (int)glist.size();
            std::vector<SetDesc> sets;
            for (int pos = 0; pos + 1 < m; ++pos) sets.push_back(SetDesc{scratch, pos, scratch, pos + 1, 0});
            std::vector<double> gc;
            std::vector<int64_t> smem;
            std::vector<int32_t> scount;
            std::vector<uint8_t> sconv;
            if (int rc = co.comps_eval(scratch, m, gc, sets, smem, scount, sconv)) return rc;
            // groups of glist are disjoint, so level `scratch` indexes them by position
            std::vector<int> order(m);
            for (int i = 0; i < m; ++i) order[i] = i;
            auto key_less = [&](int a, int b) {
                if (gc[a] != gc[b]) return gc[a] < gc[b];
                return glist[a][0] < glist[b][0];
            };
            std::sort(order.begin(), order.end(), key_less);
            int merged_at = -1;
            for (int pos : order) {
                std::vector<int> sides;
                if (pos - 1 >= 0) sides.push_back(pos - 1);
                if (pos + 1 < m) sides.push_back(pos + 1);
                std::sort(sides.begin(), sides.end(), key_less);
                for (int side : sides) {
                    const int lo = std::min(pos, side);
                    if (smem[lo] < budget) {                    // fits(union)
                        std::vector<int> u = glist[lo];
                        u.insert(u.end(), glist[lo + 1].begin(), glist[lo + 1].end());
                        std::sort(u.begin(), u.end());
                        glist[lo] = u;
                        glist.erase(glist.begin() + lo + 1);
                        merged_at = lo;
                        break;
                    }
                }
                if (merged_at >= 0) break;
            }
            if (merged_at < 0) {
                err[0] = (int64_t)glist.size();
                return fail(ctx, PC_ERR_STUCK, "compaction stuck");
            }
        }
        glist = topo(glist);
    }

    phase("compact");
    // ---- outputs: blocks and their profiles (blocks.py:387-397)
    const int nbk = (int)glist.size();
    const int fin = (int)co.levels.size();
    if (int rc = co.upload_level(fin, glist)) return rc;
    if (int rc = co.profiles(fin, nbk, false, tf, tb, comp, mem)) return rc;
    *n_blocks = nbk;
    int pos = 0;
    block_off[0] = 0;
    for (int b = 0; b < nbk; ++b) {
        for (int a : glist[b]) block_atoms[pos++] = a;
        block_off[b + 1] = pos;
        out_tf[b] = tf[b];
        out_tb[b] = tb[b];
        out_mem[b] = mem[b];
    }
    phase("outputs");
    return PC_OK;
}
