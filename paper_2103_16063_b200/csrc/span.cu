// K1/K2: span-cost and cut-time tables.
//
// Replaces _Profiler.record -> CostModel.profile(BlockSet.span(lo, hi), m, ckpt)
// (pkg/src/pipecut/stages.py:138-145, costs.py:97-160, blocks.py:333-343) and
// _Profiler.cut_time (stages.py:147-157) for every span of a BlockSet and every
// (m, ckpt) key a batch of DP calls needs.  The flat restatement the kernels
// evaluate is documented in paper_2103_16063_b200/flatten.py.
#include "common.cuh"

namespace pcb {

// ---------------------------------------------------------------- input tables
// in(lo, hi) = sum over span-input values v of (fix, ps):
//   v counts iff ob(v) < lo and cstar(v, lo) < hi, cstar = first consumer block >= lo
// One CTA per lo scatters every value into a delta array over cstar and
// prefix-sums it over hi.  Integer sums: order-free, exact.
__global__ void k_in_tables(DevProblem p, int64_t *out_fix, int64_t *out_ps) {
    extern __shared__ int64_t sm[];
    const int nb = p.nb;
    const int lo = blockIdx.x;
    int64_t *dfix = sm;            // [nb]
    int64_t *dps = sm + nb;        // [nb]
    for (int i = threadIdx.x; i < nb; i += blockDim.x) { dfix[i] = 0; dps[i] = 0; }
    __syncthreads();
    for (int v = threadIdx.x; v < p.n_in; v += blockDim.x) {
        if (p.in_ob[v] >= lo) continue;
        for (int k = p.in_cons_off[v]; k < p.in_cons_off[v + 1]; ++k) {
            int c = p.in_cons[k];
            if (c >= lo) {
                atomicAdd((unsigned long long *)&dfix[c], (unsigned long long)p.in_fix[v]);
                atomicAdd((unsigned long long *)&dps[c], (unsigned long long)p.in_ps[v]);
                break;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t af = 0, ap = 0;
        const int64_t row = tri_row(lo, nb);
        for (int hi = lo + 1; hi <= nb; ++hi) {
            af += dfix[hi - 1];
            ap += dps[hi - 1];
            out_fix[row + (hi - lo - 1)] = af;
            out_ps[row + (hi - lo - 1)] = ap;
        }
    }
}

void launch_in_tables(const DevProblem &p, int64_t *in_fix, int64_t *in_ps, cudaStream_t st) {
    size_t smem = sizeof(int64_t) * 2 * (size_t)p.nb;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_in_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_in_tables<<<p.nb, 256, smem, st>>>(p, in_fix, in_ps);
}

// ---------------------------------------------------------------- time folds
// General (non-monotone) fold: one warp per (key, lo, 32 consecutive hi).
// All lanes walk the sorted task list together (costs.py:120) and each lane
// adds the tasks with lo <= block < its hi, so the fp64 fold order is the
// reference's exactly.
__global__ void k_span_time_general(DevProblem p, int n_keys, const int64_t *keys_m,
                                    double *raw_tf, double *raw_tb) {
    const int nb = p.nb;
    const int chunks = (nb + 31) / 32;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    const int64_t per_key = (int64_t)nb * chunks;
    if (gw >= per_key * n_keys) return;
    const int k = (int)(gw / per_key);
    const int rem = (int)(gw % per_key);
    const int lo = rem / chunks;
    const int chunk = rem % chunks;
    if (lo + 1 + chunk * 32 > nb) return;
    const int hi = lo + 1 + chunk * 32 + lane;
    const double m = (double)keys_m[k];
    const int ov = ov_index(p, keys_m[k]);
    double tf = 0.0, tb = 0.0;
    for (int t = 0; t < p.n_tasks; ++t) {
        const int b = p.task_block[t];
        if (b < lo) continue;
        double x, y;
        task_times(p, ov, t, m, x, y);
        if (b < hi) {
            tf = __dadd_rn(tf, x);
            tb = __dadd_rn(tb, y);
        }
    }
    if (hi <= nb) {
        const int64_t idx = (int64_t)k * tri_size(nb) + tri_idx(lo, hi, nb);
        raw_tf[idx] = tf;
        raw_tb[idx] = tb;
    }
}

void launch_span_time_general(const DevProblem &p, int n_keys, const int64_t *keys_m,
                              double *raw_tf, double *raw_tb, cudaStream_t st) {
    const int chunks = (p.nb + 31) / 32;
    const int64_t warps = (int64_t)n_keys * p.nb * chunks;
    const int wpb = 8;
    const int64_t blocks = (warps + wpb - 1) / wpb;
    k_span_time_general<<<(unsigned)blocks, wpb * 32, 0, st>>>(p, n_keys, keys_m, raw_tf, raw_tb);
}

// ---------------------------------------------------------------- span rows
// One thread per (key, lo) sweeps hi = lo+1..nb:
//   * running max of task footprints (costs.py:150-155), each task's
//     footprint counting only predecessors owned in blocks >= lo;
//   * in the monotone case the time fold itself (blocks in sorted-id order,
//     so extending hi continues the reference's fold exactly) over the key's
//     task times (raw_tf / raw_tb: [key][task], k_key_task_times); otherwise
//     raw_tf / raw_tb hold the general fold's span times ([key][tri]);
//   * memory (costs.py:157-159) -> feasibility (stages.py:230) folded into the
//     table as NaN;
//   * its row of the per-key cut-time table (stages.py:147-157).
// Output layout is hi-major (lo contiguous), the DP's predecessor order.
// With beta a power of two, t_bwd == beta * t_fwd exactly (scaling by 2^k
// commutes with every rounding of the fold); the DP then derives it and only
// t_fwd is stored -- verified here for every span, flag set on any mismatch.
template <bool MONO>
__global__ void k_span_rows(DevProblem p, int n_keys, const int64_t *keys_m,
                            const int32_t *keys_ckpt, const double *raw_tf,
                            const double *raw_tb, double *const *tf_out, double *const *tb_out,
                            double *const *cut_out, int derived, int *mismatch) {
    const int nb = p.nb;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)n_keys * nb) return;
    const int k = (int)(gid / nb);
    const int lo = (int)(gid % nb);
    const int64_t m = keys_m[k];
    const int ckpt = keys_ckpt[k];
    const int64_t tri = tri_size(nb);
    double *out_f = tf_out[k];
    double *out_b = derived ? nullptr : tb_out[k];
    double *cut = cut_out[k];
    for (int i = 0; i < 2; ++i) {
        cut[(int64_t)i * (nb + 1) + lo] = cut_time_dev(p, lo, m, i);
        if (lo == nb - 1) cut[(int64_t)i * (nb + 1) + nb] = cut_time_dev(p, nb, m, i);
    }
    const int ov = ov_index(p, m);
    double tf = 0.0, tb = 0.0;
    int64_t run_fp = 0;
    bool bad = false;
    const int64_t row = tri_row(lo, nb);
    // The block -> task indirection is loaded one block ahead (the row is a
    // chain of dependent loads otherwise: offsets, task, its dependencies).
    int q0 = p.blk_off[lo], q1 = p.blk_off[lo + 1];
    int t0 = q0 < q1 ? p.blk_tasks[q0] : 0;
    int e0 = q0 < q1 ? p.dep_off[t0] : 0, e1 = q0 < q1 ? p.dep_off[t0 + 1] : 0;
    for (int hi = lo + 1; hi <= nb; ++hi) {
        const int c0 = q0, c1 = q1, ct = t0, ce0 = e0, ce1 = e1;
        if (hi < nb) {
            q0 = c1;
            q1 = p.blk_off[hi + 1];
            t0 = q0 < q1 ? p.blk_tasks[q0] : 0;
            e0 = q0 < q1 ? p.dep_off[t0] : 0;
            e1 = q0 < q1 ? p.dep_off[t0 + 1] : 0;
        }
        for (int q = c0; q < c1; ++q) {
            const int t = q == c0 ? ct : p.blk_tasks[q];
            int64_t fp = task_fp(p, ov, t, m);
            const int d0 = q == c0 ? ce0 : p.dep_off[t], d1 = q == c0 ? ce1 : p.dep_off[t + 1];
            for (int d = d0; d < d1; ++d)
                if (p.dep_ob[d] >= lo) fp += p.dep_fix[d] + m * p.dep_ps[d];
            run_fp = fp > run_fp ? fp : run_fp;
            if (MONO) {                 // this key's task times (k_key_task_times)
                tf = __dadd_rn(tf, raw_tf[(int64_t)k * p.n_tasks + t]);
                tb = __dadd_rn(tb, raw_tb[(int64_t)k * p.n_tasks + t]);
            }
        }
        const int64_t idx = row + (hi - lo - 1);
        double f = tf, b = tb;
        if (!MONO) {
            f = raw_tf[(int64_t)k * tri + idx];
            b = raw_tb[(int64_t)k * tri + idx];
        }
        const int64_t param = p.pre_param[hi] - p.pre_param[lo];
        const int64_t inb = p.in_tab_fix[idx] + m * p.in_tab_ps[idx];
        const int64_t res = (p.pre_res_fix[hi] - p.pre_res_fix[lo]) +
                            m * (p.pre_res_ps[hi] - p.pre_res_ps[lo]) + res_corr(p, ov, lo, hi);
        const int64_t act = inb + (ckpt ? run_fp : res);
        const double memd = __dadd_rn(__dmul_rn((double)param, p.factor), (double)act);
        const int64_t mem = (int64_t)memd;
        const bool ok = mem <= p.mem_budget;                   // stages.py:230
        const int64_t o = hm_idx(lo, hi);
        out_f[o] = span_mark(f, ok, p.nonneg);
        if (derived) {
            // every span, feasible or not: the DP's skip search reads
            // beta * |t_fwd| as t_bwd on infeasible spans too
            bad |= __dmul_rn(p.beta, f) != b;
        } else {
            out_b[o] = b;
        }
    }
    if (bad) atomicOr(mismatch, 1);
}

// Per (key, task): the task's forward / backward time at the key's share
// (task_times, costs.py:130-140).  Monotone graphs fold them along every
// span row; computing them once per key keeps the fp64 division out of the
// O(nb^2) fold (same operation, same value).
__global__ void k_key_task_times(DevProblem p, int n_keys, const int64_t *keys_m, double *x,
                                 double *y) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)n_keys * p.n_tasks) return;
    const int k = (int)(gid / p.n_tasks);
    const int t = (int)(gid % p.n_tasks);
    const int64_t m = keys_m[k];
    task_times(p, ov_index(p, m), t, (double)m, x[gid], y[gid]);
}

void launch_key_task_times(const DevProblem &p, int n_keys, const int64_t *keys_m, double *x,
                           double *y, cudaStream_t st) {
    const int64_t n = (int64_t)n_keys * p.n_tasks;
    if (n <= 0) return;
    k_key_task_times<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n_keys, keys_m, x, y);
}

void launch_span_dp_tables(const DevProblem &p, int n_keys, const int64_t *keys_m,
                           const int32_t *keys_ckpt, const double *raw_tf, const double *raw_tb,
                           double *const *tf, double *const *tb, double *const *cut,
                           int derived, int *mismatch, cudaStream_t st) {
    const int64_t n = (int64_t)n_keys * p.nb;
    const int tpb = 128;
    const unsigned blocks = (unsigned)((n + tpb - 1) / tpb);
    if (p.monotone)
        k_span_rows<true><<<blocks, tpb, 0, st>>>(p, n_keys, keys_m, keys_ckpt, raw_tf, raw_tb,
                                                 tf, tb, cut, derived, mismatch);
    else
        k_span_rows<false><<<blocks, tpb, 0, st>>>(p, n_keys, keys_m, keys_ckpt, raw_tf, raw_tb,
                                                  tf, tb, cut, derived, mismatch);
}

// First feasible lo >= 1 of every hi (per key; hi when none): the DP reads it
// at levels s >= 2, whose predecessors are b' >= s - 1 >= 1, and skips the b'
// below it, all infeasible by construction (no monotonicity assumed); level 1
// reads the span from lo = 0 directly (that span's only input can be a small
// model input, so it may fit where [1, hi) does not).  One warp per (key, hi)
// row, 32 lo per ballot.  With `check` the whole row is read and open[k]
// flagged when some lo above the first feasible one is infeasible
// (feasibility not suffix-closed in lo >= 1): the DP's objective bound counts
// non-empty predecessors by range and needs it closed.
__global__ void k_first_feasible(int nb, int n_keys, int nonneg, int check,
                                 const double *const *tf, int32_t *const *ffb, int *open) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (int64_t)n_keys * (nb + 1)) return;
    const int k = (int)(gw / (nb + 1));
    const int hi = (int)(gw % (nb + 1));
    const double *row = tf[k] + hm_idx(0, hi);
    int first = hi;
    bool gap = false;
    for (int lo0 = 1; lo0 < hi; lo0 += 32) {
        const int lo = lo0 + lane;
        const bool in = lo < hi;
        const bool ok = in && span_ok(row[lo], nonneg);
        const uint32_t m = __ballot_sync(0xffffffffu, ok);
        const uint32_t inr = __ballot_sync(0xffffffffu, in);
        if (first == hi) {
            if (m) {
                const int f = __ffs(m) - 1;
                first = lo0 + f;
                if (!check) break;
                gap = gap || ((~m & inr) >> f) != 0;
            }
        } else {
            gap = gap || (~m & inr) != 0;
        }
    }
    if (lane == 0) {
        ffb[k][hi] = first;
        if (check && gap) atomicOr(&open[k], 1);
    }
}

void launch_first_feasible(int nb, int n_keys, int nonneg, int check, const double *const *tf,
                           int32_t *const *ffb, int *open, cudaStream_t st) {
    const int64_t n = (int64_t)n_keys * (nb + 1) * 32;
    k_first_feasible<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(nb, n_keys, nonneg, check, tf,
                                                                  ffb, open);
}

// ---------------------------------------------------------------- queries
// CostModel.profile(BlockSet.span(lo, hi), m, ckpt) for arbitrary queries,
// one thread each (stage records of a plan, BlockSet.costs, tests).
__global__ void k_profile_queries(DevProblem p, int n, const int32_t *qlo, const int32_t *qhi,
                                  const int64_t *qm, const int32_t *qckpt, double *otf,
                                  double *otb, int64_t *omem) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int lo = qlo[i], hi = qhi[i];
    const int64_t m = qm[i];
    const double md = (double)m;
    const int ov = ov_index(p, m);
    double tf = 0.0, tb = 0.0;
    int t0 = 0, t1 = p.n_tasks;
    if (p.monotone) { t0 = p.blk_off[lo]; t1 = p.blk_off[hi]; }
    for (int t = t0; t < t1; ++t) {
        const int b = p.task_block[t];
        if (b < lo || b >= hi) continue;
        double x, y;
        task_times(p, ov, t, md, x, y);
        tf = __dadd_rn(tf, x);
        tb = __dadd_rn(tb, y);
    }
    int64_t run_fp = 0;
    for (int blk = lo; blk < hi; ++blk)
        for (int q = p.blk_off[blk]; q < p.blk_off[blk + 1]; ++q) {
            const int t = p.blk_tasks[q];
            int64_t fp = task_fp(p, ov, t, m);
            for (int d = p.dep_off[t]; d < p.dep_off[t + 1]; ++d)
                if (p.dep_ob[d] >= lo) fp += p.dep_fix[d] + m * p.dep_ps[d];
            run_fp = fp > run_fp ? fp : run_fp;
        }
    const int64_t idx = tri_idx(lo, hi, p.nb);
    const int64_t param = p.pre_param[hi] - p.pre_param[lo];
    const int64_t inb = p.in_tab_fix[idx] + m * p.in_tab_ps[idx];
    const int64_t res = (p.pre_res_fix[hi] - p.pre_res_fix[lo]) +
                        m * (p.pre_res_ps[hi] - p.pre_res_ps[lo]) + res_corr(p, ov, lo, hi);
    const int64_t act = inb + (qckpt[i] ? run_fp : res);
    const double memd = __dadd_rn(__dmul_rn((double)param, p.factor), (double)act);
    otf[i] = tf;
    otb[i] = tb;
    omem[i] = (int64_t)memd;
}

void launch_profile_queries(const DevProblem &p, int n, const int32_t *lo, const int32_t *hi,
                            const int64_t *m, const int32_t *ckpt, double *tf, double *tb,
                            int64_t *mem, cudaStream_t st) {
    if (n <= 0) return;
    k_profile_queries<<<(n + 127) / 128, 128, 0, st>>>(p, n, lo, hi, m, ckpt, tf, tb, mem);
}

// ---------------------------------------------------------------- sharding weights
// Thread per (call, b): sum over device counts of the feasible predecessor
// count b - ffb(key(dev))[b], weighted by the (d, d') pairs with that count.
__global__ void k_call_weights(int nb, int n, const int32_t *calls, const int32_t *koff,
                               const int16_t *keyidx, const int32_t *const *ffb,
                               unsigned long long *w) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n * nb) return;
    const int c = (int)(g / nb);
    const int b = 1 + (int)(g % nb);
    const int S = calls[4 * c], D = calls[4 * c + 1];
    const int B = D - S + 1;
    unsigned long long acc = 0;
    for (int dev = 1; dev <= B; ++dev) {
        const int kk = keyidx[koff[c] + dev];
        if (kk < 0) continue;
        const int f = b - ffb[kk][b];
        if (f > 0) acc += (unsigned long long)(B - dev + 1) * (unsigned long long)f;
    }
    if (acc) atomicAdd(&w[c], acc * (unsigned long long)S);
}

void launch_call_weights(int nb, int n, const int32_t *calls, const int32_t *koff,
                         const int16_t *keyidx, const int32_t *const *ffb, unsigned long long *w,
                         cudaStream_t st) {
    const int64_t t = (int64_t)n * nb;
    if (t > 0) k_call_weights<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(nb, n, calls, koff, keyidx, ffb, w);
}

}  // namespace pcb
