// Shared declarations of the pipecut_b200 CUDA library (sm_100a).
//
// Numeric parity rules, enforced everywhere here:
//   * every fp64 operation is an explicit __d*_rn intrinsic and the library
//     is compiled with -fmad=false, so nothing is contracted into an FMA;
//   * (f*m)/F in that order (costs.py:137), beta*x (costs.py:138);
//   * comm_time = lat + (double)bytes / bw, division first (costs.py:86);
//   * boundary bytes = trunc(fixed + m*ps) in fp64 (blocks.py:331);
//   * mem = (int64)((double)param * ((1+g)+o) + (double)act) (costs.py:158).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pipecut_b200.h"

namespace pcb {

// ------------------------------------------------------------------ device problem
struct DevProblem {
    int nb = 0, n_tasks = 0, n_in = 0;
    int num_nodes = 1, dpn = 1, checkpointing = 0, monotone = 0;
    int nonneg = 1;                  // every task time >= 0 (span_mark encoding below)
    int n_inter = 1;                 // 2 when num_nodes > 1 (intra / inter cut variants)
    int64_t mem_budget = 0;
    double flops = 1, beta = 2, factor = 4, bw_intra = 1, bw_inter = 1, lat = 0;
    // tasks (sorted node-id order)
    const int32_t *task_block = nullptr;
    const double *task_flops = nullptr;
    const int64_t *fp_fix = nullptr, *fp_ps = nullptr;
    const int64_t *prod_fix = nullptr, *prod_ps = nullptr;   // produced bytes alone
    const int32_t *dep_off = nullptr, *dep_ob = nullptr;
    const int64_t *dep_fix = nullptr, *dep_ps = nullptr;
    // block -> task CSR (task indices ascending)
    const int32_t *blk_off = nullptr, *blk_tasks = nullptr;
    // span-input values
    const int32_t *in_ob = nullptr, *in_cons_off = nullptr, *in_cons = nullptr;
    const int64_t *in_fix = nullptr, *in_ps = nullptr;
    // prefix sums over blocks [nb+1]
    const int64_t *pre_param = nullptr, *pre_res_fix = nullptr, *pre_res_ps = nullptr;
    // boundary arrays [nb+1]
    const int64_t *cut_fixed = nullptr;
    const double *cut_ps = nullptr;
    // span input tables, triangular [tri(nb)]
    const int64_t *in_tab_fix = nullptr, *in_tab_ps = nullptr;
    // measured cost-table overrides (costs.py:130-148), per resolved share m
    int n_ov = 0;
    const int64_t *ov_m = nullptr;       // [n_ov]
    const uint8_t *ov_has = nullptr;     // [n_ov][n_tasks]
    const double *ov_tf = nullptr, *ov_tb = nullptr;
    const int64_t *ov_act = nullptr;
    const int64_t *ov_corr = nullptr;    // [n_ov][nb+1] prefix of resident corrections
};

__device__ inline int ov_index(const DevProblem &p, int64_t m) {
    for (int i = 0; i < p.n_ov; ++i)
        if (p.ov_m[i] == m) return i;
    return -1;
}

// per-task forward/backward time at share m (costs.py:130-140)
__device__ inline void task_times(const DevProblem &p, int ov, int t, double md, double &x, double &y) {
    if (ov >= 0 && p.ov_has[(int64_t)ov * p.n_tasks + t]) {
        x = p.ov_tf[(int64_t)ov * p.n_tasks + t];
        const double b = p.ov_tb[(int64_t)ov * p.n_tasks + t];
        y = isnan(b) ? __dmul_rn(p.beta, x) : b;
    } else {
        x = __ddiv_rn(__dmul_rn(p.task_flops[t], md), p.flops);
        y = __dmul_rn(p.beta, x);
    }
}

// base footprint of a task (produced + span-independent preds), with the
// cost table's act_bytes replacing the produced bytes (costs.py:147-148)
__device__ inline int64_t task_fp(const DevProblem &p, int ov, int t, int64_t m) {
    int64_t fp = p.fp_fix[t] + m * p.fp_ps[t];
    if (ov >= 0 && p.ov_has[(int64_t)ov * p.n_tasks + t]) {
        const int64_t a = p.ov_act[(int64_t)ov * p.n_tasks + t];
        if (a >= 0) fp += a - (p.prod_fix[t] + m * p.prod_ps[t]);
    }
    return fp;
}

__device__ inline int64_t res_corr(const DevProblem &p, int ov, int lo, int hi) {
    if (ov < 0) return 0;
    const int64_t *c = p.ov_corr + (int64_t)ov * (p.nb + 1);
    return c[hi] - c[lo];
}

// Triangular span index, rows by lo with hi contiguous:
// row lo holds hi = lo+1 .. nb.
__host__ __device__ inline int64_t tri_row(int64_t lo, int64_t nb) {
    return lo * nb - (lo * (lo - 1)) / 2;
}
__host__ __device__ inline int64_t tri_idx(int64_t lo, int64_t hi, int64_t nb) {
    return tri_row(lo, nb) + (hi - lo - 1);
}
__host__ __device__ inline int64_t tri_size(int64_t nb) { return nb * (nb + 1) / 2; }
// hi-major triangular index (row hi holds lo = 0 .. hi-1): the DP reads a
// cell's predecessors lo = b' contiguously.
__host__ __device__ inline int64_t hm_idx(int64_t lo, int64_t hi) { return hi * (hi - 1) / 2 + lo; }

// _Profiler.cut_time (stages.py:147-157) given the inter-node flag.
__device__ inline double cut_time_dev(const DevProblem &p, int cut, int64_t m, int inter) {
    double s = __dadd_rn((double)p.cut_fixed[cut], __dmul_rn((double)m, p.cut_ps[cut]));
    double nbytes = trunc(s);
    double bw = inter ? p.bw_inter : p.bw_intra;
    return __dadd_rn(p.lat, __ddiv_rn(nbytes, bw));
}

__host__ __device__ inline int inter_of(int num_nodes, int dpn, int64_t cum) {
    return (num_nodes > 1 && (cum % dpn) == 0) ? 1 : 0;
}

// ------------------------------------------------------------------ key tables
// Span feasibility (mem <= budget, stages.py:230) is carried in the t_fwd
// table itself.  With non-negative task times (the FLOP model, or cost tables
// without negative entries) an infeasible span keeps |t_fwd| with the sign bit
// set: the DP's prefix-skip search reads the magnitude of every span.  When
// some time can be negative the sign is data, the skip is off, and an
// infeasible span holds NaN instead (NaN inputs are rejected on the host).
__device__ __forceinline__ double span_mark(double tf, bool ok, int nonneg) {
    return ok ? tf : (nonneg ? -tf : __longlong_as_double(0x7ff8000000000000ll));
}
__device__ __forceinline__ bool span_ok(double tf, int nonneg) {
    return nonneg ? !signbit(tf) : !isnan(tf);
}

// One (microbatch share m, checkpointing) key:
//   tf[hm_idx(lo,hi)]  t_fwd of span [lo,hi) at m, marked by span_mark
//   tb[hm_idx(lo,hi)]  t_bwd (absent when it is derived as beta * t_fwd)
//   cut[inter][c]      cut_time(c, m, inter) for c in [0, nb]

// ------------------------------------------------------------------ DP batch
// One DP call in a level-synchronous batch.  Calls are ordered by S
// descending so the calls still active at level s are a prefix.
struct CallDesc {
    int32_t S, D, R, MB;
    int32_t A, B;              // b-range and d-range sizes: nb-S+1, D-S+1
    int32_t ckpt;
    int32_t key_off;           // keyidx[key_off + dev], dev in [1, B]
    int64_t val_off;           // cell offset of this call in the ping-pong value arrays
    int64_t hist_off;          // cell offset of level 1 in the history arrays
    int64_t vpool_base;        // entry offset of this call in each value pool
    int64_t vpool_cap;
    int64_t hpool_base;        // entry offset of this call in the history pool
    int64_t hpool_cap;
    int64_t col_off;           // offset of this call's d columns in the column-bound arrays
    int32_t orig;              // index in the caller's call list
    int32_t pad;
    double U;                  // objective upper bound (+inf: none); candidates whose
                               // every completion exceeds it are dropped (dp.cu: bound)
};

// Warps (cells) per CTA of the level kernel: 4 warps x 12 CTAs per SM (40
// registers, DP_MIN_BLOCKS in dp.cu) -- small CTAs free their slot as soon as
// their few cells finish; the occupancy/register split is re-measured whenever
// the kernel changes (round 2 sweep, 7 / 8 / 10 / 12 CTAs per SM =
// 1258 / 1180 / 1159 / 1116 ms of DP on 4096 x 256)
#ifndef PC_DP_WARPS
#define PC_DP_WARPS 4
#endif
constexpr int DP_WARPS = PC_DP_WARPS;
#ifndef DP_MIN_BLOCKS
#define DP_MIN_BLOCKS 12
#endif
// the bounded batches' persistent list kernel: 8 CTAs per SM (64 registers)
// measured best there (r2w: 813 vs 861 ms of DP on 4096 x 256 at 12)
#ifndef DP_LIST_MIN_BLOCKS
#define DP_LIST_MIN_BLOCKS 8
#endif
constexpr int DP_MIN_CTAS = DP_LIST_MIN_BLOCKS;   // resident list-kernel CTAs per SM
constexpr int DP_LIST_MIN_BLOCKS_DEEP = 10;       // ... on batches of DP_DEEP_LEVELS levels or more
constexpr int DP_DEEP_LEVELS = 512;
constexpr int WORK_SLOTS = 64;  // work counters spread over slots (no same-address atomics)
constexpr int FMAX = 64;       // Pareto frontier capacity per cell (two slots per lane)
constexpr int FMAX_BIG = 126;  // the re-run variant (four slots per lane; 127 = CNT_REACH)

struct DPBatch {
    int nb;
    int n_calls;
    const CallDesc *calls;
    const int64_t *cta_prefix;      // [n_calls+1] CTAs per call: ceil(A * B / DP_WARPS)
    const int32_t *cta_call;        // [cta_prefix[n_calls]] call of each CTA
    const int16_t *keyidx;          // -1 = zero share
    const double *const *key_tf;    // per-key table pointers (device arrays)
    const double *const *key_tb;
    const double *const *key_cut;
    const int32_t *const *key_ffb;  // per key: first feasible lo for each hi
    double beta;
    int64_t batch_size;             // BS of every call of the batch
    int num_nodes, dpn;
    int mono_skip;                  // task times >= 0: t_fwd(b', b) non-increasing in b' (the
                                    // prefix skip) and the span_mark sign-bit encoding
    // per level, per (call, d column): smallest / largest b of a non-empty cell
    int32_t *col_min[2];
    int32_t *col_max[2];
    // ping-pong level values: per cell count + offset into the call's pool
    // region (exact-size allocation by one atomic per cell)
    uint8_t *val_cnt[2];
    uint32_t *val_off[2];
    // bounded batches: per (call, column) inclusive prefix count over b of the
    // cells the reference holds non-empty (count > 0 or CNT_REACH)
    int32_t *reach_pre[2];
    int bounded;                    // some call of the batch has a finite U
    // bounded batches: the live cells of the level (call << 40 | cell index),
    // listed by k_dp_triage, walked by k_dp_level_list
    unsigned long long *live;
    unsigned long long *live_count;  // [0] cells listed, [1] cells taken (k_dp_level_list)
    float2 *live_lb;                 // each live cell's suffix lower bounds (lbf, lbb), rounded down
    // bounded batches, per level: per (call, column) the suffix / prefix
    // group-bound factors and keys (k_level_factors; group_bounds' arithmetic)
    double2 *lvl_kk;                 // [col_total] (suffix, prefix) factor
    short2 *lvl_kx;                  // [col_total] (suffix, prefix) key, -1: no bound
    double *pool_tf[2];
    double *pool_tb[2];
    unsigned long long *vpool_used[2];  // [n_calls] per parity
    double *spill_tf[2];                // shared spill pool when a call region is full
    double *spill_tb[2];
    unsigned long long *vspill_used;    // [2]
    int64_t vspill_cap;
    int64_t val_cells;
    // back-pointer history of every level, same scheme
    uint8_t *hist_cnt;
    uint32_t *hist_off;
    uint32_t *hpool;
    unsigned long long *hpool_used;     // [n_calls]
    uint32_t *hspill;
    unsigned long long *hspill_used;
    int64_t hspill_cap;
    int64_t hist_cells;
    int *overflow;                  // 1: frontier > fmax_limit, 2: a pool region ran out
    int fmax_limit;                 // frontier entries a cell may hold in this pass
    unsigned long long *counters;   // [0] pairs, [1] candidates, [2] inserts, [3..] sizes
};

// pool offsets: bit 31 set = entry offset into the shared spill pool
constexpr uint32_t SPILL_BIT = 0x80000000u;

// count byte: bits 0-6 entries, bit 7 saw_zero_share
constexpr uint8_t CNT_MASK = 0x7f;
constexpr uint8_t CNT_ZERO = 0x80;
// count value of a cell the reference holds non-empty whose every entry the
// objective bound dropped (dp.cu: bound); FMAX < CNT_REACH, so never a count
constexpr uint8_t CNT_REACH = 0x7f;
__host__ __device__ inline int cnt_entries(uint8_t v) {
    const int c = v & CNT_MASK;
    return c == CNT_REACH ? 0 : c;
}

// packed back-pointer (bp, dp, idx): lexicographic order == integer order
__host__ __device__ inline uint32_t pack_key(uint32_t bp, uint32_t dp, uint32_t idx) {
    return (bp << 18) | (dp << 6) | idx;
}
__host__ __device__ inline int key_bp(uint32_t k) { return (int)(k >> 18); }
__host__ __device__ inline int key_dp(uint32_t k) { return (int)((k >> 6) & 0xfff); }
__host__ __device__ inline int key_idx(uint32_t k) { return (int)(k & 63); }
constexpr int MAX_NB_KEY = (1 << 14) - 1;
constexpr int MAX_D_KEY = (1 << 12) - 1;

// ------------------------------------------------------------------ launchers
// span.cu
void launch_in_tables(const DevProblem &p, int64_t *in_fix, int64_t *in_ps, cudaStream_t st);
void launch_span_time_general(const DevProblem &p, int n_keys, const int64_t *keys_m,
                              double *raw_tf, double *raw_tb, cudaStream_t st);
void launch_key_task_times(const DevProblem &p, int n_keys, const int64_t *keys_m, double *x,
                           double *y, cudaStream_t st);
void launch_span_dp_tables(const DevProblem &p, int n_keys, const int64_t *keys_m,
                           const int32_t *keys_ckpt, const double *raw_tf, const double *raw_tb,
                           double *const *tf, double *const *tb, double *const *cut,
                           int derived, int *mismatch, cudaStream_t st);
void launch_first_feasible(int nb, int n_keys, int nonneg, int check, const double *const *tf,
                           int32_t *const *ffb, int *open, cudaStream_t st);
// dp.cu: objective bound of a batch's calls from a plan of each (the optimum of
// its (S, D, R, MB/2) partner), and the non-empty prefix counts per level
void launch_plan_bound(const DPBatch &b, int n, const int32_t *pos, const int32_t *seg_off,
                       const int32_t *lo, const int32_t *hi, const int32_t *dev, double *U,
                       bool derived, cudaStream_t st);
void launch_reach_prefix(const DPBatch &b, int s, int n_active, int64_t n_cols,
                         const int64_t *col_prefix, cudaStream_t st);
constexpr int GB_SPLITS = 2;    // greedy-bound device splits per call (extras first / last; spread: r2cm, no gain)
void launch_greedy_bound(const DPBatch &b, int n, const int32_t *pos, double *U, bool derived,
                         cudaStream_t st);
void launch_level_factors(const DPBatch &b, int s, int n_active, int64_t n_cols,
                          const int64_t *col_prefix, cudaStream_t st);
void launch_dp_triage(const DPBatch &b, int s, int n_active, int64_t n_cells,
                      const int64_t *cell_prefix, bool derived, cudaStream_t st);
void launch_dp_level_list(const DPBatch &b, int s, int sm_count, bool deep, bool derived, bool big,
                          cudaStream_t st);
void launch_profile_queries(const DevProblem &p, int n, const int32_t *lo, const int32_t *hi,
                            const int64_t *m, const int32_t *ckpt, double *tf, double *tb,
                            int64_t *mem, cudaStream_t st);
void launch_call_weights(int nb, int n, const int32_t *calls, const int32_t *koff,
                         const int16_t *keyidx, const int32_t *const *ffb, unsigned long long *w,
                         cudaStream_t st);
// dp.cu
void launch_cta_call(const int64_t *prefix, int n, int64_t total, int32_t *out, cudaStream_t st);
void launch_dp_level(const DPBatch &b, int s, int n_active, int64_t n_ctas, bool derived,
                     bool big, cudaStream_t st);
// cost tables: the reference's pruning break applied to the level's cells;
// returns the number of kernels launched
int launch_prune_cut(const DPBatch &b, int s, int n_active, int64_t n_rows, int64_t n_cols,
                     const int64_t *row_prefix, const int64_t *col_prefix, int32_t *row_e,
                     cudaStream_t st);
void launch_row_visits(const DPBatch &b, int pruning, int64_t *level_sums, int64_t *row_sums,
                       const int64_t *level_row_off, int64_t n_rows_total, cudaStream_t st);
void launch_backtrack(const DPBatch &b, int64_t batch_size, const int32_t *plan_off,
                      int32_t *seg_lo, int32_t *seg_hi, int32_t *seg_dev, double *objective,
                      int32_t *feasible, cudaStream_t st);
// sim.cu: full schedule and validate_plan's charged times
void launch_schedule(const DevProblem &p, int S, int R, int MB, int64_t BS, const int32_t *lo,
                     const int32_t *hi, const int32_t *dev, const double *tf, const double *tb,
                     int32_t *lane_off, int32_t *ev_mb, int8_t *ev_phase, double *ev_start,
                     double *ev_end, double *summary, cudaStream_t st);
void launch_charge_plan(const DevProblem &p, int S, const int32_t *lo, const int32_t *hi,
                        const int32_t *dev, const int64_t *m, const double *rtf, const double *rtb,
                        double *ctf, double *ctb, double *objective, cudaStream_t st);
// brute.cu: exhaustive (cuts x compositions) search, brute_force_partition
constexpr int BF_MAXS = 64;       // stages per enumerated assignment
constexpr int BF_CHUNK = 64;      // composition ranks per work item
constexpr int BF_THREADS = 256;
struct BruteArgs {
    const double *const *key_tf;
    const double *const *key_tb;
    const double *const *key_cut;
    const int16_t *keyidx;        // [D - S + 2] key of each device count (-1: m == 0)
    const int64_t *binom;         // [(n_max + 1) * kcols] C(a, j), saturated
    int kcols;
    int nb, S, D, derived, num_nodes, dpn;
    int nonneg;                   // span_mark encoding of the key tables
    double beta;
    int64_t n_comb, n_comp, n_chunks;
    unsigned long long *out_key;  // per block winner
    long long *out_idx;
    double *out_obj;
};
void launch_brute(const BruteArgs &a, int blocks, cudaStream_t st);
// peak.cu
double measure_fp64_gops(cudaStream_t st, int sm_count);
double measure_dadd_gops(cudaStream_t st, int sm_count);
// sim.cu
void launch_simulate(const DevProblem &p, int n_plans, const int32_t *plan_off,
                     const int32_t *plan_S, const int32_t *plan_R, const int32_t *plan_MB,
                     int64_t batch_size, const int32_t *seg_lo, const int32_t *seg_hi,
                     const int32_t *seg_dev, const double *st_tf, const double *st_tb,
                     double *iteration, cudaStream_t st, int max_S);

}  // namespace pcb
