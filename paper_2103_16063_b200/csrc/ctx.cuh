// Library context shared by the translation units of the C-ABI.
#pragma once

#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace pcb {

struct DBuf {
    void *p = nullptr;
    size_t n = 0;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t ensure(size_t bytes) {
        if (bytes <= n && p) return cudaSuccess;
        release();
        size_t want = bytes + bytes / 4 + 256;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return e;
        }
        n = want;
        return cudaSuccess;
    }
    template <class T>
    T *as() const { return (T *)p; }
};

// partition_blocks' device buffers, kept across calls (allocation and the
// pinned staging would otherwise cost more than a small coarsening)
struct CoarsenBufs {
    DBuf atoms_d, lev_grp, lev_off, lev_at, sets_d, scratch_d, out_d, comp_d;
    DBuf refine_d;            // device refinement: pairs, scratch, labels out
    int refine_cluster = 0;   // k_refine's cluster size (0 = not chosen yet)
    DBuf gc_d;                // group compute times of a coarsening level
    char *pout = nullptr;     // pinned read-back staging
    size_t pout_bytes = 0;
    int lev_cap = 0;          // level slots valid for lev_n atoms
    int lev_n = -1;
    int32_t *pin = nullptr;   // pinned level staging [lev_cap][3 * lev_n + 1]
    size_t pin_bytes = 0;
    ~CoarsenBufs() {
        if (pin) cudaFreeHost(pin);
        if (pout) cudaFreeHost(pout);
    }
};

struct CachedKey {
    int64_t m;
    int ckpt;
    double *tf = nullptr;    // [tri] hi-major, NaN = infeasible
    double *tb = nullptr;    // [tri] or null when derived as beta * tf
    double *cut = nullptr;   // [2][nb+1], then ffb int32 [nb+1]
    int slot = -1;           // slot in the key arena
    bool closed = false;     // feasible lo form a suffix [ffb, hi) for every hi
};

}  // namespace pcb

struct pc_ctx {
    using DBuf = pcb::DBuf;
    using CachedKey = pcb::CachedKey;
    using DevProblem = pcb::DevProblem;
    using DPBatch = pcb::DPBatch;
    using CallDesc = pcb::CallDesc;
    int device = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
    std::string err;
    int sm_count = 0;
    // problem
    bool has_problem = false;
    DevProblem P;
    int nb = 0;
    std::vector<int64_t> pre_param;
    DBuf prob;       // all problem arrays in one allocation
    DBuf in_tab;     // in_tab_fix | in_tab_ps
    // key cache
    std::vector<CachedKey> keys;
    std::map<std::pair<int64_t, int>, int> key_map;
    DBuf key_arena;  // fixed-size key slots (grow-only; a reset forgets keys, keeps memory)
    size_t key_slot = 0;
    int key_cap = 0;
    std::vector<char> slot_used;
    DBuf key_ptrs;   // [3][n_keys] device pointers (tf, tb, cut)
    size_t key_bytes = 0;
    bool derived = false;    // t_bwd derived as beta * t_fwd (beta a power of two)
    bool mono_skip = false;  // span times monotone (non-negative flops): DP prefix skip
    bool mono_flops = false; // the flops part of mono_skip
    bool has_cost_table = false;
    std::vector<int32_t> h_task_block;
    std::vector<int64_t> h_prod_fix, h_prod_ps;
    std::vector<int64_t> ov_m;           // resolved shares (host copy)
    DBuf ov_d;
    DBuf mismatch_d;
    // batch scratch
    DBuf cta_call_d;
    DBuf calls_d, warp_prefix_d, keyidx_d, val_d, hist_d, overflow_d;
    DBuf level_off_d, level_sums_d, row_prefix_d;
    DBuf plan_off_d, seg_d, objective_d, feasible_d;
    DBuf q_d, q_out_d, sim_d;
    DBuf raw_d, keys_m_d, keys_ckpt_d, colb_d;
    pcb::CoarsenBufs cb;  // partition_blocks
    DBuf bf_d;       // brute force: binomials, keys, per-block winners
    DBuf cut_d;      // pruning cut (cost tables): row/column prefixes, row_e
    // last batch (for budget crossing queries)
    std::vector<CallDesc> last_calls;   // sorted order
    std::vector<int> last_pos;          // orig -> sorted position
    std::vector<double> bb_U;           // per call of the current run_calls_impl (bound)
    std::vector<int> bb_partner;        // per call: call whose optimum bounds it, or -1
    bool bb_off = false;                // re-running calls whose bound was too tight
    const void *bb_outs = nullptr;      // the CallOut list those indices refer to
    DBuf bound_d;                       // plan-bound inputs / outputs
    DBuf reach_d;                       // non-empty prefix counts (two levels)
    DBuf live_d;                        // live-cell list of a bounded level + its count
    DBuf open_d;                        // first_feasible: per fresh key, not suffix-closed
    int64_t bounded_calls = 0, bound_reruns = 0;   // diagnostics of the last run
    int64_t frontier_reruns = 0;                     // calls re-run with FMAX_BIG frontiers
    std::vector<std::vector<int64_t>> last_level_sums;  // by orig
    int last_pruning = 1;
    int last_FL = 4;
    DPBatch last_batch{};
    // timing of the last batch
    double last_dp_ms = 0, last_span_ms = 0, last_post_ms = 0;
    int64_t last_dp_launches = 0;
    int64_t last_pairs = 0, last_cands = 0, last_inserts = 0;
    int64_t launches = 0;   // all kernel launches since the last reset
    DBuf counters_d;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    size_t mem_free = 0;    // last cudaMemGetInfo reading (run_calls_impl)
};

namespace pcb {

#define CUDA_TRY(ctx, expr)                                                       \
    do {                                                                          \
        cudaError_t e__ = (expr);                                                 \
        if (e__ != cudaSuccess) {                                                 \
            (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(e__);    \
            return PC_ERR_CUDA;                                                   \
        }                                                                         \
    } while (0)

inline int fail(pc_ctx *ctx, int code, const std::string &msg) {
    ctx->err = msg;
    return code;
}

inline int check_launch(pc_ctx *ctx, const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, PC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return PC_OK;
}

}  // namespace pcb
