/*
 * pipecut_b200 — C-ABI of the B200-native partition-search hot path.
 *
 * Drop-in boundary for the reference package `pipecut` (pure Python,
 * /root/reference/pkg).  The reference has no native code, so there is no
 * existing FFI; these entry points are what its Python call sites bind via
 * ctypes (INTEGRATION.md shows the stubs).  Each entry point names the
 * reference function it replaces:
 *
 *   pc_set_problem      BlockSet + CostModel + ClusterSpec, flattened
 *                       (pkg/src/pipecut/blocks.py:295-343, costs.py:89-164,
 *                        graph.py:176-199)
 *   pc_profile_spans    CostModel.profile(BlockSet.span(lo, hi), m, ckpt)
 *                       (costs.py:97-160 via stages.py:138-145)
 *   pc_form_stage_dp    form_stage_dp (stages.py:282-291 -> _run_dp 188-279)
 *   pc_run_calls        the per-(n, S, MB) _run_dp calls of form_stage plus
 *                       simulate()-based ranking keys (stages.py:389-411,
 *                       simulate.py:79-165) -- the unit sharded across GPUs
 *   pc_form_stage       form_stage (stages.py:372-413), single GPU
 *   pc_last_crossing    the SearchBudgetExceeded visit count (stages.py:214-216)
 *   pc_partition_blocks partition_blocks (blocks.py:361-397)
 *   pc_set_overrides    measured cost-table entries (costs.py:43-80, 130-148)
 *   pc_brute_force      brute_force_partition (stages.py:304-369)
 *   pc_check_plan       validate_plan's fresh records (stages.py:416-492)
 *   pc_simulate         simulate (simulate.py:79-179)
 *   pc_call_weights     sharding weights of form_stage's call enumeration
 *                       (stages.py:389-403); no reference counterpart
 *   pc_ctx_*, pc_device_info, pc_reset_cache, pc_timer_*, pc_measure_fp64_peak,
 *   pc_measure_dadd_peak, pc_bound_info
 *                       library plumbing and measurement; no reference
 *                       counterpart
 *
 * Conventions: plain pointers and sizes, caller-owned host buffers, valid for
 * the duration of the call; the library owns device memory behind an opaque
 * context.  Calls are blocking.  There is no CPU fallback: without a usable
 * sm_100 device every compute entry point returns PC_ERR_CUDA.
 */
#ifndef PIPECUT_B200_H
#define PIPECUT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (mapped to the reference exception classes in Python) */
#define PC_OK                 0
#define PC_INFEASIBLE         1   /* plan is None (stages.py:122-125) */
#define PC_ERR_INVALID       (-1) /* InvalidArgs (stages.py:160-168, 382-384) */
#define PC_ERR_BUDGET        (-2) /* SearchBudgetExceeded (stages.py:33-37, 214-216) */
#define PC_ERR_ATOM          (-3) /* InfeasibleAtom (blocks.py:22-31, 366-369) */
#define PC_ERR_STUCK         (-4) /* CompactionStuck (blocks.py:34-42, 291) */
#define PC_ERR_CUDA          (-5) /* CUDA / device error; see pc_last_error */
#define PC_ERR_CAPACITY      (-6) /* frontier (> 126 entries) / table capacity exceeded (never truncated) */

typedef struct pc_ctx pc_ctx;

/*
 * Flattened span-profile problem (paper_2103_16063_b200/flatten.py builds it).
 * Arrays are read-only for the call of pc_set_problem, which copies them to
 * the device.
 */
typedef struct pc_problem {
    int32_t nb;                 /* len(BlockSet) */
    int32_t n_tasks;            /* tasks in sorted node-id order (costs.py:120) */
    const int32_t *task_block;  /* [n_tasks] */
    const double  *task_flops;  /* [n_tasks] flops_per_sample (costs.py:137) */
    const int64_t *task_fp_fix; /* [n_tasks] produced + span-independent preds */
    const int64_t *task_fp_ps;  /* [n_tasks] per-sample part */
    const int64_t *task_prod_fix; /* [n_tasks] produced bytes alone (cost tables replace it) */
    const int64_t *task_prod_ps;
    const int32_t *task_dep_off;/* [n_tasks+1] CSR: preds owned in block dep_ob */
    const int32_t *dep_ob;      /*   count in the footprint iff dep_ob >= lo  */
    const int64_t *dep_fix;
    const int64_t *dep_ps;
    int32_t n_in;               /* values listed in some atom's input_values */
    const int32_t *in_ob;       /* [n_in] owner block, -1 model input/unowned */
    const int32_t *in_cons_off; /* [n_in+1] CSR of sorted consumer blocks */
    const int32_t *in_cons;
    const int64_t *in_fix;      /* [n_in] */
    const int64_t *in_ps;       /* [n_in] */
    const int64_t *blk_param;   /* [nb] parameter bytes owned per block */
    const int64_t *blk_res_fix; /* [nb] resident bytes per block */
    const int64_t *blk_res_ps;  /* [nb] */
    const int64_t *cut_fixed;   /* [nb+1] BlockSet._cut_fixed (blocks.py:310) */
    const double  *cut_ps;      /* [nb+1] BlockSet._cut_per_sample (blocks.py:311) */
    /* CostModelConfig (costs.py:27-40) */
    double flops_per_sec;
    double bwd_fwd_ratio;
    double grad_factor;
    double opt_factor;
    int32_t checkpointing;
    /* ClusterSpec (graph.py:176-199) */
    int32_t num_nodes;
    int32_t devices_per_node;
    int32_t monotone;           /* task_block non-decreasing: incremental folds */
    int32_t has_cost_table;     /* CostModelConfig.cost_table set: every microbatch share
                                   used must be resolved by pc_set_overrides */
    int64_t mem_budget;
    double bw_intra;
    double bw_inter;
    double latency;
} pc_problem;

/*
 * Flattened atomic partition for partition_blocks (blocks.py:73-124): what the
 * memory of any atom set at microbatch 1 with checkpointing, convexity and
 * cut traffic need (paper_2103_16063_b200/flatten.py: flatten_atoms).
 */
typedef struct pc_atoms {
    int32_t n;                  /* atoms (topological order) */
    int32_t n_tasks;
    int32_t n_in;               /* values listed in some atom's input_values */
    int32_t n_traffic;          /* value traffic entries (blocks.py:96-102) */
    const int64_t *atom_param;  /* [n] parameter bytes owned by each atom */
    const int32_t *task_atom;   /* [n_tasks] sorted node-id order */
    const double  *task_flops;  /* [n_tasks] */
    const int64_t *task_fp1;    /* [n_tasks] produced + always-counted preds at m=1 */
    const int32_t *dep_off;     /* [n_tasks+1] anchor inputs owned by atom dep_owner */
    const int32_t *dep_owner;
    const int64_t *dep_size;
    const int32_t *atom_task_off, *atom_tasks;   /* tasks of each atom, ascending */
    const int32_t *atom_in_off, *atom_in;        /* input values of each atom */
    const int32_t *in_owner;    /* [n_in] owner atom, -1 model input / unowned */
    const int64_t *in_size;     /* [n_in] size at m=1 */
    const int32_t *in_atoms_off, *in_atoms;      /* atoms listing each input, ascending */
    const int32_t *succ_off, *succ;              /* partition.dependencies() */
    const int32_t *pred_off, *pred;
    const int32_t *nbr_off, *nbr;                /* sorted(succ | pred) */
    const int32_t *tr_owner;    /* [n_traffic] */
    const int64_t *tr_size;
    const int32_t *tr_cons_off, *tr_cons;        /* foreign consumer atoms */
    const int32_t *atom_tr_off, *atom_tr;        /* traffic entries touching each atom */
    const int64_t *task_prod1;  /* [n_tasks] produced bytes alone at m=1 */
    const uint8_t *ov_has;      /* [n_tasks] or NULL: cost-table entry at m=1 (costs.py:130-148) */
    const double  *ov_tf, *ov_tb;               /* ov_tb NaN: bwd_fwd_ratio * ov_tf */
    const int64_t *ov_act;                      /* -1: keep the produced bytes */
    int64_t budget;             /* ClusterSpec.device_memory_bytes */
    double flops_per_sec, bwd_fwd_ratio, grad_factor, opt_factor;
} pc_atoms;

/* One DP call of _run_dp (stages.py:188): S stages on D devices. */
typedef struct pc_call {
    int32_t S, D, R, MB;        /* stage count, devices, replica factor, microbatches */
} pc_call;

/* Plan output (StagePlan/Plan, stages.py:40-57) into caller arrays of
 * capacity cap_stages.  iteration_time is simulate(plan).iteration_time_sec
 * (simulate.py:165) when requested. */
typedef struct pc_plan {
    int32_t cap_stages;
    int32_t n_stages;           /* 0 when infeasible */
    int32_t *lo, *hi, *devices; /* [cap_stages] */
    double  *t_fwd, *t_bwd;     /* [cap_stages] profile at the plan microbatch, no comm */
    int64_t *mem;               /* [cap_stages] */
    int32_t S, D, R, MB;
    double objective;           /* max fwd + max bwd with comm (stages.py:277-278) */
    double iteration_time;      /* simulate(plan).iteration_time_sec, or NaN */
} pc_plan;

typedef struct pc_stats {
    int64_t visits;             /* SearchStats.visits, pruned as the reference counts */
    int64_t dp_calls;           /* SearchStats.dp_calls */
    int64_t visits_unpruned;    /* closed form: the throughput unit */
    int64_t cells;              /* (s, b, d) table cells computed on device */
    int64_t pairs;              /* feasible (cell, predecessor) pairs evaluated */
    int64_t candidates;         /* frontier candidates generated (stages.py:238-239) */
    int64_t dp_launches;        /* DP level kernel launches */
    int64_t kernel_launches;    /* all library kernel launches of the call */
    double  device_ms;          /* device time of the DP level kernels (CUDA events) */
    double  span_ms;            /* device time of span/cut table kernels */
    double  post_ms;            /* device time after the DP levels: visit counts, backtrack,
                                   stage records, simulate and the result copies (CUDA events) */
} pc_stats;

/* Per-call result of pc_run_calls (one record per pc_call). */
typedef struct pc_call_result {
    int32_t feasible;
    int32_t n_stages;
    double  objective;
    double  iteration_time;
    int64_t visits;             /* pruned reference visits of this call */
    int64_t visits_unpruned;
    int64_t budget_cross;       /* running visits at the first cell exceeding the
                                   budget within this call given visits_before, or -1 */
} pc_call_result;

/* ---- context ---------------------------------------------------------- */
int  pc_ctx_create(int device, pc_ctx **out);
void pc_ctx_destroy(pc_ctx *ctx);
const char *pc_last_error(pc_ctx *ctx);
int  pc_device_info(pc_ctx *ctx, int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor);

/* ---- problem ------------------------------------------------------------ */
int pc_set_problem(pc_ctx *ctx, const pc_problem *p);

/* Measured cost-table overrides (costs.py:130-148) resolved on the host for
 * n_m microbatch shares m_values[i]: for task t (sorted-id order) with
 * has[i*n_tasks + t] != 0, t_fwd = tf[...], t_bwd = tb[...] (NaN: bwd_fwd_ratio
 * * t_fwd) and, when act[...] >= 0, produced bytes = act[...].  Replaces the
 * previous set; drops cached span tables. */
int pc_set_overrides(pc_ctx *ctx, int32_t n_m, const int64_t *m_values, const uint8_t *has,
                     const double *tf, const double *tb, const int64_t *act);

/* brute_force_partition (pkg/src/pipecut/stages.py:304-369): every (cut
 * combination, composition of D into S parts) pair, objective
 * max(tf) + max(tb), ties by the reference's lex (bounds, devs) order;
 * stats->visits = number of pairs.  The reference's nb <= 12 / D <= 8 guard
 * (TooLarge) is the caller's; here the cap is 1e12 pairs and S <= 64
 * (PC_ERR_CAPACITY beyond).  Returns PC_OK or PC_INFEASIBLE. */
int pc_brute_force(pc_ctx *ctx, int32_t S, int32_t D, int64_t batch_size, int32_t R,
                   int32_t MB, pc_plan *plan, pc_stats *stats);

/* validate_plan's fresh records (pkg/src/pipecut/stages.py:416-492) for the
 * plan's stages: span profile at each stage's share (NaN / -1 where the share
 * is zero), the comm-charged times and objective = max(tf) + max(tb) over the
 * stages with a positive share (NaN if none).  Arrays are [plan->n_stages]. */
int pc_check_plan(pc_ctx *ctx, const pc_plan *plan, int64_t batch_size, double *rec_tf,
                  double *rec_tb, int64_t *rec_mem, double *charged_tf, double *charged_tb,
                  double *objective);

/* simulate (pkg/src/pipecut/simulate.py:79-179) of a plan: every lane event,
 * stage-major, lane_off[n_stages+1]; phases 0 fwd, 1 recompute, 2 bwd, 3 comm,
 * 4 allreduce; microbatch -1 for the gradient sync.  summary[5] = {iteration
 * time, busy device-seconds, bubble fraction, samples/s, devices}.  ev_cap must
 * be >= n_stages * (5 * MB + 1). */
int pc_simulate(pc_ctx *ctx, const pc_plan *plan, int64_t batch_size, int32_t ev_cap,
                int32_t *lane_off, int32_t *ev_mb, int8_t *ev_phase, double *ev_start,
                double *ev_end, double *summary);

/* Sharding weights for n calls (the LPT key of form_stage_sharded): per call
 * S * sum_b sum_dev (B - dev + 1) * #{1 <= lo < b : span (lo, b) fits at the share
 * of dev devices}, from the key tables (built for every call's shares).
 * Exact integers: every rank computes the same assignment. */
int pc_call_weights(pc_ctx *ctx, int32_t n, const pc_call *calls, int64_t batch_size,
                    int64_t *weights);

/* CostModel.profile over block spans (costs.py:97-160 via stages.py:138-145):
 * n queries (lo, hi, m, ckpt). */
int pc_profile_spans(pc_ctx *ctx, int32_t n, const int32_t *lo, const int32_t *hi,
                     const int64_t *m, const int32_t *ckpt,
                     double *t_fwd, double *t_bwd, int64_t *mem);

/* form_stage_dp (stages.py:282-291 -> _run_dp 188-279): one DP call.
 * visit_budget < 0 means none.  Returns PC_OK,
 * PC_INFEASIBLE, PC_ERR_BUDGET (stats->visits = visits at the crossing). */
int pc_form_stage_dp(pc_ctx *ctx, int32_t S, int32_t D, int64_t batch_size,
                     int32_t R, int32_t MB, int32_t disable_pruning,
                     int64_t visit_budget, pc_plan *plan, pc_stats *stats);

/* Batch of independent DP calls (the sharded unit of form_stage,
 * stages.py:389-411).  Every
 * call's plan is simulated for its ranking key when want_iteration != 0.
 * plans may be NULL (results only); otherwise n entries. */
int pc_run_calls(pc_ctx *ctx, int32_t n, const pc_call *calls, int64_t batch_size,
                 int32_t disable_pruning, int32_t want_iteration,
                 pc_call_result *results, pc_plan *plans, pc_stats *stats);

/* form_stage (stages.py:372-413) on one GPU.  Batching of the widening
 * levels: speculative = 1 all in one batch, 0 one batch per level, 2 the first
 * level and then the rest together.  The reference's first-feasible-level
 * rule is applied afterwards; results and stats are identical in every mode. */
int pc_form_stage(pc_ctx *ctx, int32_t num_nodes, int32_t devices_per_node,
                  int64_t batch_size, int32_t disable_pruning, int64_t visit_budget,
                  int32_t speculative, pc_plan *plan, pc_stats *stats);

/* Budget crossing inside call `index` of the last pc_run_calls batch given
 * the visits accumulated before it (stages.py:214-216): -1 if not crossed,
 * -2 if that call ran in an earlier memory chunk / wave of the batch (its
 * flags are gone: run it alone and ask again). */
int pc_last_crossing(pc_ctx *ctx, int32_t index, int64_t visits_before, int64_t budget,
                     int64_t *visits_at_cross);

/* partition_blocks (blocks.py:361-397): at most k convex, memory-feasible
 * blocks in dependency order.  Outputs (caller capacity n atoms): n_blocks,
 * block_off[n_blocks+1], block_atoms[n] (ascending within a block), and per
 * block t_fwd, t_bwd, mem = CostModel.profile(block, 1, ckpt=True)
 * (blocks.py:390).  PC_ERR_ATOM: err[0] = atom index, err[1] = its memory
 * (InfeasibleAtom); PC_ERR_STUCK: err[0] = groups left (CompactionStuck);
 * PC_ERR_INVALID: k < 1. */
int pc_partition_blocks(pc_ctx *ctx, const pc_atoms *atoms, int32_t k, int32_t *n_blocks,
                        int32_t *block_off, int32_t *block_atoms, double *t_fwd,
                        double *t_bwd, int64_t *mem, int64_t *err);

/* Drop the cached span/cut tables (they are rebuilt on demand). */
int pc_reset_cache(pc_ctx *ctx);

/* CUDA events on the library stream bracketing host-visible work. */
int pc_timer_start(pc_ctx *ctx);
int pc_timer_stop(pc_ctx *ctx, double *ms);

/* Measured fp64 add/max issue rate of this device (Gop/s), the roofline
 * denominator of the DP kernel (no tensor-core roof: min/max/add recurrence). */
int pc_measure_fp64_peak(pc_ctx *ctx, double *gops);

/* Diagnostics of the last pc_run_calls / pc_form_stage* call: calls that ran
 * with a finite objective bound, calls re-run unbounded because their bound
 * was below the optimum, and calls re-run with the 126-entry frontier kernels
 * because some cell outgrew 64 entries (frontier_reruns may be NULL).  No
 * reference counterpart. */
int pc_bound_info(pc_ctx *ctx, int64_t *bounded_calls, int64_t *reruns, int64_t *frontier_reruns);

/* Measured pure-DADD rate of this device (Gop/s): the fp64 pipe's peak op rate,
 * the denominator of the DP kernel's algorithmic-fp64 roofline. */
int pc_measure_dadd_peak(pc_ctx *ctx, double *gops);

#ifdef __cplusplus
}
#endif
#endif /* PIPECUT_B200_H */
