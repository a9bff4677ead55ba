/*
 * ORACLE — test infrastructure only.  Not part of the product path.
 *
 * Plain-C, single-threaded restatement of the reference's partition-search
 * hot path over the flat arrays of include/pipecut_b200.h (built by
 * paper_2103_16063_b200/flatten.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker or
 * the timed CPU baseline ("kind": "port").
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * function below with /root/reference (or the unmodified install in
 * baseline/_ref) on the reference's own test families and on the committed
 * golden fixtures in tests/golden/.
 *
 * Each function cites the reference lines it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/pipecut_b200.h"

/* ---------------------------------------------------------------------- */
/* CostModel.profile(BlockSet.span(lo, hi), m, ckpt)  (costs.py:97-160)     */
/* ---------------------------------------------------------------------- */
void orc_span_record(const pc_problem *p, int lo, int hi, int64_t m, int ckpt,
                     double *tf_out, double *tb_out, int64_t *mem_out)
{
    /* time: fold in sorted node-id order (costs.py:120, 137-140) */
    double tf = 0.0, tb = 0.0;
    for (int t = 0; t < p->n_tasks; ++t) {
        int b = p->task_block[t];
        if (b < lo || b >= hi) continue;
        double x = (p->task_flops[t] * (double)m) / p->flops_per_sec;
        double y = p->bwd_fwd_ratio * x;
        tf = tf + x;
        tb = tb + y;
    }
    /* parameters (costs.py:124-125) */
    int64_t param = 0, res = 0;
    for (int b = lo; b < hi; ++b) {
        param += p->blk_param[b];
        res += p->blk_res_fix[b] + m * p->blk_res_ps[b];   /* costs.py:126-127, 149 */
    }
    /* span inputs (atoms.py:136-138, costs.py:118) */
    int64_t inb = 0;
    for (int v = 0; v < p->n_in; ++v) {
        if (p->in_ob[v] >= lo) continue;
        for (int k = p->in_cons_off[v]; k < p->in_cons_off[v + 1]; ++k) {
            int c = p->in_cons[k];
            if (c >= lo) {
                if (c < hi) inb += p->in_fix[v] + m * p->in_ps[v];
                break;
            }
        }
    }
    /* largest single-task working set (costs.py:150-155) */
    int64_t maxfp = 0;
    for (int t = 0; t < p->n_tasks; ++t) {
        int b = p->task_block[t];
        if (b < lo || b >= hi) continue;
        int64_t fp = p->task_fp_fix[t] + m * p->task_fp_ps[t];
        for (int k = p->task_dep_off[t]; k < p->task_dep_off[t + 1]; ++k)
            if (p->dep_ob[k] >= lo) fp += p->dep_fix[k] + m * p->dep_ps[k];
        if (fp > maxfp) maxfp = fp;
    }
    int64_t act = inb + (ckpt ? maxfp : res);                /* costs.py:157 */
    double factor = (1.0 + p->grad_factor) + p->opt_factor;  /* costs.py:158 */
    double memd = (double)param * factor + (double)act;
    *tf_out = tf;
    *tb_out = tb;
    *mem_out = (int64_t)memd;                                 /* int() truncation */
}

/* _Profiler.cut_time (stages.py:147-157) with BlockSet.boundary_bytes
 * (blocks.py:326-331) and comm_time (costs.py:83-86, 162-164). */
double orc_cut_time(const pc_problem *p, int cut, int64_t m, int64_t cum)
{
    double nbytes = trunc((double)p->cut_fixed[cut] + (double)m * p->cut_ps[cut]);
    int inter = p->num_nodes > 1 && (cum % p->devices_per_node) == 0;
    double bw = inter ? p->bw_inter : p->bw_intra;
    return p->latency + nbytes / bw;
}

/* ---------------------------------------------------------------------- */
/* _run_dp (stages.py:188-279) with _pareto (stages.py:176-185)             */
/* ---------------------------------------------------------------------- */
typedef struct { double tf, tb; int bp, dp, idx; int ord; } orc_entry;
typedef struct { int n; orc_entry *e; } orc_cell;

/* frontier-size histogram of the cells computed (diagnostics) */
static int64_t g_fhist[65];
void orc_frontier_hist(int64_t *out)
{
    for (int i = 0; i < 65; ++i) { out[i] = g_fhist[i]; g_fhist[i] = 0; }
}

/* sorted(range(n), key=(tf, tb, i)) of _pareto (stages.py:177): a stable
 * bottom-up merge sort on (tf, tb); stability keeps insertion order (ord) on
 * equal (tf, tb), so the order equals qsort with cmp_entry. */
static inline int entry_less(const orc_entry *x, const orc_entry *y)
{
    return x->tf < y->tf || (x->tf == y->tf && x->tb < y->tb);
}

static void sort_cands(orc_entry *a, size_t n, orc_entry **tmp, size_t *tmp_cap)
{
    if (*tmp_cap < n) {
        *tmp_cap = n;
        *tmp = (orc_entry *)realloc(*tmp, n * sizeof(orc_entry));
    }
    /* insertion sort runs of 16, then merge passes */
    const size_t RUN = 16;
    for (size_t lo = 0; lo < n; lo += RUN) {
        size_t hi = lo + RUN < n ? lo + RUN : n;
        for (size_t i = lo + 1; i < hi; ++i) {
            orc_entry v = a[i];
            size_t j = i;
            while (j > lo && entry_less(&v, &a[j - 1])) { a[j] = a[j - 1]; --j; }
            a[j] = v;
        }
    }
    orc_entry *src = a, *dst = *tmp;
    for (size_t w = RUN; w < n; w *= 2) {
        for (size_t lo = 0; lo < n; lo += 2 * w) {
            size_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            size_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) dst[k++] = entry_less(&src[j], &src[i]) ? src[j++] : src[i++];
            while (i < mid) dst[k++] = src[i++];
            while (j < hi) dst[k++] = src[j++];
        }
        orc_entry *t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, n * sizeof(orc_entry));
}

typedef struct {
    int filled;
    double tf, tb;
    int64_t mem;
} orc_rec;

typedef struct {
    const pc_problem *p;
    int ckpt;
    int n_keys;
    int64_t keys[64];
    orc_rec *memo[64];          /* [nb+1][nb+1] per key */
} orc_prof;

/* One memo row: every hi > lo of span [lo, hi) at share m in one pass.  Only
 * for monotone task_block (non-decreasing along the sorted task list, the C5
 * chains): the tasks of [lo, hi+1) are then those of [lo, hi) followed by the
 * tasks of block hi, so continuing the fold of t_fwd / t_bwd over hi performs
 * exactly the additions of orc_span_record's fold (costs.py:137-140); the
 * byte sums are integers (order-free) and the footprint is a running max
 * (costs.py:150-155).  Pinned against orc_span_record and CostModel.profile
 * by tests/test_oracle.py. */
static void span_row(const pc_problem *p, int lo, int64_t m, int ckpt, orc_rec *row)
{
    int nb = p->nb;
    int64_t *in_add = (int64_t *)calloc((size_t)nb + 2, sizeof(int64_t));
    /* inputs: v counts in [lo, hi) iff in_ob[v] < lo and its first consumer
     * block c >= lo has c < hi, i.e. for every hi > c */
    for (int v = 0; v < p->n_in; ++v) {
        if (p->in_ob[v] >= lo) continue;
        for (int k = p->in_cons_off[v]; k < p->in_cons_off[v + 1]; ++k) {
            int c = p->in_cons[k];
            if (c >= lo) {
                in_add[c + 1] += p->in_fix[v] + m * p->in_ps[v];
                break;
            }
        }
    }
    double factor = (1.0 + p->grad_factor) + p->opt_factor;
    double tf = 0.0, tb = 0.0;
    int64_t param = 0, res = 0, inb = 0, maxfp = 0;
    int t = 0;
    while (t < p->n_tasks && p->task_block[t] < lo) ++t;
    for (int hi = lo + 1; hi <= nb; ++hi) {
        int b = hi - 1;                       /* block joining the span */
        for (; t < p->n_tasks && p->task_block[t] == b; ++t) {
            double x = (p->task_flops[t] * (double)m) / p->flops_per_sec;
            double y = p->bwd_fwd_ratio * x;
            tf = tf + x;
            tb = tb + y;
            int64_t fp = p->task_fp_fix[t] + m * p->task_fp_ps[t];
            for (int k = p->task_dep_off[t]; k < p->task_dep_off[t + 1]; ++k)
                if (p->dep_ob[k] >= lo) fp += p->dep_fix[k] + m * p->dep_ps[k];
            if (fp > maxfp) maxfp = fp;
        }
        param += p->blk_param[b];
        res += p->blk_res_fix[b] + m * p->blk_res_ps[b];
        inb += in_add[hi];
        int64_t act = inb + (ckpt ? maxfp : res);
        double memd = (double)param * factor + (double)act;
        orc_rec *r = &row[hi];
        r->tf = tf;
        r->tb = tb;
        r->mem = (int64_t)memd;
        r->filled = 1;
    }
    free(in_add);
}

/* The memo row path above, exposed for the pinning test. */
void orc_span_record_row(const pc_problem *p, int lo, int hi, int64_t m, int ckpt,
                         double *tf_out, double *tb_out, int64_t *mem_out)
{
    orc_rec *row = (orc_rec *)calloc((size_t)p->nb + 1, sizeof(orc_rec));
    span_row(p, lo, m, ckpt, row);
    *tf_out = row[hi].tf;
    *tb_out = row[hi].tb;
    *mem_out = row[hi].mem;
    free(row);
}

static const orc_rec *prof_record(orc_prof *pf, int lo, int hi, int64_t m)
{
    int k;
    for (k = 0; k < pf->n_keys; ++k)
        if (pf->keys[k] == m) break;
    if (k == pf->n_keys) {
        if (k == 64) abort();
        pf->keys[k] = m;
        pf->memo[k] = (orc_rec *)calloc((size_t)(pf->p->nb + 1) * (pf->p->nb + 1), sizeof(orc_rec));
        pf->n_keys++;
    }
    orc_rec *r = &pf->memo[k][(size_t)lo * (pf->p->nb + 1) + hi];
    if (!r->filled) {
        if (pf->p->monotone)
            span_row(pf->p, lo, m, pf->ckpt, &pf->memo[k][(size_t)lo * (pf->p->nb + 1)]);
        else
            orc_span_record(pf->p, lo, hi, m, pf->ckpt, &r->tf, &r->tb, &r->mem);
        r->filled = 1;
    }
    return r;
}

static void prof_free(orc_prof *pf)
{
    for (int k = 0; k < pf->n_keys; ++k) free(pf->memo[k]);
    pf->n_keys = 0;
}

/* Simulated iteration time of a plan (simulate.py:79-165). */
double orc_simulate(const pc_problem *p, int S, const int32_t *lo, const int32_t *hi,
                    const int32_t *dev, const double *tfs, const double *tbs,
                    int64_t BS, int R, int MB)
{
    int ckpt = p->checkpointing && S > 1;
    int64_t denom = (int64_t)MB * R;
    int64_t *m = (int64_t *)malloc(sizeof(int64_t) * S);
    int64_t *cum = (int64_t *)malloc(sizeof(int64_t) * (S + 1));
    double *cf = (double *)malloc(sizeof(double) * S);
    double *cb = (double *)malloc(sizeof(double) * S);
    double *lane = (double *)calloc(S, sizeof(double));
    cum[0] = 0;
    for (int s = 0; s < S; ++s) {
        m[s] = BS / (denom * dev[s]);
        cum[s + 1] = cum[s] + dev[s];
    }
    for (int s = 0; s < S; ++s) {
        cf[s] = s < S - 1 ? orc_cut_time(p, hi[s], m[s], cum[s + 1]) : 0.0;  /* :107-108 */
        cb[s] = s > 0 ? orc_cut_time(p, lo[s], m[s], cum[s]) : 0.0;          /* :109-110 */
    }
    /* forward fill (simulate.py:116-127); arrival[mb][s] is only read for
     * the same mb right after it is written, so one row suffices */
    for (int mb = 0; mb < MB; ++mb) {
        double carry = 0.0;
        for (int s = 0; s < S; ++s) {
            double a = s == 0 ? 0.0 : carry;                 /* arrival[mb][s] */
            double start = a > lane[s] ? a : lane[s];        /* max(lane_free, arrival) */
            double end = start + tfs[s];
            lane[s] = end;
            if (s < S - 1) {
                double send_end = end + cf[s];
                lane[s] = send_end;
                carry = send_end;
            }
        }
    }
    /* backward drain in reverse microbatch order (simulate.py:129-146) */
    for (int mb = MB - 1; mb >= 0; --mb) {
        double carry = 0.0;
        for (int s = S - 1; s >= 0; --s) {
            if (ckpt) lane[s] = lane[s] + tfs[s];
            double g = s == S - 1 ? 0.0 : carry;             /* grad_arrival[mb][s] */
            double start = g > lane[s] ? g : lane[s];
            double end = start + tbs[s];
            lane[s] = end;
            if (s > 0) {
                double send_end = end + cb[s];
                lane[s] = send_end;
                carry = send_end;
            }
        }
    }
    /* gradient sync (simulate.py:148-163) */
    for (int s = 0; s < S; ++s) {
        int64_t group = (int64_t)dev[s] * R;
        if (group <= 1) continue;
        int64_t params = 0;
        for (int b = lo[s]; b < hi[s]; ++b) params += p->blk_param[b];
        if (params == 0) continue;
        int64_t nbytes = 2 * params * (group - 1) / group;
        int64_t first_node = cum[s] / p->devices_per_node;
        int64_t last_node = (cum[s + 1] - 1) / p->devices_per_node;
        int spans = R > 1 || first_node != last_node;
        double bw = spans ? p->bw_inter : p->bw_intra;
        double dur = p->latency + (double)nbytes / bw;
        if (dur > 0.0) lane[s] = lane[s] + dur;
    }
    double it = lane[0];
    for (int s = 1; s < S; ++s)
        if (lane[s] > it) it = lane[s];                       /* :165 */
    free(m); free(cum); free(cf); free(cb); free(lane);
    return it;
}

/* One _run_dp call.  Returns PC_OK / PC_INFEASIBLE / PC_ERR_BUDGET.
 * *visits is incremented as the reference increments stats.visits. */
int orc_run_dp(const pc_problem *p, orc_prof *pf, int S, int D, int64_t BS, int R, int MB,
               int disable_pruning, int64_t budget, int64_t *visits, pc_plan *out)
{
    int nb = p->nb;
    int ckpt = p->checkpointing && S > 1;                   /* :193 */
    int64_t denom = (int64_t)MB * R;
    /* levels[s][b][d] */
    size_t ncell = (size_t)(nb + 1) * (D + 1);
    orc_cell **lv = (orc_cell **)calloc(S + 1, sizeof(orc_cell *));
    for (int s = 0; s <= S; ++s) lv[s] = (orc_cell *)calloc(ncell, sizeof(orc_cell));
    lv[0][0].n = 1;
    lv[0][0].e = (orc_entry *)calloc(1, sizeof(orc_entry));
    lv[0][0].e[0].bp = lv[0][0].e[0].dp = lv[0][0].e[0].idx = -1;
    size_t cap = 1024;
    orc_entry *cands = (orc_entry *)malloc(cap * sizeof(orc_entry));
    orc_entry *tmp = NULL;
    size_t tmp_cap = 0;
    int rc = PC_OK;
    int d_min = 1;
    for (int s = 1; s <= S && rc == PC_OK; ++s) {
        if (s > 1) d_min = 1;                                 /* :205-209 */
        orc_cell *prev = lv[s - 1], *cur = lv[s];
        for (int b = s; b <= nb - S + s && rc == PC_OK; ++b) {
            int dlo = d_min > s ? d_min : s;
            for (int d = D - (S - s); d >= dlo; --d) {
                *visits += (int64_t)(b - s + 1) * (d - s + 1);     /* :214 */
                if (budget >= 0 && *visits > budget) { rc = PC_ERR_BUDGET; break; }
                size_t nc = 0;
                int saw_zero = 0;
                /* prev cells in sorted (bp, dp) order (stages.py:220); level
                 * s-1 holds cells only at bp in [s-1, nb-S+s-1], dp in
                 * [s-1, D-S+s-1], so the scan starts and ends there */
                int dp_end = d < D - S + s ? d : D - S + s;
                for (int bp = s - 1; bp < b; ++bp) {
                    for (int dp = s - 1; dp < dp_end; ++dp) {
                        orc_cell *pc = &prev[(size_t)bp * (D + 1) + dp];
                        if (pc->n == 0) continue;
                        int64_t dev = d - dp;
                        int64_t m = BS / (denom * dev);
                        if (m == 0) { saw_zero = 1; continue; }      /* :224-228 */
                        const orc_rec *r = prof_record(pf, bp, b, m);
                        if (r->mem > p->mem_budget) continue;       /* :230 */
                        double tf = r->tf;
                        if (b < nb) tf = tf + orc_cut_time(p, b, m, d);
                        double tb = r->tb;
                        if (bp > 0) tb = tb + orc_cut_time(p, bp, m, dp);
                        for (int i = 0; i < pc->n; ++i) {
                            if (nc == cap) {
                                cap *= 2;
                                cands = (orc_entry *)realloc(cands, cap * sizeof(orc_entry));
                            }
                            orc_entry *c = &cands[nc];
                            double ptf = pc->e[i].tf, ptb = pc->e[i].tb;
                            c->tf = tf > ptf ? tf : ptf;              /* max(ptf, tf) */
                            c->tb = tb > ptb ? tb : ptb;
                            c->bp = bp; c->dp = dp; c->idx = i; c->ord = (int)nc;
                            ++nc;
                        }
                    }
                }
                if (nc) {
                    sort_cands(cands, nc, &tmp, &tmp_cap);          /* _pareto */
                    orc_cell *cc = &cur[(size_t)b * (D + 1) + d];
                    cc->e = (orc_entry *)malloc(nc * sizeof(orc_entry));
                    double best = INFINITY;
                    for (size_t i = 0; i < nc; ++i) {
                        if (cands[i].tb < best) {
                            cc->e[cc->n++] = cands[i];
                            best = cands[i].tb;
                        }
                    }
                    cc->e = (orc_entry *)realloc(cc->e, (size_t)cc->n * sizeof(orc_entry));
                    g_fhist[cc->n < 64 ? cc->n : 64]++;
                } else if (!disable_pruning && !saw_zero) {   /* :242-249 */
                    if (s == 1) d_min = d + 1;
                    break;
                }
            }
        }
    }
    free(cands);
    free(tmp);
    out->n_stages = 0;
    out->objective = NAN;
    out->iteration_time = NAN;
    if (rc == PC_OK) {
        orc_cell *fin = &lv[S][(size_t)nb * (D + 1) + D];
        if (fin->n == 0) {
            rc = PC_INFEASIBLE;
        } else {
            orc_entry best = fin->e[0];                                /* :256-259 */
            for (int i = 1; i < fin->n; ++i)
                if (fin->e[i].tf + fin->e[i].tb < best.tf + best.tb) best = fin->e[i];
            int s = S, b = nb, d = D;
            orc_entry e = best;
            while (s > 0) {                                             /* :260-268 */
                int k = s - 1;
                out->lo[k] = e.bp;
                out->hi[k] = b;
                out->devices[k] = d - e.dp;
                if (s > 1) e = lv[s - 1][(size_t)e.bp * (D + 1) + e.dp].e[e.idx];
                int nbp = out->lo[k], ndp = d - out->devices[k];
                s -= 1; b = nbp; d = ndp;
            }
            for (int k = 0; k < S; ++k) {                               /* :269-276 */
                int64_t m = BS / (denom * out->devices[k]);
                const orc_rec *r = prof_record(pf, out->lo[k], out->hi[k], m);
                out->t_fwd[k] = r->tf;
                out->t_bwd[k] = r->tb;
                out->mem[k] = r->mem;
            }
            out->n_stages = S;
            out->objective = best.tf + best.tb;
        }
    }
    out->S = S; out->D = D; out->R = R; out->MB = MB;
    for (int s = 0; s <= S; ++s) {
        for (size_t i = 0; i < ncell; ++i) free(lv[s][i].e);
        free(lv[s]);
    }
    free(lv);
    return rc;
}

/* form_stage_dp (stages.py:282-291).  Fresh profiler per call. */
int orc_form_stage_dp(const pc_problem *p, int S, int D, int64_t BS, int R, int MB,
                      int disable_pruning, int64_t budget, pc_plan *out, int64_t *visits)
{
    if (S < 1 || D < 1 || BS < 1 || R < 1 || MB < 1) return PC_ERR_INVALID;
    if (S > D || S > p->nb) return PC_ERR_INVALID;
    if (S > out->cap_stages) return PC_ERR_CAPACITY;
    orc_prof pf;
    memset(&pf, 0, sizeof pf);
    pf.p = p;
    pf.ckpt = p->checkpointing && S > 1;
    *visits = 0;
    int rc = orc_run_dp(p, &pf, S, D, BS, R, MB, disable_pruning, budget, visits, out);
    prof_free(&pf);
    return rc;
}

/* form_stage (stages.py:372-413).  scratch must hold cap_stages entries per
 * array like out.  Returns PC_OK, PC_INFEASIBLE, PC_ERR_BUDGET. */
int orc_form_stage(const pc_problem *p, int N, int dpn, int64_t BS, int disable_pruning,
                   int64_t budget, pc_plan *out, pc_plan *scratch,
                   int64_t *visits, int64_t *dp_calls)
{
    if (N < 1 || dpn < 1 || BS < 1) return PC_ERR_INVALID;
    int nb = p->nb;
    *visits = 0;
    *dp_calls = 0;
    orc_prof pf[2];
    memset(pf, 0, sizeof pf);
    pf[0].p = pf[1].p = p;
    pf[0].ckpt = 0;
    pf[1].ckpt = p->checkpointing;
    for (int n = 1; n <= N; n *= 2) {
        if (N % n) continue;
        int D = dpn * n, R = N / n;
        int have = 0;
        double best_it = 0, best_obj = 0;
        int best_mb = 0;
        for (int S = dpn * (n - 1) + 1; S <= D; ++S) {
            if (S > nb) continue;
            if (S > out->cap_stages) { prof_free(&pf[0]); prof_free(&pf[1]); return PC_ERR_CAPACITY; }
            for (int64_t MB = 1; MB * R <= BS; MB *= 2) {
                ++*dp_calls;
                orc_prof *use = &pf[p->checkpointing && S > 1];
                int rc = orc_run_dp(p, use, S, D, BS, R, (int)MB, disable_pruning, budget,
                                    visits, scratch);
                if (rc == PC_ERR_BUDGET) { prof_free(&pf[0]); prof_free(&pf[1]); return rc; }
                if (rc != PC_OK) continue;
                double it = orc_simulate(p, S, scratch->lo, scratch->hi, scratch->devices,
                                         scratch->t_fwd, scratch->t_bwd, BS, R, (int)MB);
                scratch->iteration_time = it;
                /* min by (iteration_time, objective, microbatches), first wins */
                int better = !have || it < best_it ||
                             (it == best_it && (scratch->objective < best_obj ||
                              (scratch->objective == best_obj && MB < best_mb)));
                if (better) {
                    have = 1;
                    best_it = it; best_obj = scratch->objective; best_mb = (int)MB;
                    out->n_stages = scratch->n_stages;
                    for (int k = 0; k < S; ++k) {
                        out->lo[k] = scratch->lo[k]; out->hi[k] = scratch->hi[k];
                        out->devices[k] = scratch->devices[k];
                        out->t_fwd[k] = scratch->t_fwd[k]; out->t_bwd[k] = scratch->t_bwd[k];
                        out->mem[k] = scratch->mem[k];
                    }
                    out->S = S; out->D = D; out->R = R; out->MB = (int)MB;
                    out->objective = scratch->objective;
                    out->iteration_time = it;
                }
            }
        }
        if (have) { prof_free(&pf[0]); prof_free(&pf[1]); return PC_OK; }
    }
    prof_free(&pf[0]); prof_free(&pf[1]);
    out->n_stages = 0;
    return PC_INFEASIBLE;
}
