// Host orchestration and the C-ABI of include/pipecut_b200.h.
//
// The device does all search arithmetic (span tables, DP levels, visit
// accounting, backtrack, stage records, simulation); the host code here only
// sizes buffers, orders launches and applies the reference's enumeration and
// selection rules over per-call records (form_stage, stages.py:372-413).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace pcb;

// =========================================================================== context
extern "C" int pc_ctx_create(int device, pc_ctx **out) {
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n <= device) {
        cudaGetLastError();
        return PC_ERR_CUDA;
    }
    pc_ctx *ctx = new pc_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return PC_ERR_CUDA;
    }
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    cudaEventCreate(&ctx->ev2);
    cudaEventCreate(&ctx->ev3);
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major != 10) {
        ctx->err = "pipecut_b200 is built for sm_100a only";
        pc_ctx_destroy(ctx);
        return PC_ERR_CUDA;
    }
    *out = ctx;
    return PC_OK;
}

static void free_keys(pc_ctx *ctx) {
    ctx->keys.clear();
    ctx->key_map.clear();
    ctx->key_bytes = 0;
    ctx->slot_used.assign(ctx->key_cap, 0);
}

extern "C" void pc_ctx_destroy(pc_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->st);
    free_keys(ctx);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev2) cudaEventDestroy(ctx->ev2);
    if (ctx->ev3) cudaEventDestroy(ctx->ev3);
    if (ctx->t0) cudaEventDestroy(ctx->t0);
    if (ctx->t1) cudaEventDestroy(ctx->t1);
    if (ctx->st) cudaStreamDestroy(ctx->st);
    delete ctx;
}

extern "C" const char *pc_last_error(pc_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

extern "C" int pc_device_info(pc_ctx *ctx, int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor) {
    int ma = 0, mi = 0;
    cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, ctx->device);
    cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, ctx->device);
    *sm_count = ctx->sm_count;
    *cc_major = ma;
    *cc_minor = mi;
    return PC_OK;
}

// =========================================================================== problem
extern "C" int pc_set_problem(pc_ctx *ctx, const pc_problem *p) {
    cudaSetDevice(ctx->device);
    if (p->nb < 1 || p->nb > MAX_NB_KEY) return fail(ctx, PC_ERR_CAPACITY, "block count out of range");
    if (p->n_tasks < 0 || p->n_in < 0) return fail(ctx, PC_ERR_INVALID, "negative sizes");
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    free_keys(ctx);
    ctx->has_problem = false;
    const int nb = p->nb, T = p->n_tasks, V = p->n_in;
    const int ndep = p->task_dep_off[T];
    const int ncons = p->in_cons_off[V];
    // block -> task CSR (stable: task indices ascending within a block)
    std::vector<int32_t> blk_off(nb + 1, 0), blk_tasks(T);
    for (int t = 0; t < T; ++t) {
        int b = p->task_block[t];
        if (b < 0 || b >= nb) return fail(ctx, PC_ERR_INVALID, "task block out of range");
        blk_off[b + 1]++;
    }
    for (int b = 0; b < nb; ++b) blk_off[b + 1] += blk_off[b];
    {
        std::vector<int32_t> fill(blk_off.begin(), blk_off.end() - 1);
        for (int t = 0; t < T; ++t) blk_tasks[fill[p->task_block[t]]++] = t;
    }
    std::vector<int64_t> pre_param(nb + 1, 0), pre_rf(nb + 1, 0), pre_rp(nb + 1, 0);
    for (int b = 0; b < nb; ++b) {
        pre_param[b + 1] = pre_param[b] + p->blk_param[b];
        pre_rf[b + 1] = pre_rf[b] + p->blk_res_fix[b];
        pre_rp[b + 1] = pre_rp[b] + p->blk_res_ps[b];
    }
    // one allocation, 8-byte aligned sub-arrays
    struct Part { const void *src; size_t bytes; size_t off; };
    std::vector<Part> parts;
    size_t total = 0;
    auto add = [&](const void *src, size_t bytes) {
        size_t off = (total + 15) & ~size_t(15);
        parts.push_back({src, bytes, off});
        total = off + bytes;
        return parts.size() - 1;
    };
    size_t i_tb = add(p->task_block, 4 * (size_t)T);
    size_t i_tf = add(p->task_flops, 8 * (size_t)T);
    size_t i_ff = add(p->task_fp_fix, 8 * (size_t)T);
    size_t i_fp = add(p->task_fp_ps, 8 * (size_t)T);
    size_t i_qf = add(p->task_prod_fix, 8 * (size_t)T);
    size_t i_qp = add(p->task_prod_ps, 8 * (size_t)T);
    size_t i_do = add(p->task_dep_off, 4 * (size_t)(T + 1));
    size_t i_dob = add(p->dep_ob, 4 * (size_t)ndep);
    size_t i_df = add(p->dep_fix, 8 * (size_t)ndep);
    size_t i_dp = add(p->dep_ps, 8 * (size_t)ndep);
    size_t i_bo = add(blk_off.data(), 4 * (size_t)(nb + 1));
    size_t i_bt = add(blk_tasks.data(), 4 * (size_t)T);
    size_t i_io = add(p->in_ob, 4 * (size_t)V);
    size_t i_ico = add(p->in_cons_off, 4 * (size_t)(V + 1));
    size_t i_ic = add(p->in_cons, 4 * (size_t)ncons);
    size_t i_if = add(p->in_fix, 8 * (size_t)V);
    size_t i_ip = add(p->in_ps, 8 * (size_t)V);
    size_t i_pp = add(pre_param.data(), 8 * (size_t)(nb + 1));
    size_t i_prf = add(pre_rf.data(), 8 * (size_t)(nb + 1));
    size_t i_prp = add(pre_rp.data(), 8 * (size_t)(nb + 1));
    size_t i_cf = add(p->cut_fixed, 8 * (size_t)(nb + 1));
    size_t i_cp = add(p->cut_ps, 8 * (size_t)(nb + 1));
    CUDA_TRY(ctx, ctx->prob.ensure(total + 16));
    std::vector<char> staging(total + 16, 0);
    for (auto &pt : parts)
        if (pt.bytes) memcpy(staging.data() + pt.off, pt.src, pt.bytes);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->prob.p, staging.data(), total, cudaMemcpyHostToDevice, ctx->st));
    char *base = (char *)ctx->prob.p;
    auto at = [&](size_t i) { return (void *)(base + parts[i].off); };
    DevProblem &D = ctx->P;
    D = DevProblem();
    D.nb = nb;
    D.n_tasks = T;
    D.n_in = V;
    D.num_nodes = p->num_nodes;
    D.dpn = p->devices_per_node;
    D.checkpointing = p->checkpointing;
    D.monotone = p->monotone;
    D.n_inter = p->num_nodes > 1 ? 2 : 1;
    D.mem_budget = p->mem_budget;
    D.flops = p->flops_per_sec;
    D.beta = p->bwd_fwd_ratio;
    D.factor = (1.0 + p->grad_factor) + p->opt_factor;   // costs.py:158
    D.bw_intra = p->bw_intra;
    D.bw_inter = p->bw_inter;
    D.lat = p->latency;
    D.task_block = (const int32_t *)at(i_tb);
    D.task_flops = (const double *)at(i_tf);
    D.fp_fix = (const int64_t *)at(i_ff);
    D.fp_ps = (const int64_t *)at(i_fp);
    D.prod_fix = (const int64_t *)at(i_qf);
    D.prod_ps = (const int64_t *)at(i_qp);
    D.n_ov = 0;
    D.dep_off = (const int32_t *)at(i_do);
    D.dep_ob = (const int32_t *)at(i_dob);
    D.dep_fix = (const int64_t *)at(i_df);
    D.dep_ps = (const int64_t *)at(i_dp);
    D.blk_off = (const int32_t *)at(i_bo);
    D.blk_tasks = (const int32_t *)at(i_bt);
    D.in_ob = (const int32_t *)at(i_io);
    D.in_cons_off = (const int32_t *)at(i_ico);
    D.in_cons = (const int32_t *)at(i_ic);
    D.in_fix = (const int64_t *)at(i_if);
    D.in_ps = (const int64_t *)at(i_ip);
    D.pre_param = (const int64_t *)at(i_pp);
    D.pre_res_fix = (const int64_t *)at(i_prf);
    D.pre_res_ps = (const int64_t *)at(i_prp);
    D.cut_fixed = (const int64_t *)at(i_cf);
    D.cut_ps = (const double *)at(i_cp);
    const int64_t tri = tri_size(nb);
    CUDA_TRY(ctx, ctx->in_tab.ensure(sizeof(int64_t) * 2 * (size_t)tri));
    int64_t *inf = ctx->in_tab.as<int64_t>();
    D.in_tab_fix = inf;
    D.in_tab_ps = inf + tri;
    launch_in_tables(D, inf, inf + tri, ctx->st);
    if (int rc = check_launch(ctx, "in_tables")) return rc;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    ctx->pre_param = pre_param;
    ctx->nb = nb;
    {
        int ex = 0;
        const double fr = frexp(p->bwd_fwd_ratio, &ex);
        ctx->derived = p->bwd_fwd_ratio > 0 && fr == 0.5;
        // span times are folds of (f*m)/F: non-negative terms make them monotone
        // in the span, which the DP's prefix skip relies on
        bool nonneg = p->flops_per_sec > 0 && p->bwd_fwd_ratio >= 0;
        for (int t = 0; t < T; ++t) {
            if (std::isnan(p->task_flops[t]))   // NaN is the infeasible-span marker (span_mark)
                return fail(ctx, PC_ERR_INVALID, "NaN flops_per_sample is not supported");
            nonneg = nonneg && p->task_flops[t] >= 0.0;
        }
        ctx->mono_flops = nonneg;
        ctx->mono_skip = nonneg;
        D.nonneg = nonneg ? 1 : 0;
    }
    ctx->has_cost_table = p->has_cost_table != 0;
    ctx->ov_m.clear();
    ctx->h_task_block.assign(p->task_block, p->task_block + T);
    ctx->h_prod_fix.assign(p->task_prod_fix, p->task_prod_fix + T);
    ctx->h_prod_ps.assign(p->task_prod_ps, p->task_prod_ps + T);
    ctx->has_problem = true;
    return PC_OK;
}

// =========================================================================== key tables
static int ensure_keys(pc_ctx *ctx, const std::vector<std::pair<int64_t, int>> &want) {
    const DevProblem &P = ctx->P;
    const int64_t tri = tri_size(P.nb);
    std::vector<std::pair<int64_t, int>> fresh;
    for (auto &k : want)
        if (!ctx->key_map.count(k)) fresh.push_back(k);
    if (fresh.empty()) return PC_OK;
    if (ctx->has_cost_table)
        for (auto &k : fresh)
            if (std::find(ctx->ov_m.begin(), ctx->ov_m.end(), k.first) == ctx->ov_m.end())
                return fail(ctx, PC_ERR_INVALID, "cost table: microbatch share not resolved by pc_set_overrides");
    for (int attempt = 0; attempt < 2; ++attempt) {
        const size_t raw_key = sizeof(double) * ((ctx->derived ? 1 : 2) * (size_t)tri + 2 * (size_t)(P.nb + 1)) + sizeof(int32_t) * (size_t)(P.nb + 1);
        const size_t per_key = (raw_key + 255) & ~size_t(255);
        if (per_key != ctx->key_slot) {          // new layout (nb or derived changed):
            free_keys(ctx);                       // re-slice the arena, keep the memory
            ctx->key_slot = per_key;
            ctx->key_cap = (int)(ctx->key_arena.n / per_key);
            ctx->slot_used.assign(ctx->key_cap, 0);
            fresh = want;
        }
        if (ctx->keys.size() + fresh.size() > (size_t)ctx->key_cap) {
            // drop cached keys this batch does not need
            std::map<std::pair<int64_t, int>, int> need;
            for (auto &k : want) need[k] = 1;
            std::vector<CachedKey> kept;
            for (auto &k : ctx->keys) {
                if (need.count({k.m, k.ckpt})) kept.push_back(k);
                else ctx->slot_used[k.slot] = 0;
            }
            ctx->keys = kept;
            ctx->key_map.clear();
            for (size_t i = 0; i < ctx->keys.size(); ++i)
                ctx->key_map[{ctx->keys[i].m, ctx->keys[i].ckpt}] = (int)i;
        }
        if (ctx->keys.size() + fresh.size() > (size_t)ctx->key_cap) {
            // grow the arena (bounded by a third of device memory) and rebuild
            // every key of the batch in it
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            const size_t limit = (free_b + ctx->key_arena.n) / 3;
            size_t slots = std::max(want.size(), (size_t)ctx->key_cap * 3 / 2);
            if (slots * per_key > limit) slots = std::max(want.size(), limit / per_key);
            free_keys(ctx);
            ctx->key_arena.release();
            ctx->key_cap = 0;
            CUDA_TRY(ctx, ctx->key_arena.ensure(slots * per_key));
            ctx->key_cap = (int)(ctx->key_arena.n / per_key);
            ctx->slot_used.assign(ctx->key_cap, 0);
            fresh = want;
        }
        const int nf = (int)fresh.size();
        std::vector<int64_t> km(nf);
        std::vector<int32_t> kc(nf);
        std::vector<double *> pf(nf), pb(nf, nullptr), pcut(nf);
        std::vector<int> slot(nf);
        int cursor = 0;
        for (int i = 0; i < nf; ++i) {
            km[i] = fresh[i].first;
            kc[i] = fresh[i].second;
            while (ctx->slot_used[cursor]) ++cursor;     // capacity checked above
            ctx->slot_used[cursor] = 1;
            slot[i] = cursor;
            char *base = ctx->key_arena.as<char>() + (size_t)cursor * per_key;
            pf[i] = (double *)base;
            if (!ctx->derived) pb[i] = pf[i] + tri;
            pcut[i] = pf[i] + (ctx->derived ? 1 : 2) * (size_t)tri;
            ctx->key_bytes += per_key;
        }
        const size_t hdr = (sizeof(int64_t) * nf + sizeof(int32_t) * nf + 15) & ~size_t(15);
        CUDA_TRY(ctx, ctx->keys_m_d.ensure(hdr + sizeof(double *) * 4 * nf + 64));
        char *kb = ctx->keys_m_d.as<char>();
        int64_t *d_km = (int64_t *)kb;
        int32_t *d_kc = (int32_t *)(kb + sizeof(int64_t) * nf);
        double **d_pf = (double **)(kb + hdr);
        double **d_pb = d_pf + nf;
        double **d_pc = d_pb + nf;
        int32_t **d_pff = (int32_t **)(d_pc + nf);
        std::vector<int32_t *> pff(nf);
        for (int i = 0; i < nf; ++i) pff[i] = (int32_t *)(pcut[i] + 2 * (size_t)(P.nb + 1));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_km, km.data(), sizeof(int64_t) * nf, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_kc, kc.data(), sizeof(int32_t) * nf, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_pf, pf.data(), sizeof(double *) * nf, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_pb, pb.data(), sizeof(double *) * nf, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_pc, pcut.data(), sizeof(double *) * nf, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_pff, pff.data(), sizeof(int32_t *) * nf, cudaMemcpyHostToDevice, ctx->st));
        const double *raw_tf = nullptr, *raw_tb = nullptr;
        if (P.monotone) {
            // per-key task times, read by the span fold (k_span_rows)
            CUDA_TRY(ctx, ctx->raw_d.ensure(sizeof(double) * 2 * (size_t)nf * P.n_tasks + 64));
            double *r = ctx->raw_d.as<double>();
            launch_key_task_times(P, nf, d_km, r, r + (size_t)nf * P.n_tasks, ctx->st);
            ctx->launches++;
            if (int rc = check_launch(ctx, "key_task_times")) return rc;
            raw_tf = r;
            raw_tb = r + (size_t)nf * P.n_tasks;
        } else {
            CUDA_TRY(ctx, ctx->raw_d.ensure(sizeof(double) * 2 * (size_t)nf * tri));
            double *r = ctx->raw_d.as<double>();
            launch_span_time_general(P, nf, d_km, r, r + (size_t)nf * tri, ctx->st);
            ctx->launches++;
            if (int rc = check_launch(ctx, "span_time_general")) return rc;
            raw_tf = r;
            raw_tb = r + (size_t)nf * tri;
        }
        CUDA_TRY(ctx, ctx->mismatch_d.ensure(sizeof(int)));
        CUDA_TRY(ctx, cudaMemsetAsync(ctx->mismatch_d.p, 0, sizeof(int), ctx->st));
        launch_span_dp_tables(P, nf, d_km, d_kc, raw_tf, raw_tb, d_pf, d_pb, d_pc, ctx->derived ? 1 : 0,
                              ctx->mismatch_d.as<int>(), ctx->st);
        ctx->launches++;
        if (int rc = check_launch(ctx, "span_dp_tables")) return rc;
        // the bound (run_chunk) needs suffix-closed feasibility: checked where it can apply
        const int check = (!ctx->has_cost_table && ctx->mono_skip) ? 1 : 0;
        CUDA_TRY(ctx, ctx->open_d.ensure(sizeof(int) * (size_t)nf + 16));
        CUDA_TRY(ctx, cudaMemsetAsync(ctx->open_d.p, 0, sizeof(int) * (size_t)nf, ctx->st));
        launch_first_feasible(P.nb, nf, P.nonneg, check, d_pf, d_pff, ctx->open_d.as<int>(), ctx->st);
        ctx->launches++;
        if (int rc = check_launch(ctx, "first_feasible")) return rc;
        int mism = 0;
        std::vector<int> open(nf, 1);
        CUDA_TRY(ctx, cudaMemcpyAsync(&mism, ctx->mismatch_d.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
        if (check)
            CUDA_TRY(ctx, cudaMemcpyAsync(open.data(), ctx->open_d.p, sizeof(int) * (size_t)nf,
                                          cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        for (int i = 0; i < nf; ++i) {
            CachedKey ck;
            ck.m = km[i];
            ck.ckpt = kc[i];
            ck.tf = pf[i];
            ck.tb = pb[i];
            ck.cut = pcut[i];
            ck.slot = slot[i];
            ck.closed = check && !open[i];
            ctx->key_map[{km[i], kc[i]}] = (int)ctx->keys.size();
            ctx->keys.push_back(ck);
        }
        if (mism && ctx->derived) {
            // t_bwd is not exactly beta * t_fwd here: store it explicitly
            free_keys(ctx);
            ctx->derived = false;
            fresh = want;
            continue;
        }
        break;
    }
    // device pointer arrays for the DP kernels
    const size_t nk = ctx->keys.size();
    std::vector<const void *> ptrs(4 * nk);
    for (size_t i = 0; i < nk; ++i) {
        ptrs[i] = ctx->keys[i].tf;
        ptrs[nk + i] = ctx->keys[i].tb;
        ptrs[2 * nk + i] = ctx->keys[i].cut;
        ptrs[3 * nk + i] = ctx->keys[i].cut + 2 * (size_t)(P.nb + 1);
    }
    CUDA_TRY(ctx, ctx->key_ptrs.ensure(sizeof(void *) * 4 * nk));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->key_ptrs.p, ptrs.data(), sizeof(void *) * 4 * nk,
                                  cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    return PC_OK;
}

// =========================================================================== batch
struct CallOut {
    int feasible = 0;
    double objective = NAN;
    double iteration = NAN;
    int64_t visits = 0, visits_unpruned = 0;
    double bound = INFINITY;     // the objective bound the call ran with
    std::vector<int32_t> lo, hi, dev;
    std::vector<double> tf, tb;
    std::vector<int64_t> mem;
    std::vector<int64_t> level_sums;
};

static int validate_call(pc_ctx *ctx, const pc_call &c, int64_t BS) {
    if (c.S < 1 || c.D < 1 || BS < 1 || c.R < 1 || c.MB < 1)
        return fail(ctx, PC_ERR_INVALID, "stage count, devices, batch size, replicas and microbatches must all be at least 1");
    if (c.S > c.D) return fail(ctx, PC_ERR_INVALID, "cannot run more stages than devices");
    if (c.S > ctx->nb) return fail(ctx, PC_ERR_INVALID, "cannot cut the blocks into that many stages");
    if (c.D > MAX_D_KEY) return fail(ctx, PC_ERR_CAPACITY, "device count beyond the packed back-pointer range");
    return PC_OK;
}

static inline int64_t tri_sum(int64_t n) { return n * (n + 1) / 2; }

// largest pool offset (entries) a 31-bit frontier offset can hold
constexpr int64_t OFF_MAX = (int64_t)SPILL_BIT - 1;
// history cells per chunk: the shared history spill pool is sized from them
// (one entry per cell at first) and must stay within OFF_MAX (the pools are
// capped there anyway; fewer chunks means fewer passes over the levels)
constexpr int64_t CHUNK_HIST_CELLS = 1900000000;
// objective bound (dp.cu) only for batches of at least this many unpruned visits
constexpr double BOUND_MIN_VISITS = 2e8;

// Runs one batch of DP calls whose buffers fit; fills outs[orig] for each.
static int run_chunk(pc_ctx *ctx, const std::vector<pc_call> &calls, const std::vector<int> &idx,
                     int64_t BS, int pruning, int want_iter, std::vector<CallOut> &outs) {
    const DevProblem &P = ctx->P;
    const int nb = ctx->nb;
    const int n = (int)idx.size();
    // order by S descending (stable)
    std::vector<int> order(idx);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return calls[a].S > calls[b].S; });
    // keys
    std::vector<std::pair<int64_t, int>> want;
    std::vector<std::vector<std::pair<int64_t, int>>> call_keys(n);
    for (int i = 0; i < n; ++i) {
        const pc_call &c = calls[order[i]];
        const int ckpt = P.checkpointing && c.S > 1;
        const int B = c.D - c.S + 1;
        call_keys[i].resize(B + 1, {0, -1});
        for (int dev = 1; dev <= B; ++dev) {
            const int64_t m = BS / ((int64_t)c.MB * c.R * dev);
            if (m >= 1) {
                call_keys[i][dev] = {m, ckpt};
                want.push_back({m, ckpt});
            }
        }
    }
    std::sort(want.begin(), want.end());
    want.erase(std::unique(want.begin(), want.end()), want.end());
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->st));
    if (int rc = ensure_keys(ctx, want)) return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->st));
    // call descriptors
    std::vector<CallDesc> cds(n);
    std::vector<int16_t> keyidx;
    std::vector<int64_t> cta_prefix(n + 1, 0);
    int64_t val_cells = 0, hist_cells = 0;
    int maxS = 0;
    for (int i = 0; i < n; ++i) {
        const pc_call &c = calls[order[i]];
        CallDesc &cd = cds[i];
        cd.S = c.S; cd.D = c.D; cd.R = c.R; cd.MB = c.MB;
        cd.A = nb - c.S + 1;
        cd.B = c.D - c.S + 1;
        cd.ckpt = P.checkpointing && c.S > 1;
        cd.key_off = (int32_t)keyidx.size();
        for (int dev = 0; dev <= cd.B; ++dev) {
            int16_t k = -1;
            if (dev >= 1 && call_keys[i][dev].second >= 0) k = (int16_t)ctx->key_map[call_keys[i][dev]];
            keyidx.push_back(k);
        }
        cd.val_off = val_cells;
        cd.hist_off = hist_cells;
        cd.orig = order[i];
        cd.pad = 0;
        cd.U = INFINITY;
        const int64_t cells = (int64_t)cd.A * cd.B;
        val_cells += cells;
        hist_cells += cells * cd.S;
        cta_prefix[i + 1] = cta_prefix[i] + ((int64_t)cd.A * cd.B + DP_WARPS - 1) / DP_WARPS;
        maxS = std::max(maxS, cd.S);
    }
    CUDA_TRY(ctx, ctx->calls_d.ensure(sizeof(CallDesc) * n));
    CUDA_TRY(ctx, ctx->warp_prefix_d.ensure(sizeof(int64_t) * (n + 1)));
    CUDA_TRY(ctx, ctx->keyidx_d.ensure(sizeof(int16_t) * keyidx.size() + 16));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->calls_d.p, cds.data(), sizeof(CallDesc) * n, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->warp_prefix_d.p, cta_prefix.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, ctx->cta_call_d.ensure(sizeof(int32_t) * (size_t)cta_prefix[n] + 16));
    launch_cta_call(ctx->warp_prefix_d.as<int64_t>(), n, cta_prefix[n], ctx->cta_call_d.as<int32_t>(), ctx->st);
    ctx->launches++;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->keyidx_d.p, keyidx.data(), sizeof(int16_t) * keyidx.size(), cudaMemcpyHostToDevice, ctx->st));

    const size_t nk = ctx->keys.size();
    DPBatch bt{};
    bt.nb = nb;
    bt.n_calls = n;
    bt.calls = ctx->calls_d.as<CallDesc>();
    bt.keyidx = ctx->keyidx_d.as<int16_t>();
    bt.key_tf = (const double *const *)ctx->key_ptrs.p;
    bt.key_tb = ((const double *const *)ctx->key_ptrs.p) + nk;
    bt.key_cut = ((const double *const *)ctx->key_ptrs.p) + 2 * nk;
    bt.key_ffb = ((const int32_t *const *)ctx->key_ptrs.p) + 3 * nk;
    bt.beta = P.beta;
    bt.batch_size = BS;
    bt.mono_skip = ctx->mono_skip ? 1 : 0;
    bt.num_nodes = P.num_nodes;
    bt.dpn = P.dpn;

    // ---- objective bound (dp.cu): only with non-negative times, no cost
    // table and suffix-closed feasibility in every key of the batch.  A call's
    // U is the DP objective of its (S, D, R, MB/2) partner's optimal plan
    // under this call's shares (run_calls_impl runs the partners first), or the
    // explicit ctx->bb_U (measurement hook).
    bool bounded = false;
    if (!ctx->has_cost_table && ctx->mono_skip && !ctx->bb_off &&
        (!ctx->bb_U.empty() || !ctx->bb_partner.empty())) {
        bool closed = true;
        for (auto &k : want) closed = closed && ctx->keys[ctx->key_map[k]].closed;
        if (closed) {
            std::vector<int32_t> pos, seg_off, slo, shi, sdev;
            for (int i = 0; i < n; ++i) {
                const int o = order[i];
                if (!ctx->bb_U.empty()) cds[i].U = ctx->bb_U[o];
                const int p = ctx->bb_partner.empty() ? -1 : ctx->bb_partner[o];
                if (p < 0 || !outs[p].feasible || (int)outs[p].lo.size() != cds[i].S) continue;
                pos.push_back(i);
                seg_off.push_back((int32_t)slo.size());
                slo.insert(slo.end(), outs[p].lo.begin(), outs[p].lo.end());
                shi.insert(shi.end(), outs[p].hi.begin(), outs[p].hi.end());
                sdev.insert(sdev.end(), outs[p].dev.begin(), outs[p].dev.end());
            }
            const int nbd = (int)pos.size();
            if (nbd > 0) {
                const size_t ns = slo.size();
                CUDA_TRY(ctx, ctx->bound_d.ensure(4 * (2 * (size_t)nbd + 3 * ns) + 8 * (size_t)nbd + 64));
                char *bb = ctx->bound_d.as<char>();
                double *d_U = (double *)bb;
                int32_t *d_pos = (int32_t *)(bb + 8 * (size_t)nbd);
                int32_t *d_so = d_pos + nbd, *d_lo = d_so + nbd, *d_hi = d_lo + ns, *d_dv = d_hi + ns;
                CUDA_TRY(ctx, cudaMemcpyAsync(d_pos, pos.data(), 4 * (size_t)nbd, cudaMemcpyHostToDevice, ctx->st));
                CUDA_TRY(ctx, cudaMemcpyAsync(d_so, seg_off.data(), 4 * (size_t)nbd, cudaMemcpyHostToDevice, ctx->st));
                CUDA_TRY(ctx, cudaMemcpyAsync(d_lo, slo.data(), 4 * ns, cudaMemcpyHostToDevice, ctx->st));
                CUDA_TRY(ctx, cudaMemcpyAsync(d_hi, shi.data(), 4 * ns, cudaMemcpyHostToDevice, ctx->st));
                CUDA_TRY(ctx, cudaMemcpyAsync(d_dv, sdev.data(), 4 * ns, cudaMemcpyHostToDevice, ctx->st));
                launch_plan_bound(bt, nbd, d_pos, d_so, d_lo, d_hi, d_dv, d_U, ctx->derived, ctx->st);
                ctx->launches++;
                if (int rc = check_launch(ctx, "plan_bound")) return rc;
                std::vector<double> U(nbd);
                CUDA_TRY(ctx, cudaMemcpyAsync(U.data(), d_U, 8 * (size_t)nbd, cudaMemcpyDeviceToHost, ctx->st));
                CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
                for (int t = 0; t < nbd; ++t) cds[pos[t]].U = std::min(cds[pos[t]].U, U[t]);
            }
            // calls still unbounded (no partner, or an infeasible one): a greedy plan
            std::vector<int32_t> gpos;
            for (int i = 0; i < n; ++i)
                if (!(cds[i].U < INFINITY) && ctx->bb_U.empty()) gpos.push_back(i);
            const int ng = (int)gpos.size();
            if (ng > 0 && getenv("PIPECUT_B200_NO_GREEDY") == nullptr) {
                CUDA_TRY(ctx, ctx->bound_d.ensure((8 * GB_SPLITS + 4) * (size_t)ng + 64));
                double *d_U = ctx->bound_d.as<double>();          // [GB_SPLITS][ng]
                int32_t *d_pos = (int32_t *)(d_U + GB_SPLITS * ng);
                CUDA_TRY(ctx, cudaMemcpyAsync(d_pos, gpos.data(), 4 * (size_t)ng, cudaMemcpyHostToDevice, ctx->st));
                launch_greedy_bound(bt, ng, d_pos, d_U, ctx->derived, ctx->st);
                ctx->launches++;
                if (int rc = check_launch(ctx, "greedy_bound")) return rc;
                std::vector<double> U(GB_SPLITS * (size_t)ng);
                CUDA_TRY(ctx, cudaMemcpyAsync(U.data(), d_U, 8 * GB_SPLITS * (size_t)ng, cudaMemcpyDeviceToHost, ctx->st));
                CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
                for (int t = 0; t < ng; ++t)                        // the best device split
                    for (int k = 1; k < GB_SPLITS; ++k) U[t] = std::min(U[t], U[(size_t)k * ng + t]);
                // No greedy plan (nothing packed: most such calls fit nowhere):
                // U = -inf keeps only what the visit counts need -- the
                // reference's emptiness of every cell, settled by k_dp_triage
                // without frontiers.  A call that turns out feasible leaves its
                // final cell non-empty but without entries (k_backtrack: -1)
                // and is re-run unbounded below, like any too-tight bound.
                for (int t = 0; t < ng; ++t) cds[gpos[t]].U = U[t] < INFINITY ? U[t] : -INFINITY;
            }
            // PIPECUT_B200_BOUND_SCALE (tests only): scale U, below 1 forcing the
            // too-tight path (final cell empty, the call re-run unbounded)
            if (const char *sc = getenv("PIPECUT_B200_BOUND_SCALE"))
                for (int i = 0; i < n; ++i) cds[i].U *= atof(sc);
            for (int i = 0; i < n; ++i) bounded = bounded || cds[i].U < INFINITY;
            if (bounded) {
                for (int i = 0; i < n; ++i) ctx->bounded_calls += cds[i].U < INFINITY;
                CUDA_TRY(ctx, cudaMemcpyAsync(ctx->calls_d.p, cds.data(), sizeof(CallDesc) * n, cudaMemcpyHostToDevice, ctx->st));
            }
        }
    }
    float dp_ms = 0;
    bool first_pass = true;
    int vcap = 8, hcap = 4;     // pool entries reserved per cell (grown on overflow)
    bool big = false;           // four-slot (FMAX_BIG) kernels after a frontier overflow
    // PIPECUT_B200_FMAX_LIMIT (tests only): a lower capacity for the two-slot
    // kernels, so the four-slot re-run path runs on ordinary inputs
    const char *lim_env = getenv("PIPECUT_B200_FMAX_LIMIT");
    const int small_limit = lim_env ? std::max(1, std::min(FMAX, atoi(lim_env))) : FMAX;
    for (;;) {
        int64_t vpool_total = 0, hpool_total = 0, col_total = 0;
        std::vector<int64_t> col_prefix(n + 1, 0);
        for (int i = 0; i < n; ++i) {
            cds[i].col_off = col_total;
            col_total += cds[i].B;
            col_prefix[i + 1] = col_total;
            const int64_t cells = (int64_t)cds[i].A * cds[i].B;
            // pool offsets are stored in 31 bits (bit 31 = SPILL_BIT): every
            // region and spill pool is capped below 2^31 entries; a cell that
            // does not fit raises the overflow flag (never a wrapped offset)
            cds[i].vpool_base = vpool_total;
            cds[i].vpool_cap = std::min<int64_t>(cells * vcap + 64, OFF_MAX);
            vpool_total += cds[i].vpool_cap;
            cds[i].hpool_base = hpool_total;
            cds[i].hpool_cap = std::min<int64_t>(cells * cds[i].S * hcap + 64, OFF_MAX);
            hpool_total += cds[i].hpool_cap;
        }
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->calls_d.p, cds.data(), sizeof(CallDesc) * n, cudaMemcpyHostToDevice, ctx->st));
        const size_t a256 = 255;
        const size_t vmeta = ((size_t)val_cells * 5 + a256) & ~a256;      // cnt u8 + off u32
        const size_t vpool = ((size_t)vpool_total * 16 + a256) & ~a256;   // tf + tb
        const size_t hmeta = ((size_t)hist_cells * 5 + a256) & ~a256;
        // shared spill pools for calls whose frontiers outgrow their region:
        // values 4 entries per cell of the batch, history 1 per cell
        const int64_t vspill = std::min<int64_t>(std::max<int64_t>(1 << 20, 4 * val_cells) * vcap / 8, OFF_MAX);
        const int64_t hspill = std::min<int64_t>(std::max<int64_t>(1 << 22, hist_cells) * hcap / 4, OFF_MAX);
        const size_t vsp = ((size_t)vspill * 16 + a256) & ~a256;
        CUDA_TRY(ctx, ctx->val_d.ensure(2 * (vmeta + vpool + vsp) + 256));
        CUDA_TRY(ctx, ctx->hist_d.ensure(hmeta + 4 * (size_t)(hpool_total + hspill) + 512));
        CUDA_TRY(ctx, ctx->overflow_d.ensure(64 + 3 * sizeof(unsigned long long) * (size_t)n + 64));
        CUDA_TRY(ctx, ctx->colb_d.ensure(4 * sizeof(int32_t) * (size_t)col_total + 64));
        for (int par = 0; par < 2; ++par) {
            bt.col_min[par] = ctx->colb_d.as<int32_t>() + (size_t)(2 * par) * col_total;
            bt.col_max[par] = ctx->colb_d.as<int32_t>() + (size_t)(2 * par + 1) * col_total;
        }
        char *vb = ctx->val_d.as<char>();
        bt.nb = nb;
        bt.n_calls = n;
        bt.calls = ctx->calls_d.as<CallDesc>();
        bt.cta_prefix = ctx->warp_prefix_d.as<int64_t>();
        bt.cta_call = ctx->cta_call_d.as<int32_t>();
        bt.keyidx = ctx->keyidx_d.as<int16_t>();
        bt.key_tf = (const double *const *)ctx->key_ptrs.p;
        bt.key_tb = ((const double *const *)ctx->key_ptrs.p) + nk;
        bt.key_cut = ((const double *const *)ctx->key_ptrs.p) + 2 * nk;
        bt.key_ffb = ((const int32_t *const *)ctx->key_ptrs.p) + 3 * nk;
        bt.beta = P.beta;
        bt.batch_size = BS;
        bt.mono_skip = ctx->mono_skip ? 1 : 0;
        bt.num_nodes = P.num_nodes;
        bt.dpn = P.dpn;
        bt.val_cells = val_cells;
        char *ob = ctx->overflow_d.as<char>();
        bt.overflow = (int *)ob;
        unsigned long long *used = (unsigned long long *)(ob + 64);
        for (int par = 0; par < 2; ++par) {
            char *base = vb + par * (vmeta + vpool + vsp);
            bt.val_off[par] = (uint32_t *)base;
            bt.val_cnt[par] = (uint8_t *)(base + 4 * (size_t)val_cells);
            bt.pool_tf[par] = (double *)(base + vmeta);
            bt.pool_tb[par] = (double *)(base + vmeta + 8 * (size_t)vpool_total);
            bt.spill_tf[par] = (double *)(base + vmeta + vpool);
            bt.spill_tb[par] = (double *)(base + vmeta + vpool + 8 * (size_t)vspill);
            bt.vpool_used[par] = used + (size_t)par * n;
        }
        bt.vspill_cap = vspill;
        char *hb = ctx->hist_d.as<char>();
        bt.hist_off = (uint32_t *)hb;
        bt.hist_cnt = (uint8_t *)(hb + 4 * (size_t)hist_cells);
        bt.hpool = (uint32_t *)(hb + hmeta);
        bt.hspill = bt.hpool + hpool_total;
        bt.hspill_cap = hspill;
        bt.hpool_used = used + 2 * (size_t)n;
        bt.vspill_used = used + 3 * (size_t)n;
        bt.hspill_used = used + 3 * (size_t)n + 2;
        bt.hist_cells = hist_cells;
        bt.bounded = bounded ? 1 : 0;
        bt.fmax_limit = big ? FMAX_BIG : small_limit;
        int64_t *d_colpre = nullptr, *d_cellpre = nullptr;
        std::vector<int64_t> cell_prefix(n + 1, 0);
        if (bounded) {
            for (int i = 0; i < n; ++i) cell_prefix[i + 1] = cell_prefix[i] + (int64_t)cds[i].A * cds[i].B;
            CUDA_TRY(ctx, ctx->reach_d.ensure(2 * 4 * (size_t)val_cells + 16 * (size_t)(n + 1) + 64));
            bt.reach_pre[0] = ctx->reach_d.as<int32_t>();
            bt.reach_pre[1] = bt.reach_pre[0] + val_cells;
            d_colpre = (int64_t *)(((uintptr_t)(bt.reach_pre[1] + val_cells) + 15) & ~uintptr_t(15));
            d_cellpre = d_colpre + (n + 1);
            CUDA_TRY(ctx, cudaMemcpyAsync(d_colpre, col_prefix.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, ctx->st));
            CUDA_TRY(ctx, cudaMemcpyAsync(d_cellpre, cell_prefix.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, ctx->st));
            CUDA_TRY(ctx, ctx->live_d.ensure(16 * (size_t)val_cells + 20 * (size_t)col_total + 256));
            bt.live_count = ctx->live_d.as<unsigned long long>();
            bt.live = bt.live_count + 8;
            bt.live_lb = (float2 *)(bt.live + val_cells);
            bt.lvl_kk = (double2 *)(((uintptr_t)(bt.live_lb + val_cells) + 15) & ~uintptr_t(15));
            bt.lvl_kx = (short2 *)(bt.lvl_kk + col_total);
        }
        CUDA_TRY(ctx, cudaMemsetAsync(ob, 0, 64 + 3 * sizeof(unsigned long long) * (size_t)n + 64, ctx->st));
        CUDA_TRY(ctx, ctx->counters_d.ensure((8 + FMAX + 3 * WORK_SLOTS) * sizeof(unsigned long long)));
        bt.counters = ctx->counters_d.as<unsigned long long>();
        CUDA_TRY(ctx, cudaMemsetAsync(bt.counters, 0, (8 + FMAX + 3 * WORK_SLOTS) * sizeof(unsigned long long), ctx->st));
        int64_t launches = 0;
        // the reference's pruning break drops cells only when a cost table can
        // make memory non-monotone in the share (dp.cu: pruning cut)
        const bool cut = pruning && ctx->has_cost_table;
        int64_t *cut_rows = nullptr, *cut_cols = nullptr;
        int32_t *row_e = nullptr;
        std::vector<int64_t> row_prefix(n + 1, 0);
        if (cut) {
            for (int i = 0; i < n; ++i) row_prefix[i + 1] = row_prefix[i] + cds[i].A;
            CUDA_TRY(ctx, ctx->cut_d.ensure(16 * (size_t)(n + 1) + 4 * (size_t)row_prefix[n] + 64));
            cut_rows = ctx->cut_d.as<int64_t>();
            cut_cols = cut_rows + (n + 1);
            row_e = (int32_t *)(cut_cols + (n + 1));
            CUDA_TRY(ctx, cudaMemcpyAsync(cut_rows, row_prefix.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, ctx->st));
            CUDA_TRY(ctx, cudaMemcpyAsync(cut_cols, col_prefix.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, ctx->st));
        }
        // PIPECUT_B200_LEVELS: per-level kernel time (debug; one event pair per level)
        const bool level_times = getenv("PIPECUT_B200_LEVELS") != nullptr;
        std::vector<cudaEvent_t> lev_ev;
        if (level_times) {
            lev_ev.resize(maxS + 1);
            for (auto &e : lev_ev) cudaEventCreate(&e);
            cudaEventRecord(lev_ev[0], ctx->st);
        }
        // PIPECUT_B200_DEEP_LEVELS (tests): the level count from which the
        // 10-CTA list kernel runs
        const char *deep_env = getenv("PIPECUT_B200_DEEP_LEVELS");
        const int deep_levels = deep_env ? atoi(deep_env) : DP_DEEP_LEVELS;
        for (int s = 1; s <= maxS; ++s) {
            int n_active = 0;
            while (n_active < n && cds[n_active].S >= s) ++n_active;
            CUDA_TRY(ctx, cudaMemsetAsync(bt.vpool_used[s & 1], 0, sizeof(unsigned long long) * n_active, ctx->st));
            CUDA_TRY(ctx, cudaMemsetAsync(bt.vspill_used + (s & 1), 0, sizeof(unsigned long long), ctx->st));
            CUDA_TRY(ctx, cudaMemsetAsync(bt.col_min[s & 1], 0x7f, sizeof(int32_t) * col_prefix[n_active], ctx->st));
            CUDA_TRY(ctx, cudaMemsetAsync(bt.col_max[s & 1], 0xff, sizeof(int32_t) * col_prefix[n_active], ctx->st));
            if (bounded) {
                // settle the cells above the bound by a thread each, then a
                // persistent grid of warps over the live ones (dp.cu)
                CUDA_TRY(ctx, cudaMemsetAsync(bt.live_count, 0, 2 * sizeof(unsigned long long), ctx->st));
                launch_level_factors(bt, s, n_active, col_prefix[n_active], d_colpre, ctx->st);
                launch_dp_triage(bt, s, n_active, cell_prefix[n_active], d_cellpre, ctx->derived, ctx->st);
                launch_dp_level_list(bt, s, ctx->sm_count, maxS >= deep_levels, ctx->derived, big, ctx->st);
                ctx->launches += 3;
            } else {
                launch_dp_level(bt, s, n_active, cta_prefix[n_active], ctx->derived, big, ctx->st);
                ctx->launches++;
            }
            ++launches;
            if (bounded && s < maxS) {
                launch_reach_prefix(bt, s, n_active, col_prefix[n_active], d_colpre, ctx->st);
                ctx->launches++;
            }
            if (cut)
                ctx->launches += launch_prune_cut(bt, s, n_active, row_prefix[n_active], col_prefix[n_active],
                                                  cut_rows, cut_cols, row_e, ctx->st);
            if (level_times) cudaEventRecord(lev_ev[s], ctx->st);
        }
        if (level_times) {
            cudaEventSynchronize(lev_ev[maxS]);
            const int edges[] = {1, 2, 9, 33, 65, 129, 249, maxS + 1};
            fprintf(stderr, "[pipecut_b200] level times:");
            for (int e = 0; e + 1 < 8; ++e) {
                float tot = 0;
                int s0 = edges[e], s1 = std::min(edges[e + 1], maxS + 1);
                for (int s = s0; s < s1; ++s) {
                    float ms = 0;
                    cudaEventElapsedTime(&ms, lev_ev[s - 1], lev_ev[s]);
                    tot += ms;
                }
                if (s1 > s0) fprintf(stderr, " s%d-%d %.1fms", s0, s1 - 1, tot);
            }
            fprintf(stderr, "\n");
            for (auto &e : lev_ev) cudaEventDestroy(e);
        }
        if (int rc = check_launch(ctx, "dp_level")) return rc;
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev2, ctx->st));
        int ovf = 0;
        unsigned long long cnt[8 + FMAX + 3 * WORK_SLOTS] = {0};
        CUDA_TRY(ctx, cudaMemcpyAsync(&ovf, bt.overflow, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(cnt, bt.counters, sizeof(cnt), cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        for (int q = 0; q < WORK_SLOTS; ++q)
            for (int j = 0; j < 3; ++j) cnt[j] += cnt[8 + FMAX + 3 * q + j];
        ctx->last_pairs += (int64_t)cnt[0];
        ctx->last_cands += (int64_t)cnt[1];
        ctx->last_inserts += (int64_t)cnt[2];
        if (getenv("PIPECUT_B200_DEBUG")) {
            fprintf(stderr, "[pipecut_b200] batch: %d calls, pairs %llu cands %llu inserts %llu ovf %d vcap %d hcap %d\n  frontier sizes:",
                    n, cnt[0], cnt[1], cnt[2], ovf, vcap, hcap);
            for (int q = 0; q <= FMAX; ++q)
                if (cnt[3 + q]) fprintf(stderr, " %d:%llu", q, cnt[3 + q]);
            fprintf(stderr, "\n  warp rounds %llu, warp iterations %llu, corner-pruned pairs %llu, window entries %llu\n",
                    cnt[4 + FMAX], cnt[5 + FMAX], cnt[6 + FMAX], cnt[7 + FMAX]);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev1, ctx->ev2);
        dp_ms += ms;
        if (first_pass) {
            float sms = 0;
            cudaEventElapsedTime(&sms, ctx->ev0, ctx->ev1);
            ctx->last_span_ms += sms;
            first_pass = false;
        }
        ctx->last_dp_launches += launches;
        if (ovf & 1) {
            // a cell outgrew the frontier capacity: re-run the pass with the
            // four-slot kernels (126 entries, never truncated); beyond that
            // the call is refused
            if (big) return fail(ctx, PC_ERR_CAPACITY, "a Pareto frontier exceeded 126 entries");
            big = true;
            ctx->frontier_reruns += n;
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->st));
            continue;
        }
        if (!ovf) break;
        // a pool region ran out: grow and rerun the batch.  With FMAX_BIG
        // entries reserved per cell every frontier fits its region unless the
        // 31-bit offset cap clipped it: then the batch is beyond the offset range.
        if (vcap >= FMAX_BIG && hcap >= FMAX_BIG)
            return fail(ctx, PC_ERR_CAPACITY, "frontier pools beyond the 31-bit offset range");
        vcap *= 2;
        hcap *= 2;
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->st));
    }
    ctx->last_dp_ms += dp_ms;
    if (getenv("PIPECUT_B200_BOUND_DEBUG"))
        fprintf(stderr, "[pipecut_b200] chunk: %d calls, MB %d..%d, bounded %d, dp %.1f ms\n", n,
                cds[0].MB, cds[n - 1].MB, (int)bounded, dp_ms);

    // ---- visits per (call, level)
    std::vector<int64_t> level_off(n + 1, 0), row_prefix(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        level_off[i + 1] = level_off[i] + cds[i].S;
        row_prefix[i + 1] = row_prefix[i] + (int64_t)cds[i].S * cds[i].A;
    }
    CUDA_TRY(ctx, ctx->level_off_d.ensure(sizeof(int64_t) * (n + 1)));
    CUDA_TRY(ctx, ctx->row_prefix_d.ensure(sizeof(int64_t) * (n + 1)));
    CUDA_TRY(ctx, ctx->level_sums_d.ensure(sizeof(int64_t) * level_off[n] + 8));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->level_off_d.p, level_off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->row_prefix_d.p, row_prefix.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->level_sums_d.p, 0, sizeof(int64_t) * level_off[n], ctx->st));
    launch_row_visits(bt, pruning, ctx->level_sums_d.as<int64_t>(), ctx->row_prefix_d.as<int64_t>(),
                      ctx->level_off_d.as<int64_t>(), row_prefix[n], ctx->st);
    ctx->launches += 2;
    if (int rc = check_launch(ctx, "visits")) return rc;

    // ---- backtrack (plan offsets in sorted order, compact)
    std::vector<int32_t> plan_off_orig(calls.size(), 0);
    int32_t seg_total = 0;
    for (int i = 0; i < n; ++i) {
        plan_off_orig[cds[i].orig] = seg_total;
        seg_total += cds[i].S;
    }
    CUDA_TRY(ctx, ctx->plan_off_d.ensure(sizeof(int32_t) * calls.size()));
    CUDA_TRY(ctx, ctx->seg_d.ensure(sizeof(int32_t) * 3 * (size_t)seg_total + 16));
    CUDA_TRY(ctx, ctx->objective_d.ensure(sizeof(double) * calls.size()));
    CUDA_TRY(ctx, ctx->feasible_d.ensure(sizeof(int32_t) * calls.size()));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->plan_off_d.p, plan_off_orig.data(), sizeof(int32_t) * calls.size(), cudaMemcpyHostToDevice, ctx->st));
    int32_t *seg = ctx->seg_d.as<int32_t>();
    launch_backtrack(bt, BS, ctx->plan_off_d.as<int32_t>(), seg, seg + seg_total, seg + 2 * seg_total,
                     ctx->objective_d.as<double>(), ctx->feasible_d.as<int32_t>(), ctx->st);
    ctx->launches++;
    if (int rc = check_launch(ctx, "backtrack")) return rc;
    std::vector<int64_t> level_sums(level_off[n]);
    std::vector<int32_t> segs(3 * (size_t)seg_total), feas(calls.size(), 0);
    std::vector<double> objs(calls.size(), NAN);
    CUDA_TRY(ctx, cudaMemcpyAsync(level_sums.data(), ctx->level_sums_d.p, sizeof(int64_t) * level_off[n], cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(segs.data(), seg, sizeof(int32_t) * 3 * (size_t)seg_total, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(feas.data(), ctx->feasible_d.p, sizeof(int32_t) * calls.size(), cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(objs.data(), ctx->objective_d.p, sizeof(double) * calls.size(), cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    // a bound below the optimum leaves the final cell with no entry although
    // the reference holds it non-empty (k_backtrack: -1); a partner plan cannot
    // do that, but such calls are re-run unbounded rather than trusted
    std::vector<int> retry;
    for (int i = 0; i < n; ++i)
        if (feas[cds[i].orig] < 0) {
            feas[cds[i].orig] = 0;
            retry.push_back(cds[i].orig);
        }

    // ---- stage records + simulation for feasible calls
    std::vector<int32_t> qlo, qhi, qck, poff, pS, pR, pMB;
    std::vector<int64_t> qm;
    std::vector<int> feas_orig;
    int maxS_f = 1;
    for (int i = 0; i < n; ++i) {
        const int o = cds[i].orig;
        if (!feas[o]) continue;
        feas_orig.push_back(o);
        poff.push_back((int32_t)qlo.size());
        pS.push_back(cds[i].S);
        pR.push_back(cds[i].R);
        pMB.push_back(cds[i].MB);
        maxS_f = std::max(maxS_f, cds[i].S);
        const int32_t off = plan_off_orig[o];
        for (int k = 0; k < cds[i].S; ++k) {
            const int32_t dev = segs[2 * (size_t)seg_total + off + k];
            qlo.push_back(segs[off + k]);
            qhi.push_back(segs[(size_t)seg_total + off + k]);
            qm.push_back(BS / ((int64_t)cds[i].MB * cds[i].R * dev));
            qck.push_back(cds[i].ckpt);
        }
    }
    const int nq = (int)qlo.size();
    const int np = (int)feas_orig.size();
    std::vector<double> qtf(nq), qtb(nq), iters(np, NAN);
    std::vector<int64_t> qmem(nq);
    if (nq > 0) {
        // inputs: lo hi ck poff pS pR pMB (int32), m (int64); outputs tf tb (f64) mem (i64) iter (f64)
        size_t in_bytes = 4 * ((size_t)3 * nq + 4 * (size_t)np) + 8 * (size_t)nq + 64;
        size_t out_bytes = 8 * (3 * (size_t)nq + (size_t)np) + 64;
        CUDA_TRY(ctx, ctx->q_d.ensure(in_bytes));
        CUDA_TRY(ctx, ctx->q_out_d.ensure(out_bytes));
        char *qb = ctx->q_d.as<char>();
        int64_t *d_m = (int64_t *)qb;
        int32_t *d_lo = (int32_t *)(qb + 8 * (size_t)nq);
        int32_t *d_hi = d_lo + nq;
        int32_t *d_ck = d_hi + nq;
        int32_t *d_poff = d_ck + nq;
        int32_t *d_S = d_poff + np;
        int32_t *d_R = d_S + np;
        int32_t *d_MB = d_R + np;
        double *o_tf = ctx->q_out_d.as<double>();
        double *o_tb = o_tf + nq;
        int64_t *o_mem = (int64_t *)(o_tb + nq);
        double *o_it = (double *)(o_mem + nq);
        CUDA_TRY(ctx, cudaMemcpyAsync(d_m, qm.data(), 8 * (size_t)nq, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_lo, qlo.data(), 4 * (size_t)nq, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_hi, qhi.data(), 4 * (size_t)nq, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_ck, qck.data(), 4 * (size_t)nq, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_poff, poff.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_S, pS.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_R, pR.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(d_MB, pMB.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, ctx->st));
        launch_profile_queries(P, nq, d_lo, d_hi, d_m, d_ck, o_tf, o_tb, o_mem, ctx->st);
        ctx->launches++;
        if (int rc = check_launch(ctx, "profile_queries")) return rc;
        if (want_iter) {
            // seg_dev of the compact layout: rebuild from queries' m? use a device copy
            std::vector<int32_t> qdev(nq);
            for (int pi = 0, q = 0; pi < np; ++pi) {
                const int o = feas_orig[pi];
                const int32_t off = plan_off_orig[o];
                for (int k = 0; k < pS[pi]; ++k, ++q) qdev[q] = segs[2 * (size_t)seg_total + off + k];
            }
            CUDA_TRY(ctx, ctx->sim_d.ensure(4 * (size_t)nq + 16));
            CUDA_TRY(ctx, cudaMemcpyAsync(ctx->sim_d.p, qdev.data(), 4 * (size_t)nq, cudaMemcpyHostToDevice, ctx->st));
            launch_simulate(P, np, d_poff, d_S, d_R, d_MB, BS, d_lo, d_hi, ctx->sim_d.as<int32_t>(),
                            o_tf, o_tb, o_it, ctx->st, maxS_f);
            ctx->launches++;
            if (int rc = check_launch(ctx, "simulate")) return rc;
            CUDA_TRY(ctx, cudaMemcpyAsync(iters.data(), o_it, 8 * (size_t)np, cudaMemcpyDeviceToHost, ctx->st));
            CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
        }
        CUDA_TRY(ctx, cudaMemcpyAsync(qtf.data(), o_tf, 8 * (size_t)nq, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(qtb.data(), o_tb, 8 * (size_t)nq, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaMemcpyAsync(qmem.data(), o_mem, 8 * (size_t)nq, cudaMemcpyDeviceToHost, ctx->st));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    }

    // everything after the DP levels (ev2: end of the last DP pass)
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev3, ctx->st));
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev3));
    {
        float pms = 0;
        cudaEventElapsedTime(&pms, ctx->ev2, ctx->ev3);
        ctx->last_post_ms += pms;
    }

    // ---- fill outputs
    std::vector<int> fpos(calls.size(), -1);
    for (int pi = 0; pi < np; ++pi) fpos[feas_orig[pi]] = pi;
    for (int i = 0; i < n; ++i) {
        const CallDesc &cd = cds[i];
        const int o = cd.orig;
        CallOut &out = outs[o];
        out.level_sums.assign(level_sums.begin() + level_off[i], level_sums.begin() + level_off[i + 1]);
        out.visits = 0;
        for (auto v : out.level_sums) out.visits += v;
        out.visits_unpruned = (int64_t)cd.S * tri_sum(cd.A) * tri_sum(cd.B);
        out.bound = cd.U;
        out.feasible = feas[o];
        out.lo.clear(); out.hi.clear(); out.dev.clear(); out.tf.clear(); out.tb.clear(); out.mem.clear();
        if (feas[o]) {
            const int pi = fpos[o];
            out.objective = objs[o];
            out.iteration = iters[pi];
            const int32_t off = plan_off_orig[o];
            for (int k = 0; k < cd.S; ++k) {
                out.lo.push_back(segs[off + k]);
                out.hi.push_back(segs[(size_t)seg_total + off + k]);
                out.dev.push_back(segs[2 * (size_t)seg_total + off + k]);
                out.tf.push_back(qtf[poff[pi] + k]);
                out.tb.push_back(qtb[poff[pi] + k]);
                out.mem.push_back(qmem[poff[pi] + k]);
            }
        }
    }
    if (getenv("PIPECUT_B200_BOUND_DEBUG"))
        for (int i = 0; i < n; ++i) {
            const CallOut &o = outs[cds[i].orig];
            if (o.feasible)
                fprintf(stderr, "[pipecut_b200]   S %d D %d R %d MB %d: U/opt %.4f\n", cds[i].S,
                        cds[i].D, cds[i].R, cds[i].MB, o.bound / o.objective);
        }
    ctx->last_calls = cds;
    ctx->last_batch = bt;
    ctx->last_pruning = pruning;
    ctx->last_pos.assign(calls.size(), -1);
    for (int i = 0; i < n; ++i) ctx->last_pos[cds[i].orig] = i;
    if (!retry.empty()) {
        for (int o : retry) {
            if (!ctx->bb_partner.empty()) ctx->bb_partner[o] = -1;
            if (!ctx->bb_U.empty()) ctx->bb_U[o] = INFINITY;
        }
        ctx->bound_reruns += (int64_t)retry.size();
        ctx->bb_off = true;                       // the re-run is unbounded
        const int rc = run_chunk(ctx, calls, retry, BS, pruning, want_iter, outs);
        ctx->bb_off = false;
        return rc;
    }
    return PC_OK;
}

// Memory-bounded batching: consecutive calls (list order) are grouped while
// their level buffers fit in half of the free device memory.
static int run_calls_impl(pc_ctx *ctx, const std::vector<pc_call> &calls, int64_t BS, int pruning,
                          int want_iter, std::vector<CallOut> &outs, int *n_chunks) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    for (auto &c : calls)
        if (int rc = validate_call(ctx, c, BS)) return rc;
    outs.assign(calls.size(), CallOut());
    ctx->last_dp_ms = 0;
    ctx->last_span_ms = 0;
    ctx->last_post_ms = 0;
    ctx->last_dp_launches = 0;
    ctx->last_pairs = 0;
    ctx->last_cands = 0;
    ctx->last_inserts = 0;
    ctx->launches = 0;
    // free device memory bounds the batch (chunks below).  cudaMemGetInfo
    // itself sporadically stalls for 5-40 ms (measured on the pool's boxes:
    // the C1-C4 latencies' outliers, and up to ~25 ms of a headline step), so
    // a batch well below the last reading (under a quarter: 4096 x 256's
    // estimate is 22 GB) reuses it; only a batch that could come near it
    // queries again.
    size_t est = 0;
    for (auto &c : calls) {
        const int64_t A = ctx->nb - c.S + 1, B = c.D - c.S + 1;
        est += (size_t)A * B * (2 * (5 + 16 * 12) + (size_t)c.S * (5 + 4 * 5));
    }
    if (ctx->mem_free == 0 || est > ctx->mem_free / 4) {
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        ctx->mem_free = free_b;
    }
    const size_t cap = ctx->mem_free / 2;
    // Objective bound (dp.cu): every call of the batch gets U from a greedy
    // plan (k_greedy_bound; within 1% of the optimum at the median on the C5
    // chains).  PIPECUT_B200_BOUND_WAVES=1 instead runs the calls in waves of
    // equal MB, ascending, and bounds a call by its (S, D, R, MB/2) partner's
    // optimal plan -- still a valid plan at half the share: memory only
    // shrinks -- measured slower (12 sequential batches: 1.43 s vs 1.21 s of DP
    // on 4096 x 256, r2j).  Results are the same either way;
    // PIPECUT_B200_NO_BOUND=1 turns the bound off.
    // Small batches skip it: the waves' extra launches and the greedy plans
    // cost more than the bound saves below ~2e8 closed-form visits (r2cj sweep:
    // nb = 256 searches 3x faster bounded, nb = 64 ones 0.5 ms slower; the
    // floor was 2e10 before calls without a greedy plan were bounded at -inf).
    double batch_visits = 0;
    for (auto &c : calls) {
        const double A = ctx->nb - c.S + 1, B = c.D - c.S + 1;
        batch_visits += (double)c.S * A * (A + 1) / 2 * B * (B + 1) / 2;
    }
    // (PIPECUT_B200_BOUND_MIN_VISITS overrides the size floor: the parity suite
    // runs once with 0 so every eligible batch of its families is bounded)
    const char *floor_env = getenv("PIPECUT_B200_BOUND_MIN_VISITS");
    const double min_visits = floor_env ? atof(floor_env) : BOUND_MIN_VISITS;
    const bool bound_ok = !ctx->has_cost_table && ctx->mono_skip && ctx->bb_U.empty() &&
                          batch_visits >= min_visits &&
                          getenv("PIPECUT_B200_NO_BOUND") == nullptr;
    std::vector<int> seq(calls.size());
    for (size_t i = 0; i < calls.size(); ++i) seq[i] = (int)i;
    ctx->bb_partner.clear();
    const bool waves = bound_ok && getenv("PIPECUT_B200_BOUND_WAVES") != nullptr;
    if (bound_ok && !waves) ctx->bb_partner.assign(calls.size(), -1);   // greedy bounds only
    if (waves) {
        std::map<std::array<int, 4>, int> where;
        for (size_t i = 0; i < calls.size(); ++i)
            where[std::array<int, 4>{calls[i].S, calls[i].D, calls[i].R, calls[i].MB}] = (int)i;
        ctx->bb_partner.assign(calls.size(), -1);
        for (size_t i = 0; i < calls.size(); ++i) {
            const pc_call &c = calls[i];
            if (c.MB % 2) continue;
            auto it = where.find(std::array<int, 4>{c.S, c.D, c.R, c.MB / 2});
            if (it != where.end()) ctx->bb_partner[i] = it->second;
        }
        std::stable_sort(seq.begin(), seq.end(),
                         [&](int a, int b) { return calls[a].MB < calls[b].MB; });
    }
    std::vector<int> cur;
    size_t cur_bytes = 0;
    int64_t cur_hist = 0;
    *n_chunks = 0;
    for (int i : seq) {
        const pc_call &c = calls[i];
        const int64_t A = ctx->nb - c.S + 1, B = c.D - c.S + 1;
        const size_t bytes = (size_t)A * B * (2 * (5 + 16 * 12) + (size_t)c.S * (5 + 4 * 5));
        const int64_t hist = A * B * c.S;
        const bool new_wave = waves && !cur.empty() && calls[cur.back()].MB != c.MB;
        if (!cur.empty() && (new_wave || cur_bytes + bytes > cap || cur_hist + hist > CHUNK_HIST_CELLS)) {
            if (int rc = run_chunk(ctx, calls, cur, BS, pruning, want_iter, outs)) return rc;
            ++*n_chunks;
            cur.clear();
            cur_bytes = 0;
            cur_hist = 0;
        }
        cur.push_back(i);
        cur_bytes += bytes;
        cur_hist += hist;
    }
    if (!cur.empty()) {
        if (int rc = run_chunk(ctx, calls, cur, BS, pruning, want_iter, outs)) return rc;
        ++*n_chunks;
    }
    // PIPECUT_B200_BB_ORACLE (measurement only): rerun the calls with each
    // call's own optimum as the bound and report both DP times
    if (getenv("PIPECUT_B200_BB_ORACLE") && ctx->bb_U.empty() && !ctx->has_cost_table && ctx->mono_skip) {
        const double dp0 = ctx->last_dp_ms;
        std::vector<CallOut> first = outs;
        ctx->bb_U.assign(calls.size(), -INFINITY);     // infeasible: reachability only
        for (size_t i = 0; i < calls.size(); ++i)
            if (first[i].feasible) ctx->bb_U[i] = first[i].objective;
        ctx->last_dp_ms = 0;
        int ch = 0;
        int rc = run_calls_impl(ctx, calls, BS, pruning, want_iter, outs, &ch);
        ctx->bb_U.clear();
        if (rc) return rc;
        int bad = 0;
        for (size_t i = 0; i < calls.size(); ++i)
            if (first[i].feasible != outs[i].feasible || (first[i].feasible &&
                (first[i].objective != outs[i].objective || first[i].lo != outs[i].lo ||
                 first[i].dev != outs[i].dev || first[i].iteration != outs[i].iteration)))
                ++bad;
        fprintf(stderr, "[pipecut_b200] bound oracle: %zu calls, dp %.1f ms -> %.1f ms, %d mismatches\n",
                calls.size(), dp0, ctx->last_dp_ms, bad);
    }
    return PC_OK;
}

// Exact visits at the first cell where the running count exceeds budget,
// scanning call `orig` of the last chunk in the reference order
// (stages.py:212-216).  Returns -1 if the budget is not crossed in it.
static int64_t crossing_in_call(pc_ctx *ctx, int orig, int64_t before, int64_t budget) {
    if (orig < 0 || orig >= (int)ctx->last_pos.size() || ctx->last_pos[orig] < 0) return -2;
    const CallDesc cd = ctx->last_calls[ctx->last_pos[orig]];
    const int64_t cells = (int64_t)cd.A * cd.B;
    std::vector<uint8_t> flags((size_t)cells * cd.S);
    if (cudaMemcpy(flags.data(), ctx->last_batch.hist_cnt + cd.hist_off, flags.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -3;
    int64_t run = before;
    int d_min = 1;
    for (int s = 1; s <= cd.S; ++s) {
        if (s > 1) d_min = 1;
        const uint8_t *lvl = flags.data() + (size_t)(s - 1) * cells;
        for (int bi = 0; bi < cd.A; ++bi) {
            const int b = s + bi;
            const int bottom = std::max(d_min, s);
            for (int d = cd.D - (cd.S - s); d >= bottom; --d) {
                run += (int64_t)(b - s + 1) * (d - s + 1);
                if (run > budget) return run;
                const uint8_t v = lvl[(size_t)(d - s) * cd.A + bi];
                if ((v & CNT_MASK) == 0 && ctx->last_pruning && !(v & CNT_ZERO)) {
                    if (s == 1) d_min = d + 1;
                    break;
                }
            }
        }
    }
    return -1;
}

static void fill_plan(const CallOut &o, const pc_call &c, pc_plan *plan) {
    plan->S = c.S;
    plan->D = c.D;
    plan->R = c.R;
    plan->MB = c.MB;
    plan->objective = o.objective;
    plan->iteration_time = o.iteration;
    plan->n_stages = o.feasible ? (int32_t)o.lo.size() : 0;
    if (!o.feasible) return;
    for (size_t k = 0; k < o.lo.size() && (int)k < plan->cap_stages; ++k) {
        plan->lo[k] = o.lo[k];
        plan->hi[k] = o.hi[k];
        plan->devices[k] = o.dev[k];
        plan->t_fwd[k] = o.tf[k];
        plan->t_bwd[k] = o.tb[k];
        plan->mem[k] = o.mem[k];
    }
}

static void fill_stats(pc_ctx *ctx, pc_stats *stats, int64_t visits, int64_t calls, int64_t unpruned,
                       int64_t cells) {
    if (!stats) return;
    stats->visits = visits;
    stats->dp_calls = calls;
    stats->visits_unpruned = unpruned;
    stats->cells = cells;
    stats->pairs = ctx->last_pairs;
    stats->candidates = ctx->last_cands;
    stats->dp_launches = ctx->last_dp_launches;
    stats->kernel_launches = ctx->launches;
    stats->device_ms = ctx->last_dp_ms;
    stats->span_ms = ctx->last_span_ms;
    stats->post_ms = ctx->last_post_ms;
}

// =========================================================================== entry points
extern "C" int pc_form_stage_dp(pc_ctx *ctx, int32_t S, int32_t D, int64_t batch_size, int32_t R,
                                int32_t MB, int32_t disable_pruning, int64_t visit_budget,
                                pc_plan *plan, pc_stats *stats) {
    ctx->bounded_calls = ctx->bound_reruns = ctx->frontier_reruns = 0;
    std::vector<pc_call> calls = {{S, D, R, MB}};
    if (plan && S > plan->cap_stages && S <= ctx->nb) return fail(ctx, PC_ERR_CAPACITY, "plan capacity");
    std::vector<CallOut> outs;
    int chunks = 0;
    if (int rc = run_calls_impl(ctx, calls, batch_size, !disable_pruning, 0, outs, &chunks)) return rc;
    const CallOut &o = outs[0];
    const int64_t cells = (int64_t)S * (ctx->nb - S + 1) * (D - S + 1);
    if (visit_budget >= 0 && o.visits > visit_budget) {
        const int64_t cross = crossing_in_call(ctx, 0, 0, visit_budget);
        if (cross < 0) return fail(ctx, PC_ERR_CUDA, "budget crossing not found");
        fill_stats(ctx, stats, cross, 1, o.visits_unpruned, cells);
        return PC_ERR_BUDGET;
    }
    fill_stats(ctx, stats, o.visits, 1, o.visits_unpruned, cells);
    if (plan) fill_plan(o, calls[0], plan);
    return o.feasible ? PC_OK : PC_INFEASIBLE;
}

extern "C" int pc_run_calls(pc_ctx *ctx, int32_t n, const pc_call *calls, int64_t batch_size,
                            int32_t disable_pruning, int32_t want_iteration,
                            pc_call_result *results, pc_plan *plans, pc_stats *stats) {
    ctx->bounded_calls = ctx->bound_reruns = ctx->frontier_reruns = 0;
    std::vector<pc_call> cv(calls, calls + n);
    std::vector<CallOut> outs;
    int chunks = 0;
    if (int rc = run_calls_impl(ctx, cv, batch_size, !disable_pruning, want_iteration, outs, &chunks)) return rc;
    int64_t vis = 0, unp = 0, cells = 0;
    for (int i = 0; i < n; ++i) {
        const CallOut &o = outs[i];
        results[i].feasible = o.feasible;
        results[i].n_stages = o.feasible ? cv[i].S : 0;
        results[i].objective = o.objective;
        results[i].iteration_time = o.iteration;
        results[i].visits = o.visits;
        results[i].visits_unpruned = o.visits_unpruned;
        results[i].budget_cross = -1;
        if (plans) fill_plan(o, cv[i], &plans[i]);
        vis += o.visits;
        unp += o.visits_unpruned;
        cells += (int64_t)cv[i].S * (ctx->nb - cv[i].S + 1) * (cv[i].D - cv[i].S + 1);
    }
    fill_stats(ctx, stats, vis, n, unp, cells);
    return PC_OK;
}

// Budget crossing inside call `index` of the last pc_run_calls.  Only the
// last chunk's flags are kept: -2 when the call ran in an earlier chunk (the
// caller re-runs it alone and asks again).
extern "C" int pc_last_crossing(pc_ctx *ctx, int32_t index, int64_t visits_before, int64_t budget,
                                int64_t *visits_at_cross) {
    int64_t r = crossing_in_call(ctx, index, visits_before, budget);
    *visits_at_cross = r;
    return r >= -2 ? PC_OK : fail(ctx, PC_ERR_CUDA, "reading the visit flags failed");
}

extern "C" int pc_form_stage(pc_ctx *ctx, int32_t N, int32_t dpn, int64_t BS, int32_t disable_pruning,
                             int64_t visit_budget, int32_t speculative, pc_plan *plan, pc_stats *stats) {
    ctx->bounded_calls = ctx->bound_reruns = ctx->frontier_reruns = 0;
    if (N < 1 || dpn < 1 || BS < 1)
        return fail(ctx, PC_ERR_INVALID, "node count, devices per node and batch size must be at least 1");
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    const int nb = ctx->nb;
    // enumeration in the reference's order (stages.py:389-403)
    std::vector<pc_call> calls;
    std::vector<int> level_of;
    std::vector<int> level_n;
    for (int n = 1; n <= N; n *= 2) {
        if (N % n) continue;
        const int D = dpn * n, R = N / n;
        const int lv = (int)level_n.size();
        level_n.push_back(n);
        for (int S = dpn * (n - 1) + 1; S <= D; ++S) {
            if (S > nb) continue;
            for (int64_t MB = 1; MB * R <= BS; MB *= 2) {
                calls.push_back({S, D, R, (int32_t)MB});
                level_of.push_back(lv);
            }
        }
    }
    const int n_levels = (int)level_n.size();
    int64_t running = 0, calls_counted = 0, unpruned = 0, cells = 0;
    int best = -1;
    std::vector<CallOut> outs_all(calls.size());
    auto process_level = [&](int lv, const std::vector<CallOut> &outs, const std::vector<int> &map) -> int {
        // map: call index (global) -> index in outs
        int lvl_best = -1;
        for (size_t ci = 0; ci < calls.size(); ++ci) {
            if (level_of[ci] != lv) continue;
            const CallOut &o = outs[map[ci]];
            ++calls_counted;
            unpruned += o.visits_unpruned;
            cells += (int64_t)calls[ci].S * (nb - calls[ci].S + 1) * (calls[ci].D - calls[ci].S + 1);
            if (visit_budget >= 0 && running + o.visits > visit_budget) {
                int64_t cross = crossing_in_call(ctx, map[ci], running, visit_budget);
                if (cross < -1) {
                    // flags of an earlier chunk are gone: recompute this call alone
                    std::vector<pc_call> one = {calls[ci]};
                    std::vector<CallOut> o1;
                    int ch = 0;
                    if (int rc = run_calls_impl(ctx, one, BS, !disable_pruning, 0, o1, &ch)) return rc;
                    cross = crossing_in_call(ctx, 0, running, visit_budget);
                }
                if (cross < 0) return fail(ctx, PC_ERR_CUDA, "budget crossing not found");
                fill_stats(ctx, stats, cross, calls_counted, unpruned, cells);
                return PC_ERR_BUDGET;
            }
            running += o.visits;
            if (!o.feasible) continue;
            if (lvl_best < 0) {
                lvl_best = (int)ci;
                continue;
            }
            // min by (iteration_time, objective, microbatches), first wins (stages.py:407-411)
            const CallOut &b = outs[map[lvl_best]];
            const bool better = o.iteration < b.iteration ||
                                (o.iteration == b.iteration &&
                                 (o.objective < b.objective ||
                                  (o.objective == b.objective && calls[ci].MB < calls[lvl_best].MB)));
            if (better) lvl_best = (int)ci;
        }
        best = lvl_best;
        return PC_OK;
    };
    int chunks = 0;
    if (speculative == 1) {
        std::vector<CallOut> outs;
        if (int rc = run_calls_impl(ctx, calls, BS, !disable_pruning, 1, outs, &chunks)) return rc;
        if (chunks > 1 && visit_budget >= 0) {
            // crossing lookups need the flags resident: fall back to per-level batches
            speculative = 0;
        } else {
            std::vector<int> map(calls.size());
            std::iota(map.begin(), map.end(), 0);
            for (int lv = 0; lv < n_levels; ++lv) {
                if (int rc = process_level(lv, outs, map)) return rc;
                if (best >= 0) {
                    fill_stats(ctx, stats, running, calls_counted, unpruned, cells);
                    if (plan) fill_plan(outs[best], calls[best], plan);
                    return PC_OK;
                }
            }
            fill_stats(ctx, stats, running, calls_counted, unpruned, cells);
            if (plan) plan->n_stages = 0;
            return PC_INFEASIBLE;
        }
    }
    running = calls_counted = unpruned = cells = 0;
    double dp_ms = 0, span_ms = 0, post_ms = 0;
    int64_t pairs = 0, cands = 0, launches = 0;
    // batches of widening levels: one per level (0), or adaptive (2): the first
    // level alone (it is usually feasible), then later levels grouped while a
    // group stays under LEVEL_GROUP_VISITS closed-form visits -- small levels
    // gain from one batch, large ones from stopping at the first feasible level
    // (tools/form_stage_modes.py: C4 3.7 vs 4.8 ms per level; 4096 x 256 184 ms
    // per level vs 839 ms for the first level and then all the rest)
    std::vector<std::pair<int, int>> groups;
    if (speculative == 2) {
        constexpr double LEVEL_GROUP_VISITS = 2e9;
        std::vector<double> lv_visits(n_levels, 0.0);
        for (size_t ci = 0; ci < calls.size(); ++ci) {
            const double A = nb - calls[ci].S + 1, Bc = calls[ci].D - calls[ci].S + 1;
            lv_visits[level_of[ci]] += (double)calls[ci].S * A * (A + 1) / 2 * Bc * (Bc + 1) / 2;
        }
        if (n_levels > 0) groups.push_back({0, 1});
        int lv = 1;
        while (lv < n_levels) {
            int end = lv + 1;
            double acc = lv_visits[lv];
            while (end < n_levels && acc + lv_visits[end] < LEVEL_GROUP_VISITS) acc += lv_visits[end++];
            groups.push_back({lv, end});
            lv = end;
        }
    } else {
        for (int lv = 0; lv < n_levels; ++lv) groups.push_back({lv, lv + 1});
    }
    for (const auto &grp : groups) {
        std::vector<pc_call> sub;
        std::vector<int> map(calls.size(), -1);
        for (size_t ci = 0; ci < calls.size(); ++ci)
            if (level_of[ci] >= grp.first && level_of[ci] < grp.second) {
                map[ci] = (int)sub.size();
                sub.push_back(calls[ci]);
            }
        if (sub.empty()) continue;
        std::vector<CallOut> outs;
        if (int rc = run_calls_impl(ctx, sub, BS, !disable_pruning, 1, outs, &chunks)) return rc;
        dp_ms += ctx->last_dp_ms;
        span_ms += ctx->last_span_ms;
        post_ms += ctx->last_post_ms;
        pairs += ctx->last_pairs;
        cands += ctx->last_cands;
        launches += ctx->last_dp_launches;
        ctx->last_dp_ms = dp_ms;
        ctx->last_span_ms = span_ms;
        ctx->last_post_ms = post_ms;
        ctx->last_pairs = pairs;
        ctx->last_cands = cands;
        ctx->last_dp_launches = launches;
        for (int lv = grp.first; lv < grp.second; ++lv) {
            if (int rc = process_level(lv, outs, map)) return rc;
            if (best >= 0) {
                fill_stats(ctx, stats, running, calls_counted, unpruned, cells);
                if (plan) fill_plan(outs[map[best]], calls[best], plan);
                return PC_OK;
            }
        }
    }
    fill_stats(ctx, stats, running, calls_counted, unpruned, cells);
    if (plan) plan->n_stages = 0;
    return PC_INFEASIBLE;
}

extern "C" int pc_profile_spans(pc_ctx *ctx, int32_t n, const int32_t *lo, const int32_t *hi,
                                const int64_t *m, const int32_t *ckpt, double *t_fwd, double *t_bwd,
                                int64_t *mem) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    for (int i = 0; i < n; ++i) {
        if (lo[i] < 0 || hi[i] <= lo[i] || hi[i] > ctx->nb || m[i] < 0)
            return fail(ctx, PC_ERR_INVALID, "span out of range");
        if (ctx->has_cost_table && std::find(ctx->ov_m.begin(), ctx->ov_m.end(), m[i]) == ctx->ov_m.end())
            return fail(ctx, PC_ERR_INVALID, "cost table: microbatch share not resolved by pc_set_overrides");
    }
    if (n == 0) return PC_OK;
    size_t in_bytes = (8 + 4 * 3) * (size_t)n + 64;
    CUDA_TRY(ctx, ctx->q_d.ensure(in_bytes));
    CUDA_TRY(ctx, ctx->q_out_d.ensure(24 * (size_t)n + 64));
    char *qb = ctx->q_d.as<char>();
    int64_t *d_m = (int64_t *)qb;
    int32_t *d_lo = (int32_t *)(qb + 8 * (size_t)n);
    int32_t *d_hi = d_lo + n;
    int32_t *d_ck = d_hi + n;
    double *o_tf = ctx->q_out_d.as<double>();
    double *o_tb = o_tf + n;
    int64_t *o_mem = (int64_t *)(o_tb + n);
    CUDA_TRY(ctx, cudaMemcpyAsync(d_m, m, 8 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_lo, lo, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_hi, hi, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_ck, ckpt, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
    launch_profile_queries(ctx->P, n, d_lo, d_hi, d_m, d_ck, o_tf, o_tb, o_mem, ctx->st);
    if (int rc = check_launch(ctx, "profile_queries")) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(t_fwd, o_tf, 8 * (size_t)n, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(t_bwd, o_tb, 8 * (size_t)n, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(mem, o_mem, 8 * (size_t)n, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    return PC_OK;
}

// brute_force_partition (stages.py:304-369) over the DP's key tables: every
// (cut combination, composition) pair on the device (brute.cu), then the
// winner's stage records as profile queries.
extern "C" int pc_brute_force(pc_ctx *ctx, int32_t S, int32_t D, int64_t batch_size, int32_t R,
                              int32_t MB, pc_plan *plan, pc_stats *stats) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    const pc_call call{S, D, R, MB};
    if (int rc = validate_call(ctx, call, batch_size)) return rc;
    if (S > BF_MAXS) return fail(ctx, PC_ERR_CAPACITY, "brute force: more than 64 stages");
    if (plan && S > plan->cap_stages) return fail(ctx, PC_ERR_CAPACITY, "plan capacity");
    const DevProblem &P = ctx->P;
    const int nb = ctx->nb, k = S - 1, kcols = S;
    const int nmax = std::max(nb, D);
    const int64_t SAT = (int64_t)1 << 62;
    std::vector<int64_t> binom((size_t)(nmax + 1) * kcols, 0);
    for (int a = 0; a <= nmax; ++a) {
        binom[(size_t)a * kcols] = 1;
        for (int j = 1; j < kcols && a > 0; ++j) {
            const int64_t x = binom[(size_t)(a - 1) * kcols + j - 1], y = binom[(size_t)(a - 1) * kcols + j];
            binom[(size_t)a * kcols + j] = (x >= SAT - y) ? SAT : x + y;
        }
    }
    const int64_t n_comb = binom[(size_t)(nb - 1) * kcols + k];
    const int64_t n_comp = binom[(size_t)(D - 1) * kcols + k];
    if (n_comb >= SAT || n_comp >= SAT || (double)n_comb * (double)n_comp > 1e12)
        return fail(ctx, PC_ERR_CAPACITY, "brute force: more than 1e12 assignments");
    // keys of every device count (stages.py:326-330)
    const int ckpt = (P.checkpointing && S > 1) ? 1 : 0;
    const int B = D - S + 1;
    std::vector<std::pair<int64_t, int>> want, dkey(B + 1, {0, -1});
    for (int dev = 1; dev <= B; ++dev) {
        const int64_t m = batch_size / ((int64_t)MB * R * dev);
        if (m >= 1) {
            dkey[dev] = {m, ckpt};
            want.push_back(dkey[dev]);
        }
    }
    std::sort(want.begin(), want.end());
    want.erase(std::unique(want.begin(), want.end()), want.end());
    ctx->launches = 0;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->st));
    if (int rc = ensure_keys(ctx, want)) return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->st));
    std::vector<int16_t> keyidx(B + 1, -1);
    for (int dev = 1; dev <= B; ++dev)
        if (dkey[dev].second >= 0) keyidx[dev] = (int16_t)ctx->key_map[dkey[dev]];
    const int64_t n_chunks = (n_comp + BF_CHUNK - 1) / BF_CHUNK;
    const int64_t items = n_comb * n_chunks;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((items + BF_THREADS - 1) / BF_THREADS,
                                                                   (int64_t)ctx->sm_count * 8));
    const size_t b_bytes = 8 * binom.size(), k_bytes = 2 * keyidx.size();
    const size_t off_k = (b_bytes + 255) & ~size_t(255);
    const size_t off_o = (off_k + k_bytes + 255) & ~size_t(255);
    CUDA_TRY(ctx, ctx->bf_d.ensure(off_o + 24 * (size_t)blocks + 64));
    char *base = ctx->bf_d.as<char>();
    CUDA_TRY(ctx, cudaMemcpyAsync(base, binom.data(), b_bytes, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(base + off_k, keyidx.data(), k_bytes, cudaMemcpyHostToDevice, ctx->st));
    const size_t nk = ctx->keys.size();
    BruteArgs a{};
    a.key_tf = (const double *const *)ctx->key_ptrs.p;
    a.key_tb = ((const double *const *)ctx->key_ptrs.p) + nk;
    a.key_cut = ((const double *const *)ctx->key_ptrs.p) + 2 * nk;
    a.keyidx = (const int16_t *)(base + off_k);
    a.binom = (const int64_t *)base;
    a.kcols = kcols;
    a.nb = nb; a.S = S; a.D = D;
    a.derived = ctx->derived ? 1 : 0;
    a.nonneg = ctx->P.nonneg;
    a.num_nodes = P.num_nodes; a.dpn = P.dpn;
    a.beta = P.beta;
    a.n_comb = n_comb; a.n_comp = n_comp; a.n_chunks = n_chunks;
    a.out_key = (unsigned long long *)(base + off_o);
    a.out_idx = (long long *)(a.out_key + blocks);
    a.out_obj = (double *)(a.out_idx + blocks);
    launch_brute(a, blocks, ctx->st);
    ctx->launches++;
    if (int rc = check_launch(ctx, "brute")) return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev2, ctx->st));
    std::vector<unsigned long long> okey(blocks);
    std::vector<long long> oidx(blocks);
    std::vector<double> oobj(blocks);
    CUDA_TRY(ctx, cudaMemcpyAsync(okey.data(), a.out_key, 8 * (size_t)blocks, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(oidx.data(), a.out_idx, 8 * (size_t)blocks, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(oobj.data(), a.out_obj, 8 * (size_t)blocks, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    int win = -1;
    for (int i = 0; i < blocks; ++i) {
        if (oidx[i] < 0) continue;
        if (win < 0 || okey[i] < okey[win] || (okey[i] == okey[win] && oidx[i] < oidx[win])) win = i;
    }
    float span_ms = 0, bf_ms = 0;
    cudaEventElapsedTime(&span_ms, ctx->ev0, ctx->ev1);
    cudaEventElapsedTime(&bf_ms, ctx->ev1, ctx->ev2);
    if (stats) {
        *stats = pc_stats{};
        stats->visits = n_comb * n_comp;           // every pair counts (stages.py:321)
        stats->dp_calls = 0;
        stats->kernel_launches = ctx->launches;
        stats->device_ms = bf_ms;
        stats->span_ms = span_ms;
    }
    if (plan) {
        plan->S = S; plan->D = D; plan->R = R; plan->MB = MB;
        plan->iteration_time = NAN;
        plan->n_stages = 0;
        plan->objective = NAN;
    }
    if (win < 0) return PC_INFEASIBLE;
    // the winner's bounds and devices (host unrank of the same lex ranks)
    auto unrank_h = [&](int64_t r, int n, int *out) {
        int v = 1;
        for (int i = 0; i < k; ++i)
            for (;;) {
                const int64_t c = binom[(size_t)(n - v) * kcols + (k - 1 - i)];
                if (r < c) { out[i] = v++; break; }
                r -= c;
                ++v;
            }
    };
    std::vector<int> cuts(std::max(k, 1)), cps(std::max(k, 1));
    unrank_h(oidx[win] / n_comp, nb - 1, cuts.data());
    unrank_h(oidx[win] % n_comp, D - 1, cps.data());
    std::vector<int32_t> qlo(S), qhi(S), qck(S, ckpt), qdev(S);
    std::vector<int64_t> qm(S);
    for (int i = 0, prev = 0; i < S; ++i) {
        qlo[i] = i == 0 ? 0 : cuts[i - 1];
        qhi[i] = i == k ? nb : cuts[i];
        const int cum = i == k ? D : cps[i];
        qdev[i] = cum - prev;
        prev = cum;
        qm[i] = batch_size / ((int64_t)MB * R * qdev[i]);
    }
    std::vector<double> tf(S), tb(S);
    std::vector<int64_t> mem(S);
    if (int rc = pc_profile_spans(ctx, S, qlo.data(), qhi.data(), qm.data(), qck.data(), tf.data(),
                                  tb.data(), mem.data()))
        return rc;
    if (plan) {
        plan->n_stages = S;
        plan->objective = oobj[win];
        for (int i = 0; i < S; ++i) {
            plan->lo[i] = qlo[i];
            plan->hi[i] = qhi[i];
            plan->devices[i] = qdev[i];
            plan->t_fwd[i] = tf[i];
            plan->t_bwd[i] = tb[i];
            plan->mem[i] = mem[i];
        }
    }
    return PC_OK;
}

// validate_plan's fresh records (stages.py:452-492): per stage the span
// profile at its share (stages with a zero share are skipped: NaN / -1), the
// comm-charged times and the recomputed objective.
extern "C" int pc_check_plan(pc_ctx *ctx, const pc_plan *plan, int64_t batch_size, double *rec_tf,
                             double *rec_tb, int64_t *rec_mem, double *charged_tf,
                             double *charged_tb, double *objective) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    const int S = plan->n_stages;
    if (S < 1 || plan->MB < 1 || plan->R < 1 || batch_size < 1) return fail(ctx, PC_ERR_INVALID, "empty plan or counts below 1");
    const int ckpt = (ctx->P.checkpointing && S > 1) ? 1 : 0;
    std::vector<int32_t> lo(S), hi(S), dv(S), qlo, qhi, qck;
    std::vector<int64_t> m(S), qm;
    std::vector<int> qi;
    for (int i = 0; i < S; ++i) {
        lo[i] = plan->lo[i];
        hi[i] = plan->hi[i];
        dv[i] = plan->devices[i];
        if (lo[i] < 0 || hi[i] > ctx->nb || hi[i] <= lo[i] || dv[i] < 1)
            return fail(ctx, PC_ERR_INVALID, "stage bounds or devices out of range");
        m[i] = batch_size / ((int64_t)plan->MB * plan->R * dv[i]);
        rec_tf[i] = rec_tb[i] = charged_tf[i] = charged_tb[i] = NAN;
        rec_mem[i] = -1;
        if (m[i] >= 1) {
            qi.push_back(i);
            qlo.push_back(lo[i]);
            qhi.push_back(hi[i]);
            qm.push_back(m[i]);
            qck.push_back(ckpt);
        }
    }
    const int nq = (int)qi.size();
    std::vector<double> tf(S, 0.0), tb(S, 0.0);
    if (nq) {
        std::vector<double> qtf(nq), qtb(nq);
        std::vector<int64_t> qmem(nq);
        if (int rc = pc_profile_spans(ctx, nq, qlo.data(), qhi.data(), qm.data(), qck.data(),
                                      qtf.data(), qtb.data(), qmem.data()))
            return rc;
        for (int j = 0; j < nq; ++j) {
            tf[qi[j]] = rec_tf[qi[j]] = qtf[j];
            tb[qi[j]] = rec_tb[qi[j]] = qtb[j];
            rec_mem[qi[j]] = qmem[j];
        }
    }
    const size_t b4 = 4 * (size_t)S, b8 = 8 * (size_t)S;
    CUDA_TRY(ctx, ctx->sim_d.ensure(3 * b4 + 5 * b8 + 64));
    char *base = ctx->sim_d.as<char>();
    double *d_tf = (double *)base, *d_tb = d_tf + S, *d_ctf = d_tb + S, *d_ctb = d_ctf + S;
    int64_t *d_m = (int64_t *)(d_ctb + S);
    double *d_obj = (double *)(d_m + S);
    int32_t *d_lo = (int32_t *)(d_obj + 1), *d_hi = d_lo + S, *d_dv = d_hi + S;
    CUDA_TRY(ctx, cudaMemcpyAsync(d_tf, tf.data(), b8, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_tb, tb.data(), b8, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_m, m.data(), b8, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_lo, lo.data(), b4, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_hi, hi.data(), b4, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_dv, dv.data(), b4, cudaMemcpyHostToDevice, ctx->st));
    launch_charge_plan(ctx->P, S, d_lo, d_hi, d_dv, d_m, d_tf, d_tb, d_ctf, d_ctb, d_obj, ctx->st);
    if (int rc = check_launch(ctx, "charge_plan")) return rc;
    std::vector<double> ctf(S), ctb(S);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctf.data(), d_ctf, b8, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctb.data(), d_ctb, b8, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(objective, d_obj, 8, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    for (int i = 0; i < S; ++i)
        if (m[i] >= 1) {
            charged_tf[i] = ctf[i];
            charged_tb[i] = ctb[i];
        }
    return PC_OK;
}

// simulate() (simulate.py:79-179) of a validated plan: every lane event
// (stage-major, lane_off[S+1]) and summary = {iteration time, busy device
// time, bubble fraction, samples/s, devices}.
extern "C" int pc_simulate(pc_ctx *ctx, const pc_plan *plan, int64_t batch_size, int32_t ev_cap,
                           int32_t *lane_off, int32_t *ev_mb, int8_t *ev_phase, double *ev_start,
                           double *ev_end, double *summary) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    const int S = plan->n_stages, MB = plan->MB, R = plan->R;
    if (S < 1 || MB < 1 || R < 1 || batch_size < 1) return fail(ctx, PC_ERR_INVALID, "empty plan or counts below 1");
    const int64_t cap = (int64_t)S * (5 * (int64_t)MB + 1);
    if (cap > ev_cap || cap > (int64_t)1 << 30) return fail(ctx, PC_ERR_CAPACITY, "event capacity");
    for (int i = 0; i < S; ++i)
        if (plan->lo[i] < 0 || plan->hi[i] > ctx->nb || plan->hi[i] <= plan->lo[i] || plan->devices[i] < 1)
            return fail(ctx, PC_ERR_INVALID, "stage bounds or devices out of range");
    const size_t b4 = 4 * (size_t)S, b8 = 8 * (size_t)S;
    const size_t ev_bytes = (size_t)cap * (4 + 1 + 8 + 8);
    CUDA_TRY(ctx, ctx->q_d.ensure(3 * b4 + 2 * b8 + 4 * (size_t)(S + 1) + 64 + 256));
    CUDA_TRY(ctx, ctx->q_out_d.ensure(ev_bytes + 256));
    char *qb = ctx->q_d.as<char>();
    double *d_tf = (double *)qb, *d_tb = d_tf + S, *d_sum = d_tb + S;
    int32_t *d_lo = (int32_t *)(d_sum + 8), *d_hi = d_lo + S, *d_dv = d_hi + S, *d_off = d_dv + S;
    char *eb = ctx->q_out_d.as<char>();
    double *d_st = (double *)eb, *d_en = d_st + cap;
    int32_t *d_mb = (int32_t *)(d_en + cap);
    int8_t *d_ph = (int8_t *)(d_mb + cap);
    CUDA_TRY(ctx, cudaMemcpyAsync(d_tf, plan->t_fwd, b8, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_tb, plan->t_bwd, b8, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_lo, plan->lo, b4, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_hi, plan->hi, b4, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(d_dv, plan->devices, b4, cudaMemcpyHostToDevice, ctx->st));
    launch_schedule(ctx->P, S, R, MB, batch_size, d_lo, d_hi, d_dv, d_tf, d_tb, d_off, d_mb, d_ph,
                    d_st, d_en, d_sum, ctx->st);
    if (int rc = check_launch(ctx, "schedule")) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(lane_off, d_off, 4 * (size_t)(S + 1), cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(summary, d_sum, 5 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    const int64_t n_ev = lane_off[S];
    CUDA_TRY(ctx, cudaMemcpyAsync(ev_mb, d_mb, 4 * (size_t)n_ev, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ev_phase, d_ph, (size_t)n_ev, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ev_start, d_st, 8 * (size_t)n_ev, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ev_end, d_en, 8 * (size_t)n_ev, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    return PC_OK;
}

// Sharding weights: per call, a feasible-pair count from the key tables,
// S * sum_b sum_dev (B - dev + 1) * #{lo < b : span (lo, b) fits at share(dev)}
// (the first feasible lo per (key, hi) is already in the table).  Exact
// integers, so every rank derives the same assignment.
extern "C" int pc_call_weights(pc_ctx *ctx, int32_t n, const pc_call *calls, int64_t batch_size,
                               int64_t *weights) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    if (n <= 0) return PC_OK;
    const DevProblem &P = ctx->P;
    std::vector<std::pair<int64_t, int>> want;
    std::vector<int32_t> koff(n + 1, 0);
    std::vector<std::pair<int64_t, int>> flat_keys;
    for (int i = 0; i < n; ++i) {
        if (int rc = validate_call(ctx, calls[i], batch_size)) return rc;
        const int ckpt = P.checkpointing && calls[i].S > 1;
        const int B = calls[i].D - calls[i].S + 1;
        koff[i + 1] = koff[i] + B + 1;
        for (int dev = 0; dev <= B; ++dev) {
            const int64_t m = dev >= 1 ? batch_size / ((int64_t)calls[i].MB * calls[i].R * dev) : 0;
            flat_keys.push_back(m >= 1 ? std::make_pair(m, ckpt) : std::make_pair((int64_t)0, -1));
            if (m >= 1) want.push_back({m, ckpt});
        }
    }
    std::sort(want.begin(), want.end());
    want.erase(std::unique(want.begin(), want.end()), want.end());
    if (int rc = ensure_keys(ctx, want)) return rc;
    std::vector<int16_t> keyidx(flat_keys.size(), -1);
    for (size_t q = 0; q < flat_keys.size(); ++q)
        if (flat_keys[q].second >= 0) keyidx[q] = (int16_t)ctx->key_map[flat_keys[q]];
    const size_t c_bytes = sizeof(pc_call) * (size_t)n, o_bytes = 4 * (size_t)(n + 1);
    const size_t k_bytes = 2 * keyidx.size(), w_bytes = 8 * (size_t)n;
    const size_t off_o = (c_bytes + 255) & ~size_t(255);
    const size_t off_k = (off_o + o_bytes + 255) & ~size_t(255);
    const size_t off_w = (off_k + k_bytes + 255) & ~size_t(255);
    CUDA_TRY(ctx, ctx->bf_d.ensure(off_w + w_bytes + 64));
    char *base = ctx->bf_d.as<char>();
    CUDA_TRY(ctx, cudaMemcpyAsync(base, calls, c_bytes, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(base + off_o, koff.data(), o_bytes, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemcpyAsync(base + off_k, keyidx.data(), k_bytes, cudaMemcpyHostToDevice, ctx->st));
    CUDA_TRY(ctx, cudaMemsetAsync(base + off_w, 0, w_bytes, ctx->st));
    const size_t nk = ctx->keys.size();
    launch_call_weights(ctx->nb, n, (const int32_t *)base, (const int32_t *)(base + off_o),
                        (const int16_t *)(base + off_k),
                        ((const int32_t *const *)ctx->key_ptrs.p) + 3 * nk,
                        (unsigned long long *)(base + off_w), ctx->st);
    ctx->launches++;
    if (int rc = check_launch(ctx, "call_weights")) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(weights, base + off_w, w_bytes, cudaMemcpyDeviceToHost, ctx->st));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    return PC_OK;
}

extern "C" int pc_reset_cache(pc_ctx *ctx) {
    cudaSetDevice(ctx->device);
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    free_keys(ctx);
    return PC_OK;
}

extern "C" int pc_timer_start(pc_ctx *ctx) {
    cudaSetDevice(ctx->device);
    if (!ctx->t0) {
        CUDA_TRY(ctx, cudaEventCreate(&ctx->t0));
        CUDA_TRY(ctx, cudaEventCreate(&ctx->t1));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->t0, ctx->st));
    return PC_OK;
}

extern "C" int pc_timer_stop(pc_ctx *ctx, double *ms) {
    cudaSetDevice(ctx->device);
    CUDA_TRY(ctx, cudaEventRecord(ctx->t1, ctx->st));
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->t1));
    float f = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&f, ctx->t0, ctx->t1));
    *ms = f;
    return PC_OK;
}

extern "C" int pc_bound_info(pc_ctx *ctx, int64_t *bounded_calls, int64_t *reruns,
                             int64_t *frontier_reruns) {
    *bounded_calls = ctx->bounded_calls;
    *reruns = ctx->bound_reruns;
    if (frontier_reruns) *frontier_reruns = ctx->frontier_reruns;
    return PC_OK;
}

extern "C" int pc_measure_dadd_peak(pc_ctx *ctx, double *gops) {
    cudaSetDevice(ctx->device);
    *gops = measure_dadd_gops(ctx->st, ctx->sm_count);
    if (*gops <= 0) return fail(ctx, PC_ERR_CUDA, "DADD peak kernel failed");
    return PC_OK;
}

extern "C" int pc_measure_fp64_peak(pc_ctx *ctx, double *gops) {
    cudaSetDevice(ctx->device);
    *gops = measure_fp64_gops(ctx->st, ctx->sm_count);
    if (*gops <= 0) return fail(ctx, PC_ERR_CUDA, "fp64 peak kernel failed");
    return PC_OK;
}

extern "C" int pc_set_overrides(pc_ctx *ctx, int32_t n_m, const int64_t *m_values, const uint8_t *has,
                                const double *tf, const double *tb, const int64_t *act) {
    if (!ctx->has_problem) return fail(ctx, PC_ERR_INVALID, "no problem set");
    cudaSetDevice(ctx->device);
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->st));
    free_keys(ctx);
    const int T = ctx->P.n_tasks, nb = ctx->nb;
    // resident corrections: act_bytes replaces the produced bytes of a task
    std::vector<int64_t> corr((size_t)n_m * (nb + 1), 0);
    bool nonneg = ctx->mono_flops;
    for (int i = 0; i < n_m; ++i) {
        int64_t *c = corr.data() + (size_t)i * (nb + 1);
        for (int t = 0; t < T; ++t) {
            const size_t q = (size_t)i * T + t;
            if (!has[q]) continue;
            if (std::isnan(tf[q]))              // NaN is the infeasible-span marker (span_mark)
                return fail(ctx, PC_ERR_INVALID, "NaN t_fwd in a cost-table entry is not supported");
            if (!(tf[q] >= 0.0) || (!std::isnan(tb[q]) && !(tb[q] >= 0.0))) nonneg = false;
            if (act[q] >= 0)
                c[ctx->h_task_block[t] + 1] += act[q] - (ctx->h_prod_fix[t] + m_values[i] * ctx->h_prod_ps[t]);
        }
        for (int b = 0; b < nb; ++b) c[b + 1] += c[b];
    }
    ctx->mono_skip = nonneg;
    ctx->P.nonneg = nonneg ? 1 : 0;      // free_keys above: tables are rebuilt in this encoding
    const size_t KT = (size_t)n_m * T;
    const size_t bytes = 8 * (size_t)n_m + KT + 8 * KT * 3 + 8 * corr.size() + 256;
    CUDA_TRY(ctx, ctx->ov_d.ensure(bytes));
    char *base = ctx->ov_d.as<char>();
    size_t off = 0;
    auto put = [&](const void *src, size_t nbytes) {
        void *dst = base + off;
        if (nbytes) cudaMemcpy(dst, src, nbytes, cudaMemcpyHostToDevice);
        off = (off + nbytes + 15) & ~size_t(15);
        return dst;
    };
    DevProblem &D = ctx->P;
    D.ov_m = (const int64_t *)put(m_values, 8 * (size_t)n_m);
    D.ov_has = (const uint8_t *)put(has, KT);
    D.ov_tf = (const double *)put(tf, 8 * KT);
    D.ov_tb = (const double *)put(tb, 8 * KT);
    D.ov_act = (const int64_t *)put(act, 8 * KT);
    D.ov_corr = (const int64_t *)put(corr.data(), 8 * corr.size());
    D.n_ov = n_m;
    ctx->ov_m.assign(m_values, m_values + n_m);
    CUDA_TRY(ctx, cudaGetLastError());
    return PC_OK;
}
