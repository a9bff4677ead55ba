// K5: simulated iteration time of candidate plans, the ranking key of
// form_stage (stages.py:404-411 -> simulate.py:79-165).
//
// The fill/drain recurrence is a true 2-D wavefront over (microbatch, stage):
// cell (mb, s) of the forward pass needs (mb-1, s) through lane_free[s] and
// (mb, s-1) through arrival.  One CTA per plan, threads own stages, and step
// t processes every cell with mb + s == t; the operations per cell are the
// reference's, in the reference's order, so the result is bit-identical.
#include "common.cuh"

namespace pcb {

__global__ void k_simulate(DevProblem p, const int32_t *plan_off, const int32_t *plan_S,
                           const int32_t *plan_R, const int32_t *plan_MB, int64_t BS,
                           const int32_t *seg_lo, const int32_t *seg_hi, const int32_t *seg_dev,
                           const double *st_tf, const double *st_tb, double *iteration) {
    extern __shared__ double sm[];
    const int pi = blockIdx.x;
    const int S = plan_S[pi];
    const int R = plan_R[pi];
    const int MB = plan_MB[pi];
    const int off = plan_off[pi];
    double *lane = sm;               // [S]
    double *cf = lane + S;           // [S]
    double *cb = cf + S;             // [S]
    double *arr = cb + S;            // [2][S]
    double *red = arr + 2 * S;       // [blockDim]
    int64_t *cum = (int64_t *)(red + blockDim.x);   // [S+1]
    const int ckpt = p.checkpointing && S > 1;
    const int64_t denom = (int64_t)MB * R;
    if (threadIdx.x == 0) {
        cum[0] = 0;
        for (int s = 0; s < S; ++s) cum[s + 1] = cum[s] + seg_dev[off + s];
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const int64_t m = BS / (denom * seg_dev[off + s]);            // simulate.py:93
        cf[s] = s < S - 1 ? cut_time_dev(p, seg_hi[off + s], m,
                                         inter_of(p.num_nodes, p.dpn, cum[s + 1])) : 0.0;
        cb[s] = s > 0 ? cut_time_dev(p, seg_lo[off + s], m,
                                     inter_of(p.num_nodes, p.dpn, cum[s])) : 0.0;
        lane[s] = 0.0;
        arr[s] = 0.0;
        arr[S + s] = 0.0;
    }
    __syncthreads();
    // forward fill (simulate.py:116-127)
    for (int t = 0; t < MB + S - 1; ++t) {
        const double *ain = arr + (t & 1) * S;
        double *aout = arr + ((t + 1) & 1) * S;
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            const int mb = t - s;
            if (mb < 0 || mb >= MB) continue;
            const double a = s == 0 ? 0.0 : ain[s];
            const double ls = lane[s];
            const double start = a > ls ? a : ls;
            const double end = __dadd_rn(start, st_tf[off + s]);
            lane[s] = end;
            if (s < S - 1) {
                const double send_end = __dadd_rn(end, cf[s]);
                lane[s] = send_end;
                aout[s + 1] = send_end;
            }
        }
        __syncthreads();
    }
    // backward drain, reverse microbatch order (simulate.py:129-146)
    for (int t = 0; t < MB + S - 1; ++t) {
        const double *gin = arr + (t & 1) * S;
        double *gout = arr + ((t + 1) & 1) * S;
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            const int r = t - (S - 1 - s);        // reverse microbatch rank
            if (r < 0 || r >= MB) continue;
            double ls = lane[s];
            if (ckpt) ls = __dadd_rn(ls, st_tf[off + s]);
            const double g = s == S - 1 ? 0.0 : gin[s];
            const double start = g > ls ? g : ls;
            const double end = __dadd_rn(start, st_tb[off + s]);
            ls = end;
            if (s > 0) {
                const double send_end = __dadd_rn(end, cb[s]);
                ls = send_end;
                gout[s - 1] = send_end;
            }
            lane[s] = ls;
        }
        __syncthreads();
    }
    // gradient sync (simulate.py:148-163)
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const int64_t group = (int64_t)seg_dev[off + s] * R;
        if (group <= 1) continue;
        const int64_t params = p.pre_param[seg_hi[off + s]] - p.pre_param[seg_lo[off + s]];
        if (params == 0) continue;
        const int64_t nbytes = 2 * params * (group - 1) / group;
        const int64_t first_node = cum[s] / p.dpn;
        const int64_t last_node = (cum[s + 1] - 1) / p.dpn;
        const bool spans = R > 1 || first_node != last_node;
        const double dur = __dadd_rn(p.lat, __ddiv_rn((double)nbytes, spans ? p.bw_inter : p.bw_intra));
        if (dur > 0.0) lane[s] = __dadd_rn(lane[s], dur);
    }
    __syncthreads();
    double mx = -1.0;
    for (int s = threadIdx.x; s < S; s += blockDim.x) mx = lane[s] > mx ? lane[s] : mx;
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            const double o = red[threadIdx.x + w];
            if (o > red[threadIdx.x]) red[threadIdx.x] = o;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) iteration[pi] = red[0];
}

void launch_simulate(const DevProblem &p, int n_plans, const int32_t *plan_off,
                     const int32_t *plan_S, const int32_t *plan_R, const int32_t *plan_MB,
                     int64_t batch_size, const int32_t *seg_lo, const int32_t *seg_hi,
                     const int32_t *seg_dev, const double *st_tf, const double *st_tb,
                     double *iteration, cudaStream_t st, int max_S) {
    if (n_plans <= 0) return;
    int threads = ((max_S + 31) / 32) * 32;
    if (threads > 1024) threads = 1024;
    if (threads < 32) threads = 32;
    // power of two for the reduction
    int t2 = 32;
    while (t2 < threads) t2 <<= 1;
    threads = t2;
    const size_t smem = sizeof(double) * (5 * (size_t)max_S + threads) + sizeof(int64_t) * (max_S + 1);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_simulate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_simulate<<<n_plans, threads, smem, st>>>(p, plan_off, plan_S, plan_R, plan_MB, batch_size,
                                               seg_lo, seg_hi, seg_dev, st_tf, st_tb, iteration);
}


// ---------------------------------------------------------------- full schedule
// simulate() itself (simulate.py:79-179): the same recurrence as k_simulate,
// but every lane event is written out -- per stage s, in the reference's
// append order: fwd [+ comm] per microbatch, then per microbatch in reverse
// [recompute,] bwd [+ comm], then the gradient sync -- with lane_off[s] its
// first event.  Busy time is folded in the reference's order (stage, device of
// the stage, lane event), then bubble and samples/s.  One CTA, threads own
// stages.  Phases: 0 fwd, 1 recompute, 2 bwd, 3 comm, 4 allreduce.
__global__ void k_schedule(DevProblem p, int S, int R, int MB, int64_t BS, const int32_t *lo,
                           const int32_t *hi, const int32_t *dev, const double *tf,
                           const double *tb, int32_t *lane_off, int32_t *ev_mb, int8_t *ev_phase,
                           double *ev_start, double *ev_end, double *summary) {
    extern __shared__ double sm[];
    double *lane = sm;                // [S]
    double *cf = lane + S;            // [S]
    double *cb = cf + S;              // [S]
    double *ar = cb + S;              // [S] gradient-sync duration (0: none)
    double *arr = ar + S;             // [2][S]
    int64_t *cum = (int64_t *)(arr + 2 * S);        // [S+1]
    int32_t *pos = (int32_t *)(cum + S + 1);        // [S] next event slot
    const int ckpt = p.checkpointing && S > 1;
    const int64_t denom = (int64_t)MB * R;
    if (threadIdx.x == 0) {
        cum[0] = 0;
        for (int s = 0; s < S; ++s) cum[s + 1] = cum[s] + dev[s];
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const int64_t m = BS / (denom * dev[s]);
        cf[s] = s < S - 1 ? cut_time_dev(p, hi[s], m, inter_of(p.num_nodes, p.dpn, cum[s + 1])) : 0.0;
        cb[s] = s > 0 ? cut_time_dev(p, lo[s], m, inter_of(p.num_nodes, p.dpn, cum[s])) : 0.0;
        double dur = 0.0;
        const int64_t group = (int64_t)dev[s] * R;
        const int64_t params = p.pre_param[hi[s]] - p.pre_param[lo[s]];
        if (group > 1 && params != 0) {
            const int64_t nbytes = 2 * params * (group - 1) / group;
            const bool spans = R > 1 || cum[s] / p.dpn != (cum[s + 1] - 1) / p.dpn;
            dur = __dadd_rn(p.lat, __ddiv_rn((double)nbytes, spans ? p.bw_inter : p.bw_intra));
        }
        ar[s] = dur;
        lane[s] = 0.0;
        arr[s] = 0.0;
        arr[S + s] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t o = 0;
        for (int s = 0; s < S; ++s) {
            lane_off[s] = o;
            pos[s] = o;
            o += MB * (1 + (s < S - 1 && cf[s] > 0.0)) +
                 MB * (ckpt + 1 + (s > 0 && cb[s] > 0.0)) + (ar[s] > 0.0);
        }
        lane_off[S] = o;
    }
    __syncthreads();
    auto put = [&](int s, int mb, int ph, double a, double b) {
        const int q = pos[s]++;
        ev_mb[q] = mb;
        ev_phase[q] = (int8_t)ph;
        ev_start[q] = a;
        ev_end[q] = b;
    };
    for (int t = 0; t < MB + S - 1; ++t) {                       // simulate.py:116-127
        const double *ain = arr + (t & 1) * S;
        double *aout = arr + ((t + 1) & 1) * S;
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            const int mb = t - s;
            if (mb < 0 || mb >= MB) continue;
            const double a = s == 0 ? 0.0 : ain[s];
            const double start = a > lane[s] ? a : lane[s];
            const double end = __dadd_rn(start, tf[s]);
            put(s, mb, 0, start, end);
            lane[s] = end;
            if (s < S - 1) {
                const double send_end = __dadd_rn(end, cf[s]);
                if (cf[s] > 0.0) put(s, mb, 3, end, send_end);
                lane[s] = send_end;
                aout[s + 1] = send_end;
            }
        }
        __syncthreads();
    }
    for (int t = 0; t < MB + S - 1; ++t) {                       // simulate.py:129-146
        const double *gin = arr + (t & 1) * S;
        double *gout = arr + ((t + 1) & 1) * S;
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            const int r = t - (S - 1 - s);
            if (r < 0 || r >= MB) continue;
            const int mb = MB - 1 - r;
            double ls = lane[s];
            if (ckpt) {
                const double e = __dadd_rn(ls, tf[s]);
                put(s, mb, 1, ls, e);
                ls = e;
            }
            const double g = s == S - 1 ? 0.0 : gin[s];
            const double start = g > ls ? g : ls;
            const double end = __dadd_rn(start, tb[s]);
            put(s, mb, 2, start, end);
            ls = end;
            if (s > 0) {
                const double send_end = __dadd_rn(end, cb[s]);
                if (cb[s] > 0.0) put(s, mb, 3, end, send_end);
                ls = send_end;
                gout[s - 1] = send_end;
            }
            lane[s] = ls;
        }
        __syncthreads();
    }
    for (int s = threadIdx.x; s < S; s += blockDim.x)             // simulate.py:148-163
        if (ar[s] > 0.0) {
            put(s, -1, 4, lane[s], __dadd_rn(lane[s], ar[s]));
            lane[s] = __dadd_rn(lane[s], ar[s]);
        }
    __syncthreads();
    if (threadIdx.x == 0) {                                       // simulate.py:165-179
        double it = lane[0];
        for (int s = 1; s < S; ++s) it = lane[s] > it ? lane[s] : it;
        double busy = 0.0;
        for (int s = 0; s < S; ++s)
            for (int64_t d = cum[s]; d < cum[s + 1]; ++d)
                for (int q = lane_off[s]; q < lane_off[s + 1]; ++q)
                    busy = __dadd_rn(busy, __dsub_rn(ev_end[q], ev_start[q]));
        const double n_dev = (double)cum[S];
        summary[0] = it;
        summary[1] = busy;
        summary[2] = it > 0.0 ? __dsub_rn(1.0, __ddiv_rn(busy, __dmul_rn(n_dev, it))) : 0.0;
        summary[3] = it > 0.0 ? __ddiv_rn((double)BS, it) : 0.0;
        summary[4] = n_dev;
    }
}

size_t schedule_smem(int S) {
    return sizeof(double) * 6 * (size_t)S + sizeof(int64_t) * (S + 1) + sizeof(int32_t) * S + 64;
}

void launch_schedule(const DevProblem &p, int S, int R, int MB, int64_t BS, const int32_t *lo,
                     const int32_t *hi, const int32_t *dev, const double *tf, const double *tb,
                     int32_t *lane_off, int32_t *ev_mb, int8_t *ev_phase, double *ev_start,
                     double *ev_end, double *summary, cudaStream_t st) {
    int threads = ((S + 31) / 32) * 32;
    if (threads > 1024) threads = 1024;
    const size_t smem = schedule_smem(S);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_schedule<<<1, threads, smem, st>>>(p, S, R, MB, BS, lo, hi, dev, tf, tb, lane_off, ev_mb,
                                         ev_phase, ev_start, ev_end, summary);
}

// validate_plan's fresh records (stages.py:452-492): charged stage times with
// the cut transfers and the recomputed objective max(tfs) + max(tbs) over the
// stages with a positive share, folded like Python's max (first of equals).
__global__ void k_charge_plan(DevProblem p, int S, const int32_t *lo, const int32_t *hi,
                              const int32_t *dev, const int64_t *m, const double *rtf,
                              const double *rtb, double *ctf, double *ctb, double *objective) {
    extern __shared__ int64_t cum_s[];
    if (threadIdx.x == 0) {
        cum_s[0] = 0;
        for (int s = 0; s < S; ++s) cum_s[s + 1] = cum_s[s] + dev[s];
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        if (m[s] < 1) continue;
        double f = rtf[s], b = rtb[s];
        if (hi[s] < p.nb) f = __dadd_rn(f, cut_time_dev(p, hi[s], m[s], inter_of(p.num_nodes, p.dpn, cum_s[s + 1])));
        if (lo[s] > 0) b = __dadd_rn(b, cut_time_dev(p, lo[s], m[s], inter_of(p.num_nodes, p.dpn, cum_s[s])));
        ctf[s] = f;
        ctb[s] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        bool any = false;
        double mf = 0.0, mb = 0.0;
        for (int s = 0; s < S; ++s) {
            if (m[s] < 1) continue;
            if (!any || ctf[s] > mf) mf = ctf[s];
            if (!any || ctb[s] > mb) mb = ctb[s];
            any = true;
        }
        *objective = any ? __dadd_rn(mf, mb) : NAN;
    }
}

void launch_charge_plan(const DevProblem &p, int S, const int32_t *lo, const int32_t *hi,
                        const int32_t *dev, const int64_t *m, const double *rtf, const double *rtb,
                        double *ctf, double *ctb, double *objective, cudaStream_t st) {
    int threads = ((S + 31) / 32) * 32;
    if (threads > 1024) threads = 1024;
    const size_t smem = sizeof(int64_t) * (S + 1);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_charge_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_charge_plan<<<1, threads, smem, st>>>(p, S, lo, hi, dev, m, rtf, rtb, ctf, ctb, objective);
}

}  // namespace pcb
