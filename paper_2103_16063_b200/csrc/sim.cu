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

}  // namespace pcb
