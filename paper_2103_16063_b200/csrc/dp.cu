// K3/K4/K7: the level-synchronous Pareto-frontier stage DP, its backtrack and
// the reference's pruned visit accounting.
//
// Replaces _run_dp and _pareto (pkg/src/pipecut/stages.py:176-279).
//
// Within a level s every cell (b, d) depends only on level s-1
// (stages.py:204-251), so one launch per level covers every active DP call of
// a batch.  Thread = one cell (b, d); a warp holds 32 consecutive b of one d,
// so
//   * the predecessor cells (b', d') of level s-1 are warp-uniform
//     (broadcast loads, every lane walks the same b' and d'),
//   * the span records (lo=b', hi=b) are contiguous across lanes
//     (hi-contiguous triangular tables: coalesced 256 B loads),
//   * each thread visits its candidates in ascending (b', d', idx) order, the
//     reference's insertion order, so its private Pareto frontier is exactly
//     _pareto's output without any cross-thread merge.
// The frontier lives in registers (capacity FL); a cell that would exceed FL
// sets a flag and the host reruns the batch with a larger FL -- entries are
// never dropped silently.
#include <math.h>

#include "common.cuh"

namespace pcb {

// Pareto frontier of (max fwd, max bwd) pairs for candidates that arrive in
// strictly increasing key order.  With keys increasing, the reference's
// (tf, tb, index) lexicographic filter (stages.py:176-185) reduces to weak
// dominance: a newcomer is dropped iff some entry has x <= cx and y <= cy,
// and it removes every entry with cx <= x and cy <= y.
template <int FL>
struct Front {
    double x[FL], y[FL];
    uint32_t k[FL];
    uint32_t valid;
    bool ovf;

    __device__ __forceinline__ void init() {
        valid = 0;
        ovf = false;
    }

    __device__ __forceinline__ void insert(double cx, double cy, uint32_t ck) {
#pragma unroll
        for (int j = 0; j < FL; ++j)
            if (((valid >> j) & 1u) && x[j] <= cx && y[j] <= cy) return;
#pragma unroll
        for (int j = 0; j < FL; ++j)
            if (((valid >> j) & 1u) && cx <= x[j] && cy <= y[j]) valid &= ~(1u << j);
        bool placed = false;
#pragma unroll
        for (int j = 0; j < FL; ++j) {
            if (!placed && !((valid >> j) & 1u)) {
                x[j] = cx;
                y[j] = cy;
                k[j] = ck;
                valid |= 1u << j;
                placed = true;
            }
        }
        if (!placed) ovf = true;
    }
};

__device__ __forceinline__ double dmax_ref(double a, double b) {
    // Python max(a, b): b if b > a else a (stages.py:239)
    return b > a ? b : a;
}

template <int FL>
__global__ void __launch_bounds__(256) k_dp_level(DPBatch B, int s, int n_active) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= B.warp_prefix[n_active]) return;
    int lo = 0, hi = n_active;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (B.warp_prefix[mid] <= gw) lo = mid; else hi = mid;
    }
    const int c = lo;
    const CallDesc cd = B.calls[c];
    const int64_t wl = gw - B.warp_prefix[c];
    const int di = (int)(wl % cd.B);
    const int bchunk = (int)(wl / cd.B);
    const int d = s + di;
    const int bi = bchunk * 32 + lane;
    const int b = s + bi;
    const bool active = bi < cd.A;
    const int nb = B.nb;
    const int64_t tri = B.tri;
    const int64_t cells = (int64_t)cd.A * cd.B;
    const int cur = s & 1, prv = (s - 1) & 1;
    const int16_t *keyidx = B.keyidx + cd.key_off;
    const int inter_d = inter_of(B.num_nodes, B.dpn, d);

    Front<FL> F;
    F.init();
    bool zero = false;
    uint32_t n_pairs = 0, n_cands = 0;

    if (s == 1) {
        // level 0 holds the single cell (0, 0) with entry (0.0, 0.0) (stages.py:201)
        const int kk = keyidx[d];
        if (kk < 0) {
            zero = true;
        } else if (active) {
            const int64_t ti = tri_idx(0, b, nb);
            const double tfc = B.key_tfc[kk][inter_d * tri + ti];
            if (!isnan(tfc)) {
                const double tbc = B.key_tbc[kk][ti];
                F.insert(dmax_ref(0.0, tfc), dmax_ref(0.0, tbc), pack_key(0, 0, 0));
                n_pairs = 1;
                n_cands = 1;
            }
        }
    } else {
        const int base = s - 1;
        const int bmax = s + min(bchunk * 32 + 31, cd.A - 1);
        const double *ptf = B.val_tf[prv] + cd.val_off;
        const double *ptb = B.val_tb[prv] + cd.val_off;
        const uint8_t *pcnt = B.val_cnt[prv] + cd.val_off;
        const int64_t vstride = B.val_cells;
        for (int bp = base; bp < bmax; ++bp) {
            const bool lane_ok = active && bp < b;
            const int64_t ti = lane_ok ? tri_idx(bp, b, nb) : 0;
            for (int dp = base; dp < d; ++dp) {
                const int64_t pc = (int64_t)(dp - base) * cd.A + (bp - base);
                const int cnt = pcnt[pc] & CNT_MASK;
                if (cnt == 0) continue;
                const int kk = keyidx[d - dp];
                if (kk < 0) {                      // m == 0 (stages.py:224-228)
                    zero |= lane_ok;
                    continue;
                }
                if (!lane_ok) continue;
                const double tfc = B.key_tfc[kk][inter_d * tri + ti];
                if (isnan(tfc)) continue;          // mem > budget (stages.py:230)
                const int inter_dp = inter_of(B.num_nodes, B.dpn, dp);
                const double tbc = B.key_tbc[kk][inter_dp * tri + ti];
                ++n_pairs;
                n_cands += cnt;
                for (int i = 0; i < cnt; ++i) {
                    const double a = ptf[i * vstride + pc];
                    const double bb = ptb[i * vstride + pc];
                    F.insert(dmax_ref(a, tfc), dmax_ref(bb, tbc), pack_key(bp, dp, i));
                }
            }
        }
    }
    // algorithmic work counters (one atomic per warp)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
        n_cands += __shfl_xor_sync(0xffffffffu, n_cands, o);
    }
    if (lane == 0) {
        atomicAdd(&B.counters[0], (unsigned long long)n_pairs);
        atomicAdd(&B.counters[1], (unsigned long long)n_cands);
    }
    if (!active) return;

    // emit in tf-ascending order (entries have distinct tf)
    const int64_t cell = (int64_t)di * cd.A + bi;
    int n = 0;
    uint8_t byte = 0;
#pragma unroll
    for (int j = 0; j < FL; ++j) {
        if (!((F.valid >> j) & 1u)) continue;
        int rank = 0;
#pragma unroll
        for (int i = 0; i < FL; ++i)
            if (((F.valid >> i) & 1u) && F.x[i] < F.x[j]) ++rank;
        B.val_tf[cur][rank * B.val_cells + cd.val_off + cell] = F.x[j];
        B.val_tb[cur][rank * B.val_cells + cd.val_off + cell] = F.y[j];
        B.hist_key[rank * B.hist_cells + cd.hist_off + (int64_t)(s - 1) * cells + cell] = F.k[j];
        ++n;
    }
    byte = (uint8_t)n | (zero ? CNT_ZERO : 0) | (F.ovf ? CNT_OVF : 0);
    B.val_cnt[cur][cd.val_off + cell] = byte;
    B.hist_cnt[cd.hist_off + (int64_t)(s - 1) * cells + cell] = byte;
    if (F.ovf) atomicOr(B.overflow, 1);
}

void launch_dp_level(const DPBatch &b, int s, int n_active, int64_t n_warps, int FL,
                     cudaStream_t st) {
    const int tpb = 256;
    const int64_t blocks = (n_warps * 32 + tpb - 1) / tpb;
    switch (FL) {
        case 4: k_dp_level<4><<<(unsigned)blocks, tpb, 0, st>>>(b, s, n_active); break;
        case 16: k_dp_level<16><<<(unsigned)blocks, tpb, 0, st>>>(b, s, n_active); break;
        default: k_dp_level<32><<<(unsigned)blocks, tpb, 0, st>>>(b, s, n_active); break;
    }
}

// ---------------------------------------------------------------- visits (K7)
// Pruned SearchStats.visits (stages.py:212-249) from the per-cell flags:
// a row (s, b) is scanned from d = D-(S-s) down; the first cell that is
// empty without a zero-share candidate ends it (inclusive).  Level 1 carries
// d_min across rows, handled by one thread per call afterwards.
__device__ __forceinline__ int64_t row_visits(const uint8_t *row, int stride, int s, int b,
                                              int B, int bottom_di, int pruning, int *dead) {
    // cells d = s + di, di in [bottom_di, B-1], scanned from the top
    int stop = bottom_di;
    *dead = -1;
    if (pruning) {
        for (int di = B - 1; di >= bottom_di; --di) {
            const uint8_t v = row[(int64_t)di * stride];
            if ((v & CNT_MASK) == 0 && !(v & CNT_ZERO)) {
                stop = di;
                *dead = di;
                break;
            }
        }
    }
    // sum_{di=stop}^{B-1} (b-s+1)(di+1)
    const int64_t w = (int64_t)(b - s + 1);
    const int64_t a = stop + 1, z = B;
    return w * ((z * (z + 1) - (a - 1) * a) / 2);
}

__global__ void k_visit_rows(DPBatch Bt, int pruning, const int64_t *call_row_prefix,
                             const int64_t *level_off, int64_t *level_sums) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= call_row_prefix[Bt.n_calls]) return;
    int lo = 0, hi = Bt.n_calls;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (call_row_prefix[mid] <= r) lo = mid; else hi = mid;
    }
    const int c = lo;
    const CallDesc cd = Bt.calls[c];
    const int64_t rl = r - call_row_prefix[c];
    const int s = 1 + (int)(rl / cd.A);
    const int bi = (int)(rl % cd.A);
    if (s == 1) return;  // level 1 carries d_min: k_visit_level1
    const int64_t cells = (int64_t)cd.A * cd.B;
    const uint8_t *row = Bt.hist_cnt + cd.hist_off + (int64_t)(s - 1) * cells + bi;
    int dead;
    const int64_t v = row_visits(row, cd.A, s, s + bi, cd.B, 0, pruning, &dead);
    atomicAdd((unsigned long long *)&level_sums[level_off[c] + s - 1], (unsigned long long)v);
}

__global__ void k_visit_level1(DPBatch Bt, int pruning, const int64_t *level_off,
                               int64_t *level_sums) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Bt.n_calls) return;
    const CallDesc cd = Bt.calls[c];
    const uint8_t *lvl = Bt.hist_cnt + cd.hist_off;
    int64_t total = 0;
    int d_min = 1;
    for (int bi = 0; bi < cd.A; ++bi) {
        const int bottom = d_min > 1 ? d_min : 1;      // max(d_min, s) with s = 1
        const int bottom_di = bottom - 1;
        if (bottom_di > cd.B - 1) continue;            // empty d range: no visits
        int dead;
        total += row_visits(lvl + bi, cd.A, 1, 1 + bi, cd.B, bottom_di, pruning, &dead);
        if (dead >= 0) d_min = dead + 1 + 1;           // d_min = d + 1, d = 1 + dead
    }
    level_sums[level_off[c]] = total;
}

void launch_row_visits(const DPBatch &b, int pruning, int64_t *level_sums, int64_t *row_prefix,
                       const int64_t *level_off, int64_t n_rows_total, cudaStream_t st) {
    if (n_rows_total > 0)
        k_visit_rows<<<(unsigned)((n_rows_total + 255) / 256), 256, 0, st>>>(
            b, pruning, row_prefix, level_off, level_sums);
    k_visit_level1<<<(b.n_calls + 127) / 128, 128, 0, st>>>(b, pruning, level_off, level_sums);
}

// ---------------------------------------------------------------- backtrack (K4)
// Final pick by (tf + tb), first wins (stages.py:253-259), then the
// back-pointer chase through the history (stages.py:260-268).
__global__ void k_backtrack(DPBatch Bt, int64_t batch_size, const int32_t *plan_off,
                            int32_t *seg_lo, int32_t *seg_hi, int32_t *seg_dev,
                            double *objective, int32_t *feasible) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Bt.n_calls) return;
    const CallDesc cd = Bt.calls[c];
    const int S = cd.S;
    const int64_t cells = (int64_t)cd.A * cd.B;
    const int64_t fcell = (int64_t)(cd.B - 1) * cd.A + (cd.A - 1);   // (nb, D)
    const int par = S & 1;
    const uint8_t byte = Bt.val_cnt[par][cd.val_off + fcell];
    const int n = byte & CNT_MASK;
    const int o = cd.orig;
    if (n == 0) {
        feasible[o] = 0;
        return;
    }
    int best = 0;
    double bx = Bt.val_tf[par][cd.val_off + fcell];
    double by = Bt.val_tb[par][cd.val_off + fcell];
    for (int j = 1; j < n; ++j) {
        const double x = Bt.val_tf[par][j * Bt.val_cells + cd.val_off + fcell];
        const double y = Bt.val_tb[par][j * Bt.val_cells + cd.val_off + fcell];
        if (__dadd_rn(x, y) < __dadd_rn(bx, by)) {
            best = j;
            bx = x;
            by = y;
        }
    }
    feasible[o] = 1;
    objective[o] = __dadd_rn(bx, by);
    int s = S, b = Bt.nb, d = cd.D, j = best;
    int64_t cell = fcell;
    const int32_t off = plan_off[o];
    while (s > 0) {
        const uint32_t key =
            Bt.hist_key[(int64_t)j * Bt.hist_cells + cd.hist_off + (int64_t)(s - 1) * cells + cell];
        const int bp = key_bp(key), dp = key_dp(key);
        seg_lo[off + s - 1] = bp;
        seg_hi[off + s - 1] = b;
        seg_dev[off + s - 1] = d - dp;
        j = key_idx(key);
        s -= 1;
        b = bp;
        d = dp;
        if (s > 0) cell = (int64_t)(d - s) * cd.A + (b - s);
    }
}

void launch_backtrack(const DPBatch &b, int FL, int64_t batch_size, const int32_t *plan_off,
                      int32_t *seg_lo, int32_t *seg_hi, int32_t *seg_dev, double *objective,
                      int32_t *feasible, cudaStream_t st) {
    (void)FL;
    k_backtrack<<<(b.n_calls + 127) / 128, 128, 0, st>>>(b, batch_size, plan_off, seg_lo, seg_hi,
                                                         seg_dev, objective, feasible);
}

}  // namespace pcb
