// K8: exhaustive stage assignment -- replaces brute_force_partition
// (pkg/src/pipecut/stages.py:294-369), the reference's second oracle.
//
// The reference walks every cut combination (itertools.combinations of
// range(1, nb), lex order) times every composition of D into S positive parts
// (_compositions, head ascending = lex order), counts each pair as a visit and
// keeps the smallest (max(tfs) + max(tbs), bounds, devs) tuple.  Both lists
// are combinations in lex order (a composition is its S-1 partial sums), so
// the pair at enumeration index  comb_rank * n_comp + comp_rank  is fixed and
// the reference's tuple order is (objective, index).  Work item = (comb rank,
// chunk of BF_CHUNK composition ranks): a thread unranks both, then walks the
// chunk by lex successor keeping its first minimum; warps and the block reduce
// (objective, index) lexicographically, the host the per-block winners.
//
// Stage times come from the DP's key tables (span t_fwd with the sign bit for
// mem > budget, t_bwd derived or stored, per-key cut tables), so every value
// is the DP's own: stages.py:333-349 on the same records.
#include <math.h>

#include "common.cuh"

namespace pcb {

// total order on doubles for the (objective, index) min; -0.0 ties +0.0 as in
// Python's tuple comparison
__device__ __forceinline__ unsigned long long order_key(double v) {
    if (v == 0.0) v = 0.0;
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// lex rank r -> k increasing values from {1 .. n}; binom[(a) * kcols + j] = C(a, j)
__device__ __forceinline__ void unrank(int64_t r, int n, int k, const int64_t *binom, int kcols,
                                       int *out) {
    int v = 1;
    for (int i = 0; i < k; ++i) {
        for (;;) {
            const int64_t c = binom[(int64_t)(n - v) * kcols + (k - 1 - i)];
            if (r < c) {
                out[i] = v++;
                break;
            }
            r -= c;
            ++v;
        }
    }
}

__global__ void k_brute(BruteArgs a) {
    const int S = a.S, k = S - 1, nb = a.nb, D = a.D;
    const int64_t n_items = a.n_comb * a.n_chunks;
    unsigned long long best_key = ~0ull;
    long long best_idx = -1;
    double best_obj = 0.0;
    int bnd[BF_MAXS + 1], cp[BF_MAXS];
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t comb = it / a.n_chunks;
        const int64_t c0 = (it % a.n_chunks) * BF_CHUNK;
        const int64_t c1 = min(a.n_comp, c0 + BF_CHUNK);
        bnd[0] = 0;
        unrank(comb, nb - 1, k, a.binom, a.kcols, bnd + 1);
        bnd[S] = nb;
        unrank(c0, D - 1, k, a.binom, a.kcols, cp);
        for (int64_t cr = c0; cr < c1; ++cr) {
            int cum = 0;
            bool feasible = true;
            double mtf = 0.0, mtb = 0.0;
            for (int i = 0; i < S; ++i) {
                const int lo = bnd[i], hi = bnd[i + 1];
                const int prev = cum;
                cum = i < k ? cp[i] : D;
                const int dv = cum - prev;
                const int kk = a.keyidx[dv];
                if (kk < 0) { feasible = false; break; }               // m == 0
                const int64_t o = hm_idx(lo, hi);
                double tf = a.key_tf[kk][o];
                if (!span_ok(tf, a.nonneg)) { feasible = false; break; }  // mem > budget
                double tb = a.derived ? __dmul_rn(a.beta, tf) : a.key_tb[kk][o];
                const double *cut = a.key_cut[kk];
                if (hi < nb) {
                    const int inter = (a.num_nodes > 1 && cum % a.dpn == 0) ? 1 : 0;
                    tf = __dadd_rn(tf, cut[inter * (nb + 1) + hi]);
                }
                if (lo > 0) {
                    const int inter = (a.num_nodes > 1 && prev % a.dpn == 0) ? 1 : 0;
                    tb = __dadd_rn(tb, cut[inter * (nb + 1) + lo]);
                }
                // Python max over the list: the first of equal maxima
                if (i == 0 || tf > mtf) mtf = tf;
                if (i == 0 || tb > mtb) mtb = tb;
            }
            if (feasible) {
                const double obj = __dadd_rn(mtf, mtb);
                const unsigned long long key = order_key(obj);
                if (key < best_key) {          // indices only grow: first minimum wins
                    best_key = key;
                    best_idx = comb * a.n_comp + cr;
                    best_obj = obj;
                }
            }
            // lex successor of cp (k values in 1..D-1)
            int j = k - 1;
            while (j >= 0 && cp[j] == D - 1 - (k - 1 - j)) --j;
            if (j < 0) break;
            ++cp[j];
            for (int q = j + 1; q < k; ++q) cp[q] = cp[q - 1] + 1;
        }
    }
    // (key, index) lexicographic min over the block
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long ok = __shfl_down_sync(0xffffffffu, best_key, off);
        const long long oi = __shfl_down_sync(0xffffffffu, best_idx, off);
        const double oo = __shfl_down_sync(0xffffffffu, best_obj, off);
        if (ok < best_key || (ok == best_key && oi >= 0 && (best_idx < 0 || oi < best_idx))) {
            best_key = ok;
            best_idx = oi;
            best_obj = oo;
        }
    }
    __shared__ unsigned long long s_key[32];
    __shared__ long long s_idx[32];
    __shared__ double s_obj[32];
    if (lane == 0) {
        s_key[w] = best_key;
        s_idx[w] = best_idx;
        s_obj[w] = best_obj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
            if (s_key[q] < best_key ||
                (s_key[q] == best_key && s_idx[q] >= 0 && (best_idx < 0 || s_idx[q] < best_idx))) {
                best_key = s_key[q];
                best_idx = s_idx[q];
                best_obj = s_obj[q];
            }
        a.out_key[blockIdx.x] = best_key;
        a.out_idx[blockIdx.x] = best_idx;
        a.out_obj[blockIdx.x] = best_obj;
    }
}

void launch_brute(const BruteArgs &a, int blocks, cudaStream_t st) {
    k_brute<<<blocks, BF_THREADS, 0, st>>>(a);
}

}  // namespace pcb
