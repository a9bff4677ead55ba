// K3/K4/K7: the level-synchronous Pareto-frontier stage DP, its backtrack and
// the reference's pruned visit accounting.
//
// Replaces _run_dp and _pareto (pkg/src/pipecut/stages.py:176-279).
//
// Within a level s every cell (b, d) depends only on level s-1
// (stages.py:204-251), so one launch per level covers every active DP call of
// a batch.  One warp owns one cell (b, d); a CTA holds the cells of one b for
// up to DP_WARPS consecutive d, which share the span row of b and the
// predecessor cells in L1.  Lanes stride over the predecessor blocks b', so
// every global load is coalesced and independent of the previous one:
//   * predecessor counts / frontier values of level s-1 ([d'][b'] layout),
//   * the span row t_fwd(b', b) (hi-major tables, b' contiguous),
//   * cut times cut(b', m, inter(d')) (per-key [inter][c] tables).
//
// Exact _pareto (stages.py:176-185) without ordering constraints: an entry e
// dominates a candidate c iff e precedes c in the (tf, tb, key) order and
// e.tb <= c.tb.  That relation is a strict partial order, so the frontier is
// the set of its maximal elements whatever the insertion order.  The cell's
// frontier lives in shared memory sorted by tf (capacity FMAX = 64); lanes
// build candidates in parallel and test them against it by binary search,
// and only the few survivors are inserted, one warp-cooperative step each.
#include <math.h>

#include "common.cuh"

// diagnostic counters (frontier-size histogram, rounds, chunks, corner-pruned
// pairs, window entries) for PIPECUT_B200_DEBUG: build with -DPC_DP_DIAG=1
#ifndef PC_DP_DIAG
#define PC_DP_DIAG 0
#endif

namespace pcb {

__device__ __forceinline__ double dmax_ref(double a, double b) {
    // Python max(a, b): b if b > a else a (stages.py:239)
    return b > a ? b : a;
}

// e dominates c: e before c in (x, y, key) order and e.y <= c.y
__device__ __forceinline__ bool dominates(double ex, double ey, uint32_t ek, double cx, double cy,
                                          uint32_t ck) {
    return ey <= cy && (ex < cx || (ex == cx && (ey < cy || ek < ck)));
}

// Per-warp Pareto frontiers in shared memory, each sorted by x ascending
// (y strictly descending), 32 * SLOTS entries per warp: SLOTS = 2 (FMAX) in
// the kernels every search runs, 4 (FMAX_BIG) in the variant a pass is re-run
// with when some cell outgrew FMAX.  Accessed through one 32-bit shared-window
// base per warp (ld/st.shared), so no generic addressing and no per-access
// rematerialization of the warp index.

__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

struct WarpFront {
    uint32_t bx, by, bk;   // shared-window addresses of this warp's arrays
    __device__ __forceinline__ double x(int j) const { return lds_f64(bx + 8u * j); }
    __device__ __forceinline__ double y(int j) const { return lds_f64(by + 8u * j); }
    __device__ __forceinline__ uint32_t k(int j) const { return lds_u32(bk + 4u * j); }
    __device__ __forceinline__ void put(int j, double vx, double vy, uint32_t vk) const {
        sts_f64(bx + 8u * j, vx);
        sts_f64(by + 8u * j, vy);
        sts_u32(bk + 4u * j, vk);
    }
};

template <int SLOTS>
__device__ __forceinline__ WarpFront warp_front(int w) {
    __shared__ double fx[DP_WARPS][32 * SLOTS];
    __shared__ double fy[DP_WARPS][32 * SLOTS];
    __shared__ uint32_t fk[DP_WARPS][32 * SLOTS];
    return WarpFront{(uint32_t)__cvta_generic_to_shared(&fx[w][0]),
                     (uint32_t)__cvta_generic_to_shared(&fy[w][0]),
                     (uint32_t)__cvta_generic_to_shared(&fk[w][0])};
}

__device__ __forceinline__ int log2_steps(int n) {
    // number of binary-search halvings covering n entries (n >= 1)
    return 32 - __clz(n);
}

// Is c dominated by the sorted frontier (n entries)?  Binary search for
// p = #entries before c in (x, y, key) order; dominated iff p > 0 and
// y[p-1] <= cy (y strictly decreases along the frontier).
__device__ __forceinline__ bool front_dominated(const WarpFront &f, int n, double cx, double cy,
                                                uint32_t ck) {
    int pos = 0;
    for (int st = 1 << (log2_steps(n) - 1); st > 0; st >>= 1)
        if (pos + st <= n && f.x(pos + st - 1) < cx) pos += st;
    if (pos < n && f.x(pos) == cx && (f.y(pos) < cy || (f.y(pos) == cy && f.k(pos) < ck))) ++pos;
    return pos > 0 && f.y(pos - 1) <= cy;
}

// Is the corner (tx, ty) strictly dominated: some entry with x <= tx,
// y <= ty and (x, y) != (tx, ty)?  Every candidate of a predecessor pair is
// componentwise >= its corner (max(ptf, tfc), max(ptb, tbc)), so a strictly
// dominated corner settles the whole pair without per-candidate tests.
__device__ __forceinline__ bool corner_dominated(const WarpFront &f, int n, double tx, double ty) {
    int pos = 0;   // #entries with x <= tx
    for (int st = 1 << (log2_steps(n) - 1); st > 0; st >>= 1)
        if (pos + st <= n && f.x(pos + st - 1) <= tx) pos += st;
    if (pos == 0) return false;
    const double ex = f.x(pos - 1), ey = f.y(pos - 1);
    return ey <= ty && (ex < tx || ey < ty);
}

// Warp-cooperative exact insert of c (same c in every lane); lane l owns
// slots l and l + 32 (the second only once the frontier exceeds 32).
// Returns the new size, or -1 beyond FMAX.
template <int SLOTS>
__device__ __forceinline__ int front_insert(const WarpFront &f, int n, int lane, double cx, double cy,
                                            uint32_t ck);

// the same for SLOTS = 4 (lane l owns slots l + 32 j), capacity FMAX_BIG
template <>
__device__ __forceinline__ int front_insert<4>(const WarpFront &f, int n, int lane, double cx,
                                               double cy, uint32_t ck) {
    double xs[4], ys[4];
    uint32_t ks[4], m[4];
    bool keep[4], lt[4];
    int pos_c = 0, tot = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int q = lane + 32 * j;
        const bool h = q < n;
        xs[j] = 0; ys[j] = 0; ks[j] = 0;
        if (h) { xs[j] = f.x(q); ys[j] = f.y(q); ks[j] = f.k(q); }
        keep[j] = h && !dominates(cx, cy, ck, xs[j], ys[j], ks[j]);
        m[j] = __ballot_sync(0xffffffffu, keep[j]);
        lt[j] = keep[j] && xs[j] < cx;
        pos_c += __popc(__ballot_sync(0xffffffffu, lt[j]));
        tot += __popc(m[j]);
    }
    const int nn = tot + 1;
    if (nn > FMAX_BIG) return -1;
    const uint32_t below = (1u << lane) - 1u;
    int p[4], acc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        p[j] = acc + __popc(m[j] & below) + (lt[j] ? 0 : 1);
        acc += __popc(m[j]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (keep[j]) f.put(p[j], xs[j], ys[j], ks[j]);
    if (lane == 0) f.put(pos_c, cx, cy, ck);
    __syncwarp();
    return nn;
}

template <>
__device__ __forceinline__ int front_insert<2>(const WarpFront &f, int n, int lane, double cx,
                                               double cy, uint32_t ck) {
    const bool h0 = lane < n;
    double x0 = 0, y0 = 0;
    uint32_t k0 = 0;
    if (h0) { x0 = f.x(lane); y0 = f.y(lane); k0 = f.k(lane); }
    if (n <= 32) {
        // c is not dominated here: it passed front_dominated against the
        // round's frontier, and every insert since was checked against it
        const bool keep0 = h0 && !dominates(cx, cy, ck, x0, y0, k0);
        const uint32_t m0 = __ballot_sync(0xffffffffu, keep0);
        const bool lt0 = keep0 && x0 < cx;
        const int pos_c = __popc(__ballot_sync(0xffffffffu, lt0));
        const int nn = __popc(m0) + 1;
        if (nn > FMAX) return -1;
        const int p0 = __popc(m0 & ((1u << lane) - 1u)) + (lt0 ? 0 : 1);
        __syncwarp();
        if (keep0) f.put(p0, x0, y0, k0);
        if (lane == 0) f.put(pos_c, cx, cy, ck);
        __syncwarp();
        return nn;
    }
    const bool h1 = lane + 32 < n;
    double x1 = 0, y1 = 0;
    uint32_t k1 = 0;
    if (h1) { x1 = f.x(lane + 32); y1 = f.y(lane + 32); k1 = f.k(lane + 32); }
    const bool keep0 = h0 && !dominates(cx, cy, ck, x0, y0, k0);
    const bool keep1 = h1 && !dominates(cx, cy, ck, x1, y1, k1);
    const uint32_t m0 = __ballot_sync(0xffffffffu, keep0);
    const uint32_t m1 = __ballot_sync(0xffffffffu, keep1);
    const bool lt0 = keep0 && x0 < cx, lt1 = keep1 && x1 < cx;
    const int pos_c = __popc(__ballot_sync(0xffffffffu, lt0)) + __popc(__ballot_sync(0xffffffffu, lt1));
    const int nn = __popc(m0) + __popc(m1) + 1;
    if (nn > FMAX) return -1;
    const uint32_t below = (1u << lane) - 1u;
    const int p0 = __popc(m0 & below) + (lt0 ? 0 : 1);
    const int p1 = __popc(m0) + __popc(m1 & below) + (lt1 ? 0 : 1);
    __syncwarp();
    if (keep0) f.put(p0, x0, y0, k0);
    if (keep1) f.put(p1, x1, y1, k1);
    if (lane == 0) f.put(pos_c, cx, cy, ck);
    __syncwarp();
    return nn;
}

// Lane of the lexicographically smallest (x, y, key) among lanes with
// `live`.  x, y >= 0, so their IEEE bit patterns order like the values: a
// cascade of 32-bit warp min-reductions (x high/low word, y high/low word,
// key) settles it, stopping as soon as one lane is left.
__device__ __forceinline__ bool lex_stage(bool &live, uint32_t &m, unsigned part) {
    const unsigned v = live ? part : 0xffffffffu;
    const unsigned mn = __reduce_min_sync(0xffffffffu, v);
    live = live && v == mn;
    m = __ballot_sync(0xffffffffu, live);
    return __popc(m) <= 1;
}

__device__ __forceinline__ int lex_min_lane(bool live, double x, double y, uint32_t k) {
    const unsigned long long xb = (unsigned long long)__double_as_longlong(x);
    const unsigned long long yb = (unsigned long long)__double_as_longlong(y);
    uint32_t m = __ballot_sync(0xffffffffu, live);
    if (__popc(m) > 1 && !lex_stage(live, m, (unsigned)(xb >> 32)) &&
        !lex_stage(live, m, (unsigned)xb) && !lex_stage(live, m, (unsigned)(yb >> 32)) &&
        !lex_stage(live, m, (unsigned)yb))
        lex_stage(live, m, k);
    return __ffs(m) - 1;
}

// Lower bounds on the largest raw forward / backward stage time of a group of
// stages (see dp_cell): k stages over span [lo, hi) with `dev` devices in all,
// so one of them holds at most devmax = dev - (k - 1).  Stage i runs at share
// m_i = BS // (q dev_i), q = MB R; with T >= m_i w_i for every stage (w_i its
// time per unit share), T >= sum w_i / sum 1/m_i and sum 1/m_i <=
// q dev / (BS - q devmax + 1) (floor(x/y) >= (x - y + 1)/y); also
// T >= t(lo, hi; m(devmax)) / k (times are monotone in the share), and
// sum w_i ~ t(lo, hi; m(devmax)) / m(devmax).  The factor (1 - 1e-9) absorbs
// the folds' rounding.  False when no share is positive at devmax.
template <bool DERIVED>
__device__ __forceinline__ bool group_bounds(const DPBatch &B, const CallDesc &cd,
                                             const int16_t *keyidx, int lo, int hi, int k, int dev,
                                             double &lf, double &lb) {
    const int devmax = dev - (k - 1);
    const int kx = keyidx[devmax];
    if (kx < 0) return false;
    const int64_t o = hm_idx(lo, hi);
    const int64_t q = (int64_t)cd.MB * cd.R;
    const int64_t mx = B.batch_size / (q * devmax);
    const double k1 = 1.0 / (double)k;
    const double k2 = (double)(B.batch_size - q * devmax + 1) / ((double)(q * dev) * (double)mx);
    const double kk = (1.0 - 1e-9) * (k1 > k2 ? k1 : k2);
    lf = __dmul_rn(fabs(B.key_tf[kx][o]), kk);
    lb = DERIVED ? __dmul_rn(B.beta, lf) : __dmul_rn(fabs(B.key_tb[kx][o]), kk);
    return true;
}

// the S - s stages after cell (b, d): [b, nb) on D - d devices
template <bool DERIVED>
__device__ __forceinline__ void suffix_bounds(const DPBatch &B, const CallDesc &cd,
                                              const int16_t *keyidx, int s, int b, int d,
                                              double &lf, double &lb) {
    if (!group_bounds<DERIVED>(B, cd, keyidx, b, B.nb, cd.S - s, cd.D - d, lf, lb)) lf = lb = 0.0;
}

// the s stages of cell (b, d): [0, b) on d devices
template <bool DERIVED>
__device__ __forceinline__ bool prefix_bounds(const DPBatch &B, const CallDesc &cd,
                                              const int16_t *keyidx, int s, int b, int d,
                                              double &lf, double &lb) {
    return group_bounds<DERIVED>(B, cd, keyidx, 0, b, s, d, lf, lb);
}

// One cell (b, d) = (s + idx / B, s + idx % B) of call c at level s, by one
// warp (w = its warp in the CTA), frontier capacity 32 * SLOTS.
template <bool DERIVED, int SLOTS>
__device__ __forceinline__ void dp_cell(const DPBatch &B, int s, int c, int64_t idx,
                                        const float2 *lbp = nullptr) {
    const CallDesc cd = B.calls[c];
    const int w = threadIdx.x >> 5;
    const int bi = (int)(idx / cd.B);
    const int di = (int)(idx % cd.B);
    const int lane = threadIdx.x & 31;
    const int b = s + bi;
    const int d = s + di;
    const int nb = B.nb;
    const int64_t cells = (int64_t)cd.A * cd.B;
    const int cur = s & 1, prv = (s - 1) & 1;
    const int16_t *keyidx = B.keyidx + cd.key_off;
    const int inter_d = (B.num_nodes > 1 && (unsigned)d % (unsigned)B.dpn == 0) ? 1 : 0;
    const int64_t row = (int64_t)b * (b - 1) / 2;       // hm_idx(0, b)
    const double beta = B.beta;
    const WarpFront F = warp_front<SLOTS>(w);
    // Objective bound (CallDesc.U, finite only with non-negative times and no
    // cost table): every completion of an entry (x, y) of this cell costs at
    // least max(x, lbf) + max(y, lbb), lbf a lower bound on the largest raw
    // forward time of the S - s stages still to come over [b, nb) with the
    // D - d devices left.  Stage i with dev_i devices runs at share
    // m_i = BS // (q dev_i), q = MB R, so its raw time is ~ m_i w_i with w_i
    // its time per unit share; T >= m_i w_i for all i gives
    //   T >= sum w_i / sum 1/m_i,   sum 1/m_i <= q (D - d) / (BS - q devmax + 1)
    // (floor(x/y) >= (x - y + 1)/y, dev_i <= devmax), and also
    //   T >= t(b, nb; m(devmax)) / (S - s)          (times monotone in m);
    // sum w_i ~ t(b, nb; m(devmax)) / m(devmax).  The factor (1 - 1e-9)
    // absorbs the folds' rounding.  Entries above U cannot lead to a plan at or
    // below U, so they are dropped; level S keeps only the final cell (nb, D).
    const double U = cd.U;
    const bool bounded = U < INFINITY;
    double lbf = 0.0, lbb = 0.0;
    if (bounded) {
        if (s == cd.S) {
            if (b != nb || d != cd.D) lbf = INFINITY;
        } else if (lbp) {               // listed by k_dp_triage with its suffix bounds
            const float2 v = *lbp;
            lbf = v.x;
            lbb = v.y;
        } else {
            suffix_bounds<DERIVED>(B, cd, keyidx, s, b, d, lbf, lbb);
        }
    }
    auto over = [&](double x, double y) {
        return bounded && __dadd_rn(dmax_ref(x, lbf), dmax_ref(y, lbb)) > U;
    };
    // (Cells whose whole frontier is above the bound -- the prefix lower bound,
    // see k_dp_triage -- never get here: bounded batches run only the cells
    // k_dp_triage listed.)
    int n = 0;
    bool ovf = false;
    bool zero = false;
    bool reach = false;    // bounded calls: the reference holds this cell non-empty
    uint32_t n_pairs = 0, n_cands = 0, n_ins = 0;
    uint32_t n_corner = 0, n_win = 0, n_rounds = 0, n_iters = 0;

    if (s == 1) {
        // level 0 holds the single cell (0, 0) with entry (0.0, 0.0) (stages.py:201)
        const int kk = keyidx[d];
        if (kk < 0) {
            zero = true;
        } else {
            const double tf = B.key_tf[kk][row];
            if (span_ok(tf, B.mono_skip)) {
                reach = true;
                double tfc = tf;
                if (b < nb) tfc = __dadd_rn(tf, B.key_cut[kk][inter_d * (nb + 1) + b]);
                const double tbc = DERIVED ? __dmul_rn(beta, tf) : B.key_tb[kk][row];
                if (!over(dmax_ref(0.0, tfc), dmax_ref(0.0, tbc))) {
                    if (lane == 0) F.put(0, dmax_ref(0.0, tfc), dmax_ref(0.0, tbc), pack_key(0, 0, 0));
                    __syncwarp();
                    n = 1;
                }
                n_pairs = lane == 0;
                n_cands = lane == 0;
            }
        }
    } else {
        // Predecessor columns d' in order; within a column only b' from
        // max(first non-empty b' of the column, first feasible lo of the key)
        // to min(last non-empty b', b - 1) can yield a candidate.  The frontier
        // is order-independent (see top), so this order is as good as the
        // reference's.
        const int base = s - 1;
        const uint8_t *pcnt = B.val_cnt[prv] + cd.val_off;
        const uint32_t *poff = B.val_off[prv] + cd.val_off;
        const double *qtf = B.pool_tf[prv] + cd.vpool_base;
        const double *qtb = B.pool_tb[prv] + cd.vpool_base;
        const double *stf = B.spill_tf[prv];
        const double *stb = B.spill_tb[prv];
        const int32_t *cmin = B.col_min[prv] + cd.col_off;
        const int32_t *cmax = B.col_max[prv] + cd.col_off;
        const double *tfrow_base = nullptr;
        // columns d' in descending order: the short last stages (dev = d - d'
        // small) come first and build a frontier that prunes the rest -- ~4x
        // fewer frontier inserts than ascending on the C5 chains (order does not
        // change the result: the dominance relation is order-independent)
        const int dpn = B.dpn;
        const bool multi_node = B.num_nodes > 1;
        int rem = (int)((unsigned)(d - 1) % (unsigned)dpn);
        for (int dp = d - 1; dp >= base; --dp, rem = rem == 0 ? dpn - 1 : rem - 1) {
            const int lo_col = cmin[dp - base];
            const int hi_col = cmax[dp - base];
            if (lo_col > hi_col || lo_col >= b) continue;           // no predecessor cell
            const int kk = keyidx[d - dp];                          // warp-uniform
            if (kk < 0) {                                           // m == 0 (stages.py:224-228)
                zero = true;
                continue;
            }
            const int bp_lo = max(lo_col, B.key_ffb[kk][b]);
            const int bp_hi = min(hi_col, b - 1);
            if (bp_lo > bp_hi) continue;                            // all spans infeasible
            const double *tfrow = B.key_tf[kk] + row;
            const double *tbrow = DERIVED ? nullptr : B.key_tb[kk] + row;
            const double cutf = b < nb ? B.key_cut[kk][inter_d * (nb + 1) + b] : 0.0;
            const double *cutb = B.key_cut[kk] + ((multi_node && rem == 0) ? (nb + 1) : 0);
            const uint8_t *ccol = pcnt + (int64_t)(dp - base) * cd.A - base;
            const uint32_t *ocol = poff + (int64_t)(dp - base) * cd.A - base;
            int lim = bp_lo - 1;          // b' <= lim are settled
            int lim_v = -1;               // insert count lim was computed at
            // One chunk of 32 predecessors b' in (top-32, top], minus an already
            // processed window [ex_lo, ex_hi].
            auto chunk = [&](int top, int ex_lo, int ex_hi) {
                const int bp = top - lane;
                int cnt = (bp > lim && bp >= bp_lo && (bp < ex_lo || bp > ex_hi))
                              ? cnt_entries(ccol[bp]) : 0;
                double tfc = 0.0, tbc = 0.0;
                int wlo = 0, whi = -1;
                const double *etf = qtf, *etb = qtb;
                int64_t pbase = 0;
                if (cnt > 0) {
                    const double tf = tfrow[bp];
                    if (span_ok(tf, B.mono_skip)) {                             // mem <= budget (stages.py:230)
                        tfc = b < nb ? __dadd_rn(tf, cutf) : tf;
                        tbc = DERIVED ? __dmul_rn(beta, tf) : tbrow[bp];
                        if (bp > 0) tbc = __dadd_rn(tbc, cutb[bp]);
                        ++n_pairs;
                        n_cands += cnt;
                        const uint32_t praw = ocol[bp];
                        pbase = (int64_t)(praw & ~SPILL_BIT);
                        if (praw & SPILL_BIT) { etf = stf; etb = stb; }
                        // every candidate of the pair is >= its ideal point: the
                        // predecessor frontier's smallest tf (entry 0) and smallest
                        // tb (last entry), each clipped by the new stage
                        const double ix = dmax_ref(etf[pbase], tfc);
                        const double iy = dmax_ref(etb[pbase + cnt - 1], tbc);
                        if ((n > 0 && corner_dominated(F, n, ix, iy)) || over(ix, iy)) {
                            if (PC_DP_DIAG) ++n_corner;
                        }
                        else {
                            // exact window: entries with ptf <= tfc collapse onto the
                            // last of them, entries with ptb <= tbc onto the first
                            // (ptf strictly ascending, ptb strictly descending:
                            // two branch-free binary searches)
                            int c0 = 0, c1 = 0;   // #{ptf <= tfc}, #{ptb > tbc}
                            for (int st = 1 << (log2_steps(cnt) - 1); st > 0; st >>= 1) {
                                if (c0 + st <= cnt && etf[pbase + c0 + st - 1] <= tfc) c0 += st;
                                if (c1 + st <= cnt && etb[pbase + c1 + st - 1] > tbc) c1 += st;
                            }
                            const int i0 = c0 - 1, i1 = c1;
                            if (i1 <= i0) { wlo = i1; whi = i1; }
                            else { wlo = i0 < 0 ? 0 : i0; whi = i1 < cnt ? i1 : cnt - 1; }
                        }
                    }
                }
                // Candidate work items (lane, window entry) compacted over the
                // warp: 32 per round whatever the lanes' window sizes (an
                // exclusive prefix over the lanes, then a 5-step shuffle search
                // for each item's owner).  The frontier does not depend on the
                // order candidates arrive in.
                const int cntw = whi - wlo + 1;
                int incl = cntw;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                const int excl = incl - cntw;
                const uint32_t pb32 = (uint32_t)pbase;           // pool offsets < 2^31
                const int spill = etf == stf ? 1 : 0;
                if (PC_DP_DIAG) {
                    n_win += cntw;
                    n_rounds += (total + 31) / 32;
                    ++n_iters;
                }
                for (int q0 = 0; q0 < total; q0 += 32) {
                    const int q = q0 + lane;
                    int ow = 0;                                  // lanes with incl <= q
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {
                        const int v = __shfl_sync(0xffffffffu, incl, ow + st - 1);
                        if (v <= q) ow += st;
                    }
                    const int o_excl = __shfl_sync(0xffffffffu, excl, ow);
                    const int o_wlo = __shfl_sync(0xffffffffu, wlo, ow);
                    const double o_tfc = __shfl_sync(0xffffffffu, tfc, ow);
                    const double o_tbc = __shfl_sync(0xffffffffu, tbc, ow);
                    const uint32_t o_pb = __shfl_sync(0xffffffffu, pb32, ow);
                    const int o_sp = __shfl_sync(0xffffffffu, spill, ow);
                    const int o_bp = __shfl_sync(0xffffffffu, bp, ow);
                    double cx = 0.0, cy = 0.0;
                    uint32_t ck = 0;
                    bool surv = false;
                    if (q < total) {
                        const int i = o_wlo + (q - o_excl);
                        const double *xt = o_sp ? stf : qtf;
                        const double *yt = o_sp ? stb : qtb;
                        cx = dmax_ref(xt[o_pb + i], o_tfc);
                        cy = dmax_ref(yt[o_pb + i], o_tbc);
                        ck = pack_key(o_bp, dp, i);
                        surv = (n == 0 || !front_dominated(F, n, cx, cy, ck)) && !over(cx, cy);
                    }
                    while (__any_sync(0xffffffffu, surv)) {
                        // insert the lexicographically smallest survivor first: nothing
                        // among the survivors can dominate it, and it removes the most
                        const int t = lex_min_lane(surv, cx, cy, ck);
                        const double tx = __shfl_sync(0xffffffffu, cx, t);
                        const double ty = __shfl_sync(0xffffffffu, cy, t);
                        const uint32_t tk = __shfl_sync(0xffffffffu, ck, t);
                        ++n_ins;
                        const int nn = front_insert<SLOTS>(F, n, lane, tx, ty, tk);
                        if (nn < 0 || nn > B.fmax_limit) ovf = true; else n = nn;
                        surv = surv && lane != t && !dominates(tx, ty, tk, cx, cy, ck);
                    }
                }
            };
            const int ex_lo = 1, ex_hi = 0;   // no excluded window
            // Scan b' downward from bp_hi.  Every candidate of pair b' is >= its
            // corner (tfc, tbc) and tbc >= t_bwd(b', b); t_fwd(b', b) and t_bwd
            // only grow as b' falls (a fold of non-negative terms), so "some
            // frontier entry strictly dominates (tf + cut(b), t_bwd)" holds on
            // a prefix of b': a 32-ary warp search finds its end, and b' up to
            // there are skipped without loading their predecessors.
            for (int top = bp_hi; top > lim; top -= 32) {
                if (B.mono_skip && (n > 0 || bounded) && (int)n_ins != lim_v) {
                    int lo_b = lim, hi_b = top + 1;   // cond true <= lo_b, false >= hi_b
                    while (hi_b - lo_b > 1) {
                        const int span = hi_b - lo_b - 1;
                        const int step = (span + 31) / 32;
                        const int p = lo_b + (lane + 1) * step;
                        bool cond = false;
                        if (p < hi_b) {
                            const double tv = fabs(tfrow[p]);
                            const double tfc = b < nb ? __dadd_rn(tv, cutf) : tv;
                            const double tbl = DERIVED ? __dmul_rn(beta, tv) : fabs(tbrow[p]);
                            cond = (n > 0 && corner_dominated(F, n, tfc, tbl)) || over(tfc, tbl);
                        }
                        const uint32_t m = __ballot_sync(0xffffffffu, cond);
                        const int k = __popc(m);              // a prefix of the lanes
                        if (k > 0) lo_b = lo_b + k * step;
                        const int nh = lo_b + step;           // first false sample
                        if (k < 32 && nh < hi_b) hi_b = nh;
                        if (lo_b >= hi_b - 1) break;
                    }
                    lim = lo_b;
                    lim_v = (int)n_ins;
                    if (top <= lim) break;
                }
                chunk(top, ex_lo, ex_hi);
            }
        }
        (void)tfrow_base;
    }
    // algorithmic work counters (one atomic per warp)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
        n_cands += __shfl_xor_sync(0xffffffffu, n_cands, o);
    }
    if (lane == 0) {
        unsigned long long *wk = B.counters + 8 + FMAX + 3 * (blockIdx.x & (WORK_SLOTS - 1));
        atomicAdd(&wk[0], (unsigned long long)n_pairs);
        atomicAdd(&wk[1], (unsigned long long)n_cands);
        atomicAdd(&wk[2], (unsigned long long)n_ins);
        if (PC_DP_DIAG) {
            atomicAdd(&B.counters[3 + min(n, FMAX)], 1ull);     // frontier-size histogram
            atomicAdd(&B.counters[4 + FMAX + 0], (unsigned long long)n_rounds);
            atomicAdd(&B.counters[4 + FMAX + 1], (unsigned long long)n_iters);
        }
    }
    if (PC_DP_DIAG) {
        unsigned a = n_corner, bw = n_win;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            bw += __shfl_xor_sync(0xffffffffu, bw, o);
        }
        if (lane == 0) {
            atomicAdd(&B.counters[4 + FMAX + 2], (unsigned long long)a);
            atomicAdd(&B.counters[4 + FMAX + 3], (unsigned long long)bw);
        }
    }
    if (bounded && s > 1 && n == 0) {
        // A bounded cell left without entries: the reference's emptiness and
        // zero-share flag come from the previous level's non-empty prefix
        // counts -- some non-empty (b' < b, d') with m == 0, and some with a
        // feasible span (b', b): b' >= first feasible lo, feasibility being
        // suffix-closed in b' for every key of a bounded batch (api.cu checks
        // it).  (With entries the cell is non-empty and the zero-share flag
        // is never read: the visit scan only asks it of empty cells.)
        const int base = s - 1;
        const int32_t *rp = B.reach_pre[prv] + cd.val_off;
        bool zl = false, rl = false;
        for (int dp = base + lane; dp < d; dp += 32) {
            const int32_t *col = rp + (int64_t)(dp - base) * cd.A - base;
            const int32_t upto = col[b - 1] & 0xffff;
            if (upto == 0) continue;
            const int kk = keyidx[d - dp];
            if (kk < 0) { zl = true; continue; }
            const int x = max(base, B.key_ffb[kk][b]);
            if (x <= b - 1 && upto > (x > base ? col[x - 1] & 0xffff : 0)) rl = true;
        }
        zero = __any_sync(0xffffffffu, zl);
        reach = __any_sync(0xffffffffu, rl);
    }
    const bool any_zero = __any_sync(0xffffffffu, zero);

    // emit the frontier (sorted by tf) into exact-size pool slots
    const int64_t cell = (int64_t)di * cd.A + bi;
    const int64_t hcell = cd.hist_off + (int64_t)(s - 1) * cells + cell;
    const int64_t vcell = cd.val_off + cell;
    if (ovf) n = 0;
    if (n > 0) {
        // exact-size slots in the call's region, or the shared spill pool
        unsigned long long vo = 0, ho = 0;
        if (lane == 0) {
            vo = atomicAdd(&B.vpool_used[cur][c], (unsigned long long)n);
            if ((int64_t)(vo + n) > cd.vpool_cap)
                vo = SPILL_BIT | atomicAdd(&B.vspill_used[cur], (unsigned long long)n);
            ho = atomicAdd(&B.hpool_used[c], (unsigned long long)n);
            if ((int64_t)(ho + n) > cd.hpool_cap)
                ho = SPILL_BIT | atomicAdd(B.hspill_used, (unsigned long long)n);
        }
        vo = __shfl_sync(0xffffffffu, vo, 0);
        ho = __shfl_sync(0xffffffffu, ho, 0);
        const bool vs = (vo & SPILL_BIT) != 0, hs = (ho & SPILL_BIT) != 0;
        const int64_t vi = (int64_t)(vo & ~(unsigned long long)SPILL_BIT);
        const int64_t hi2 = (int64_t)(ho & ~(unsigned long long)SPILL_BIT);
        if ((vs && vi + n > B.vspill_cap) || (hs && hi2 + n > B.hspill_cap)) {
            if (lane == 0) atomicOr(B.overflow, 2);
            n = 0;
        } else {
            double *otf = vs ? B.spill_tf[cur] + vi : B.pool_tf[cur] + cd.vpool_base + vi;
            double *otb = vs ? B.spill_tb[cur] + vi : B.pool_tb[cur] + cd.vpool_base + vi;
            uint32_t *okk = hs ? B.hspill + hi2 : B.hpool + cd.hpool_base + hi2;
            for (int j = lane; j < n; j += 32) {
                otf[j] = F.x(j);
                otb[j] = F.y(j);
                okk[j] = F.k(j);
            }
            if (lane == 0) {
                B.val_off[cur][vcell] = (uint32_t)vi | (vs ? SPILL_BIT : 0u);
                B.hist_off[hcell] = (uint32_t)hi2 | (hs ? SPILL_BIT : 0u);
                atomicMin(&B.col_min[cur][cd.col_off + di], b);
                atomicMax(&B.col_max[cur][cd.col_off + di], b);
            }
        }
    }
    if (lane == 0) {
        const uint8_t cnt_byte = n > 0 ? (uint8_t)n : (bounded && reach ? CNT_REACH : 0);
        const uint8_t byte = cnt_byte | (any_zero ? CNT_ZERO : 0);
        B.val_cnt[cur][vcell] = byte;
        B.hist_cnt[hcell] = byte;
        if (ovf) atomicOr(B.overflow, 1);
    }
}

template <bool DERIVED, int SLOTS>
__global__ void __launch_bounds__(DP_WARPS * 32, DP_MIN_BLOCKS) k_dp_level(DPBatch B, int s, int n_active) {
    const int64_t cta = blockIdx.x;                  // grid = cta_prefix[n_active]
    const int c = B.cta_call[cta];
    // warps take consecutive cells of the call in (b, d) order, so every warp
    // of the CTA has a cell whatever B is; heaviest cells (largest b: most
    // predecessors) are dispatched first so the level's tail is short
    const int64_t idx = (int64_t)B.calls[c].A * B.calls[c].B - 1 -
                        ((cta - B.cta_prefix[c]) * DP_WARPS + (threadIdx.x >> 5));
    if (idx < 0) return;                              // whole warp
    dp_cell<DERIVED, SLOTS>(B, s, c, idx);
}

// Bounded batches: a warp per LIVE cell only.  k_dp_triage settled every cell
// whose whole frontier is above its call's bound (thread per cell: flags
// only) and listed the others, heaviest first within each call; a persistent
// grid takes them in list order, one cell per warp per atomic pop (dynamic, so
// a warp that drew a heavy cell does not hold up the level's tail).
#ifndef PC_LIST_ATOMIC
#define PC_LIST_ATOMIC 1
#endif
#ifndef PC_LIST_GRAB
#define PC_LIST_GRAB 1          // consecutive list cells a warp takes per pop
#endif
template <bool DERIVED, int SLOTS, int MINB>
__global__ void __launch_bounds__(DP_WARPS * 32, MINB) k_dp_level_list(DPBatch B, int s) {
    const unsigned long long n = B.live_count[0];
    const int lane = threadIdx.x & 31;
    if (PC_LIST_ATOMIC) {
        for (;;) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(B.live_count + 1, (unsigned long long)PC_LIST_GRAB);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n) break;
            for (int g = 0; g < PC_LIST_GRAB && t + g < n; ++g) {
                const unsigned long long e = B.live[t + g];
                dp_cell<DERIVED, SLOTS>(B, s, (int)(e >> 40), (int64_t)(e & ((1ull << 40) - 1)),
                                        B.live_lb + t + g);
            }
        }
    } else {
        const unsigned long long stride = (unsigned long long)gridDim.x * DP_WARPS;
        for (unsigned long long t = (unsigned long long)blockIdx.x * DP_WARPS + (threadIdx.x >> 5);
             t < n; t += stride) {
            const unsigned long long e = B.live[t];
            dp_cell<DERIVED, SLOTS>(B, s, (int)(e >> 40), (int64_t)(e & ((1ull << 40) - 1)),
                                    B.live_lb + t);
        }
    }
}

// One thread per cell of the active calls of a bounded batch at level s: a
// cell that can only end without entries gets its count byte here --
// CNT_REACH or 0 for the reference's emptiness, plus the zero-share flag, from
// the previous level's non-empty prefix counts -- and every other cell is
// appended to the live list (warp-aggregated).  "Only without entries": for a
// bounded call, level S off the final cell, the prefix lower bound above U, or
// no column whose shortest feasible last stage from a predecessor with
// entries stays within U; for an unbounded call of the batch, no predecessor
// with entries in any column's feasible range.  (U = -inf, a call without a
// greedy plan, settles every cell but level 1's and the final one here.)
constexpr int TRIAGE_CALLS = 64;     // calls a triage CTA caches (cells of more: global search)
template <bool DERIVED>
__global__ void k_dp_triage(DPBatch B, int s, int n_active, const int64_t *cell_prefix) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    // the calls this CTA's cells belong to: their range of cell_prefix, found
    // once, then searched in shared memory
    __shared__ int s_c0, s_c1;
    __shared__ int64_t s_pre[TRIAGE_CALLS + 1];
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    if (threadIdx.x == 0) {
        int lo = 0, hi = n_active;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (cell_prefix[mid] <= g0) lo = mid; else hi = mid;
        }
        int c1 = lo;
        while (c1 + 1 < n_active && cell_prefix[c1 + 1] < g0 + blockDim.x && c1 - lo < TRIAGE_CALLS - 1) ++c1;
        s_c0 = lo;
        s_c1 = c1;
    }
    __syncthreads();
    const int c0 = s_c0, c1 = s_c1;
    for (int i = threadIdx.x; i <= c1 - c0 + 1; i += blockDim.x) s_pre[i] = cell_prefix[c0 + i];
    __syncthreads();
    bool live = false;
    int c = 0;
    int64_t idx = 0;
    float2 lb = make_float2(0.f, 0.f);
    if (g < cell_prefix[n_active]) {
        int lo = 0, hi = c1 - c0 + 1;
        if (g >= s_pre[hi]) {                      // past the cached calls (rare: many tiny calls)
            lo = c1 + 1;
            hi = n_active;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (cell_prefix[mid] <= g) lo = mid; else hi = mid;
            }
            c = lo;
        } else {
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= g) lo = mid; else hi = mid;
            }
            c = c0 + lo;
        }
        const CallDesc cd = B.calls[c];
        idx = (int64_t)cd.A * cd.B - 1 - (g - cell_prefix[c]);     // heaviest first
        const int bi = (int)(idx / cd.B), di = (int)(idx % cd.B);
        const int b = s + bi, d = s + di, nb = B.nb;
        const int16_t *keyidx = B.keyidx + cd.key_off;
        bool dead = false;
        if (cd.U < INFINITY) {
            if (s == cd.S) {
                dead = b != nb || d != cd.D;
            } else {
                // suffix_bounds / prefix_bounds with this level's factors
                const double2 fk = B.lvl_kk[cd.col_off + di];
                const short2 fx = B.lvl_kx[cd.col_off + di];
                double lbf = 0.0, lbb = 0.0;
                if (fx.x >= 0) {
                    const int64_t o = hm_idx(b, nb);
                    lbf = __dmul_rn(fabs(B.key_tf[fx.x][o]), fk.x);
                    lbb = DERIVED ? __dmul_rn(B.beta, lbf) : __dmul_rn(fabs(B.key_tb[fx.x][o]), fk.x);
                }
                if (s > 1 && fx.y >= 0) {
                    const int64_t o = hm_idx(0, b);
                    const double plf = __dmul_rn(fabs(B.key_tf[fx.y][o]), fk.y);
                    const double plb = DERIVED ? __dmul_rn(B.beta, plf) : __dmul_rn(fabs(B.key_tb[fx.y][o]), fk.y);
                    dead = __dadd_rn(dmax_ref(plf, lbf), dmax_ref(plb, lbb)) > cd.U;
                }
                if (s > 1 && !dead) {
                    // A column can only contribute through a predecessor with
                    // entries among its feasible spans, and every candidate of
                    // it is >= the corner of its shortest such span, (b_max, b)
                    // with b_max the column's last non-empty b' (below b): if
                    // that corner is already above the bound -- or no column
                    // has such a predecessor -- dp_cell would load no pair and
                    // end empty (the reference's emptiness, below, is the
                    // same either way).
                    const int base = s - 1;
                    const int32_t *rp = B.reach_pre[(s - 1) & 1] + cd.val_off;
                    const int32_t *cmax = B.col_max[(s - 1) & 1] + cd.col_off;
                    const int64_t row = (int64_t)b * (b - 1) / 2;
                    const int inter_d = (B.num_nodes > 1 && (unsigned)d % (unsigned)B.dpn == 0) ? 1 : 0;
                    bool alive = false;
                    for (int dp = d - 1; dp >= base && !alive; --dp) {
                        const int32_t *col = rp + (int64_t)(dp - base) * cd.A - base;
                        const int32_t upto = col[b - 1] >> 16;
                        if (upto == 0) continue;
                        const int kk = keyidx[d - dp];
                        if (kk < 0) continue;
                        const int x = max(base, B.key_ffb[kk][b]);
                        if (!(x <= b - 1 && upto > (x > base ? col[x - 1] >> 16 : 0))) continue;
                        const int bp = min(cmax[dp - base], b - 1);
                        const double tf = B.key_tf[kk][row + bp];
                        const double tfc = b < nb ? __dadd_rn(tf, B.key_cut[kk][inter_d * (nb + 1) + b]) : tf;
                        double tbc = DERIVED ? __dmul_rn(B.beta, tf) : B.key_tb[kk][row + bp];
                        if (bp > 0) {
                            const int inter_p = (B.num_nodes > 1 && (unsigned)dp % (unsigned)B.dpn == 0) ? 1 : 0;
                            tbc = __dadd_rn(tbc, B.key_cut[kk][inter_p * (nb + 1) + bp]);
                        }
                        alive = !(__dadd_rn(dmax_ref(tfc, lbf), dmax_ref(tbc, lbb)) > cd.U);
                    }
                    dead = !alive;
                }
                // handed to dp_cell rounded down: still lower bounds
                lb = make_float2(__double2float_rd(lbf), __double2float_rd(lbb));
            }
        } else if (s > 1) {
            // an unbounded call of the batch (no greedy plan: typically one
            // that fits nowhere): a cell without a predecessor holding entries
            // among its feasible spans ends empty -- settled here as well
            const int base = s - 1;
            const int32_t *rp = B.reach_pre[(s - 1) & 1] + cd.val_off;
            bool pred = false;
            for (int dp = d - 1; dp >= base && !pred; --dp) {
                const int32_t *col = rp + (int64_t)(dp - base) * cd.A - base;
                const int32_t upto = col[b - 1] >> 16;
                if (upto == 0) continue;
                const int kk = keyidx[d - dp];
                if (kk < 0) continue;
                const int x = max(base, B.key_ffb[kk][b]);
                pred = x <= b - 1 && upto > (x > base ? col[x - 1] >> 16 : 0);
            }
            dead = !pred;
        }
        if (dead) {
            bool reach = false, zero = false;
            if (s == 1) {
                const int kk = keyidx[d];
                if (kk < 0) zero = true;
                else reach = span_ok(B.key_tf[kk][(int64_t)b * (b - 1) / 2], B.mono_skip);
            } else {
                const int base = s - 1;
                const int32_t *rp = B.reach_pre[(s - 1) & 1] + cd.val_off;
                // columns by share: m == 0 exactly for the widest last stages
                // (dev above a threshold), so the zero-share ones come first
                // in d' ascending -- each test stops at its first hit
                int dp = base;
                for (; dp < d && keyidx[d - dp] < 0; ++dp)
                    if (!zero) zero = (rp[(int64_t)(dp - base) * cd.A - base + b - 1] & 0xffff) != 0;
                for (int dq = d - 1; dq >= dp && !reach; --dq) {
                    const int32_t *col = rp + (int64_t)(dq - base) * cd.A - base;
                    const int32_t upto = col[b - 1] & 0xffff;
                    if (upto == 0) continue;
                    const int kk = keyidx[d - dq];
                    const int x = max(base, B.key_ffb[kk][b]);
                    reach = x <= b - 1 && upto > (x > base ? col[x - 1] & 0xffff : 0);
                }
            }
            const int64_t cell = (int64_t)di * cd.A + bi;
            const uint8_t byte = (reach ? CNT_REACH : 0) | (zero ? CNT_ZERO : 0);
            B.val_cnt[s & 1][cd.val_off + cell] = byte;
            B.hist_cnt[cd.hist_off + (int64_t)(s - 1) * cd.A * cd.B + cell] = byte;
        } else {
            live = true;
        }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, live);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(B.live_count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (live) {
        const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
        B.live[at] = ((unsigned long long)c << 40) | (unsigned long long)idx;
        B.live_lb[at] = lb;
    }
}

// Per (active call, column d) of level s: group_bounds' key and factor for
// the suffix (S - s stages over [b, nb) on D - d devices) and the prefix (s
// stages over [0, b) on d devices) -- they do not depend on b, so the
// triage's cells read them instead of recomputing three divisions each.
__global__ void k_level_factors(DPBatch B, int s, int n_active, const int64_t *col_prefix) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= col_prefix[n_active]) return;
    int lo = 0, hi = n_active;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (col_prefix[mid] <= g) lo = mid; else hi = mid;
    }
    const CallDesc cd = B.calls[lo];
    const int di = (int)(g - col_prefix[lo]);
    const int d = s + di;
    const int16_t *keyidx = B.keyidx + cd.key_off;
    auto factor = [&](int k, int dev, double &kk) -> int {
        const int devmax = dev - (k - 1);
        if (k < 1 || devmax < 1) return -1;
        const int kx = keyidx[devmax];
        if (kx < 0) return -1;
        const int64_t q = (int64_t)cd.MB * cd.R;
        const int64_t mx = B.batch_size / (q * devmax);
        const double k1 = 1.0 / (double)k;
        const double k2 = (double)(B.batch_size - q * devmax + 1) / ((double)(q * dev) * (double)mx);
        kk = (1.0 - 1e-9) * (k1 > k2 ? k1 : k2);
        return kx;
    };
    double ks = 0.0, kp = 0.0;
    const int xs = s < cd.S ? factor(cd.S - s, cd.D - d, ks) : -1;
    const int xp = factor(s, d, kp);
    B.lvl_kk[cd.col_off + di] = make_double2(ks, kp);
    B.lvl_kx[cd.col_off + di] = make_short2((short)xs, (short)xp);
}

void launch_level_factors(const DPBatch &b, int s, int n_active, int64_t n_cols,
                          const int64_t *col_prefix, cudaStream_t st) {
    if (n_cols > 0)
        k_level_factors<<<(unsigned)((n_cols + 255) / 256), 256, 0, st>>>(b, s, n_active, col_prefix);
}

void launch_dp_triage(const DPBatch &b, int s, int n_active, int64_t n_cells,
                      const int64_t *cell_prefix, bool derived, cudaStream_t st) {
    if (n_cells <= 0) return;
    const unsigned blocks = (unsigned)((n_cells + 255) / 256);
    if (derived)
        k_dp_triage<true><<<blocks, 256, 0, st>>>(b, s, n_active, cell_prefix);
    else
        k_dp_triage<false><<<blocks, 256, 0, st>>>(b, s, n_active, cell_prefix);
}

// Resident CTAs per SM of the list kernel: 8 (64 registers) on the headline's
// batches, 10 (48 registers, more spills, more warps to hide the loads) on
// batches with very many levels -- r2db: 4096 x 256 499 vs 502 ms, 4096 x
// 1024 3450 vs 3258 ms of DP.
void launch_dp_level_list(const DPBatch &b, int s, int sm_count, bool deep, bool derived, bool big,
                          cudaStream_t st) {
    const int tpb = DP_WARPS * 32;
    if (big) {
        const int n = sm_count * DP_LIST_MIN_BLOCKS;
        if (derived) k_dp_level_list<true, 4, DP_LIST_MIN_BLOCKS><<<n, tpb, 0, st>>>(b, s);
        else k_dp_level_list<false, 4, DP_LIST_MIN_BLOCKS><<<n, tpb, 0, st>>>(b, s);
    } else if (deep) {
        const int n = sm_count * DP_LIST_MIN_BLOCKS_DEEP;
        if (derived) k_dp_level_list<true, 2, DP_LIST_MIN_BLOCKS_DEEP><<<n, tpb, 0, st>>>(b, s);
        else k_dp_level_list<false, 2, DP_LIST_MIN_BLOCKS_DEEP><<<n, tpb, 0, st>>>(b, s);
    } else {
        const int n = sm_count * DP_LIST_MIN_BLOCKS;
        if (derived) k_dp_level_list<true, 2, DP_LIST_MIN_BLOCKS><<<n, tpb, 0, st>>>(b, s);
        else k_dp_level_list<false, 2, DP_LIST_MIN_BLOCKS><<<n, tpb, 0, st>>>(b, s);
    }
}

// CTA -> call of a batch, once per batch: the active calls of every level are
// a prefix of the batch's calls, so the map holds for all levels.
__global__ void k_cta_call(const int64_t *prefix, int n, int32_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= prefix[n]) return;
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (prefix[mid] <= i) lo = mid; else hi = mid;
    }
    out[i] = lo;
}

void launch_cta_call(const int64_t *prefix, int n, int64_t total, int32_t *out, cudaStream_t st) {
    if (total > 0) k_cta_call<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(prefix, n, out);
}

void launch_dp_level(const DPBatch &b, int s, int n_active, int64_t n_ctas, bool derived,
                     bool big, cudaStream_t st) {
    const int tpb = DP_WARPS * 32;
    const unsigned blocks = (unsigned)n_ctas;
    if (big) {
        if (derived) k_dp_level<true, 4><<<blocks, tpb, 0, st>>>(b, s, n_active);
        else k_dp_level<false, 4><<<blocks, tpb, 0, st>>>(b, s, n_active);
    } else {
        if (derived) k_dp_level<true, 2><<<blocks, tpb, 0, st>>>(b, s, n_active);
        else k_dp_level<false, 2><<<blocks, tpb, 0, st>>>(b, s, n_active);
    }
}

// ---------------------------------------------------------------- bound: U from a plan
// The objective the DP gives one complete path -- the plan (lo, hi, devices)
// of each listed call -- with this batch's key tables: per stage the charged
// times exactly as k_dp_level forms a candidate (raw span time, + cut(hi) at
// the stage's end, + cut(lo) at its start, inter-node flags from the running
// device count), max-folded from the level-0 entry (0, 0), then tf + tb.  Any
// path is one of the DP's plans, so the result bounds the call's optimum.
// One thread per call; +inf if a stage has a zero share or an infeasible span.
template <bool DERIVED>
__global__ void k_plan_bound(DPBatch Bt, int n, const int32_t *pos, const int32_t *seg_off,
                             const int32_t *lo, const int32_t *hi, const int32_t *dev,
                             double *U) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const CallDesc cd = Bt.calls[pos[t]];
    const int16_t *keyidx = Bt.keyidx + cd.key_off;
    const int nb = Bt.nb;
    double mf = 0.0, mb = 0.0;
    int cum = 0;
    for (int k = 0; k < cd.S; ++k) {
        const int q = seg_off[t] + k;
        const int a = lo[q], z = hi[q], dv = dev[q];
        const int prev = cum;
        cum += dv;
        const int kk = (dv >= 1 && dv <= cd.B) ? keyidx[dv] : -1;
        if (kk < 0) { U[t] = INFINITY; return; }
        const int64_t o = hm_idx(a, z);
        const double tf = Bt.key_tf[kk][o];
        if (!span_ok(tf, Bt.mono_skip)) { U[t] = INFINITY; return; }
        double tfc = tf;
        if (z < nb) {
            const int inter = (Bt.num_nodes > 1 && cum % Bt.dpn == 0) ? 1 : 0;
            tfc = __dadd_rn(tf, Bt.key_cut[kk][inter * (nb + 1) + z]);
        }
        double tbc = DERIVED ? __dmul_rn(Bt.beta, tf) : Bt.key_tb[kk][o];
        if (a > 0) {
            const int inter = (Bt.num_nodes > 1 && prev % Bt.dpn == 0) ? 1 : 0;
            tbc = __dadd_rn(tbc, Bt.key_cut[kk][inter * (nb + 1) + a]);
        }
        mf = dmax_ref(mf, tfc);
        mb = dmax_ref(mb, tbc);
    }
    U[t] = __dadd_rn(mf, mb);
}

void launch_plan_bound(const DPBatch &b, int n, const int32_t *pos, const int32_t *seg_off,
                       const int32_t *lo, const int32_t *hi, const int32_t *dev, double *U,
                       bool derived, cudaStream_t st) {
    if (n <= 0) return;
    if (derived)
        k_plan_bound<true><<<(n + 127) / 128, 128, 0, st>>>(b, n, pos, seg_off, lo, hi, dev, U);
    else
        k_plan_bound<false><<<(n + 127) / 128, 128, 0, st>>>(b, n, pos, seg_off, lo, hi, dev, U);
}

// ---------------------------------------------------------------- bound: greedy plan
// Calls without a partner plan (the first MB wave, or an infeasible partner):
// a plan from bisection on a stage cost T.  Stage i gets D / S devices, one
// more for the first D % S stages (S stages, D devices, each <= B).  pack(T)
// walks the blocks left to right: stage i ends at the largest hi -- leaving a
// block for each later stage, the last stage ending at nb -- whose span fits
// and whose charged forward + backward time is <= T, scanning hi upward until
// the raw forward time alone passes T (raw times grow with the span).  The
// DP objective of the plan packed at the smallest T found (max-folded charged
// times as in k_plan_bound) bounds the optimum; +inf if nothing packs.  One
// CTA per call: the search for the smallest T that packs is GB_WARPS-wide
// (each warp packs one candidate T per round), so a call needs 1 + GB_ROUNDS
// + 1 sequential packs instead of the ~16 of a bisection.
constexpr int GB_WARPS = 8;     // T values a call tries at once
constexpr int GB_ROUNDS = 5;    // 9^5 = 59049: finer than 14 halvings
template <bool DERIVED>
__global__ void __launch_bounds__(GB_WARPS * 32) k_greedy_bound(DPBatch Bt, int n, const int32_t *pos,
                                                                double *U) {
    const int w = blockIdx.x;
    const int wi = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    __shared__ int s_res[GB_WARPS];
    if (w >= n) return;
    const CallDesc cd = Bt.calls[pos[w]];
    const int16_t *keyidx = Bt.keyidx + cd.key_off;
    const int nb = Bt.nb, S = cd.S, D = cd.D;
    const int q = D / S, r = D % S;
    const int kq = keyidx[q], kq1 = r > 0 ? keyidx[q + 1] : kq;
    // the D % S extra devices go to the first stages (blockIdx.y == 0), the
    // last ones (1) or spread evenly (2); the host keeps the best plan
    const int pat = blockIdx.y;
    U += (int64_t)pat * n;
    if (kq < 0 || kq1 < 0) {
        if (threadIdx.x == 0) U[w] = INFINITY;
        return;
    }
    auto extras_before = [&](int i) {          // extra devices among stages < i
        return pat == 0 ? min(i, r) : pat == 1 ? max(0, i - (S - r))
                                               : (int)(((int64_t)i * r) / S);
    };
    auto extra = [&](int i) { return extras_before(i + 1) > extras_before(i); };
    auto before_devs = [&](int i) { return i * q + extras_before(i); };
    // charged times of stage i = [lo, hi) (k_plan_bound's arithmetic)
    auto charged = [&](int i, int lo, int hi, double &tfc, double &tbc, double &raw) -> bool {
        const int kk = extra(i) ? kq1 : kq;
        const int before = before_devs(i), after = before + q + (extra(i) ? 1 : 0);
        const int64_t o = hm_idx(lo, hi);
        const double tf = Bt.key_tf[kk][o];
        raw = fabs(tf);
        tfc = tf;
        if (hi < nb) {
            const int inter = (Bt.num_nodes > 1 && after % Bt.dpn == 0) ? 1 : 0;
            tfc = __dadd_rn(tf, Bt.key_cut[kk][inter * (nb + 1) + hi]);
        }
        tbc = DERIVED ? __dmul_rn(Bt.beta, tf) : Bt.key_tb[kk][o];
        if (lo > 0) {
            const int inter = (Bt.num_nodes > 1 && before % Bt.dpn == 0) ? 1 : 0;
            tbc = __dadd_rn(tbc, Bt.key_cut[kk][inter * (nb + 1) + lo]);
        }
        return span_ok(tf, Bt.mono_skip);
    };
    // pack(T): true if S stages cover [0, nb); with `eval`, the plan's objective
    // pack(T): 1 if S stages cover [0, nb), 0 if T is too small, -1 to give up
    // (a stage whose one-block span does not fit and that found no fitting span
    // at all: memory, not T, is what fails -- no bound then)
    auto pack = [&](double T, bool eval, double &obj) -> int {
        int lo = 0;
        double mf = 0.0, mb = 0.0;
        for (int i = 0; i < S; ++i) {
            const int last = nb - (S - 1 - i);
            int best = -1;
            bool any_fit = false;
            if (i == S - 1) {
                double tfc, tbc, raw;
                const bool ok = charged(i, lo, nb, tfc, tbc, raw);
                any_fit = ok;
                if (ok && __dadd_rn(tfc, tbc) <= T) best = nb;
            } else {
                for (int h0 = lo + 1; h0 <= last; h0 += 32) {
                    const int h = h0 + lane;
                    bool good = false, stop = false, fit = false;
                    if (h <= last) {
                        double tfc, tbc, raw;
                        fit = charged(i, lo, h, tfc, tbc, raw);
                        good = fit && __dadd_rn(tfc, tbc) <= T;
                        stop = raw > T;
                    }
                    const uint32_t gm = __ballot_sync(0xffffffffu, good);
                    if (gm) best = h0 + 31 - __clz(gm);
                    any_fit = any_fit || __any_sync(0xffffffffu, fit);
                    if (__ballot_sync(0xffffffffu, stop)) break;
                }
            }
            if (best < 0) {
                if (!any_fit) {
                    double tfc, tbc, raw;
                    if (!charged(i, lo, lo + 1, tfc, tbc, raw)) return -1;
                }
                return 0;
            }
            if (eval) {
                double tfc, tbc, raw;
                charged(i, lo, best, tfc, tbc, raw);
                mf = dmax_ref(mf, tfc);
                mb = dmax_ref(mb, tbc);
            }
            lo = best;
        }
        obj = __dadd_rn(mf, mb);
        return 1;
    };
    double obj = INFINITY, dummy;
    // a T that packs: from the balanced estimate (1 + beta) t(0, nb) / S, the
    // warps trying its doublings at once (the first that packs wins; a give-up
    // before it ends the search); then the (GB_WARPS + 1)-ary search down
    const double total = fabs(Bt.key_tf[kq][hm_idx(0, nb)]);
    const double T0 = 1.5 * (1.0 + Bt.beta) * total / S + 1e-300;
    {
        const int r0 = pack(ldexp(T0, wi), false, dummy);
        if (lane == 0) s_res[wi] = r0;
    }
    __syncthreads();
    int tries = -1;
    for (int j = 0; j < GB_WARPS; ++j)
        if (s_res[j] != 0) {
            if (s_res[j] > 0) tries = j;
            break;
        }
    if (tries < 0) {
        if (threadIdx.x == 0) U[w] = INFINITY;
        return;
    }
    double hiT = ldexp(T0, tries);
    double loT = tries ? 0.5 * hiT : 0.0;
    for (int round = 0; round < GB_ROUNDS; ++round) {
        __syncthreads();                        // s_res of the previous round read
        const double Tw = loT + (hiT - loT) * (double)(wi + 1) / (double)(GB_WARPS + 1);
        const int r = pack(Tw, false, dummy);
        if (lane == 0) s_res[wi] = r;
        __syncthreads();
        double nlo = loT, nhi = hiT;            // the smallest packing point, the failure below it
        for (int j = GB_WARPS - 1; j >= 0; --j) {
            const double Tj = loT + (hiT - loT) * (double)(j + 1) / (double)(GB_WARPS + 1);
            if (s_res[j] > 0) {
                nhi = Tj;
            } else {
                nlo = Tj;
                break;
            }
        }
        loT = nlo;
        hiT = nhi;
    }
    if (wi == 0) {
        const bool ok = pack(hiT, true, obj) > 0;
        if (lane == 0) U[w] = ok ? obj : INFINITY;
    }
}

void launch_greedy_bound(const DPBatch &b, int n, const int32_t *pos, double *U, bool derived,
                         cudaStream_t st) {
    if (n <= 0) return;
    const dim3 grid((unsigned)n, GB_SPLITS);     // U holds [GB_SPLITS][n]
    if (derived)
        k_greedy_bound<true><<<grid, GB_WARPS * 32, 0, st>>>(b, n, pos, U);
    else
        k_greedy_bound<false><<<grid, GB_WARPS * 32, 0, st>>>(b, n, pos, U);
}

// ---------------------------------------------------------------- bound: non-empty prefix
// Bounded batches: per (call, d column) the inclusive prefix count over b of
// the cells of level s the reference holds non-empty (count > 0 or CNT_REACH),
// read by level s + 1 for its emptiness and zero-share flags.  One warp per
// column, 32 cells per step.
__global__ void k_reach_prefix(DPBatch Bt, int s, int n_active, const int64_t *col_prefix) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= col_prefix[n_active]) return;
    int lo = 0, hi = n_active;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (col_prefix[mid] <= g) lo = mid; else hi = mid;
    }
    const CallDesc cd = Bt.calls[lo];
    const int di = (int)(g - col_prefix[lo]);
    const int cur = s & 1;
    const uint8_t *vcol = Bt.val_cnt[cur] + cd.val_off + (int64_t)di * cd.A;
    int32_t *pcol = Bt.reach_pre[cur] + cd.val_off + (int64_t)di * cd.A;
    int32_t run = 0;
    for (int b0 = 0; b0 < cd.A; b0 += 32) {
        const int bi = b0 + lane;
        // low half: cells the reference holds non-empty (count > 0 or
        // CNT_REACH); high half: cells with entries (A <= 16383 keeps the
        // two prefix counts apart)
        const uint8_t byte = bi < cd.A ? vcol[bi] : 0;
        const int v = ((byte & CNT_MASK) != 0 ? 1 : 0) | (cnt_entries(byte) > 0 ? 1 << 16 : 0);
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (bi < cd.A) pcol[bi] = run + incl;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
}

void launch_reach_prefix(const DPBatch &b, int s, int n_active, int64_t n_cols,
                         const int64_t *col_prefix, cudaStream_t st) {
    if (n_cols > 0)
        k_reach_prefix<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(b, s, n_active,
                                                                             col_prefix);
}

// ---------------------------------------------------------------- pruning cut
// With pruning the reference ends a row (s, b) at its first empty cell that
// saw no zero-share candidate, scanning d down, and the cells below are never
// created (stages.py:244-251); at level 1 the floor d_min = d + 1 also holds
// for every later row.  Memory growing with the share makes those cells empty
// anyway, so the DP computes whole rows; measured cost tables break that
// (an act_bytes entry can make a larger share fit where a smaller one did
// not), and then the level is cut here before the next one reads it:
//   k_cut_rows   e(row) = largest di that ends the row (-1: none)
//   k_cut_level1 e(row) = prefix max of e over the call's rows (the carried d_min)
//   k_cut_cols   cells di <= e(row) lose their entries (count 0, zero-share
//                flag kept so the visit scan sees the reference's rows), and the
//                per-column non-empty b range the next level reads is rebuilt.
__device__ __forceinline__ int call_of(const int64_t *prefix, int n, int64_t x) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (prefix[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void k_cut_rows(DPBatch Bt, int s, int n_active, const int64_t *row_prefix,
                           int32_t *row_e) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= row_prefix[n_active]) return;
    const int c = call_of(row_prefix, n_active, r);
    const CallDesc cd = Bt.calls[c];
    const int bi = (int)(r - row_prefix[c]);
    const uint8_t *cell = Bt.val_cnt[s & 1] + cd.val_off + bi;
    int e = -1;
    for (int di = cd.B - 1; di >= 0; --di) {
        const uint8_t v = cell[(int64_t)di * cd.A];
        if ((v & CNT_MASK) == 0 && !(v & CNT_ZERO)) {
            e = di;
            break;
        }
    }
    row_e[r] = e;
}

__global__ void k_cut_level1(DPBatch Bt, int n_active, const int64_t *row_prefix, int32_t *row_e) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_active) return;
    int32_t *e = row_e + row_prefix[c];
    int run = -1;
    for (int bi = 0; bi < Bt.calls[c].A; ++bi) {
        run = max(run, e[bi]);
        e[bi] = run;
    }
}

__global__ void k_cut_cols(DPBatch Bt, int s, int n_active, const int64_t *col_prefix,
                           const int64_t *row_prefix, const int32_t *row_e) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= col_prefix[n_active]) return;
    const int c = call_of(col_prefix, n_active, g);
    const CallDesc cd = Bt.calls[c];
    const int di = (int)(g - col_prefix[c]);
    const int cur = s & 1;
    uint8_t *vcol = Bt.val_cnt[cur] + cd.val_off + (int64_t)di * cd.A;
    uint8_t *hcol = Bt.hist_cnt + cd.hist_off + (int64_t)(s - 1) * cd.A * cd.B + (int64_t)di * cd.A;
    const int32_t *e = row_e + row_prefix[c];
    int mn = 0x7f7f7f7f, mx = -1;
    for (int bi = lane; bi < cd.A; bi += 32) {
        uint8_t v = vcol[bi];
        if ((v & CNT_MASK) == 0) continue;
        if (di <= e[bi]) {
            v &= (uint8_t)CNT_ZERO;
            vcol[bi] = v;
            hcol[bi] = v;
            continue;
        }
        mn = min(mn, s + bi);
        mx = max(mx, s + bi);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
        Bt.col_min[cur][cd.col_off + di] = mn;
        Bt.col_max[cur][cd.col_off + di] = mx;
    }
}

int launch_prune_cut(const DPBatch &b, int s, int n_active, int64_t n_rows, int64_t n_cols,
                     const int64_t *row_prefix, const int64_t *col_prefix, int32_t *row_e,
                     cudaStream_t st) {
    if (n_rows <= 0) return 0;
    k_cut_rows<<<(unsigned)((n_rows + 127) / 128), 128, 0, st>>>(b, s, n_active, row_prefix, row_e);
    int launches = 1;
    if (s == 1) {
        k_cut_level1<<<(n_active + 127) / 128, 128, 0, st>>>(b, n_active, row_prefix, row_e);
        ++launches;
    }
    k_cut_cols<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(b, s, n_active, col_prefix,
                                                                      row_prefix, row_e);
    return launches + 1;
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
    int64_t key = -1;                 // level_sums slot of this row, -1: none
    unsigned long long v = 0;
    if (r < call_row_prefix[Bt.n_calls]) {
        int lo = 0, hi = Bt.n_calls;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (call_row_prefix[mid] <= r) lo = mid; else hi = mid;
        }
        const int c = lo;
        const int A = Bt.calls[c].A, B = Bt.calls[c].B;
        const int64_t rl = r - call_row_prefix[c];
        const int s = 1 + (int)(rl / A);
        const int bi = (int)(rl % A);
        if (s > 1) {                      // level 1 carries d_min: k_visit_level1
            const uint8_t *row = Bt.hist_cnt + Bt.calls[c].hist_off + (int64_t)(s - 1) * A * B + bi;
            int dead;
            v = (unsigned long long)row_visits(row, A, s, s + bi, B, 0, pruning, &dead);
            key = level_off[c] + s - 1;
        }
    }
    // consecutive rows share their (call, level) slot: one atomic per warp then
    // (every row of a level adding to one address was the kernel's bottleneck)
    const int64_t k0 = __shfl_sync(0xffffffffu, key, 0);
    if (__all_sync(0xffffffffu, key == k0)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && k0 >= 0)
            atomicAdd((unsigned long long *)&level_sums[k0], v);
    } else if (key >= 0) {
        atomicAdd((unsigned long long *)&level_sums[key], v);
    }
}

// Level 1 carries d_min from row to row (stages.py:205-209, 247-248): one
// warp per call walks the rows in order, each row scanned 32 cells per ballot
// from the top for its first dead cell.
__global__ void k_visit_level1(DPBatch Bt, int pruning, const int64_t *level_off,
                               int64_t *level_sums) {
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= Bt.n_calls) return;
    const CallDesc cd = Bt.calls[c];
    const uint8_t *lvl = Bt.hist_cnt + cd.hist_off;
    int64_t total = 0;
    int d_min = 1;
    for (int bi = 0; bi < cd.A; ++bi) {
        const int bottom_di = d_min - 1;               // max(d_min, s) - 1 with s = 1
        if (bottom_di > cd.B - 1) continue;            // empty d range: no visits
        int stop = bottom_di, dead = -1;
        if (pruning) {
            for (int top = cd.B - 1; top >= bottom_di; top -= 32) {
                const int di = top - lane;
                bool is_dead = false;
                if (di >= bottom_di) {
                    const uint8_t v = lvl[(int64_t)di * cd.A + bi];
                    is_dead = (v & CNT_MASK) == 0 && !(v & CNT_ZERO);
                }
                const uint32_t m = __ballot_sync(0xffffffffu, is_dead);
                if (m) {
                    dead = top - (__ffs(m) - 1);
                    stop = dead;
                    break;
                }
            }
        }
        // sum_{di=stop}^{B-1} (b-s+1)(di+1), b - s + 1 = bi + 1
        const int64_t a1 = stop + 1, z = cd.B;
        total += (int64_t)(bi + 1) * ((z * (z + 1) - (a1 - 1) * a1) / 2);
        if (dead >= 0) d_min = dead + 2;               // d_min = d + 1, d = 1 + dead
    }
    if (lane == 0) level_sums[level_off[c]] = total;
}

void launch_row_visits(const DPBatch &b, int pruning, int64_t *level_sums, int64_t *row_prefix,
                       const int64_t *level_off, int64_t n_rows_total, cudaStream_t st) {
    if (n_rows_total > 0)
        k_visit_rows<<<(unsigned)((n_rows_total + 255) / 256), 256, 0, st>>>(
            b, pruning, row_prefix, level_off, level_sums);
    k_visit_level1<<<(unsigned)((b.n_calls * 32 + 127) / 128), 128, 0, st>>>(b, pruning, level_off, level_sums);
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
    const int64_t vcell = cd.val_off + fcell;
    const uint8_t fb = Bt.val_cnt[par][vcell];
    const int n = cnt_entries(fb);
    const int o = cd.orig;
    if (n == 0) {
        // non-empty for the reference but every entry above the bound: the
        // bound was below the optimum (the host reruns the call unbounded)
        feasible[o] = (fb & CNT_MASK) == CNT_REACH ? -1 : 0;
        return;
    }
    const uint32_t vo = Bt.val_off[par][vcell];
    const int64_t vi = vo & ~SPILL_BIT;
    const double *vx = (vo & SPILL_BIT) ? Bt.spill_tf[par] + vi : Bt.pool_tf[par] + cd.vpool_base + vi;
    const double *vy = (vo & SPILL_BIT) ? Bt.spill_tb[par] + vi : Bt.pool_tb[par] + cd.vpool_base + vi;
    int best = 0;
    double bx = vx[0], by = vy[0];
    for (int j = 1; j < n; ++j) {
        if (__dadd_rn(vx[j], vy[j]) < __dadd_rn(bx, by)) {
            best = j;
            bx = vx[j];
            by = vy[j];
        }
    }
    feasible[o] = 1;
    objective[o] = __dadd_rn(bx, by);
    int s = S, b = Bt.nb, d = cd.D, j = best;
    int64_t cell = fcell;
    const int32_t off = plan_off[o];
    while (s > 0) {
        const int64_t hcell = cd.hist_off + (int64_t)(s - 1) * cells + cell;
        const uint32_t ho = Bt.hist_off[hcell];
        const uint32_t key = (ho & SPILL_BIT) ? Bt.hspill[(ho & ~SPILL_BIT) + j]
                                              : Bt.hpool[cd.hpool_base + ho + j];
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

void launch_backtrack(const DPBatch &b, int64_t batch_size, const int32_t *plan_off,
                      int32_t *seg_lo, int32_t *seg_hi, int32_t *seg_dev, double *objective,
                      int32_t *feasible, cudaStream_t st) {
    k_backtrack<<<(b.n_calls + 127) / 128, 128, 0, st>>>(b, batch_size, plan_off, seg_lo, seg_hi,
                                                         seg_dev, objective, feasible);
}

}  // namespace pcb
