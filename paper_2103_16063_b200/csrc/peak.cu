// fp64 rate microbenchmarks: the roofline denominators of the DP level kernel
// (a min/max/add recurrence; no tensor-core or HBM roof binds it).
//   MIX  -- one op per DADD / fp64 max (DSETP.MAX + select on sm_100) / DSETP,
//           the three fp64 operations of a DP visit, back to back
//   DADD -- pure DADD chains: the fp64 pipe's peak op rate
// Independent chains at full occupancy, best of 5 launches (CUDA events).
#include "common.cuh"

namespace pcb {

constexpr int PEAK_ITERS = 4096;
constexpr int PEAK_CHAINS = 8;

template <bool MIX>
__global__ void __launch_bounds__(256) k_fp64_peak(double seed, double *out) {
    double a[PEAK_CHAINS], c[PEAK_CHAINS];
#pragma unroll
    for (int i = 0; i < PEAK_CHAINS; ++i) {
        a[i] = seed * (threadIdx.x + i);
        c[i] = seed - i;
    }
    const double inc = seed * 1e-9;
    int flag = 0;
    for (int it = 0; it < PEAK_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < PEAK_CHAINS; ++i) {
            a[i] = __dadd_rn(a[i], inc);              // DADD
            if (MIX) {
                c[i] = fmax(c[i], a[i]);              // fp64 max
                flag += (a[i] <= c[i]) ? 1 : 0;       // DSETP
            } else {
                c[i] = __dadd_rn(c[i], inc);          // DADD
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < PEAK_CHAINS; ++i) s += a[i] + c[i];
    if (s == 12345.678 || flag == -1) out[0] = s;
}

template <bool MIX>
static double measure(cudaStream_t st, int sm_count) {
    double *out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sm_count * 8;   // 2048 threads per SM
    k_fp64_peak<MIX><<<blocks, 256, 0, st>>>(1.0000001, out);   // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, st);
        k_fp64_peak<MIX><<<blocks, 256, 0, st>>>(1.0000001 + r, out);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return -1;
    const double ops_per_iter = MIX ? 3.0 : 2.0;
    const double ops = ops_per_iter * PEAK_ITERS * PEAK_CHAINS * (double)blocks * 256;
    return ops / (best * 1e-3) / 1e9;
}

double measure_fp64_gops(cudaStream_t st, int sm_count) { return measure<true>(st, sm_count); }
double measure_dadd_gops(cudaStream_t st, int sm_count) { return measure<false>(st, sm_count); }

}  // namespace pcb
