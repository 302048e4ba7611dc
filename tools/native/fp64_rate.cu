// fp64_rate.cu — sustained FP64 instruction throughput of one B200 SM for the
// instruction mixes the tile kernels use: DMUL, DADD, DFMA, and the exact
// complex multiply (4 DMUL + 2 DADD). 8 independent chains per thread, so
// latency is hidden; results in lanes/clock/SM at the clock the run measured
// (clock64 around the loop).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/native/fp64_rate.cu -o /tmp/fp64_rate && /tmp/fp64_rate
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096, CH = 8;

template <int MODE>
__global__ void k(double *out, double a, double b, long long *cyc) {
    double x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = a + c * 1e-3 + threadIdx.x * 1e-9; y[c] = b - c * 1e-3; }
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) x[c] = __dmul_rn(x[c], a);                      // 1 DMUL
            if (MODE == 1) x[c] = __dadd_rn(x[c], b);                      // 1 DADD
            if (MODE == 2) x[c] = __fma_rn(x[c], a, b);                    // 1 DFMA
            if (MODE == 3) {                                               // cmul: 4 DMUL + 2 DADD
                const double re = __dsub_rn(__dmul_rn(a, x[c]), __dmul_rn(b, y[c]));
                const double im = __dadd_rn(__dmul_rn(a, y[c]), __dmul_rn(b, x[c]));
                x[c] = re; y[c] = im;
            }
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char *name, double per_iter_ops) {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 512;  // 64 warps per SM
    k<MODE><<<blocks, threads>>>(out, 0.999999, 1e-7, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, 0.999999, 1e-7, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double lane_ops = (double)blocks * threads * ITERS * CH * per_iter_ops;
    const double clk = (double)c / (ms * 1e-3);  // one block's clock64 span over the kernel time: ~SM clock
    printf("{\"mix\": \"%s\", \"ms\": %.3f, \"lane_ops_per_s\": %.4e, \"sm_clock_hz_est\": %.4e, \"lanes_per_clk_per_sm\": %.2f}\n",
           name, ms, lane_ops / (ms * 1e-3), clk, lane_ops / (ms * 1e-3) / clk / sms);
}

int main() {
    run<0>("DMUL", 1);
    run<1>("DADD", 1);
    run<2>("DFMA", 1);
    run<3>("cmul (4 DMUL + 2 DADD)", 6);
    return 0;
}
