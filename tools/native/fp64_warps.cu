// fp64_warps.cu — FP64 throughput of one B200 SM as a function of the warps
// resident per SM and of the independent chains per warp: what a kernel with
// few warps per SM sub-partition (the fused tile kernel runs 5) can reach.
// One block per SM; rate = lane-ops / (clock64 span of the block) in
// lanes/clock/SM. CH = 1 with 1 warp per sub-partition gives the dependent
// DFMA latency (clocks per instruction).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/native/fp64_warps.cu -o /tmp/fp64_warps && /tmp/fp64_warps
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int CH, int MODE>
__global__ void k(double *out, double a, double b, long long *cyc) {
    double x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = a + c * 1e-3 + threadIdx.x * 1e-9; y[c] = b - c * 1e-3; }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) x[c] = __fma_rn(x[c], a, b);
            if (MODE == 1) {  // exact complex multiply: 4 DMUL + 2 DADD, depth 2
                const double re = __dsub_rn(__dmul_rn(a, x[c]), __dmul_rn(b, y[c]));
                const double im = __dadd_rn(__dmul_rn(a, y[c]), __dmul_rn(b, x[c]));
                x[c] = re; y[c] = im;
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH, int MODE>
void run(int warps) {
    static double *out = nullptr;
    static long long *cyc = nullptr;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (!out) { cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024); }
    for (int rep = 0; rep < 2; ++rep) k<CH, MODE><<<sms, warps * 32>>>(out, 0.999999, 1e-7, cyc);
    cudaDeviceSynchronize();
    long long c[1024];
    cudaMemcpy(c, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)c[i] / sms;
    const double per = MODE == 0 ? 1 : 6;
    const double instr = (double)warps * ITERS * CH * per;  // warp instructions per SM
    printf("{\"mix\": \"%s\", \"warps_per_sm\": %d, \"chains\": %d, \"lanes_per_clk_per_sm\": %.2f, \"clk_per_warp_instr_per_subpartition\": %.2f}\n",
           MODE == 0 ? "DFMA" : "cmul", warps, CH, instr * 32 / mean, mean / (instr / 4));
}

template <int MODE>
void sweep() {
    for (int w : {4, 8, 12, 16, 20, 32, 64}) {
        run<1, MODE>(w);
        run<2, MODE>(w);
        run<4, MODE>(w);
        run<8, MODE>(w);
        if (w <= 32) run<16, MODE>(w);
    }
}

int main() {
    sweep<0>();
    sweep<1>();
    return 0;
}
